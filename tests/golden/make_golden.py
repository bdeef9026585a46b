#!/usr/bin/env python
"""Generate golden input/output vectors from the REAL reference (`mdbench` 0.1.0).

Runs only in the build container, where /root/reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src,
replays the fixtures its own tests use (seeds and shapes cited per block) and
stores inputs + outputs as small .npz files next to this script.  The oracle
(oracle/oracle.py + oracle/md_oracle.c) is pinned bit-for-bit against these
files by tests/test_oracle_golden.py; the GPU parity tests reuse the same files.
Nothing at test/bench time reads /root/reference.
"""
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
import mdbench as ref  # noqa: E402
from mdbench.bruteforce import forces_and_energy  # noqa: E402
from mdbench.core import COMPUTE, HOST  # noqa: E402
from mdbench.sim import TRUNCATED  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}.npz: {os.path.getsize(path) / 1024:.1f} KiB, {len(arrays)} arrays")


def ragged(nl):
    """Store a fixed-stride list compactly: counts + concatenated valid rows."""
    rows = [nl.indices[i, :nl.counts[i]] for i in range(nl.counts.size)]
    flat = np.concatenate(rows) if rows else np.zeros(0, np.int32)
    return nl.counts.astype(np.int32), flat.astype(np.int32)


# ---------------------------------------------------------------- neighbour
def neighbor_cases():
    out = {}
    cases = []
    # test_neighbor.py:87-100 : (seed, n, density) at r_list 3.0, stride 512
    for seed, n, density in [(0, 120, 0.3), (1, 250, 0.8), (2, 400, 1.0), (3, 60, 0.2)]:
        edge = (n / density) ** (1.0 / 3.0)
        cases.append((f"cube{seed}", (edge, edge, edge), n, seed, 3.0, 512))
    # test_neighbor.py:30-45 : orthorhombic (10,8,6), r_list 2 -> 5x4x3 cells
    cases.append(("ortho", (10.0, 8.0, 6.0), 200, 0, 2.0, 64))
    # test_neighbor.py:116-123 : 2 cells per axis -> brute-force fallback
    cases.append(("fallback", (4.4, 4.4, 4.4), 80, 5, 2.0, 256))
    # test_neighbor.py:126-136 : stride 4 overflows
    cases.append(("overflow", (6.0, 6.0, 6.0), 200, 6, 3.0, 4))
    # test_neighbor.py:103-113 : symmetric + sorted rows
    cases.append(("sym", (8.0, 8.0, 8.0), 300, 4, 2.5, 256))
    names = []
    for name, edges, n, seed, r_list, stride in cases:
        box = ref.SimBox(edges)
        gen = np.random.default_rng(seed)
        pos = gen.uniform(0.0, 1.0, size=(n, 3)) * box.edge_lengths
        state = ref.ParticleState(pos)
        grid = ref.bin_particles(state, box, r_list)
        nl = ref.build_neighbor_list(state, grid, r_list, stride)
        counts, flat = ragged(nl)
        perm = ref.reorder_by_cell(ref.ParticleState(pos), grid)
        names.append(name)
        out.update({
            f"{name}.pos": pos, f"{name}.edges": np.array(edges),
            f"{name}.r_list": np.float64(r_list), f"{name}.stride": np.int64(stride),
            f"{name}.ncells": grid.cells_per_axis, f"{name}.cell_edge": grid.cell_edge,
            f"{name}.cell_of": grid.cell_of_particle, f"{name}.cell_start": grid.cell_start,
            f"{name}.cell_particles": grid.cell_particles,
            f"{name}.fallback": np.bool_(grid.fallback),
            f"{name}.counts": counts, f"{name}.rows": flat,
            f"{name}.overflow": np.bool_(nl.overflow),
            f"{name}.at_build": nl.positions_at_build, f"{name}.perm": perm,
        })
    # test_neighbor.py:58-66 : top boundary clamp
    x = np.nextafter(9.0, 0.0)
    st = ref.ParticleState(np.array([[x, x, x]]))
    g = ref.bin_particles(st, ref.SimBox.cubic(9.0), 3.0)
    out["clamp.cell_of"] = g.cell_of_particle
    out["clamp.cell_start"] = g.cell_start
    out["names"] = np.array(names)
    save("neighbor", **out)


# ------------------------------------------------------------------ rebuild
def rebuild_cases():
    # test_neighbor.py:174-213
    box = ref.SimBox.cubic(10.0)
    rows = []

    def record(tag, state, nl):
        rows.append((tag, np.array(state.positions.acquire_read(COMPUTE)),
                     np.array(state.images.acquire_read(COMPUTE)),
                     nl.positions_at_build.copy(), nl.r_list, nl.r_cut,
                     ref.needs_rebuild(state, box, nl)))

    st = ref.ParticleState(np.array([[5.0, 5.0, 5.0], [1.0, 1.0, 1.0]]))
    nl = ref.build_neighbor_list(st, ref.bin_particles(st, box, 3.0), 3.0, 8, r_cut=2.5)
    record("still", st, nl)
    st.positions.acquire_update(COMPUTE)[0, 0] = 5.25
    record("exact_half_skin", st, nl)
    st.positions.acquire_update(COMPUTE)[0, 0] = 5.25 + 1e-9
    record("just_over", st, nl)

    st = ref.ParticleState(np.array([[0.05, 5.0, 5.0], [7.0, 5.0, 5.0]]))
    nl = ref.build_neighbor_list(st, ref.bin_particles(st, box, 3.0), 3.0, 8, r_cut=2.5)
    st.positions.acquire_update(COMPUTE)[0, 0] = 9.95
    st.images.acquire_update(COMPUTE)[0, 0] = -1
    record("crossed_with_image", st, nl)
    st.images.acquire_update(COMPUTE)[0, 0] = 0
    record("crossed_without_image", st, nl)

    st = ref.ParticleState(np.array([[5.0, 5.0, 5.0], [1.0, 1.0, 1.0]]))
    nl = ref.build_neighbor_list(st, ref.bin_particles(st, box, 2.5), 2.5, 8, r_cut=2.5)
    record("zero_skin_still", st, nl)
    st.positions.acquire_update(COMPUTE)[0, 0] += 1e-12
    record("zero_skin_moved", st, nl)

    # a random many-particle case around the threshold
    gen = np.random.default_rng(77)
    pos = gen.uniform(0, 10.0, size=(300, 3))
    st = ref.ParticleState(pos)
    nl = ref.build_neighbor_list(st, ref.bin_particles(st, box, 3.0), 3.0, 128, r_cut=2.7)
    p = st.positions.acquire_update(COMPUTE)
    im = st.images.acquire_update(COMPUTE)
    p += gen.normal(scale=0.05, size=p.shape)
    w, k = ref.wrap_position(p, im, box)
    p[...] = w
    im[...] = k
    record("random300", st, nl)

    save("rebuild",
         tags=np.array([r[0] for r in rows]),
         edges=box.edge_lengths,
         **{f"{r[0]}.pos": r[1] for r in rows},
         **{f"{r[0]}.img": r[2] for r in rows},
         **{f"{r[0]}.at_build": r[3] for r in rows},
         **{f"{r[0]}.r_list": np.float64(r[4]) for r in rows},
         **{f"{r[0]}.r_cut": np.float64(r[5]) for r in rows},
         **{f"{r[0]}.answer": np.bool_(r[6]) for r in rows})


# ------------------------------------------------------------------- forces
def force_cases():
    out = {}
    lj = ref.make_shifted(1.0, 1.0, 2.5)
    out["lj"] = np.array([lj.epsilon, lj.sigma, lj.r_cut, lj.energy_shift])
    seq = ref.BackendSelector()
    # test_forces.py:45-56 : truncated, n=320, L=7.5, seeds 50..54, r_list 3.0
    for seed in range(50, 55):
        box = ref.SimBox.cubic(7.5)
        pos = np.random.default_rng(seed).uniform(0.0, 7.5, size=(320, 3))
        st = ref.ParticleState(pos)
        grid = ref.bin_particles(st, box, 3.0)
        nl = ref.build_neighbor_list(st, grid, 3.0, 256, r_cut=lj.r_cut)
        ref.compute_forces_truncated(st, lj, box, nl, seq)
        bf, bpe, btot = forces_and_energy(st, lj, box)
        counts, flat = ragged(nl)
        out.update({
            f"trunc{seed}.pos": pos, f"trunc{seed}.edge": np.float64(7.5),
            f"trunc{seed}.counts": counts, f"trunc{seed}.rows": flat,
            f"trunc{seed}.forces": np.array(st.forces.acquire_read(COMPUTE)),
            f"trunc{seed}.pe": np.array(st.per_particle_potential.acquire_read(COMPUTE)),
            f"trunc{seed}.brute_forces": bf, f"trunc{seed}.brute_pe": bpe,
            f"trunc{seed}.brute_total": np.float64(btot),
        })
    # test_forces.py:32-42 : all-to-all, n=300, L=7.0, seeds 0..1
    for seed in range(2):
        box = ref.SimBox.cubic(7.0)
        pos = np.random.default_rng(seed).uniform(0.0, 7.0, size=(300, 3))
        st = ref.ParticleState(pos)
        ref.compute_forces_all_to_all(st, lj, box, seq)
        out.update({
            f"all{seed}.pos": pos, f"all{seed}.edge": np.float64(7.0),
            f"all{seed}.forces": np.array(st.forces.acquire_read(COMPUTE)),
            f"all{seed}.pe": np.array(st.per_particle_potential.acquire_read(COMPUTE)),
        })
    # test_forces.py:70-84 : pairs straddling the cutoff
    eps = np.array([-4e-15, -1e-15, 0.0, 1e-15, 4e-15])
    positions = [[1.0, 1.0 + 3 * k, 1.0] for k in range(eps.size)]
    positions += [[1.0 + 2.5 + e, 1.0 + 3 * k, 1.0] for k, e in enumerate(eps)]
    pos = np.array(positions)
    box = ref.SimBox.cubic(20.0)
    st = ref.ParticleState(pos)
    ref.compute_forces_all_to_all(st, lj, box, seq)
    out.update({"straddle.pos": pos, "straddle.edge": np.float64(20.0),
                "straddle.forces": np.array(st.forces.acquire_read(COMPUTE)),
                "straddle.pe": np.array(st.per_particle_potential.acquire_read(COMPUTE))})
    # test_forces.py:171-188 : singular pairs
    pos = np.array([[1.0, 1.0, 1.0], [3.0, 3.0, 3.0], [1.0, 1.0, 1.0]])
    try:
        ref.compute_forces_all_to_all(ref.ParticleState(pos), lj, ref.SimBox.cubic(10.0), seq)
    except ref.SingularPairError as exc:
        out["singular.pos"] = pos
        out["singular.ij"] = np.array([exc.i, exc.j])
    # test_potential.py:19-23
    out["shift_2p5"] = np.float64(lj.energy_shift)
    save("forces", **out)


# ---------------------------------------------------------------- integrate
def integrate_cases():
    gen = np.random.default_rng(2024)
    n = 240
    edges = np.array([7.0, 8.0, 9.0])
    box = ref.SimBox(edges)
    pos = gen.uniform(0, 1, size=(n, 3)) * edges
    vel = gen.normal(scale=30.0, size=(n, 3))   # some cross several boxes in one step
    vel[:8] *= 40.0
    masses = gen.uniform(0.5, 2.0, size=n)
    img = gen.integers(-3, 4, size=(n, 3))
    forces = gen.normal(scale=20.0, size=(n, 3))
    dt = 0.01
    st = ref.ParticleState(pos, velocities=vel, masses=masses, images=img)
    st.forces.acquire_write(COMPUTE)[...] = forces
    ref.vv_integrate(st, ref.IntegratorParams(dt), box)
    p1 = np.array(st.positions.acquire_read(COMPUTE))
    i1 = np.array(st.images.acquire_read(COMPUTE))
    v1 = np.array(st.velocities.acquire_read(COMPUTE))
    forces2 = gen.normal(scale=20.0, size=(n, 3))
    st.forces.acquire_write(COMPUTE)[...] = forces2
    ref.vv_finalize(st, ref.IntegratorParams(dt))
    v2 = np.array(st.velocities.acquire_read(COMPUTE))
    # wrap edge cases: core.py:72-93, test_core.py:60-66
    wb = ref.SimBox.cubic(10.0)
    r_in = np.array([[10.0, -1e-17, 25.0], [0.0, 9.999999999999998, -30.5],
                     [-10.0, 1e3 + 0.25, np.nextafter(10.0, 0.0)]])
    i_in = np.array([[0, 0, 0], [1, -1, 2], [5, 0, 0]], dtype=np.int64)
    w, k = ref.wrap_position(r_in, i_in, wb)
    # minimum image ties: test_core.py:36-44
    mi_in = np.array([[5.0, -5.0, 15.0], [2.5, 7.5, -7.5], [4.999999999999999, 0.0, 1e-300]])
    mi = ref.minimum_image(mi_in, wb)
    save("integrate", pos=pos, vel=vel, masses=masses, img=img, forces=forces,
         forces2=forces2, edges=edges, dt=np.float64(dt), pos1=p1, img1=i1,
         vel1=v1, vel2=v2, wrap_in=r_in, wrap_img=i_in, wrap_out=w,
         wrap_img_out=k, mi_in=mi_in, mi_out=mi)


# -------------------------------------------------------------- observables
def observable_cases():
    gen = np.random.default_rng(99)
    sizes = [1, 2, 3, 5, 31, 4095, 4096, 4097, 8191, 8193, 10000, 100003]
    base = gen.normal(size=max(sizes)) * np.exp(gen.normal(size=max(sizes)) * 3)
    sums = np.array([ref.reduce_sum(base[:s]) for s in sizes])
    fast = np.array([ref.reduce_sum(base[:s], mode="fast") for s in sizes])
    n = 5000
    vel = gen.normal(size=(n, 3))
    masses = gen.uniform(0.5, 2.0, size=n)
    st = ref.ParticleState(gen.uniform(0, 5, size=(n, 3)), velocities=vel, masses=masses)
    pe_in = gen.normal(size=n)
    st.per_particle_potential.acquire_write(COMPUTE)[...] = pe_in
    ke, temp = ref.kinetic_energy_and_temperature(st)
    save("observables", values=base, sizes=np.array(sizes), sums=sums, fast=fast,
         vel=vel, masses=masses, pe_in=pe_in, ke=np.float64(ke),
         temperature=np.float64(temp),
         pe=np.float64(ref.potential_energy_total(st)),
         momentum=ref.total_momentum(st))


# --------------------------------------------------------------- trajectory
def trajectory_case():
    # Same state point as BASELINE.json configs 1-2 at a size the CPU suite
    # replays in seconds: fcc + vacancies, T0=1.2, rc=2.5, skin 0.3, dt=0.001.
    n, rho, T, dt, skin, steps, every = 500, 0.75, 1.2, 0.001, 0.3, 300, 20
    st, box = ref.init_lattice_any(n, rho)
    ref.init_velocities(st, T, 42)
    pos0 = np.array(st.positions.acquire_read(HOST))
    vel0 = np.array(st.velocities.acquire_read(HOST))
    lj = ref.make_shifted(1.0, 1.0, 2.5)
    sim = ref.Simulation(st, box, lj, dt, force_mode=TRUNCATED, skin=skin,
                         sample_interval=every, sample_initial=True)
    sim.run(steps)
    s = sim.samples
    # lattice generator fixtures (integrate.py:110-171)
    lat256, box256 = ref.init_lattice_any(256, 0.8)
    save("trajectory", n=np.int64(n), density=np.float64(rho), dt=np.float64(dt),
         skin=np.float64(skin), steps=np.int64(steps), every=np.int64(every),
         edges=box.edge_lengths, pos0=pos0, vel0=vel0,
         step=np.array([x.step for x in s]),
         pe=np.array([x.potential_energy for x in s]),
         ke=np.array([x.kinetic_energy for x in s]),
         temperature=np.array([x.temperature for x in s]),
         momentum=np.array([x.total_momentum for x in s]),
         rebuilds=np.array([x.rebuild_count for x in s]),
         pos_end=np.array(st.positions.acquire_read(HOST)),
         vel_end=np.array(st.velocities.acquire_read(HOST)),
         img_end=np.array(st.images.acquire_read(HOST)),
         forces_end=np.array(st.forces.acquire_read(HOST)),
         stride_end=np.int64(sim._stride),
         lat256=np.array(lat256.positions.acquire_read(HOST)),
         lat256_edges=box256.edge_lengths)


# ------------------------------------------------ all-to-all loop (default mode)
def all2all_trajectory_case():
    """Simulation.run in the reference's DEFAULT force mode (sim.py:62-102, all_to_all,
    untruncated pair potential as in the all2all-2k preset, bench.py:147-151), at a size the
    reference finishes in seconds: an NVE run and a thermostatted one (second finalize slot,
    sim.py:86-87) from the same start."""
    n, rho, T, dt, steps, every = 300, 0.8, 1.0, 0.002, 200, 20
    out = {}
    for tag, rate in (("nve", 0.0), ("nvt", 5.0)):
        st, box = ref.init_lattice_any(n, rho)
        ref.init_velocities(st, T, 42)
        if tag == "nve":
            out["pos0"] = np.array(st.positions.acquire_read(HOST))
            out["vel0"] = np.array(st.velocities.acquire_read(HOST))
            out["edges"] = box.edge_lengths
        lj = ref.make_shifted(1.0, 1.0)                   # r_cut = inf: the bare potential
        thermostat = ref.ThermostatParams(temperature=T, rate=rate, seed=7) if rate else None
        sim = ref.Simulation(st, box, lj, dt, thermostat=thermostat, sample_interval=every,
                             sample_initial=True)
        sim.run(steps)
        s = sim.samples
        out[tag + "_step"] = np.array([x.step for x in s])
        out[tag + "_pe"] = np.array([x.potential_energy for x in s])
        out[tag + "_ke"] = np.array([x.kinetic_energy for x in s])
        out[tag + "_momentum"] = np.array([x.total_momentum for x in s])
        out[tag + "_pos_end"] = np.array(st.positions.acquire_read(HOST))
        out[tag + "_vel_end"] = np.array(st.velocities.acquire_read(HOST))
        out[tag + "_forces_end"] = np.array(st.forces.acquire_read(HOST))
    save("all2all_trajectory", n=np.int64(n), density=np.float64(rho), dt=np.float64(dt),
         steps=np.int64(steps), every=np.int64(every), temperature=np.float64(T),
         rate=np.float64(5.0), seed=np.int64(7), **out)


# ---------------------------------------------------------- rng / thermostat
def thermostat_case():
    from mdbench import rng
    # test_rng.py:9-13 address (12345, 0, 7)
    raw = rng.raw_words(12345, 0, 7, 12)
    uni = rng.uniforms(12345, 0, 7, 8, word_offset=3)
    nrm = rng.normals(12345, 1, 0, 9, word_offset=2)
    gen = np.random.default_rng(5)
    n = 3000
    vel = gen.normal(size=(n, 3))
    masses = gen.uniform(0.5, 2.0, size=n)
    st = ref.ParticleState(gen.uniform(0, 5, size=(n, 3)), velocities=vel, masses=masses)
    params = ref.ThermostatParams(temperature=1.7, rate=25.0, seed=99)
    count = ref.andersen_thermostat(st, params, 0.004, 321)
    save("thermostat", raw=raw, uniforms=uni, normals=nrm, vel=vel, masses=masses,
         temperature=np.float64(1.7), rate=np.float64(25.0), seed=np.int64(99),
         dt=np.float64(0.004), step=np.int64(321), count=np.int64(count),
         vel_after=np.array(st.velocities.acquire_read(COMPUTE)))


# ------------------------------------------------------- harness CSV files
def harness_csv_case():
    """Records / samples files WRITTEN BY THE REFERENCE's own writers (bench.py:222-285)
    from a sweep it ran itself (bench.py:372-383, smoke-sized): the B200 harness must read
    them, summarise them and write them back byte for byte.  Also the reference's
    speed-up / efficiency rows for both baselines (bench.py:393-442)."""
    from mdbench import bench
    cfg = bench.BenchConfig(n_particles=108, density=0.8, temperature=1.5, dt=0.002, steps=40,
                            r_cut=2.5, skin=0.5, thermostat_rate=5.0, seed=7,
                            sample_interval=10, equilibration_steps=10)
    records = bench.run_sweep(cfg, [1, 2, 3])
    bench.write_records_csv(os.path.join(OUT, "reference_records.csv"), records)
    _, samples = bench.run_benchmark(cfg)
    bench.write_samples_csv(os.path.join(OUT, "reference_samples.csv"), samples)
    rows = {}
    for base in ("sequential", "single"):
        sr = bench.compute_speedup_efficiency(records, baseline=base)
        rows[base] = np.array([[r.worker_count, r.wall_time_s, r.speedup, r.efficiency]
                               for r in sr])
    save("harness", speedup_sequential=rows["sequential"], speedup_single=rows["single"])
    print("reference_records.csv / reference_samples.csv written")


if __name__ == "__main__":
    print("reference mdbench", ref.__version__)
    if len(sys.argv) > 1 and sys.argv[1] == "harness":
        harness_csv_case()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "all2all":
        all2all_trajectory_case()
        sys.exit(0)
    neighbor_cases()
    rebuild_cases()
    force_cases()
    integrate_cases()
    observable_cases()
    trajectory_case()
    all2all_trajectory_case()
    thermostat_case()
    harness_csv_case()
