"""GPU tests of the assembled step loop (`-m gpu`): the native C++ runner against
the operator-by-operator loop (bitwise), both against the CPU oracle, energy
conservation, stride growth, reordering invariance, and size-independent
properties at a larger N."""
import numpy as np
import pytest

import paper_2406_04210_b200 as b2
from conftest import load_golden
from helpers import fluid_state, quantize_ds, quantize_f32
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

LJ = b2.make_shifted(1.0, 1.0, 2.5)


def lattice_sim(n, native, reorder="hilbert", dt=0.001, skin=0.3, every=20, seed=42, **kw):
    st, box = b2.init_lattice_any(n, 0.75)
    b2.init_velocities(st, 1.2, seed)
    sim = b2.Simulation(st, box, LJ, dt, force_mode=b2.TRUNCATED, skin=skin,
                        sample_interval=every, sample_initial=True, native=native,
                        reorder=reorder, **kw)
    return sim


def series(sim):
    return np.array([[s.potential_energy, s.kinetic_energy, *s.total_momentum, s.virial]
                     for s in sim.samples])


def test_native_loop_equals_operator_loop_bitwise():
    runs = {}
    for native in (True, False):
        sim = lattice_sim(2048, native, reorder=None)
        sim.run(130)      # not a multiple of the sample interval: exercises the deferred kick
        sim.run(70)
        runs[native] = (series(sim), np.array(sim.state.positions.acquire_read(b2.HOST)),
                        np.array(sim.state.velocities.acquire_read(b2.HOST)),
                        np.array(sim.state.images.acquire_read(b2.HOST)), sim.rebuild_count)
        sim.close()
    for a, b in zip(runs[True][:4], runs[False][:4]):
        assert np.array_equal(a, b)
    # the in-loop fp32 displacement test may fire one step before the exact fp64 one
    assert runs[True][4] >= 2 and abs(runs[True][4] - runs[False][4]) <= 1


def test_graphed_steps_equal_ungraphed_steps_bitwise():
    """The CUDA-graph step (conditional rebuild node) runs the same kernels on the
    same data as the host-driven loop: identical trajectories, no host round trips."""
    runs = {}
    for graph in (8, False):
        sim = lattice_sim(2048, True, reorder="hilbert", every=40, graph=graph)
        sim.run(130)
        sim.run(70)
        runs[graph] = (series(sim), np.array(sim.state.positions.acquire_read(b2.HOST)),
                       np.array(sim.state.velocities.acquire_read(b2.HOST)),
                       np.array(sim.state.images.acquire_read(b2.HOST)), sim.rebuild_count,
                       sim.graph_steps, sim.wasted_force_launches)
        sim.close()
    for a, b in zip(runs[8][:5], runs[False][:5]):
        assert np.array_equal(a, b)
    assert runs[8][5] >= 180 and runs[False][5] == 0          # most steps ran as graphs
    assert runs[8][6] == 0                                    # nothing speculative in a graph


def test_overflow_inside_a_step_graph_is_recovered():
    """stride_policy='tight' sizes rows to exactly the fullest row, so a later
    in-graph rebuild overflows: the batch freezes, the stride grows, the step is
    resumed -- same trajectory as the ungraphed loop with the same policy."""
    out = {}
    for graph in (True, False):
        sim = lattice_sim(2916, True, stride=16, stride_policy="tight", every=50, graph=graph,
                          dt=0.002)
        sim.run(400)
        out[graph] = (series(sim), sim.overflow_events, sim.stride, sim.rebuild_count)
        sim.close()
    assert out[True][1] >= 2                  # at least one overflow after construction
    assert np.array_equal(out[True][0], out[False][0])
    assert out[True][1:] == out[False][1:]


def test_reordering_does_not_change_the_physics():
    """Hilbert / cell reordering only permutes rows: energies agree to fp32
    summation-order noise and the host view stays in logical order."""
    out = {}
    for reorder in (None, "hilbert", "cell"):
        sim = lattice_sim(2048, True, reorder=reorder, every=50)
        sim.run(100)
        out[reorder] = (series(sim), np.array(sim.state.positions.acquire_read(b2.HOST)))
        if reorder:
            assert sim.reorders >= 1
            assert not np.array_equal(sim.state.particle_ids(), np.arange(2048))
        sim.close()
    for mode in ("hilbert", "cell"):
        assert np.allclose(out[mode][0][:, :2], out[None][0][:, :2], rtol=2e-6)
        assert np.max(np.abs(out[mode][1] - out[None][1])) < 1e-3


def test_trajectory_tracks_the_reference_run():
    """Same initial state as the golden reference trajectory (N=500): the first
    samples agree to fp32 accuracy, the whole series to the chaotic-divergence
    bound, and total energy is conserved as well as the reference conserves it."""
    G = load_golden("trajectory")
    st = b2.ParticleState(G["pos0"], velocities=G["vel0"])
    box = b2.SimBox(G["edges"])
    sim = b2.Simulation(st, box, LJ, float(G["dt"]), force_mode=b2.TRUNCATED,
                        skin=float(G["skin"]), sample_interval=int(G["every"]),
                        sample_initial=True)
    sim.run(int(G["steps"]))
    s = sim.samples
    assert [x.step for x in s] == list(G["step"])
    pe = np.array([x.potential_energy for x in s])
    ke = np.array([x.kinetic_energy for x in s])
    e_ref = G["pe"] + G["ke"]
    assert abs(pe[0] - G["pe"][0]) <= 2e-6 * abs(G["pe"][0])
    assert abs(ke[0] - G["ke"][0]) <= 2e-6 * abs(G["ke"][0])
    assert np.max(np.abs(pe - G["pe"])) <= 2e-3 * np.abs(G["pe"]).max()
    drift_ref = np.max(np.abs(e_ref - e_ref[0])) / abs(e_ref[0])
    drift = np.max(np.abs((pe + ke) - (pe + ke)[0])) / abs((pe + ke)[0])
    assert drift <= max(3.0 * drift_ref, 2e-5)
    mom = np.array([x.total_momentum for x in s])
    assert np.max(np.abs(mom)) <= 1e-3
    assert abs(sim.samples[-1].rebuild_count - int(G["rebuilds"][-1])) <= 3
    sim.close()


def test_nve_energy_conservation_n4096():
    """BASELINE config 1 (N=4096, rho=0.75, T0=1.2, rc=2.5, dt=0.001, 1000 steps):
    the reference drifts 7.6e-06 over this run; bound 3e-5."""
    sim = lattice_sim(4096, True, every=100)
    sim.run(1000)
    e = np.array([s.total_energy for s in sim.samples])
    assert np.max(np.abs(e - e[0])) / abs(e[0]) <= 3e-5
    t_end = sim.samples[-1].temperature
    assert 0.5 < t_end < 1.0          # lattice melts: T relaxes towards ~0.66
    assert 15 <= sim.rebuild_count <= 40      # reference: 24 per 1000 steps
    p = np.array(sim.samples[-1].total_momentum)
    assert np.max(np.abs(p)) <= 1e-2
    # small systems run their intermediate steps in batches inside ONE cooperative launch
    # (b2md_steps_persistent): far fewer launches than steps
    assert sim.persistent_steps > 0 and 100 <= sim.kernel_launches < 1000
    sim.close()


def test_persistent_step_kernel_is_bit_identical_to_one_launch_per_step():
    """b2md_steps_persistent (up to 256 MD steps per cooperative launch, grid barriers between
    them, 16 / 4 / 2 / 1 lanes per particle by size) against the gated one-launch steps and the
    separate integrate / force launches: same trajectories, energies, image counters and rebuild
    schedule bit for bit, for every lane count, across rebuilds and sample steps."""
    for n in (2048, 20_000, 50_000):
        out = []
        for kw in (dict(persistent_steps=0, advance=False), dict(persistent_steps=0, advance=True),
                   dict(persistent_steps=256), dict(persistent_steps=7)):
            sim = lattice_sim(n, True, every=37, dt=0.002, **kw)
            sim.run(150)
            sim.run(63)
            out.append((series(sim), np.array(sim.state.positions.acquire_read(b2.HOST)),
                        np.array(sim.state.velocities.acquire_read(b2.HOST)),
                        np.array(sim.state.images.acquire_read(b2.HOST)), sim.rebuild_count,
                        sim.kernel_launches))
            sim.close()
        for other in out[1:]:
            for a, b in zip(out[0][:5], other[:5]):
                assert np.array_equal(a, b), n
        assert out[0][4] >= 3
        assert out[2][5] < out[1][5] < out[0][5]          # launches: batches < one per step < two


def test_stride_growth_recovers_from_overflow():
    # DEFAULT_STRIDE-like start that is too small: the list must grow, not truncate
    for policy, native in (("fit", True), ("double", True), ("fit", False)):
        sim = lattice_sim(1372, native, stride=16, stride_policy=policy, every=10)
        assert sim.overflow_events >= 1 and sim.stride >= 66
        if policy == "double":
            assert sim.stride in (128,)
        sim.run(30)
        e = np.array([s.total_energy for s in sim.samples])
        assert np.max(np.abs(e - e[0])) / abs(e[0]) <= 1e-5
        sim.close()


def test_stride_growth_limit_raises(monkeypatch):
    import paper_2406_04210_b200.sim as simmod
    monkeypatch.setattr(simmod, "STRIDE_GROWTH_LIMIT", 0)      # test_bench.py:207-216 analogue
    with pytest.raises(b2.NeighborOverflowError):
        lattice_sim(500, True, stride=8)
    with pytest.raises(b2.NeighborOverflowError):
        lattice_sim(500, False, stride=8)


def test_singular_pair_surfaces_from_the_native_loop():
    pos = np.array([[1.0, 1.0, 1.0], [5.0, 5.0, 5.0], [1.0, 1.0, 1.0], [8.0, 2.0, 3.0]])
    st = b2.ParticleState(pos)
    with pytest.raises(b2.SingularPairError) as exc:
        b2.Simulation(st, b2.SimBox.cubic(12.0), LJ, 0.001, force_mode=b2.TRUNCATED, skin=0.3)
    assert (exc.value.i, exc.value.j) == (0, 2)


def test_kob_andersen_mixture_conserves_energy():
    n = 4000
    st, box = b2.init_lattice_any(n, 1.2)
    species = (np.random.default_rng(42).permutation(n) < n // 5).astype(np.int32)
    st = b2.ParticleState(st.positions.acquire_read(b2.HOST), species=species)
    b2.init_velocities(st, 1.0, 7)
    ka = b2.PairTable.kob_andersen()
    sim = b2.Simulation(st, box, ka, 0.001, force_mode=b2.TRUNCATED, skin=0.3,
                        sample_interval=50, sample_initial=True)
    sim.run(400)
    e = np.array([s.total_energy for s in sim.samples])
    assert np.max(np.abs(e - e[0])) / abs(e[0]) <= 5e-5
    # species travel with their particles through every reorder
    assert np.array_equal(sim.state.species.acquire_read(b2.HOST), species)
    # against the oracle's fp64 evaluation of the same final configuration
    pos = np.array(sim.state.positions.acquire_read(b2.HOST))
    og = orc.bin_particles(pos, box.edge_lengths, ka.max_r_cut + 0.3)
    onl = orc.build_neighbor_list(pos, np.zeros_like(pos, dtype=np.int64), og,
                                  ka.max_r_cut + 0.3, 512, r_cut=ka.max_r_cut,
                                  threads=orc.host_threads())
    _, rpe, rw = orc.forces_truncated(pos, box.edge_lengths, ka.table(), onl, species=species,
                                      threads=orc.host_threads())
    last = sim.samples[-1]
    assert last.potential_energy == pytest.approx(rpe.sum(), rel=2e-5)
    assert last.virial == pytest.approx(rw.sum(), rel=2e-4)
    sim.close()


def test_large_system_properties():
    """Size-independent invariants at N=256k (no oracle run needed): Hilbert keys
    sorted after a reorder, list symmetric in aggregate, total force ~ 0,
    momentum conserved, energies finite and extensive."""
    n = 262_144
    sim = lattice_sim(n, True, every=50)
    dev = sim.state.device_state()
    keys, _ = b2.hilbert_keys(sim.state, sim.box, 2.8)
    assert np.all(np.diff(keys.cpu().numpy()) >= 0)
    sim.run(100)
    s0, s1 = sim.samples[0], sim.samples[-1]
    assert abs(s1.total_energy - s0.total_energy) <= 2e-5 * abs(s0.total_energy)
    assert -8.0 * n < s0.potential_energy < -5.0 * n
    assert np.max(np.abs(s1.total_momentum)) <= 0.05
    f = sim.state.forces.acquire_read(b2.HOST)
    assert np.all(np.isfinite(f))
    assert np.max(np.abs(f.sum(axis=0))) <= 1e-4 * np.abs(f).max() * np.sqrt(n)
    counts = sim._keep["counts"][:n].cpu().numpy()
    assert counts.sum() % 2 == 0 and counts.min() > 30 and counts.max() <= sim.stride
    assert sorted(sim.state.particle_ids().tolist()) == list(range(n))
    sim.close()


def test_reference_presets_run_through_the_harness():
    """bench.py presets on the B200 backend: smoke-256 (thermostatted, truncated) and a
    shortened all2all-2k (the paper's primary benchmark, untruncated all-pairs)."""
    from dataclasses import replace
    rec, samples = b2.run_benchmark(b2.preset_config("smoke-256"))
    assert rec.steps_per_second > 0 and len(samples) == 4
    assert abs(np.mean([s.temperature for s in samples]) - 1.5) < 0.35
    cfg = replace(b2.preset_config("all2all-2k"), steps=400, equilibration_steps=100)
    rec, samples = b2.run_benchmark(cfg)
    assert rec.final_energy_drift_rel < 1e-4                  # test_acceptance.py:82-91 bound
    assert rec.rebuild_count == 0 and len(samples) == 8
    mom = np.array([s.total_momentum for s in samples])
    assert np.max(np.abs(mom)) < 1e-2


def test_config2_energy_drift_matches_the_reference_bound():
    """BASELINE config 2: N=65 536, rho=0.75, T0=1.2, rc=2.5, skin 0.3, dt=0.001,
    10^4 NVE steps with Hilbert reordering.  The fp64 reference drifts 1.29e-6 end
    to end (second-half max deviation 2.1e-7, 267 rebuilds).
    Stated bound for the fp32 / double-single engine: 1e-5 end to end, 5e-6 over the
    second half."""
    sim = lattice_sim(65_536, True, every=100)
    sim.run(10_000)
    e = np.array([s.total_energy for s in sim.samples])
    assert abs(e[-1] - e[0]) / abs(e[0]) <= 1e-5
    half = len(e) // 2
    assert np.max(np.abs(e[half:] - e[half])) / abs(e[0]) <= 5e-6
    assert 230 <= sim.rebuild_count <= 310
    assert 0.60 < sim.samples[-1].temperature < 0.68
    assert np.max(np.abs(np.array([s.total_momentum for s in sim.samples]))) < 0.05
    sim.close()


def test_orthorhombic_box_and_unequal_masses_track_the_oracle():
    """Non-cubic box, non-unit masses, particles crossing all three faces: the
    device loop follows the fp64 oracle loop (same initial state quantised to the
    device formats) sample by sample."""
    gen = np.random.default_rng(21)
    edges = np.array([13.0, 10.5, 9.2])
    n = 900
    # jittered simple-cubic start (no overlaps), hot enough to cross faces quickly
    g = np.stack(np.meshgrid(np.arange(10), np.arange(10), np.arange(9), indexing="ij"), -1)
    pos = (g.reshape(-1, 3)[:n] + 0.5) * (edges / np.array([10, 10, 9]))
    pos = quantize_f32(pos + gen.normal(scale=0.05, size=pos.shape))
    masses = quantize_f32(gen.uniform(0.5, 3.0, size=n))
    vel = quantize_f32(gen.normal(scale=1.5, size=(n, 3)) / np.sqrt(masses)[:, None])
    lj = b2.make_shifted(1.0, 1.0, 2.5)
    st = b2.ParticleState(pos, velocities=vel, masses=masses)
    sim = b2.Simulation(st, b2.SimBox(edges), lj, 0.002, force_mode=b2.TRUNCATED, skin=0.4,
                        sample_interval=20, sample_initial=True)
    sim.run(200)
    osim = orc.Sim(pos, vel, edges, lj.table(), 0.002, 0.4, masses=masses, sample_interval=20,
                   threads=orc.host_threads())
    osim.samples.insert(0, osim.measure())
    osim.run(200)
    assert len(sim.samples) == len(osim.samples) == 11
    for a, b in zip(sim.samples, osim.samples):
        assert a.potential_energy == pytest.approx(b["pe"], rel=5e-5, abs=1e-2)
        assert a.kinetic_energy == pytest.approx(b["ke"], rel=5e-5)
        assert np.allclose(a.total_momentum, b["momentum"], atol=5e-3)
    img = sim.state.images.acquire_read(b2.HOST)
    assert np.count_nonzero(img) > 20                       # faces were really crossed
    p = sim.state.positions.acquire_read(b2.HOST)
    unwrapped = p + img * edges
    d = unwrapped - (osim.pos + osim.images * edges)
    assert np.max(np.abs(d)) < 5e-3                         # trajectories still together
    sim.close()


@pytest.mark.parametrize("n", [4096, 262_144])
def test_velocity_upload_on_the_side_stream_changes_nothing(n):
    """Simulation() uploads velocities that are still on the host on a side stream and lets the
    runner wait for them behind the first list build (b2md_runner_config::vel_ready_event);
    a state whose velocities are already on the device takes the plain path.  Same bits."""
    out = []
    for presync in (False, True):
        st, box = b2.init_lattice_any(n, 0.75)
        b2.init_velocities(st, 1.2, 42)
        if presync:
            st.sync_to_compute()
        sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001,
                            force_mode=b2.TRUNCATED, skin=0.3, sample_interval=20,
                            sample_initial=True, reorder="hilbert")
        assert ("vel_ready" in sim._keep) == (not presync)
        sim.run(60)
        out.append((np.array([s.total_energy for s in sim.samples]),
                    np.array([s.kinetic_energy for s in sim.samples]),
                    np.array(st.positions.acquire_read(b2.HOST)),
                    np.array(st.velocities.acquire_read(b2.HOST))))
        sim.close()
    for a, b in zip(*out):
        assert np.array_equal(a, b)
