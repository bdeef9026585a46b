"""Native loop of the all-to-all force mode (`-m gpu`): b2md_run_all_pairs against the
operator-by-operator loop (bitwise), against the reference's own run in its default
force mode (tests/golden/all2all_trajectory.npz) and against the oracle."""
import numpy as np
import pytest

import paper_2406_04210_b200 as b2
from conftest import load_golden
from helpers import quantize_f32

pytestmark = pytest.mark.gpu


def golden_sim(G, tag, native):
    st = b2.ParticleState(G["pos0"], velocities=G["vel0"])
    box = b2.SimBox(G["edges"])
    thermostat = None
    if tag == "nvt":
        thermostat = b2.ThermostatParams(float(G["temperature"]), float(G["rate"]), int(G["seed"]))
    return b2.Simulation(st, box, b2.make_shifted(1.0, 1.0), float(G["dt"]), thermostat=thermostat,
                         sample_interval=int(G["every"]), sample_initial=True, native=native)


def host_state(sim):
    st = sim.state
    return [np.array(b.acquire_read(b2.HOST)) for b in
            (st.positions, st.velocities, st.images, st.forces, st.per_particle_potential,
             st.virial)]


@pytest.mark.parametrize("tag", ["nve", "nvt"])
def test_native_loop_is_bit_identical_to_the_operator_loop(tag):
    G = load_golden("all2all_trajectory")
    out = {}
    for native in (True, False):
        sim = golden_sim(G, tag, native)
        assert sim.native_all_pairs == native and not sim.native
        sim.run(130)                # not a multiple of the sample interval
        sim.run(70)
        out[native] = (host_state(sim), [(s.step, s.potential_energy, s.kinetic_energy)
                                          for s in sim.samples], sim.kernel_launches)
        sim.close()
    for a, b in zip(out[True][0], out[False][0]):
        assert np.array_equal(a, b)
    assert out[True][1] == out[False][1]
    # NVE: one launch per intermediate step (all pairs + finalize + integrate), and per call (a
    # call ends at each sample) the first integrate, the last force evaluation and its finalize;
    # NVT: all pairs, then finalize + thermostat + integrate in one pass -- two launches per
    # step -- plus the first integrate of every call
    assert out[True][2] == (200 + 2 * 11 if tag == "nve" else 2 * 200 + 11)


@pytest.mark.parametrize("tag", ["nve", "nvt"])
def test_native_loop_tracks_the_reference_run(tag):
    """The reference's own 200-step run in its default force mode: the first samples agree
    to fp32 accuracy, the series to the chaotic-divergence bound, NVE energy is conserved as
    well as the reference conserves it; the thermostat redraws the same particles at the same
    steps (streams are addressed by particle id and step)."""
    G = load_golden("all2all_trajectory")
    sim = golden_sim(G, tag, True)
    sim.run(int(G["steps"]))
    s = sim.samples
    assert [x.step for x in s] == list(G[tag + "_step"])
    pe = np.array([x.potential_energy for x in s])
    ke = np.array([x.kinetic_energy for x in s])
    gpe, gke = G[tag + "_pe"], G[tag + "_ke"]
    assert abs(pe[0] - gpe[0]) <= 2e-6 * abs(gpe[0])
    assert abs(ke[0] - gke[0]) <= 2e-6 * abs(gke[0])
    assert np.max(np.abs(pe - gpe)) <= 2e-3 * np.abs(gpe).max()
    assert np.max(np.abs(ke - gke)) <= 2e-3 * np.abs(gpe).max()
    if tag == "nve":
        e, ge = pe + ke, gpe + gke
        drift_ref = np.max(np.abs(ge - ge[0])) / abs(ge[0])
        assert np.max(np.abs(e - e[0])) / abs(e[0]) <= max(3.0 * drift_ref, 2e-5)
    pos = np.array(sim.state.positions.acquire_read(b2.HOST))
    d = pos - G[tag + "_pos_end"]
    d -= G["edges"] * np.rint(d / G["edges"])
    assert np.max(np.abs(d)) <= 5e-3
    sim.close()


def test_singular_pair_surfaces_through_the_native_loop():
    gen = np.random.default_rng(11)
    n, edge = 200, 8.0
    pos = quantize_f32(gen.uniform(0, edge, size=(n, 3)))
    vel = np.zeros((n, 3))
    # two particles that meet exactly after the first drift: equal and opposite velocities
    # (the pair potential is too weak to change an fp32 velocity)
    pos[17] = (1.0, 1.0, 1.0)
    pos[93] = (1.0 + 2.0 ** -4, 1.0, 1.0)
    vel[17, 0], vel[93, 0] = 1.0, -1.0
    st = b2.ParticleState(pos, velocities=vel)
    sim = b2.Simulation(st, b2.SimBox.cubic(edge), b2.make_shifted(1e-30, 0.5), 2.0 ** -5,
                        sample_interval=1000)
    with pytest.raises(b2.SingularPairError) as err:
        sim.run(3)
    assert (err.value.i, err.value.j) == (17, 93)
    sim.close()


# ---- the other shapes of the all-pairs kernel (chosen from n alone) ---------------------
def _all_pairs_vs_oracle(n, lj):
    """Untruncated potential: every particle sums n - 1 pair terms in fp32, so the bounds are
    the stated 1e-5 on the L2 error of the forces and, per particle, 1e-4 relative to the rms
    force / 2e-4 on energies and virial (measured at N = 12 500, profiles/exp/
    all_pairs_accuracy.py: L2 5.1e-7, M1 1.4e-5, M3 4.1e-5, energy 7.5e-5 -- the exact-fp32
    min-image kernel this one replaced: 3.6e-7, 1.4e-5, 2.1e-5, 7.5e-5)."""
    from helpers import fluid_state, force_error_metrics, scalar_rel_error
    from oracle import oracle as orc
    pos, _, edge = fluid_state(n, density=0.8, seed=5)
    pos = quantize_f32(pos)
    st = b2.ParticleState(pos)
    b2.compute_forces_all_to_all(st, lj, b2.SimBox.cubic(edge))
    rf, rpe, rw = orc.forces_all_pairs(pos, [edge] * 3, lj.table(), threads=orc.host_threads())
    f = np.array(st.forces.acquire_read(b2.HOST))
    m = force_error_metrics(f, rf)
    m["L2"] = float(np.linalg.norm(f - rf) / np.linalg.norm(rf))
    assert m["L2"] <= 1e-5 and m["M3"] <= 1e-4 and m["M1"] <= 1e-4, m
    assert scalar_rel_error(st.per_particle_potential.acquire_read(b2.HOST), rpe) <= 2e-4
    assert scalar_rel_error(st.virial.acquire_read(b2.HOST), rw) <= 2e-4
    return m


def test_four_warp_shape_matches_the_oracle():
    """12 288 <= N < 65 536: four warps per tile of 32 particles (fixed-point min-image)."""
    _all_pairs_vs_oracle(12500, b2.make_shifted(1.0, 1.0))


def test_one_thread_per_particle_shape_matches_the_list_kernels():
    """N >= 65 536: one thread per particle in blocks of 128.  The oracle's all-pairs scan
    takes minutes there; with a cutoff the all-pairs result must equal the neighbour-list
    result (itself pinned to the oracle at this size by test_gpu_bench_sizes.py) up to the
    fp32 summation order."""
    from helpers import fluid_state, force_error_metrics, scalar_rel_error
    n = 66000
    pos, _, edge = fluid_state(n, density=0.75, seed=9)
    pos = quantize_f32(pos)
    box = b2.SimBox.cubic(edge)
    lj = b2.make_shifted(1.0, 1.0, 2.5)
    a, b = b2.ParticleState(pos), b2.ParticleState(pos)
    b2.compute_forces_all_to_all(a, lj, box)
    grid = b2.bin_particles(b, box, 2.8)
    nl = b2.build_neighbor_list(b, grid, 2.8, 128, r_cut=2.5)
    assert not nl.overflow
    b2.compute_forces_truncated(b, lj, box, nl)
    fa, fb = a.forces.acquire_read(b2.HOST), b.forces.acquire_read(b2.HOST)
    m = force_error_metrics(fa, fb)
    m["L2"] = float(np.linalg.norm(np.array(fa) - np.array(fb)) / np.linalg.norm(fb))
    # (the jittered lattice has a few close contacts with forces of order 10^3: errors are
    # judged against the particle's own force, M1, and in the L2 norm)
    assert m["L2"] <= 1e-5 and m["M1"] <= 1e-5, m
    # energies / virial: per particle, against its own value plus the typical sum of the
    # magnitudes of its ~50 pair terms (a total near zero is a cancellation, not a scale)
    for name, scale in (("per_particle_potential", 10.0), ("virial", 100.0)):
        x = np.array(getattr(a, name).acquire_read(b2.HOST))
        y = np.array(getattr(b, name).acquire_read(b2.HOST))
        assert np.max(np.abs(x - y) / (np.abs(y) + scale)) <= 1e-5, name


def test_pair_table_loop_is_bit_identical_to_the_operator_loop():
    """Kob-Andersen tables through the all-to-all loop (table variants of the kernels,
    one-launch steps included)."""
    from helpers import fluid_state
    n = 700
    pos, vel, edge = fluid_state(n, density=1.2, temperature=0.8, seed=3, jitter=0.02)
    species = (np.random.default_rng(4).permutation(n) < n // 5).astype(np.int32)
    out = {}
    for native in (True, False):
        st = b2.ParticleState(quantize_f32(pos), velocities=quantize_f32(vel), species=species)
        sim = b2.Simulation(st, b2.SimBox.cubic(edge), b2.PairTable.kob_andersen(), 0.001,
                            sample_interval=25, native=native)
        sim.run(60)
        out[native] = host_state(sim) + [np.array([s.total_energy for s in sim.samples])]
        sim.close()
    for x, y in zip(out[True], out[False]):
        assert np.array_equal(x, y)
    e = out[True][-1]
    assert np.all(np.isfinite(e)) and np.max(np.abs(e - e[0])) <= 1e-3 * abs(e[0])      # (sane run)
