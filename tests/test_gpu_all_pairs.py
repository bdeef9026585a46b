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
