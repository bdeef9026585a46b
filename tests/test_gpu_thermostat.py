"""Andersen thermostat and counter-based streams on the device (`-m gpu`) against
the reference's golden vectors (tests/golden/thermostat.npz) and the oracle."""
import numpy as np
import pytest

import paper_2406_04210_b200 as b2
from paper_2406_04210_b200 import rng
from conftest import load_golden
from helpers import quantize_f32
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def test_stream_words_match_reference_vectors():
    G = load_golden("thermostat")
    assert np.array_equal(rng.raw_words(12345, 0, 7, 12), G["raw"])            # bit-exact
    assert np.array_equal(rng.uniforms(12345, 0, 7, 8, word_offset=3), G["uniforms"])
    got = rng.normals(12345, 1, 0, 9, word_offset=2)
    assert np.max(np.abs(got - G["normals"])) <= 4e-16 * np.max(np.abs(G["normals"]))
    # a long block: every uniform identical, normals to a few ulp, tails included
    n = 200_000
    assert np.array_equal(rng.uniforms(7, 0, 3, n), orc.stream_uniforms(7, 0, 3, n))
    z, zr = rng.normals(7, 0, 3, n), orc.stream_normals(7, 0, 3, n)
    assert np.max(np.abs(z - zr) / np.maximum(np.abs(zr), 1e-3)) <= 1e-14
    assert rng.raw_words(1, 2, 3, 0).size == 0


def test_andersen_thermostat_matches_reference():
    G = load_golden("thermostat")
    vel, masses = quantize_f32(G["vel"]), quantize_f32(G["masses"])
    params = b2.ThermostatParams(float(G["temperature"]), float(G["rate"]), int(G["seed"]))
    st = b2.ParticleState(np.zeros_like(vel), velocities=vel, masses=masses)
    count = b2.andersen_thermostat(st, params, float(G["dt"]), int(G["step"]))
    want_vel, redraw = orc.andersen_thermostat(vel, masses, params.temperature, params.rate,
                                               params.seed, float(G["dt"]), int(G["step"]))
    assert count == int(redraw.sum()) == int(G["count"])       # same particles selected
    got = st.velocities.acquire_read(b2.HOST)
    assert np.array_equal(got[~redraw], vel[~redraw])           # untouched rows bit-identical
    assert np.max(np.abs(got[redraw] - want_vel[redraw])
                  / np.maximum(np.abs(want_vel[redraw]), 1e-3)) <= 2e-7   # fp32 velocities
    # zero rate: nothing happens
    assert b2.andersen_thermostat(st, b2.ThermostatParams(1.0, 0.0, 1), 0.01, 5) == 0
    with pytest.raises(ValueError):
        b2.ThermostatParams(-1.0, 1.0, 0)


def test_thermostat_is_independent_of_device_row_order():
    """Streams are addressed by logical particle id: an internal Hilbert reorder
    must not change who is redrawn or what they receive."""
    gen = np.random.default_rng(3)
    n, edge = 4000, 17.0
    pos = gen.uniform(0, edge, size=(n, 3))
    vel = quantize_f32(gen.normal(size=(n, 3)))
    params = b2.ThermostatParams(0.9, 40.0, 1234)
    out = []
    for reorder in (False, True):
        st = b2.ParticleState(pos, velocities=vel)
        if reorder:
            b2.reorder_hilbert(st, b2.SimBox.cubic(edge), 2.8, internal=True)
        c = b2.andersen_thermostat(st, params, 0.005, 77)
        out.append((c, np.array(st.velocities.acquire_read(b2.HOST))))
    assert out[0][0] == out[1][0] > 0
    assert np.array_equal(out[0][1], out[1][1])


def test_thermostatted_simulation_holds_the_target_temperature():
    # test_acceptance.py:123-136 analogue: mean T within a few standard errors
    st, box = b2.init_lattice_any(4000, 0.75)
    b2.init_velocities(st, 1.5, 42)
    thermo = b2.ThermostatParams(temperature=1.5, rate=20.0, seed=7)
    sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.002, force_mode=b2.TRUNCATED,
                        skin=0.3, thermostat=thermo, sample_interval=10)
    assert sim.native                  # the thermostat runs inside the native step loop
    sim.run(1500)
    temps = np.array([s.temperature for s in sim.samples[50:]])
    assert abs(temps.mean() - 1.5) < 0.03
    sim.close()


@pytest.mark.parametrize("n,pair_rows", [(4000, False), (4000, True)])
def test_native_thermostat_loop_equals_the_operator_loop_bitwise(n, pair_rows):
    """sim.py:86-87,100-102: the thermostat is the second finalize slot, called with
    SignalEngine.step_count.  The native runner (integrate / force / finalize / andersen
    launched from C++) and the signal/slot loop calling the same operators one by one must
    produce the same bits: same redraw decisions (Philox words indexed by step and logical
    particle id), same rebuild steps, same samples -- across calls that split the run and
    across the stride growth of the first build."""
    out = []
    for native in (False, True):
        st, box = b2.init_lattice_any(n, 0.75)
        b2.init_velocities(st, 1.5, 42)
        thermo = b2.ThermostatParams(temperature=1.5, rate=20.0, seed=7)
        sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.002,
                            force_mode=b2.TRUNCATED, skin=0.3, thermostat=thermo,
                            sample_interval=25, native=native, pair_rows=pair_rows,
                            reorder=None)      # (a reorder changes the summation order, and
        # the in-loop fp32 displacement test may fire one step before the exact fp64 one)
        assert sim.native == native
        sim.run(60)
        sim.run(41)                    # step numbers continue across calls
        out.append((np.array(st.velocities.acquire_read(b2.HOST)),
                    np.array(st.positions.acquire_read(b2.HOST)),
                    [(s.step, s.total_energy, s.temperature) for s in sim.samples],
                    sim.rebuild_count))
        if native:
            assert sim.nlist_seconds > 0.0 and sim.force_seconds > 0.0
        sim.close()
    assert abs(out[0][3] - out[1][3]) <= 1 and out[0][3] >= 2
    assert out[0][2] == out[1][2] and len(out[0][2]) == 4
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
