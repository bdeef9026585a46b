"""Pin the CPU oracle bit-for-bit against vectors produced by the real reference
(tests/golden/make_golden.py).  CPU-only; no GPU, no /root/reference at run time."""
import numpy as np
import pytest

from conftest import load_golden, unragged
from oracle import oracle as orc


# ---------------------------------------------------------------- cells/lists
NB = load_golden("neighbor")
NB_NAMES = [str(x) for x in NB["names"]]


@pytest.mark.parametrize("name", NB_NAMES)
def test_binning_bit_exact(name):
    g = orc.bin_particles(NB[f"{name}.pos"], NB[f"{name}.edges"], float(NB[f"{name}.r_list"]))
    assert np.array_equal(g.cells_per_axis, NB[f"{name}.ncells"])
    assert np.array_equal(g.cell_edge, NB[f"{name}.cell_edge"])
    assert np.array_equal(g.cell_of_particle, NB[f"{name}.cell_of"])
    assert np.array_equal(g.cell_start, NB[f"{name}.cell_start"])
    assert np.array_equal(g.cell_particles, NB[f"{name}.cell_particles"])
    assert g.fallback == bool(NB[f"{name}.fallback"])


@pytest.mark.parametrize("name", NB_NAMES)
@pytest.mark.parametrize("threads", [1, 3])
def test_neighbor_rows_bit_exact(name, threads):
    pos, edges = NB[f"{name}.pos"], NB[f"{name}.edges"]
    r_list, stride = float(NB[f"{name}.r_list"]), int(NB[f"{name}.stride"])
    g = orc.bin_particles(pos, edges, r_list)
    nl = orc.build_neighbor_list(pos, np.zeros_like(pos, dtype=np.int64), g,
                                 r_list, stride, threads=threads)
    assert nl.overflow == bool(NB[f"{name}.overflow"])
    assert np.array_equal(nl.counts, NB[f"{name}.counts"])
    want = unragged(NB[f"{name}.counts"], NB[f"{name}.rows"], stride)
    for i in range(pos.shape[0]):
        c = nl.counts[i]
        assert np.array_equal(nl.indices[i, :c], want[i, :c]), (name, i)
    assert np.array_equal(nl.positions_at_build, NB[f"{name}.at_build"])


@pytest.mark.parametrize("name", NB_NAMES)
def test_reorder_permutation(name):
    assert np.array_equal(orc.reorder_permutation(NB[f"{name}.cell_of"]), NB[f"{name}.perm"])


def test_pair_sets_match_bruteforce():
    for name in ("cube0", "cube3", "fallback"):
        pos, edges = NB[f"{name}.pos"], NB[f"{name}.edges"]
        want = unragged(NB[f"{name}.counts"], NB[f"{name}.rows"])
        assert orc.pair_set(want, NB[f"{name}.counts"]) == \
            orc.pairs_within(pos, edges, float(NB[f"{name}.r_list"]))


def test_top_boundary_clamp():
    x = np.nextafter(9.0, 0.0)
    g = orc.bin_particles(np.array([[x, x, x]]), [9.0] * 3, 3.0)
    assert np.array_equal(g.cell_of_particle, NB["clamp.cell_of"])
    assert np.array_equal(g.cell_start, NB["clamp.cell_start"])


# -------------------------------------------------------------------- rebuild
def test_rebuild_criterion():
    G = load_golden("rebuild")
    for tag in [str(t) for t in G["tags"]]:
        nl = orc.NList(None, None, 0, False, None, float(G[f"{tag}.r_list"]),
                       float(G[f"{tag}.r_cut"]), G[f"{tag}.at_build"])
        got = orc.needs_rebuild(G[f"{tag}.pos"], G[f"{tag}.img"], G["edges"], nl)
        assert got == bool(G[f"{tag}.answer"]), tag


# --------------------------------------------------------------------- forces
FO = load_golden("forces")


def _table():
    eps, sig, rc, shift = FO["lj"]
    tab = orc.pair_table(eps, sig, rc)
    assert tab[0, 3] == shift == FO["shift_2p5"]
    assert tab[0, 3] == pytest.approx(0.016316891136, abs=1e-12)
    return tab


@pytest.mark.parametrize("seed", range(50, 55))
def test_truncated_forces_bit_exact(seed):
    k = f"trunc{seed}"
    pos, edge = FO[f"{k}.pos"], float(FO[f"{k}.edge"])
    edges = [edge] * 3
    g = orc.bin_particles(pos, edges, 3.0)
    nl = orc.build_neighbor_list(pos, np.zeros((len(pos), 3), np.int64), g, 3.0, 256, r_cut=2.5)
    assert np.array_equal(nl.counts, FO[f"{k}.counts"])
    f, pe, w = orc.forces_truncated(pos, edges, _table(), nl, threads=2)
    assert np.array_equal(f, FO[f"{k}.forces"])
    assert np.array_equal(pe, FO[f"{k}.pe"])
    # independent expression tree agrees to rounding (bruteforce.py)
    bf, bpe, bw = orc.forces_bruteforce_numpy(pos, edges, _table())
    assert np.array_equal(bf, FO[f"{k}.brute_forces"])
    assert np.array_equal(bpe, FO[f"{k}.brute_pe"])
    assert np.allclose(w, bw, rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("seed", range(2))
def test_all_pairs_forces_bit_exact(seed):
    k = f"all{seed}"
    f, pe, _ = orc.forces_all_pairs(FO[f"{k}.pos"], [float(FO[f"{k}.edge"])] * 3, _table())
    assert np.array_equal(f, FO[f"{k}.forces"])
    assert np.array_equal(pe, FO[f"{k}.pe"])


def test_cutoff_straddle_bit_exact():
    f, pe, _ = orc.forces_all_pairs(FO["straddle.pos"], [20.0] * 3, _table())
    assert np.array_equal(f, FO["straddle.forces"])
    assert np.array_equal(pe, FO["straddle.pe"])


def test_singular_pair_indices():
    with pytest.raises(orc.SingularPair) as exc:
        orc.forces_all_pairs(FO["singular.pos"], [10.0] * 3, _table())
    assert [exc.value.i, exc.value.j] == list(FO["singular.ij"])


def test_single_type_table_equals_two_identical_types():
    # pair-table extension: a 2-type table with identical rows and arbitrary
    # species labels reproduces the pinned single-type result bit for bit
    k = "trunc50"
    pos, edges = FO[f"{k}.pos"], [float(FO[f"{k}.edge"])] * 3
    g = orc.bin_particles(pos, edges, 3.0)
    nl = orc.build_neighbor_list(pos, np.zeros((len(pos), 3), np.int64), g, 3.0, 256, r_cut=2.5)
    tab2 = orc.pair_table(np.ones((2, 2)), np.ones((2, 2)), np.full((2, 2), 2.5))
    species = np.random.default_rng(1).integers(0, 2, size=len(pos)).astype(np.int32)
    f, pe, _ = orc.forces_truncated(pos, edges, tab2, nl, species=species)
    assert np.array_equal(f, FO[f"{k}.forces"])
    assert np.array_equal(pe, FO[f"{k}.pe"])


# ------------------------------------------------------------------ integrate
def test_integrate_finalize_bit_exact():
    G = load_golden("integrate")
    p1, i1, v1 = orc.vv_integrate(G["pos"], G["img"], G["vel"], G["forces"],
                                  G["masses"], G["edges"], float(G["dt"]))
    assert np.array_equal(p1, G["pos1"])
    assert np.array_equal(i1, G["img1"])
    assert np.array_equal(v1, G["vel1"])
    v2 = orc.vv_finalize(v1, G["forces2"], G["masses"], float(G["dt"]))
    assert np.array_equal(v2, G["vel2"])
    # the C kernels used by the timed CPU baseline do the same arithmetic
    import ctypes
    L = orc.lib()
    vel = np.array(G["vel"]); pos = np.array(G["pos"]); img = np.array(G["img"])
    f = np.ascontiguousarray(G["forces"]); m = np.ascontiguousarray(G["masses"])
    e = np.ascontiguousarray(G["edges"])
    dp = lambda a, t: a.ctypes.data_as(ctypes.POINTER(t))
    L.orc_vv_kick(ctypes.c_int64(len(m)), dp(vel, ctypes.c_double), dp(f, ctypes.c_double),
                  dp(m, ctypes.c_double), ctypes.c_double(float(G["dt"])), ctypes.c_int(2))
    L.orc_vv_drift_wrap(ctypes.c_int64(len(m)), dp(pos, ctypes.c_double), dp(img, ctypes.c_int64),
                        dp(vel, ctypes.c_double), dp(e, ctypes.c_double),
                        ctypes.c_double(float(G["dt"])), ctypes.c_int(2))
    assert np.array_equal(vel, G["vel1"])
    assert np.array_equal(pos, G["pos1"])
    assert np.array_equal(img, G["img1"])


def test_wrap_and_minimum_image_edge_cases():
    G = load_golden("integrate")
    w, k = orc.wrap_position(G["wrap_in"], G["wrap_img"], [10.0] * 3)
    assert np.array_equal(w, G["wrap_out"])
    assert np.array_equal(k, G["wrap_img_out"])
    assert np.array_equal(orc.minimum_image(G["mi_in"], [10.0] * 3), G["mi_out"])


# ---------------------------------------------------------------- observables
def test_deterministic_sum_bit_exact():
    G = load_golden("observables")
    for size, want, fast in zip(G["sizes"], G["sums"], G["fast"]):
        assert orc.reduce_sum(G["values"][:size]) == want, size
        assert orc.reduce_sum(G["values"][:size], deterministic=False) == fast
    assert orc.reduce_sum(np.zeros(0)) == 0.0


def test_thermo_scalars():
    G = load_golden("observables")
    t = orc.thermo(G["vel"], G["masses"], G["pe_in"])
    assert t["pe"] == float(G["pe"])
    assert np.array_equal(t["momentum"], G["momentum"])
    # einsum's row product may group differently: agree to 1 ulp-level
    assert t["ke"] == pytest.approx(float(G["ke"]), rel=1e-15)
    assert t["temperature"] == pytest.approx(float(G["temperature"]), rel=1e-15)


# ----------------------------------------------------------------- trajectory
def test_lattice_generator_bit_exact():
    G = load_golden("trajectory")
    pos, edge = orc.fcc_lattice(int(G["n"]), float(G["density"]))
    assert np.array_equal(pos, G["pos0"])
    assert np.array_equal(np.full(3, edge), G["edges"])
    pos, edge = orc.fcc_lattice(256, 0.8)
    assert np.array_equal(pos, G["lat256"])


def test_nve_trajectory_bit_exact():
    """300 NVE steps from the reference's own initial state: every sample of the
    oracle loop (energies, momentum, rebuild count) equals the reference's."""
    G = load_golden("trajectory")
    sim = orc.Sim(G["pos0"], G["vel0"], G["edges"], orc.pair_table(1.0, 1.0, 2.5),
                  float(G["dt"]), float(G["skin"]), sample_interval=int(G["every"]),
                  threads=2)
    sim.samples.append(sim.measure())   # sample_initial=True in the golden run
    sim.run(int(G["steps"]))
    s = sim.samples
    assert [x["step"] for x in s] == list(G["step"])
    assert np.array_equal([x["pe"] for x in s], G["pe"])
    assert np.array_equal([x["ke"] for x in s], G["ke"]) or \
        np.allclose([x["ke"] for x in s], G["ke"], rtol=1e-15, atol=0)
    assert np.array_equal(np.array([x["momentum"] for x in s]), G["momentum"])
    assert [x["rebuild_count"] for x in s] == list(G["rebuilds"])
    assert np.array_equal(sim.pos, G["pos_end"])
    assert np.array_equal(sim.vel, G["vel_end"])
    assert np.array_equal(sim.images, G["img_end"])
    assert np.array_equal(sim.forces, G["forces_end"])
    assert sim.stride == int(G["stride_end"])


def _oracle_all2all_run(G, rate):
    """Simulation.run in all_to_all mode (sim.py:62-102) restated with the oracle's
    operators: integrate -> all-pairs forces -> finalize [-> thermostat]."""
    n = int(G["n"])
    edges, dt = G["edges"], float(G["dt"])
    table = orc.pair_table(1.0, 1.0, np.inf)
    masses = np.ones(n)
    pos, vel = G["pos0"].copy(), G["vel0"].copy()
    images = np.zeros((n, 3), np.int64)
    f, pe, _ = orc.forces_all_pairs(pos, edges, table, threads=2)
    samples = []

    def sample(step):
        t = orc.thermo(vel, masses, pe)
        samples.append((step, t["pe"], t["ke"], t["momentum"]))
    sample(0)
    for step in range(int(G["steps"])):
        pos, images, vel = orc.vv_integrate(pos, images, vel, f, masses, edges, dt)
        f, pe, _ = orc.forces_all_pairs(pos, edges, table, threads=2)
        vel = orc.vv_finalize(vel, f, masses, dt)
        if rate:
            vel, _ = orc.andersen_thermostat(vel, masses, float(G["temperature"]), rate,
                                             int(G["seed"]), dt, step)
        if (step + 1) % int(G["every"]) == 0:
            sample(step + 1)
    return samples, pos, vel, f


@pytest.mark.parametrize("tag", ["nve", "nvt"])
def test_all_to_all_loop_bit_exact(tag):
    """The reference's default force mode, NVE and with the Andersen thermostat as second
    finalize slot: every sample and the end state of the oracle loop equal the reference's."""
    G = load_golden("all2all_trajectory")
    samples, pos, vel, f = _oracle_all2all_run(G, float(G["rate"]) if tag == "nvt" else 0.0)
    assert [x[0] for x in samples] == list(G[tag + "_step"])
    assert np.array_equal([x[1] for x in samples], G[tag + "_pe"])
    assert np.allclose([x[2] for x in samples], G[tag + "_ke"], rtol=1e-15, atol=0)
    assert np.array_equal(np.array([x[3] for x in samples]), G[tag + "_momentum"])
    assert np.array_equal(pos, G[tag + "_pos_end"])
    assert np.array_equal(vel, G[tag + "_vel_end"])
    assert np.array_equal(f, G[tag + "_forces_end"])


# ----------------------------------------------------------- rng / thermostat
def test_random_streams_and_thermostat_bit_exact():
    G = load_golden("thermostat")
    assert np.array_equal(orc.stream_raw(12345, 0, 7, 12), G["raw"])
    assert np.array_equal(orc.stream_uniforms(12345, 0, 7, 8, word_offset=3), G["uniforms"])
    assert np.array_equal(orc.stream_normals(12345, 1, 0, 9, word_offset=2), G["normals"])
    vel, redraw = orc.andersen_thermostat(G["vel"], G["masses"], float(G["temperature"]),
                                          float(G["rate"]), int(G["seed"]), float(G["dt"]),
                                          int(G["step"]))
    assert int(redraw.sum()) == int(G["count"])
    assert np.array_equal(vel, G["vel_after"])
