"""GPU parity tests (run on the B200 with `-m gpu`): every operator of the hot
path is called through the reference-shaped Python API -> ctypes -> libb2md.so and
compared with the CPU oracle on identical inputs.

Bar: bit-exact for integer-valued results (cells, CSR arrays, neighbour rows,
permutations, image counters, rebuild decision, fp64 tree sums); stated
tolerances for fp32 pair arithmetic (forces/energies/virial, 1e-5) and for the
double-single integrator.
"""
import numpy as np
import pytest

import paper_2406_04210_b200 as b2
from conftest import load_golden, unragged
from helpers import (backward_error, fluid_state, force_error_metrics, quantize_ds,
                     quantize_f32, scalar_rel_error)
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

NB = load_golden("neighbor")
NB_NAMES = [str(x) for x in NB["names"]]


def make_state(pos, **kw):
    return b2.ParticleState(pos, **kw)


# ------------------------------------------------------------ residency / formats
def test_state_round_trip_is_exact_for_device_formats():
    gen = np.random.default_rng(5)
    n = 1000
    pos = quantize_ds(gen.uniform(0, 50.0, size=(n, 3)))
    vel = quantize_f32(gen.normal(size=(n, 3)))
    masses = quantize_f32(gen.uniform(0.5, 2.0, size=n))
    img = gen.integers(-5, 6, size=(n, 3))
    species = gen.integers(0, 3, size=n).astype(np.int32)
    st = make_state(pos, velocities=vel, masses=masses, images=img, species=species)
    for name, want in [("positions", pos), ("velocities", vel), ("masses", masses),
                       ("images", img), ("species", species)]:
        buf = getattr(st, name)
        view = buf.acquire_read(b2.COMPUTE)          # host -> device conversion
        assert buf.valid_on == "both" and buf.copy_count == 1
        assert np.array_equal(view.to_numpy(), want), name
        buf.acquire_write(b2.COMPUTE)                # pretend a kernel wrote it
        assert buf.valid_on == b2.COMPUTE
        assert np.array_equal(buf.acquire_read(b2.HOST), want), name   # device -> host
        assert buf.copy_count == 2
        buf.acquire_read(b2.HOST)
        assert buf.copy_count == 2                   # no redundant transfer


def test_full_precision_positions_round_to_double_single():
    gen = np.random.default_rng(6)
    pos = gen.uniform(0, 100.0, size=(500, 3))
    st = make_state(pos)
    got = st.positions.acquire_read(b2.COMPUTE).to_numpy()
    assert np.array_equal(got, quantize_ds(pos))
    assert np.max(np.abs(got - pos)) < 100.0 * 2.0 ** -47


# ------------------------------------------------------------------- cells
@pytest.mark.parametrize("name", NB_NAMES)
def test_binning_bit_exact(name):
    pos = quantize_ds(NB[f"{name}.pos"])
    edges, r_list = NB[f"{name}.edges"], float(NB[f"{name}.r_list"])
    want = orc.bin_particles(pos, edges, r_list)
    grid = b2.bin_particles(make_state(pos), b2.SimBox(edges), r_list)
    assert np.array_equal(grid.cells_per_axis, want.cells_per_axis)
    assert np.array_equal(grid.cell_edge, want.cell_edge)
    assert grid.fallback == want.fallback
    assert np.array_equal(grid.cell_of_particle, want.cell_of_particle)
    assert np.array_equal(grid.cell_start, want.cell_start)
    assert np.array_equal(grid.cell_particles, want.cell_particles)
    assert grid.occupancy_counts().sum() == pos.shape[0]


def test_binning_clamps_top_boundary():
    # test_neighbor.py:58-66
    x = float(np.float32(np.nextafter(np.float32(9.0), np.float32(0.0))))
    grid = b2.bin_particles(make_state(np.array([[x, x, x]])), b2.SimBox.cubic(9.0), 3.0)
    assert grid.cell_of_particle[0] == grid.n_cells - 1
    assert grid.cell_start[-1] == 1
    # a high word equal to L (position just below L in fp64) must clamp too
    y = np.nextafter(9.0, 0.0)
    grid = b2.bin_particles(make_state(np.array([[y, y, y]])), b2.SimBox.cubic(9.0), 3.0)
    assert grid.cell_of_particle[0] == grid.n_cells - 1


def test_binning_large_random_bit_exact():
    gen = np.random.default_rng(11)
    n, edge = 200_000, 64.37
    pos = quantize_ds(gen.uniform(0, edge, size=(n, 3)))
    want = orc.bin_particles(pos, [edge] * 3, 2.8)
    grid = b2.bin_particles(make_state(pos), b2.SimBox.cubic(edge), 2.8)
    assert np.array_equal(grid.cell_of_particle, want.cell_of_particle)
    assert np.array_equal(grid.cell_start, want.cell_start)
    assert np.array_equal(grid.cell_particles, want.cell_particles)


# ------------------------------------------------------------------- lists
def build_both(pos, edges, r_list, stride, r_cut=None):
    box = b2.SimBox(edges)
    st = make_state(pos)
    grid = b2.bin_particles(st, box, r_list)
    nl = b2.build_neighbor_list(st, grid, r_list, stride, r_cut=r_cut)
    og = orc.bin_particles(pos, edges, r_list)
    onl = orc.build_neighbor_list(pos, np.zeros_like(pos, dtype=np.int64), og, r_list, stride,
                                  r_cut=r_cut, threads=orc.host_threads())
    return st, box, nl, onl


def assert_rows_equal(nl, onl):
    assert nl.overflow == onl.overflow
    cnt = nl.counts
    assert np.array_equal(cnt, onl.counts)
    idx = nl.indices
    width = onl.indices.shape[1]
    mask = np.arange(width)[None, :] < cnt[:, None]
    assert np.array_equal(np.where(mask, idx[:, :width], 0), np.where(mask, onl.indices, 0))


@pytest.mark.parametrize("name", NB_NAMES)
def test_neighbor_rows_bit_exact_on_reference_fixtures(name):
    pos = quantize_ds(NB[f"{name}.pos"])
    st, box, nl, onl = build_both(pos, NB[f"{name}.edges"], float(NB[f"{name}.r_list"]),
                                  int(NB[f"{name}.stride"]))
    assert_rows_equal(nl, onl)
    assert np.array_equal(nl.positions_at_build, onl.positions_at_build)
    assert nl.rebuild_count == 1
    if not onl.overflow and pos.shape[0] <= 400:
        assert nl.pair_set() == orc.pairs_within(pos, NB[f"{name}.edges"],
                                                 float(NB[f"{name}.r_list"]))
    # most fixtures survive the quantisation unchanged: compare with the
    # reference's own rows where they do
    want = unragged(NB[f"{name}.counts"], NB[f"{name}.rows"], int(NB[f"{name}.stride"]))
    if np.array_equal(onl.counts, NB[f"{name}.counts"]):
        mask = np.arange(want.shape[1])[None, :] < onl.counts[:, None]
        assert np.array_equal(np.where(mask, nl.indices[:, :want.shape[1]], 0),
                              np.where(mask, want, 0))


def test_neighbor_overflow_is_flagged_not_truncated():
    # test_neighbor.py:126-136
    pos = quantize_ds(NB["overflow.pos"])
    st, box, small, osmall = build_both(pos, NB["overflow.edges"], 3.0, 4)
    assert small.overflow and np.all(small.counts <= 4)
    assert small.max_count > 4
    st, box, big, obig = build_both(pos, NB["overflow.edges"], 3.0, 512)
    assert not big.overflow and big.counts.max() == small.max_count
    lj = b2.make_shifted(1.0, 1.0, 2.5)
    with pytest.raises(b2.NeighborOverflowError):
        b2.compute_forces_truncated(st, lj, box, small)


def test_neighbor_build_validation():
    # test_neighbor.py:139-146
    box = b2.SimBox.cubic(8.0)
    st = make_state(np.random.default_rng(7).uniform(0, 8.0, size=(10, 3)))
    grid = b2.bin_particles(st, box, 2.0)
    with pytest.raises(b2.ConfigError):
        b2.build_neighbor_list(st, grid, 2.0, 0)
    with pytest.raises(ValueError):
        b2.build_neighbor_list(st, grid, 2.0, 8, r_cut=2.5)
    first = b2.build_neighbor_list(st, grid, 2.0, 64)
    second = b2.build_neighbor_list(st, grid, 2.0, 64, prev=first)
    assert (first.rebuild_count, second.rebuild_count) == (1, 2)


@pytest.mark.parametrize("n,seed", [(4096, 1), (30_000, 2)])
def test_neighbor_rows_bit_exact_fluid(n, seed):
    """config-1-like fluid states: rows identical to the oracle's, symmetric."""
    pos, _, edge = fluid_state(n, seed=seed)
    pos = quantize_ds(pos)
    st, box, nl, onl = build_both(pos, [edge] * 3, 2.8, 128, r_cut=2.5)
    assert_rows_equal(nl, onl)
    # symmetry: i in row(j) for every j in row(i)
    idx, cnt = nl.indices, nl.counts
    rows = [set(idx[i, :cnt[i]].tolist()) for i in range(n)]
    for i in range(0, n, max(n // 500, 1)):
        for j in rows[i]:
            assert i in rows[j]


def test_neighbor_decisions_at_the_listing_radius():
    """Pairs placed within a few ulp of r_list: the fp32 pre-test must defer to
    the exact fp64 decision (strict r2 < rl2)."""
    r_list = 2.8
    base = np.array([20.0, 2.0, 20.0])
    offs = r_list + np.array([-3e-15, -2e-13, 0.0, 2e-13, 3e-15, -1e-7, 1e-7, -1e-5, 1e-5])
    pos = []
    for k, d in enumerate(offs):
        origin = base + np.array([0.0, 6.0 * k, 0.0])
        pos.append(origin)
        pos.append(origin + np.array([d, 0.0, 0.0]))
    # fill the rest of the box sparsely so the grid has >= 3 cells per axis
    pos = quantize_ds(np.array(pos))
    edges = [64.0, 64.0, 64.0]
    st, box, nl, onl = build_both(pos, edges, r_list, 16)
    assert_rows_equal(nl, onl)
    assert nl.pair_set() == orc.pairs_within(pos, edges, r_list)


# ----------------------------------------------------------------- rebuild
def test_rebuild_criterion_matches_reference_cases():
    G = load_golden("rebuild")
    for tag in [str(t) for t in G["tags"]]:
        edges = G["edges"]
        box = b2.SimBox(edges)
        r_list, r_cut = float(G[f"{tag}.r_list"]), float(G[f"{tag}.r_cut"])
        # build the list at the snapshot, then move to the probe configuration
        at = G[f"{tag}.at_build"]
        w, k = orc.wrap_position(at, np.zeros_like(at, dtype=np.int64), edges)
        st = make_state(w, images=k)
        grid = b2.bin_particles(st, box, r_list)
        nl = b2.build_neighbor_list(st, grid, r_list, 256, r_cut=r_cut)
        assert np.array_equal(nl.positions_at_build, quantize_ds(w) + k * edges)
        st.positions.acquire_write(b2.HOST)[...] = G[f"{tag}.pos"]
        st.images.acquire_write(b2.HOST)[...] = G[f"{tag}.img"]
        pos_q = quantize_ds(G[f"{tag}.pos"])
        onl = orc.NList(None, None, 0, False, None, r_list, r_cut, nl.positions_at_build)
        want = orc.needs_rebuild(pos_q, G[f"{tag}.img"], edges, onl)
        assert b2.needs_rebuild(st, box, nl) == want, tag
        assert b2.max_displacement_sq(st, box, nl) == orc.max_displacement_sq(
            pos_q, G[f"{tag}.img"], edges, nl.positions_at_build), tag
        if tag != "exact_half_skin" and tag != "just_over":
            assert want == bool(G[f"{tag}.answer"]), tag


# ----------------------------------------------------------------- reorder
def test_reorder_by_cell_permutes_all_arrays_bitwise():
    # test_neighbor.py:218-238
    gen = np.random.default_rng(10)
    n = 150
    pos = quantize_ds(gen.uniform(0.0, 8.0, size=(n, 3)))
    vel = quantize_f32(gen.normal(size=(n, 3)))
    masses = quantize_f32(gen.uniform(0.5, 2.0, size=n))
    box = b2.SimBox.cubic(8.0)
    st = make_state(pos, velocities=vel, masses=masses,
                    images=gen.integers(-2, 3, size=(n, 3)),
                    species=gen.integers(0, 2, size=n).astype(np.int32))
    b2.compute_forces_all_to_all(st, b2.make_shifted(1.0, 1.0, 2.5), box)
    before = {k: np.array(buf.acquire_read(b2.HOST)) for k, buf in st.buffers().items()}
    grid = b2.bin_particles(st, box, 3.0)
    cells = grid.cell_of_particle
    perm = b2.reorder_by_cell(st, grid)
    assert np.array_equal(perm, orc.reorder_permutation(cells))
    assert np.all(np.diff(cells[perm]) >= 0)
    for k, buf in st.buffers().items():
        assert np.array_equal(buf.acquire_read(b2.HOST), before[k][perm]), k


@pytest.mark.parametrize("sub_bits", [0, 2, 7])
def test_hilbert_keys_and_sort_bit_exact(sub_bits):
    gen = np.random.default_rng(12)
    n, edge, r_list = 50_000, 37.3, 2.8
    pos = quantize_ds(gen.uniform(0, edge, size=(n, 3)))
    st = make_state(pos)
    box = b2.SimBox.cubic(edge)
    keys, key_bits = b2.hilbert_keys(st, box, r_list, sub_bits)
    keys = keys.cpu().numpy().astype(np.uint64)
    want_perm, want_keys = orc.hilbert_permutation(pos, [edge] * 3, r_list, sub_bits)
    assert key_bits == 3 * (4 + sub_bits)          # 13 cells per axis -> 4 bits
    assert np.array_equal(keys, want_keys)
    perm = b2.reorder_hilbert(st, box, r_list, sub_bits, internal=True)
    assert np.array_equal(perm, want_perm)         # stable: ties keep index order
    # rows moved, logical (host) view unchanged
    assert np.array_equal(st.particle_ids(), want_perm.astype(np.int32))
    assert np.array_equal(st.positions.acquire_read(b2.COMPUTE).to_numpy(), pos)
    # the key is cell-aligned: after the sort every cell's particles are contiguous rows
    grid = b2.bin_particles(st, box, r_list)
    cells = grid.cell_of_particle
    changes = np.count_nonzero(np.diff(cells) != 0)
    assert changes == np.unique(cells).size - 1
    start, parts = grid.cell_start, grid.cell_particles
    occupied = np.flatnonzero(np.diff(start) > 0)
    for c in occupied[:: max(len(occupied) // 200, 1)]:
        rows = parts[start[c]:start[c + 1]]
        assert np.array_equal(rows, np.arange(rows[0], rows[0] + rows.size))


def test_hilbert_curve_is_a_space_filling_walk():
    """Property of the key function itself: consecutive keys of a full 2^b grid
    are face neighbours (unit step in exactly one axis)."""
    bits = 3
    ax = np.arange(1 << bits)
    q = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), axis=-1).reshape(-1, 3)
    keys = orc.hilbert_keys(q.astype(np.uint64), bits)
    assert sorted(keys.tolist()) == list(range(q.shape[0]))
    walk = q[np.argsort(keys)]
    assert np.all(np.abs(np.diff(walk, axis=0)).sum(axis=1) == 1)
    # and the device computes the same keys for cell-centre positions (8 cells of
    # edge 1 per axis, no sub-cell bits)
    pos = q + 0.5
    got, key_bits = b2.hilbert_keys(make_state(pos), b2.SimBox.cubic(8.0), 1.0, 0)
    assert key_bits == 9
    assert np.array_equal(got.cpu().numpy().astype(np.uint64), keys)


# ------------------------------------------------------------------ forces
FORCE_TOL = 1e-5      # stated fp32 tolerance (BASELINE.json north_star)


def check_forces(pos, edges, params, r_list, species=None, stride=256):
    """GPU truncated forces vs the fp64 oracle on fp32-representable positions."""
    box = b2.SimBox(edges)
    st = make_state(pos, species=species)
    grid = b2.bin_particles(st, box, r_list)
    nl = b2.build_neighbor_list(st, grid, r_list, stride, r_cut=params.max_r_cut)
    assert not nl.overflow
    og = orc.bin_particles(pos, edges, r_list)
    onl = orc.build_neighbor_list(pos, np.zeros_like(pos, dtype=np.int64), og, r_list, stride,
                                  r_cut=params.max_r_cut, threads=orc.host_threads())
    table = params.table()
    rf, rpe, rw = orc.forces_truncated(pos, edges, table, onl, species=species,
                                       threads=orc.host_threads())
    # Stated metric: absolute error of each per-particle
    # quantity relative to the sum of the magnitudes of its pair terms (backward-
    # error scale), plus the rms-force scale for the force vector.
    fs, us, ws = orc.pair_scales(pos, edges, table, onl, species=species,
                                 threads=orc.host_threads())
    # both force kernels: thread (or sub-warp) per particle over the list itself,
    # and thread per particle pair over the merged rows
    for pair_rows in (True, False):
        b2.compute_forces_truncated(st, params, box, nl, pair_rows=pair_rows)
        f = st.forces.acquire_read(b2.HOST)
        pe = st.per_particle_potential.acquire_read(b2.HOST)
        w = st.virial.acquire_read(b2.HOST)
        m = force_error_metrics(f, rf, fs)
        assert m["M2"] <= FORCE_TOL, m      # error / sum_j |f_ij|  (the stated per-particle metric)
        assert np.linalg.norm(f - rf) <= FORCE_TOL * np.linalg.norm(rf)   # relative L2 error
        # per-particle error against the NET force (cancellation-sensitive: the net force
        # can be 100x smaller than the pair terms it is the sum of) -- looser bound
        assert m["M1"] <= 1e-4, m
        assert backward_error(pe, rpe, us) <= FORCE_TOL
        assert backward_error(w, rw, ws) <= FORCE_TOL
        # totals (what measure() reports) are far tighter
        assert abs(pe.sum() - rpe.sum()) <= 1e-6 * np.abs(rpe).sum()
        assert abs(w.sum() - rw.sum()) <= 1e-6 * np.abs(rw).sum()
    return st, box, nl, m


@pytest.mark.parametrize("seed", range(50, 55))
def test_truncated_forces_reference_fixtures(seed):
    # test_forces.py:45-56 fixtures (n=320, L=7.5), quantised to fp32
    FO = load_golden("forces")
    pos = quantize_f32(FO[f"trunc{seed}.pos"])
    check_forces(pos, [7.5] * 3, b2.make_shifted(1.0, 1.0, 2.5), 3.0)


@pytest.mark.parametrize("n,seed", [(4096, 3), (32_000, 4)])
def test_truncated_forces_fluid(n, seed):
    pos, _, edge = fluid_state(n, seed=seed)
    pos = quantize_f32(pos)
    st, box, nl, m = check_forces(pos, [edge] * 3, b2.make_shifted(1.0, 1.0, 2.5), 2.8,
                                  stride=128)
    f = st.forces.acquire_read(b2.HOST)
    # Newton's third law in aggregate (test_forces.py:104-111)
    assert np.max(np.abs(f.sum(axis=0))) <= 1e-4 * np.abs(f).max() * np.sqrt(n)


def test_kob_andersen_pair_tables():
    n = 8192
    pos, _, edge = fluid_state(n, density=1.2, seed=9, jitter=0.03)
    pos = quantize_f32(pos)
    species = (np.random.default_rng(42).permutation(n) < n // 5).astype(np.int32)  # 20 % B
    ka = b2.PairTable.kob_andersen()
    check_forces(pos, [edge] * 3, ka, ka.max_r_cut + 0.3, species=species, stride=256)


def test_pair_table_with_identical_rows_equals_single_type_bitwise():
    pos, _, edge = fluid_state(4096, seed=5)
    pos = quantize_f32(pos)
    box = b2.SimBox.cubic(edge)
    out = []
    for params, species in [
            (b2.make_shifted(1.0, 1.0, 2.5), None),
            (b2.PairTable(np.ones((2, 2)), np.ones((2, 2)), np.full((2, 2), 2.5)),
             np.random.default_rng(1).integers(0, 2, size=4096).astype(np.int32))]:
        st = make_state(pos, species=species)
        grid = b2.bin_particles(st, box, 2.8)
        nl = b2.build_neighbor_list(st, grid, 2.8, 128, r_cut=2.5)
        b2.compute_forces_truncated(st, params, box, nl)
        out.append((np.array(st.forces.acquire_read(b2.HOST)),
                    np.array(st.per_particle_potential.acquire_read(b2.HOST))))
    # same pair terms; only the deferred prefactors are applied in another order
    assert np.max(np.abs(out[0][0] - out[1][0])) <= 1e-6 * np.abs(out[0][0]).max()
    assert np.max(np.abs(out[0][1] - out[1][1])) <= 1e-6 * np.abs(out[0][1]).max()


def test_all_pairs_forces_match_oracle_and_truncated_kernel():
    FO = load_golden("forces")
    pos = quantize_f32(FO["all0.pos"])
    box = b2.SimBox.cubic(7.0)
    lj = b2.make_shifted(1.0, 1.0, 2.5)
    st = make_state(pos)
    b2.compute_forces_all_to_all(st, lj, box)
    rf, rpe, rw = orc.forces_all_pairs(pos, [7.0] * 3, lj.table(), threads=orc.host_threads())
    f = np.array(st.forces.acquire_read(b2.HOST))
    m = force_error_metrics(f, rf)
    assert m["M3"] <= FORCE_TOL, m
    assert scalar_rel_error(st.per_particle_potential.acquire_read(b2.HOST), rpe) <= FORCE_TOL
    assert scalar_rel_error(st.virial.acquire_read(b2.HOST), rw) <= FORCE_TOL
    # untruncated potential (test_forces.py:59-67)
    st2 = make_state(pos)
    bare = b2.make_shifted(1.0, 1.0)
    b2.compute_forces_all_to_all(st2, bare, box)
    rf2, rpe2, _ = orc.forces_all_pairs(pos, [7.0] * 3, bare.table(), threads=orc.host_threads())
    assert force_error_metrics(st2.forces.acquire_read(b2.HOST), rf2)["M3"] <= FORCE_TOL
    assert scalar_rel_error(st2.per_particle_potential.acquire_read(b2.HOST), rpe2) <= FORCE_TOL


def test_singular_pairs_are_reported_like_the_reference():
    # test_forces.py:171-188: lowest i, first j; also across the periodic boundary
    lj = b2.make_shifted(1.0, 1.0, 2.5)
    box = b2.SimBox.cubic(10.0)
    pos = np.array([[1.0, 1.0, 1.0], [3.0, 3.0, 3.0], [1.0, 1.0, 1.0]])
    with pytest.raises(b2.SingularPairError) as exc:
        b2.compute_forces_all_to_all(make_state(pos), lj, box)
    assert (exc.value.i, exc.value.j) == (0, 2)
    st = make_state(pos)
    grid = b2.bin_particles(st, box, 3.0)
    nl = b2.build_neighbor_list(st, grid, 3.0, 8, r_cut=2.5)
    with pytest.raises(b2.SingularPairError) as exc:
        b2.compute_forces_truncated(st, lj, box, nl)
    assert (exc.value.i, exc.value.j) == (0, 2)


def test_cutoff_is_exclusive():
    # r == r_cut contributes nothing (forces.py:92-93), r just inside does
    lj = b2.make_shifted(1.0, 1.0, 2.5)
    box = b2.SimBox.cubic(20.0)
    pos = np.array([[1.0, 1.0, 1.0], [3.5, 1.0, 1.0], [1.0, 8.0, 1.0], [3.4990234375, 8.0, 1.0]])
    st = make_state(pos)
    grid = b2.bin_particles(st, box, 3.0)
    nl = b2.build_neighbor_list(st, grid, 3.0, 8, r_cut=2.5)
    b2.compute_forces_truncated(st, lj, box, nl)
    f = st.forces.acquire_read(b2.HOST)
    pe = st.per_particle_potential.acquire_read(b2.HOST)
    assert np.all(f[:2] == 0.0) and np.all(pe[:2] == 0.0)
    assert f[2, 0] != 0.0 and f[2, 0] == -f[3, 0]


def test_translation_invariance_across_the_periodic_faces():
    """Shifting everything by a grid-aligned vector (so that many pairs now
    straddle the faces) leaves forces unchanged to fp32 rounding: exercises the
    exact image-shift path (test_forces.py:114-132 analogue)."""
    n = 4096
    pos, _, edge_raw = fluid_state(n, seed=8)
    grid_q = 2.0 ** -10
    edge = float(np.round(edge_raw / grid_q) * grid_q)   # box edge on the grid too
    pos = np.floor(pos / grid_q) * grid_q
    pos = np.where(pos >= edge, pos - edge, pos)
    lj = b2.make_shifted(1.0, 1.0, 2.5)
    box = b2.SimBox.cubic(edge)
    results = []
    for shift in (np.zeros(3), np.array([edge / 2, 3.0, -7.25])):
        p = pos + np.floor(shift / grid_q) * grid_q
        p -= np.floor(p / edge) * edge
        p = np.where(p >= edge, p - edge, p)
        st = make_state(quantize_f32(p))
        g = b2.bin_particles(st, box, 2.8)
        nl = b2.build_neighbor_list(st, g, 2.8, 128, r_cut=2.5)
        b2.compute_forces_truncated(st, lj, box, nl)
        results.append(np.array(st.forces.acquire_read(b2.HOST)))
    m = force_error_metrics(results[1], results[0])
    assert m["M3"] <= FORCE_TOL, m


# --------------------------------------------------------------- integrator
def test_vv_integrate_and_finalize_match_reference_arithmetic():
    G = load_golden("integrate")
    pos, vel = quantize_ds(G["pos"]), quantize_f32(G["vel"])
    masses, forces = quantize_f32(G["masses"]), quantize_f32(G["forces"])
    edges, dt = G["edges"], float(G["dt"])
    st = make_state(pos, velocities=vel, masses=masses, images=G["img"])
    st.forces.acquire_write(b2.HOST)[...] = forces
    box = b2.SimBox(edges)
    b2.vv_integrate(st, b2.IntegratorParams(dt), box)
    p1, i1, v1 = orc.vv_integrate(pos, G["img"], vel, forces, masses, edges, dt)
    got_v = st.velocities.acquire_read(b2.HOST)
    got_p = st.positions.acquire_read(b2.HOST)
    got_i = st.images.acquire_read(b2.HOST)
    assert np.max(np.abs(got_v - v1) / np.maximum(np.abs(v1), 1.0)) <= 2e-7     # fp32 velocities
    # unwrapped positions agree to double-single accuracy of the drift
    # (the drift uses the fp32 velocity the device holds)
    v_dev = got_v
    want_unwrapped = (pos + G["img"] * edges) + v_dev * dt
    got_unwrapped = got_p + got_i * edges
    assert np.max(np.abs(got_unwrapped - want_unwrapped)) <= 1e-9
    assert np.all(got_p >= 0.0) and np.all(got_p < edges)
    # images: identical wherever the wrapped coordinate is not within rounding of a face
    safe = (np.minimum(p1, edges - p1) > 1e-6)
    assert np.array_equal(got_i[safe], i1[safe])
    forces2 = quantize_f32(G["forces2"])
    st.forces.acquire_write(b2.HOST)[...] = forces2
    b2.vv_finalize(st, b2.IntegratorParams(dt))
    v2 = orc.vv_finalize(got_v, forces2, masses, dt)
    got_v2 = st.velocities.acquire_read(b2.HOST)
    assert np.max(np.abs(got_v2 - v2) / np.maximum(np.abs(v2), 1.0)) <= 2e-7


def test_free_drift_crosses_boundary_and_counts_images():
    # test_integrate.py:21-31: free particle drifting across the lower face
    box = b2.SimBox.cubic(10.0)
    st = make_state(np.array([[5.0, 0.05, 5.0]]), velocities=np.array([[1.0, -1.0, 0.0]]))
    for _ in range(10):
        b2.vv_integrate(st, b2.IntegratorParams(0.01), box)
    pos = st.positions.acquire_read(b2.HOST)
    img = st.images.acquire_read(b2.HOST)
    assert np.array_equal(img, [[0, -1, 0]])
    assert pos[0] == pytest.approx([5.1, 9.95, 5.0], abs=1e-6)


def test_double_single_drift_keeps_small_increments():
    """10^4 drifts of 1e-6 at x ~ 100: fp32 alone would lose every increment."""
    box = b2.SimBox.cubic(128.0)
    st = make_state(np.array([[100.0, 100.0, 100.0]]), velocities=np.array([[1e-3, 0.0, 0.0]]))
    steps = 2000
    for _ in range(steps):
        b2.vv_integrate(st, b2.IntegratorParams(1e-3), box)
    x = st.positions.acquire_read(b2.HOST)[0, 0]
    want = 100.0 + steps * float(np.float32(1e-3)) * 1e-3
    assert abs(x - want) < 1e-9


# -------------------------------------------------------------- reductions
def test_reduce_sum_bit_exact_with_reference_tree():
    G = load_golden("observables")
    for size, want in zip(G["sizes"], G["sums"]):
        assert b2.reduce_sum(G["values"][:size]) == want, size
    assert b2.reduce_sum(np.zeros(0)) == 0.0
    big = np.random.default_rng(3).normal(size=5_000_001)
    assert b2.reduce_sum(big) == orc.reduce_sum(big)
    with pytest.raises(ValueError):
        b2.reduce_sum([1.0], mode="sloppy")


def test_thermo_bit_exact_with_oracle_on_device_formats():
    G = load_golden("observables")
    vel, masses = quantize_f32(G["vel"]), quantize_f32(G["masses"])
    pe, w = quantize_f32(G["pe_in"]), quantize_f32(G["pe_in"][::-1])
    st = make_state(np.zeros((len(masses), 3)), velocities=vel, masses=masses)
    st.per_particle_potential.acquire_write(b2.HOST)[...] = pe
    st.virial.acquire_write(b2.HOST)[...] = w
    t = b2.thermo(st)
    want = orc.thermo(vel, masses, pe, w)
    assert t.potential_energy == want["pe"]
    assert t.kinetic_energy == want["ke"]
    assert np.array_equal(np.array(t.momentum), want["momentum"])
    assert t.virial == want["virial"]
    assert t.temperature == want["temperature"]
    assert np.allclose(t.com_velocity, want["com_velocity"], rtol=1e-15)
    ke, temp = b2.kinetic_energy_and_temperature(st)
    assert (ke, temp) == (want["ke"], want["temperature"])
    assert b2.potential_energy_total(st) == want["pe"]
    assert np.array_equal(b2.total_momentum(st), want["momentum"])
    # hand values (test_observables.py:77-109)
    st = make_state(np.zeros((2, 3)), velocities=np.array([[1.0, 2.0, 2.0], [0.0, -3.0, 4.0]]),
                    masses=np.array([2.0, 0.5]))
    t = b2.thermo(st)
    assert t.kinetic_energy == 9.0 + 6.25
    assert t.temperature == 2.0 * 15.25 / 6.0
    assert t.momentum == (2.0, 2.5, 6.0)
