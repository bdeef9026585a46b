"""b2md_build_pair_list -- the step loop's list build, which emits the force kernel's pair rows
straight from the list kernel's decision masks -- against the two-stage path it replaces
(b2md_build_nlist_ex, bit-exact with the reference's rows, followed by b2md_pair_rows): pair
tiles, pair counts, row counts, boundary flags and the status words must be bit-identical, and
the plain rows it still writes (pairs that straddle two cells) must be the reference's."""
import ctypes

import numpy as np
import pytest
import torch

import paper_2406_04210_b200 as b2
from paper_2406_04210_b200 import _lib
from paper_2406_04210_b200.neighbor import reorder_hilbert
from helpers import fluid_state, quantize_f32

pytestmark = pytest.mark.gpu

LIST_ANY_PREFIX = 1


def fused_build(st, box, grid, r_list, stride, skin, n_rows=None, flags=LIST_ANY_PREFIX):
    dev = st.device_state()
    n = dev.n
    n_rows = n if n_rows is None else n_rows
    pitch = (n + 31) // 32 * 32
    rows = (stride + 15) // 16 * 16
    d = dict(device=dev.device)
    nbr = torch.full((rows, pitch), -7, dtype=torch.int32, **d)       # poison: must not matter
    counts = torch.zeros(pitch, dtype=torch.int32, **d)
    boundary = torch.zeros(pitch, dtype=torch.uint8, **d)
    pair_pitch = ((n_rows + 1) // 2 + 31) // 32 * 32
    pair_rows = 2 * rows
    pair_nbr = torch.zeros((pair_rows // 4, pair_pitch, 4), dtype=torch.int32, **d)
    pair_counts = torch.full((pair_pitch,), 12345, dtype=torch.int32, **d)
    dev.reset_status()
    _lib.call("b2md_build_pair_list", dev.pos_hi.data_ptr(), dev.pos_lo.data_ptr(), n,
              box.c_box(), grid.c_grid(), grid.d_cell_of.data_ptr(), grid.d_cell_start.data_ptr(),
              grid.d_cell_particles.data_ptr(), float(r_list), stride, pitch, nbr.data_ptr(),
              counts.data_ptr(), boundary.data_ptr(), float(r_list) + skin, n_rows, flags, rows,
              pair_nbr.data_ptr(), pair_counts.data_ptr(), pair_pitch, pair_rows,
              dev.status.data_ptr(), dev.stream)
    status = dev.read_status()
    return dict(nbr=nbr, counts=counts, boundary=boundary, pair_nbr=pair_nbr,
                pair_counts=pair_counts, pair_pitch=pair_pitch, status=status, rows=rows)


def two_stage(st, box, grid, r_list, stride, skin):
    nl = b2.build_neighbor_list(st, grid, r_list, stride, r_cut=r_list - skin)
    assert not nl.overflow
    d_pair, d_cnt, pair_pitch = nl.pair_rows()
    return nl, d_pair, d_cnt, pair_pitch


def compare(st, box, r_list, stride, skin, expect_fused_fraction=None):
    grid = b2.bin_particles(st, box, r_list)
    nl, d_pair, d_cnt, pair_pitch = two_stage(st, box, grid, r_list, stride, skin)
    got = fused_build(st, box, grid, r_list, stride, skin)
    n = st.device_state().n
    assert got["pair_pitch"] == pair_pitch
    assert got["status"].overflow == 0 and got["status"].max_count == nl.max_count
    assert torch.equal(got["counts"], nl.d_counts)
    assert torch.equal(got["boundary"], nl.d_boundary)
    assert torch.equal(got["pair_counts"], d_cnt)
    tiles = min(got["pair_nbr"].shape[0], d_pair.shape[0])
    assert torch.equal(got["pair_nbr"][:tiles], d_pair[:tiles])
    assert not got["pair_nbr"][tiles:].any() and not d_pair[tiles:].any()
    # plain rows (row-major in this mode: row i at nbr + i * list_rows): either the reference's
    # row, or untouched (the pair was emitted directly)
    rows = got["nbr"].reshape(-1)[:n * got["rows"]].reshape(n, got["rows"]).cpu().numpy()
    ref = nl.indices
    cnt = nl.counts
    touched = (rows != -7).any(axis=1)
    for i in np.flatnonzero(touched):
        assert np.array_equal(rows[i, :cnt[i]], ref[i, :cnt[i]])
    if expect_fused_fraction is not None:
        assert 1.0 - touched.mean() >= expect_fused_fraction
    return 1.0 - touched.mean()


@pytest.mark.parametrize("n,density", [(500, 0.75), (4097, 0.75), (30_000, 0.75), (8192, 1.2),
                                       (30_001, 1.2)])
def test_fused_build_matches_two_stage_after_hilbert_reorder(n, density):
    pos, _, edge = fluid_state(n, density=density, seed=n)
    st = b2.ParticleState(quantize_f32(pos))
    box = b2.SimBox.cubic(edge)
    r_list, skin = 2.8, 0.3
    reorder_hilbert(st, box, r_list)
    frac = compare(st, box, r_list, 160 if density > 1 else 112, skin,
                   expect_fused_fraction=0.6 if n > 4000 else None)
    print(f"n={n} rho={density}: {100 * frac:.1f} % of the rows emitted as pair rows directly")


def test_fused_build_on_unordered_particles_falls_back_row_by_row():
    """Lattice order (no reorder): cells are not contiguous index ranges, so every pair goes
    through the plain rows and the merge -- same result."""
    pos, _, edge = fluid_state(6000, seed=3)
    gen = np.random.default_rng(0)
    pos = pos[gen.permutation(len(pos))]
    st = b2.ParticleState(quantize_f32(pos))
    box = b2.SimBox.cubic(edge)
    frac = compare(st, box, 2.8, 112, 0.3)
    assert frac < 0.2


def test_fused_build_with_many_particles_per_cell():
    """Cells of 2 r_list: ~130 particles per cell -- several passes of 24 rows and several
    candidate batches per cell; tiles are carried across the batches."""
    pos, _, edge = fluid_state(20_000, seed=5)
    st = b2.ParticleState(quantize_f32(pos))
    box = b2.SimBox.cubic(edge)
    r_cell = 5.0
    grid_big = b2.bin_particles(st, box, r_cell)
    b2.reorder_by_cell(st, grid_big)
    grid_big = b2.bin_particles(st, box, r_cell)
    # a list of radius 2.8 over the coarse grid: the C entry points take the grid as given
    r_list, skin, stride = 2.8, 0.3, 112
    dev = st.device_state()
    n = dev.n
    pitch = (n + 31) // 32 * 32
    rows = 112
    d = dict(device=dev.device)
    nbr = torch.zeros((rows, pitch), dtype=torch.int32, **d)
    counts = torch.zeros(pitch, dtype=torch.int32, **d)
    boundary = torch.zeros(pitch, dtype=torch.uint8, **d)
    dev.reset_status()
    _lib.call("b2md_build_nlist_ex", dev.pos_hi.data_ptr(), dev.pos_lo.data_ptr(), n,
              box.c_box(), grid_big.c_grid(), grid_big.d_cell_of.data_ptr(),
              grid_big.d_cell_start.data_ptr(), grid_big.d_cell_particles.data_ptr(), r_list,
              stride, pitch, nbr.data_ptr(), counts.data_ptr(), boundary.data_ptr(),
              r_list + skin, n, LIST_ANY_PREFIX, dev.status.data_ptr(), dev.stream)
    assert dev.read_status().overflow == 0
    pair_pitch = ((n + 1) // 2 + 31) // 32 * 32
    pair_nbr = torch.zeros((2 * rows // 4, pair_pitch, 4), dtype=torch.int32, **d)
    pair_counts = torch.zeros(pair_pitch, dtype=torch.int32, **d)
    _lib.call("b2md_pair_rows", nbr.data_ptr(), counts.data_ptr(), pitch, rows, n,
              pair_nbr.data_ptr(), pair_counts.data_ptr(), pair_pitch, 2 * rows, dev.stream)
    got = fused_build(st, box, grid_big, r_list, stride, skin)
    assert torch.equal(got["counts"], counts)
    assert torch.equal(got["pair_counts"], pair_counts)
    assert torch.equal(got["pair_nbr"], pair_nbr)
    touched = (got["nbr"].reshape(-1)[:n * got["rows"]].reshape(n, got["rows"]) != -7).any(dim=1)
    assert touched.float().mean().item() < 0.2


def test_fused_build_flags_overflow_and_reports_the_longest_row():
    pos, _, edge = fluid_state(8000, seed=9)
    st = b2.ParticleState(quantize_f32(pos))
    box = b2.SimBox.cubic(edge)
    reorder_hilbert(st, box, 2.8)
    grid = b2.bin_particles(st, box, 2.8)
    nl = b2.build_neighbor_list(st, grid, 2.8, 256, r_cut=2.5)
    got = fused_build(st, box, grid, 2.8, 48, 0.3)          # rows want ~78 entries
    assert got["status"].overflow == 1 and got["status"].max_count == nl.max_count
    assert int(got["counts"].max()) == 48


def test_fused_build_leaves_ghost_rows_alone():
    """n_rows < n (slab decomposition: rows [n_rows, n) are ghosts): pairs are formed among the
    owned rows only and ghost rows get neither a row nor a pair."""
    pos, _, edge = fluid_state(9001, seed=11)
    st = b2.ParticleState(quantize_f32(pos))
    box = b2.SimBox.cubic(edge)
    reorder_hilbert(st, box, 2.8)
    grid = b2.bin_particles(st, box, 2.8)
    n = 9001
    n_rows = 7001
    dev = st.device_state()
    pitch = (n + 31) // 32 * 32
    rows = 112
    d = dict(device=dev.device)
    nbr = torch.zeros((rows, pitch), dtype=torch.int32, **d)
    counts = torch.zeros(pitch, dtype=torch.int32, **d)
    boundary = torch.zeros(pitch, dtype=torch.uint8, **d)
    dev.reset_status()
    _lib.call("b2md_build_nlist_ex", dev.pos_hi.data_ptr(), dev.pos_lo.data_ptr(), n,
              box.c_box(), grid.c_grid(), grid.d_cell_of.data_ptr(), grid.d_cell_start.data_ptr(),
              grid.d_cell_particles.data_ptr(), 2.8, 112, pitch, nbr.data_ptr(),
              counts.data_ptr(), boundary.data_ptr(), 3.1, n_rows, LIST_ANY_PREFIX,
              dev.status.data_ptr(), dev.stream)
    pair_pitch = ((n_rows + 1) // 2 + 31) // 32 * 32
    pair_nbr = torch.zeros((2 * rows // 4, pair_pitch, 4), dtype=torch.int32, **d)
    pair_counts = torch.zeros(pair_pitch, dtype=torch.int32, **d)
    _lib.call("b2md_pair_rows", nbr.data_ptr(), counts.data_ptr(), pitch, rows, n_rows,
              pair_nbr.data_ptr(), pair_counts.data_ptr(), pair_pitch, 2 * rows, dev.stream)
    got = fused_build(st, box, grid, 2.8, 112, 0.3, n_rows=n_rows)
    assert torch.equal(got["counts"], counts)
    assert torch.equal(got["pair_counts"], pair_counts)
    assert torch.equal(got["pair_nbr"], pair_nbr)


@pytest.mark.parametrize("n,steps", [(262_144, 120), (1_000_000, 80)])
def test_native_loop_is_bit_identical_with_either_list_build(monkeypatch, n, steps):
    """Whole trajectories: the runner with b2md_build_pair_list (default) and with the
    two-stage build (B2MD_LIST_PAIRS=0) produce the same bits -- also at the benchmark's size
    (39^3 cells, 500 000 pair rows)."""
    out = []
    for mode in ("1", "0"):
        monkeypatch.setenv("B2MD_LIST_PAIRS", mode)
        st, box = b2.init_lattice_any(n, 0.75)
        b2.init_velocities(st, 1.2, 42)
        sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001,
                            force_mode=b2.TRUNCATED, skin=0.3, sample_interval=40,
                            sample_initial=True, reorder="hilbert")
        assert sim.pair_rows
        sim.run(steps)
        out.append((np.array([s.total_energy for s in sim.samples]),
                    np.array(st.positions.acquire_read(b2.HOST)),
                    np.array(st.velocities.acquire_read(b2.HOST)), sim.rebuild_count))
        sim.close()
    assert out[0][3] == out[1][3] and out[0][3] >= 2
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    assert np.array_equal(out[0][2], out[1][2])
