"""Lane order of the pair kernel (b2md_pair_order, B2MD_FORCE_ORDERED): which thread of a
block walks which pair row.  The order is a permutation of every block sorted by row
length, rows are padded to the longest row of their new warp, and nothing computed from
the rows changes by a bit (forces, energies, virial, whole trajectories)."""
import numpy as np
import pytest
import torch

import paper_2406_04210_b200 as b2
from paper_2406_04210_b200 import _lib
from helpers import fluid_state, quantize_f32

pytestmark = pytest.mark.gpu

THREADS = 128            # kPairThreads
ORDERED = 8              # B2MD_FORCE_ORDERED


def pair_forces(st, box, nl, pair, counts, pitch, flags):
    dev = st.device_state()
    from paper_2406_04210_b200.forces import _table_ptr
    keep, tab_ptr, nt = _table_ptr(b2.make_shifted(1.0, 1.0, 2.5), st)
    dev.reset_status()
    _lib.call("b2md_force_lj_pairs", dev.pos_hi.data_ptr(), dev.n, box.c_box(),
              pair.data_ptr(), counts.data_ptr(), pitch, nl.d_nbr.data_ptr(),
              nl.d_counts.data_ptr(), nl.pitch, nl.d_boundary.data_ptr(), tab_ptr, nt, flags,
              dev.force.data_ptr(), dev.virial.data_ptr(), dev.status.data_ptr(), dev.stream)
    torch.cuda.synchronize()
    return dev.force.clone(), dev.virial.clone()


@pytest.mark.parametrize("n,unit,face_key", [(1, 1, 0), (255, 1, 1), (4097, 1, 0), (4097, 2, 1),
                                              (30_000, 1, 1), (30_001, 4, 0), (262_144, 1, 0)])
def test_lane_order_is_a_sorted_permutation_and_changes_no_bit(n, unit, face_key):
    if n < 1000:
        gen = np.random.default_rng(n)
        edge = 9.0
        pos = quantize_f32(gen.uniform(0, edge, size=(n, 3)))
    else:
        pos, _, edge = fluid_state(n, seed=n)
        pos = quantize_f32(pos)
    box = b2.SimBox.cubic(edge)
    st = b2.ParticleState(pos)
    grid = b2.bin_particles(st, box, 2.8)
    nl = b2.build_neighbor_list(st, grid, 2.8, 128, r_cut=2.5)
    assert not nl.overflow
    d_pair, d_cnt, pitch = nl.pair_rows()
    lib = _lib.load()
    n_pairs = (n + 1) // 2
    n_blocks = (n_pairs + THREADS - 1) // THREADS
    extra = int(lib.b2md_pair_schedule_len(n))
    assert extra >= 2 * n_blocks + THREADS * n_blocks // 4
    base_f, base_w = pair_forces(st, box, nl, d_pair, d_cnt, pitch, 0)

    tiles = d_pair.shape[0]
    counts = d_cnt.cpu().numpy()
    row_tiles = (counts + 3) // 4
    # everything behind the padding of the particle-order warps is poisoned with flagged
    # entries: a warp that walked past its own padding would change the forces
    rows = d_pair.permute(1, 0, 2).reshape(pitch, 4 * tiles).cpu().numpy().copy()
    for w in range(0, pitch, 32):
        rows[w:w + 32, 4 * int(row_tiles[w:w + 32].max()):] = 3
    pair = torch.from_numpy(rows.reshape(pitch, tiles, 4)).permute(1, 0, 2).contiguous().cuda()
    cnt_ext = torch.zeros(pitch + extra, dtype=torch.int32, device="cuda")
    cnt_ext[:pitch] = d_cnt
    dev = st.device_state()
    _lib.call("b2md_pair_order", nl.d_boundary.data_ptr(), n, pair.data_ptr(), cnt_ext.data_ptr(),
              pitch, 4 * tiles, unit, face_key, dev.stream)
    torch.cuda.synchronize()
    order = cnt_ext[pitch + 2 * n_blocks:].cpu().numpy().view(np.uint8)[:n_blocks * THREADS]
    order = order.reshape(n_blocks, THREADS).astype(np.int64)
    assert np.array_equal(np.sort(order, axis=1), np.tile(np.arange(THREADS), (n_blocks, 1)))
    padded = np.zeros(n_blocks * THREADS, dtype=np.int64)
    padded[:n_pairs] = row_tiles[:n_pairs]
    by_slot = np.take_along_axis(padded.reshape(n_blocks, THREADS), order, axis=1)
    if unit == 1 and not face_key:
        assert np.all(np.diff(by_slot, axis=1) >= 0)
    # units stay together
    assert np.all(order.reshape(n_blocks, THREADS // unit, unit)[:, :, 0] % unit == 0)
    assert np.all(np.diff(order.reshape(n_blocks, THREADS // unit, unit), axis=2) == 1)
    # the warps walk fewer tiles than in particle order, never more
    new_trips = by_slot.reshape(n_blocks, THREADS // 32, 32).max(2).sum()
    old_trips = padded.reshape(n_blocks, THREADS // 32, 32).max(2).sum()
    assert new_trips <= old_trips
    # rows are padded, flag-less, to the longest row of their new warp
    got = pair.permute(1, 0, 2).reshape(pitch, 4 * tiles).cpu().numpy()
    gmax = by_slot.reshape(n_blocks, THREADS // 32, 32).max(2)
    for b in range(n_blocks):
        for s in range(THREADS):
            t = b * THREADS + order[b, s]
            if t < n_pairs:
                assert np.array_equal(got[t, :counts[t]], rows[t, :counts[t]])
                assert np.all(got[t, counts[t]:4 * gmax[b, s // 32]] & 3 == 0)
    f, w = pair_forces(st, box, nl, pair, cnt_ext, pitch, ORDERED)
    assert torch.equal(f, base_f) and torch.equal(w, base_w)
    assert float(base_f[:, :3].abs().max()) > 0.0 or n < 3


def test_trajectory_is_bit_identical_with_the_lane_order(monkeypatch):
    n = 262_144
    series = []
    for mode in ("1", "3", "519", "0"):        # schedule; + order; + order of units of 2 with the face key; neither
        monkeypatch.setenv("B2MD_PAIR_SCHEDULE", mode)
        st, box = b2.init_lattice_any(n, 0.75)
        b2.init_velocities(st, 1.2, 42)
        sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001,
                            force_mode=b2.TRUNCATED, skin=0.3, sample_interval=40,
                            sample_initial=True)
        assert sim.pair_rows
        sim.run(120)
        series.append((np.array([s.total_energy for s in sim.samples]),
                       np.array(st.positions.acquire_read(b2.HOST)),
                       np.array(st.velocities.acquire_read(b2.HOST)), sim.rebuild_count))
        sim.close()
    assert series[0][3] >= 2
    for other in series[1:]:
        assert other[3] == series[0][3]
        for x, y in zip(series[0][:3], other[:3]):
            assert np.array_equal(x, y)
