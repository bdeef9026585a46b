"""Pruned ("inner") pair rows of the one-launch step (b2md_force_lj_pairs_advance_pruned): the
inner rows are exactly the entries of the full rows inside r_cut + delta with narrowed flags; a
step over them gives the same bits as a step over the full rows (the dropped entries contribute
exact zeros, forces.py:92); the flag bits follow the displacements; whole trajectories of the
native loop are bit-identical with and without pruning and keep the reference's rebuild schedule
(neighbor.py:243-254)."""
import ctypes

import numpy as np
import pytest
import torch

import paper_2406_04210_b200 as b2
from paper_2406_04210_b200 import _lib

pytestmark = pytest.mark.gpu

R_CUT, SKIN, DELTA = 2.5, 0.3, 0.1
INNER, NOW, OUTER = 1, 2, 3


def make_sim(n, prune_delta, steps=0, seed=42, density=0.75, sample_interval=50, lj=None):
    st, box = b2.init_lattice_any(n, density)
    if lj is not None and lj.ntypes > 1:
        species = (np.random.default_rng(seed).permutation(n) < n // 5).astype(np.int32)
        st = b2.ParticleState(st.positions.acquire_read(b2.HOST), species=species)
    b2.init_velocities(st, 1.2, seed)
    lj = lj or b2.make_shifted(1.0, 1.0, R_CUT)
    sim = b2.Simulation(st, box, lj, 0.001, force_mode=b2.TRUNCATED, skin=SKIN,
                        sample_interval=sample_interval, sample_initial=True, reorder="hilbert",
                        pair_rows=True, prune_delta=prune_delta)
    if steps:
        sim.run(steps)
    return sim, st, box, lj


def launch(sim, box, lj, mode, gates, scratch, dt=0.001):
    dev = sim.state.device_state()
    k = sim._keep
    cfg = k["cfg"]
    tab = np.ascontiguousarray(lj.table())
    _lib.call("b2md_force_lj_pairs_advance_pruned", dev.pos_hi.data_ptr(),
              scratch["out"].data_ptr(), scratch["pos_lo"].data_ptr(), scratch["vel"].data_ptr(),
              scratch["image"].data_ptr(), dev.n, box.c_box(), dt, scratch["ref"].data_ptr(),
              (0.5 * SKIN) ** 2, k["pair_nbr"].data_ptr(), k["pair_counts"].data_ptr(),
              cfg.pair_pitch, k["nbr"].data_ptr(), k["counts"].data_ptr(), k["pitch"],
              k["boundary"].data_ptr(), tab.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 1, 0,
              gates[0], gates[1], gates[2], mode, scratch["inner"].data_ptr(),
              scratch["inner_counts"].data_ptr(), cfg.pair_rows, R_CUT, SKIN, DELTA,
              scratch["status"].data_ptr(), dev.stream)
    torch.cuda.synchronize()


def fresh_scratch(sim):
    dev = sim.state.device_state()
    k = sim._keep
    return {"out": torch.zeros_like(dev.pos_hi), "pos_lo": dev.pos_lo.clone(),
            "vel": dev.vel.clone(), "image": dev.image.clone(), "ref": k["ref_pos"].clone(),
            "inner": torch.zeros_like(k["pair_nbr"]),
            "inner_counts": torch.zeros(k["cfg"].pair_pitch, dtype=torch.int32,
                                        device=dev.pos_hi.device),
            "status": torch.zeros(16, dtype=torch.int32, device=dev.pos_hi.device)}


def rows_of(tiles, pitch):
    t = tiles.shape[0]
    return tiles.permute(1, 0, 2).reshape(pitch, 4 * t).cpu().numpy()


def test_prune_launch_writes_the_subset_inside_r_cut_plus_delta():
    n = 20_000
    sim, st, box, lj = make_sim(n, 0.0, steps=30)          # moved a little since the list build
    sc = fresh_scratch(sim)
    launch(sim, box, lj, NOW, (5, 12, 14), sc, dt=1e-9)
    k = sim._keep
    pitch = k["cfg"].pair_pitch
    outer = rows_of(k["pair_nbr"], pitch)
    outer_cnt = k["pair_counts"][:pitch].cpu().numpy()
    inner = rows_of(sc["inner"], pitch)
    inner_cnt = sc["inner_counts"].cpu().numpy()
    pos = sim.state.device_state().pos_hi[:, :3].double().cpu().numpy()
    edge = float(box.edge_lengths[0])
    lim2 = (R_CUT + DELTA) ** 2
    n_pairs = (n + 1) // 2
    dropped = ambiguous = 0
    for t in range(0, n_pairs, 7):
        e = outer[t, :outer_cnt[t]]
        j = e >> 2
        keep = np.zeros(len(e), dtype=np.int64)
        fuzzy = np.zeros(len(e), dtype=bool)
        for which in (0, 1):
            i = min(2 * t + which, n - 1)
            d = pos[i] - pos[j]
            d -= edge * np.rint(d / edge)
            r2 = (d * d).sum(axis=1)
            listed = ((e >> which) & 1) == 1
            keep |= (listed & (r2 < lim2)).astype(np.int64) << which
            fuzzy |= listed & (np.abs(r2 - lim2) < 1e-4)
        got = inner[t, :inner_cnt[t]]
        if fuzzy.any():
            ambiguous += 1
            sure = ~fuzzy
            want = ((j << 2) | keep)[sure & (keep != 0)]
            assert np.isin(want, got).all()
            continue
        want = ((j << 2) | keep)[keep != 0]
        assert np.array_equal(got, want), t
        dropped += len(e) - len(want)
    assert dropped > 1000 and ambiguous < 50
    # padding up to the warp's longest inner row is flag-less
    for w in range(0, pitch, 32):
        longest = (int(inner_cnt[w:w + 32].max()) + 3) // 4 * 4
        for t in range(w, min(w + 32, pitch)):
            assert np.all(inner[t, inner_cnt[t]:longest] & 3 == 0)
    sim.close()


def test_step_over_inner_rows_is_bit_identical_to_the_full_rows():
    n = 30_000
    sim, st, box, lj = make_sim(n, 0.0, steps=20)
    base = fresh_scratch(sim)
    launch(sim, box, lj, NOW, (5, 12, 14), base)            # prune + step over the full rows
    assert base["status"][13].item() == 1
    results = {}
    for name, mode in (("inner", INNER), ("outer", OUTER)):
        sc = fresh_scratch(sim)
        sc["inner"], sc["inner_counts"] = base["inner"], base["inner_counts"]
        launch(sim, box, lj, mode, (5, 12, 14), sc)
        assert sc["status"][13].item() == 1
        results[name] = sc
    for name in ("out", "pos_lo", "vel", "image"):
        assert torch.equal(results["inner"][name], results["outer"][name]), name
        assert torch.equal(results["inner"][name], base[name]), name
    assert int(base["inner_counts"].sum()) < 0.9 * int(sim._keep["pair_counts"][:sim._keep["cfg"].pair_pitch].sum())
    sim.close()


def test_flag_bits_follow_the_displacements():
    n = 20_000
    sim, st, box, lj = make_sim(n, 0.0, steps=0)
    dev = sim.state.device_state()

    def flags_after(kick_one, dt, mode, ref_shift=0.0, first=None):
        sc = first or fresh_scratch(sim)
        if kick_one is not None:
            sc["vel"][7, 0] = kick_one
        if ref_shift:
            sc["ref"][11, 1] -= ref_shift          # particle 11 is that far from its snapshot
        sc["status"].zero_()
        launch(sim, box, lj, mode, (5, 12, 14), sc, dt=dt)
        return sc, int(sc["status"][12].item())

    # nothing moved: no flag; the gate words rotate: word 14 is cleared for the next launch
    sc, w = flags_after(None, 1e-9, NOW)
    assert w == 0
    # one particle moves 0.06 > delta / 2 in the step after the prune: inner rows expired
    # (the prune snapshot travels in ref.w; the rest of the snapshot is the list build's, so that
    # a particle the 1e-9 step carried across a face does not look displaced by a box edge)
    sc2 = fresh_scratch(sim)
    sc2["inner"], sc2["inner_counts"] = sc["inner"], sc["inner_counts"]
    sc2["ref"][:, 3] = sc["ref"][:, 3]
    _, w = flags_after(60.0, 0.001, INNER, first=sc2)
    assert w == 2
    # ... 0.04 < delta / 2: still fine
    sc3 = fresh_scratch(sim)
    sc3["inner"], sc3["inner_counts"] = sc["inner"], sc["inner_counts"]
    sc3["ref"][:, 3] = sc["ref"][:, 3]
    _, w = flags_after(40.0, 0.001, INNER, first=sc3)
    assert w == 0
    # a particle 0.12 > (skin - delta) / 2 from the list snapshot: pruning is not legal any more
    _, w = flags_after(None, 1e-9, OUTER, ref_shift=0.12)
    assert w == 6          # (... and, with no displacement recorded at "the prune", expired too)
    # ... 0.16 > skin / 2: new list
    _, w = flags_after(None, 1e-9, OUTER, ref_shift=0.16)
    assert w == 7          # (0.16 from the snapshot is also more than delta / 2 since "the prune")
    # gated launches return at once and hand the word on
    for mode, word in ((INNER, 2), (NOW, 4), (OUTER, 1), (INNER, 1)):
        sc4 = fresh_scratch(sim)
        sc4["status"][5] = word
        sc4["status"][14] = 99
        before = sc4["vel"].clone()
        launch(sim, box, lj, mode, (5, 12, 14), sc4)
        assert sc4["status"][13].item() == 0 and sc4["status"][12].item() == word
        assert sc4["status"][14].item() == 0
        assert torch.equal(sc4["vel"], before)
    sim.close()


@pytest.mark.parametrize("n,density,steps", [(262_144, 0.75, 230), (40_000, 1.2, 150)])
def test_native_loop_with_pruning_is_bit_identical_and_keeps_the_rebuild_schedule(n, density, steps):
    out = []
    for delta in (0.0, DELTA):
        lj = None
        if density > 1.0:
            lj = b2.PairTable.kob_andersen()
        sim, st, box, lj = make_sim(n, delta, density=density, lj=lj, sample_interval=40)
        sim.run(steps)
        prunes, outer_steps = sim.prune_stats()
        out.append((np.array([s.total_energy for s in sim.samples]),
                    np.array(st.positions.acquire_read(b2.HOST)),
                    np.array(st.velocities.acquire_read(b2.HOST)),
                    np.array(st.images.acquire_read(b2.HOST)), sim.rebuild_count, prunes,
                    outer_steps))
        sim.close()
    assert out[0][4] == out[1][4] and out[0][4] >= 3
    for a, b in zip(out[0][:4], out[1][:4]):
        assert np.array_equal(a, b)
    assert out[0][5] == 0 and out[1][5] >= 2 * out[1][4]
    # almost every one-launch step walked the inner rows
    assert out[1][6] <= 0.25 * steps
    print(f"n={n}: {out[1][4]} rebuilds, {out[1][5]} prunes, {out[1][6]} steps over the full rows")
