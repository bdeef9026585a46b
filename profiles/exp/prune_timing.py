"""One-launch step over the full rows, over pruned rows, and the prune launch itself, timed alone on
the molten N = 1 M fluid (CUDA events, 30 launches each); entries per pair row before / after.
    python profiles/exp/prune_timing.py [delta]"""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2406_04210_b200 as b2
from paper_2406_04210_b200 import _lib

delta = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
st, box = b2.init_lattice_any(n, 0.75)
b2.init_velocities(st, 1.2, 42)
lj = b2.make_shifted(1.0, 1.0, 2.5)
sim = b2.Simulation(st, box, lj, 0.001, force_mode=b2.TRUNCATED, skin=0.3, sample_interval=100,
                    reorder="hilbert", prune_delta=0.0)
sim.run(400)
dev = sim.state.device_state(); k = sim._keep; cfg = k["cfg"]
tab = np.ascontiguousarray(lj.table()); tp = tab.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
sc = {nm: getattr(dev, nm).clone() for nm in ("pos_lo", "vel", "image")}
ref = k["ref_pos"].clone(); out = torch.empty_like(dev.pos_hi)
inner = torch.zeros_like(k["pair_nbr"]); inner_counts = torch.zeros(cfg.pair_pitch, dtype=torch.int32, device=out.device)
status = torch.zeros(16, dtype=torch.int32, device=out.device)
def launch(mode):
    status.zero_()
    _lib.call("b2md_force_lj_pairs_advance_pruned", dev.pos_hi.data_ptr(), out.data_ptr(),
              sc["pos_lo"].data_ptr(), sc["vel"].data_ptr(), sc["image"].data_ptr(), n, box.c_box(),
              1e-9, ref.data_ptr(), 1e30, k["pair_nbr"].data_ptr(), k["pair_counts"].data_ptr(),
              cfg.pair_pitch, k["nbr"].data_ptr(), k["counts"].data_ptr(), k["pitch"],
              k["boundary"].data_ptr(), tp, 1, 4 if cfg.pair_schedule else 0, 5, 12, 14, mode,
              inner.data_ptr(), inner_counts.data_ptr(), cfg.pair_rows, 2.5, 0.3, delta,
              status.data_ptr(), dev.stream)
def legacy():
    _lib.call("b2md_force_lj_pairs_advance", dev.pos_hi.data_ptr(), out.data_ptr(),
              sc["pos_lo"].data_ptr(), sc["vel"].data_ptr(), sc["image"].data_ptr(), n, box.c_box(),
              1e-9, ref.data_ptr(), 1e30, k["pair_nbr"].data_ptr(), k["pair_counts"].data_ptr(),
              cfg.pair_pitch, k["nbr"].data_ptr(), k["counts"].data_ptr(), k["pitch"],
              k["boundary"].data_ptr(), tp, 1, 4 if cfg.pair_schedule else 0, 12, 14,
              status.data_ptr(), dev.stream)
def timeit(fn, reps=30):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize(); a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return 1e3 * a.elapsed_time(b) / reps
launch(2); torch.cuda.synchronize()
res = {"delta": delta, "n": n,
       "outer_entries_per_pair": float(k["pair_counts"][:cfg.pair_pitch].float().sum().item()) / ((n + 1) // 2),
       "inner_entries_per_pair": float(inner_counts.float().sum().item()) / ((n + 1) // 2)}
def warp_tiles(c):
    t = (c[: (len(c) // 32) * 32].view(-1, 32) + 3) // 4
    return float(t.max(dim=1).values.float().mean().item()), float(t.float().mean().item())
res["outer_tiles_warp_max_mean"] = warp_tiles(k["pair_counts"][:cfg.pair_pitch])
res["inner_tiles_warp_max_mean"] = warp_tiles(inner_counts)
res["legacy_us"] = round(timeit(legacy), 2)
res["outer_mode_us"] = round(timeit(lambda: launch(3)), 2)
res["inner_mode_us"] = round(timeit(lambda: launch(1)), 2)
res["prune_launch_us"] = round(timeit(lambda: launch(2)), 2)
import json; print(json.dumps(res))
