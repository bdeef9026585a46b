"""Fixed vs per-tile cost of the pair kernel: rows truncated to a fraction of their length
(GPU box only; the forces are then wrong on purpose)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2406_04210_b200 as b2
from paper_2406_04210_b200 import _lib

n = 1_000_000
st, box = b2.init_lattice_any(n, 0.75)
b2.init_velocities(st, 1.2, 42)
lj = b2.make_shifted(1.0, 1.0, 2.5)
sim = b2.Simulation(st, box, lj, 0.001, force_mode=b2.TRUNCATED, skin=0.3, sample_interval=100,
                    reorder="hilbert", pair_rows=True)
sim.run(500)
dev = sim.state.device_state(); k = sim._keep; cfg = k["cfg"]
tab = np.ascontiguousarray(lj.table()); tp = tab.ctypes.data_as(ctypes.POINTER(ctypes.c_double))

def launch():
    _lib.call("b2md_force_lj_pairs", dev.pos_hi.data_ptr(), n, box.c_box(), k["pair_nbr"].data_ptr(),
              k["pair_counts"].data_ptr(), cfg.pair_pitch, k["nbr"].data_ptr(), k["counts"].data_ptr(),
              k["pitch"], k["boundary"].data_ptr(), tp, 1, 1, dev.force.data_ptr(),
              dev.virial.data_ptr(), dev.status.data_ptr(), dev.stream)

def timeit(tag):
    launch(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(30): launch()
    b.record(); torch.cuda.synchronize()
    print(tag, round(a.elapsed_time(b) / 30 * 1e3, 1), "us", flush=True)

orig = k["pair_counts"].clone()
for frac in (1.0, 0.75, 0.5, 0.25, 0.0):
    k["pair_counts"].copy_((orig.float() * frac).to(torch.int32))
    timeit(f"rows x {frac}")
# every row the same length (no warp-max padding, no imbalance between warps)
k["pair_counts"].copy_(torch.full_like(orig, 88))
timeit("all rows 88 entries (22 tiles)")
k["pair_counts"].copy_(torch.full_like(orig, 108))
timeit("all rows 108 entries (27 tiles)")
