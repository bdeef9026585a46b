"""How much of the pair kernel's time is gather locality?  Times the kernel on the real
pair rows, on rows whose indices are replaced by near-diagonal ones (perfect locality,
same flags / lengths) and by uniformly random ones (no locality).  GPU box only."""
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
    print(tag, a.elapsed_time(b) / 30, flush=True)

timeit("real rows")
pn = k["pair_nbr"]                       # (tiles, pitch, 4)
tiles, pitch, _ = pn.shape
flags = pn & 3
t_idx = torch.arange(pitch, device=pn.device, dtype=torch.int64).view(1, pitch, 1)
kk = (torch.arange(tiles, device=pn.device, dtype=torch.int64).view(tiles, 1, 1) * 4
      + torch.arange(4, device=pn.device, dtype=torch.int64).view(1, 1, 4))
orig = pn.clone()
near = (2 * t_idx + kk + n // 2) % n          # far away in space: no pair inside the cutoff
pn.copy_(((near << 2) | flags).to(torch.int32))
timeit("near-diagonal indices (all lanes of a warp within ~100 rows)")
same = ((2 * (t_idx // 32) * 32 + kk + n // 2) % n).expand(tiles, pitch, 4)
pn.copy_(((same << 2) | flags).to(torch.int32))
timeit("warp-uniform indices (one line per gather)")
rnd = torch.randint(0, n, (tiles, pitch, 4), device=pn.device, dtype=torch.int64)
flags = flags * 0                              # random partners may coincide: mask everything
pn.copy_(((rnd << 2) | flags).to(torch.int32))
timeit("random indices")
pn.copy_((orig & ~3))
timeit("real rows, all flags off (no evaluation contributes)")
