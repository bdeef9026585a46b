"""Which image-shift variant the warps of the pair kernel take (molten N = 1 M)."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2406_04210_b200 as b2
n = 1_000_000
st, box = b2.init_lattice_any(n, 0.75)
b2.init_velocities(st, 1.2, 42)
sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001, force_mode=b2.TRUNCATED, skin=0.3,
                    sample_interval=100, reorder="hilbert")
sim.run(400)
bd = sim._keep["boundary"][:n].cpu().numpy().astype(np.int64)
print("byte histogram", dict(sorted(collections.Counter(bd.tolist()).items())))
w = bd[: n // 64 * 64].reshape(-1, 64)
near = np.bitwise_or.reduce(w & 7, axis=1)
clear = np.bitwise_and.reduce(w >> 3, axis=1)
ok = (near & ~clear) == 0
variant = np.where(ok, near << 3, np.where(near != 0, 7, 0))
print("warps", w.shape[0], "variant histogram", dict(sorted(collections.Counter(variant.tolist()).items())))
print("flagged warps", float((near != 0).mean()), "careful axes per warp", float(np.array([bin(int(x)).count('1') for x in near]).mean()))
