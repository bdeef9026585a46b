"""What would binning pair rows by length buy?  (GPU box, N = 1 M molten fluid.)

A warp of the pair force kernel runs as many trips as its longest row has tiles.  This
script takes the real pair-row lengths after `--steps` MD steps and reports the mean
trips per warp (a) as laid out now (pair t in lane t), (b) if the pairs of every window
of W consecutive columns were sorted by length before being dealt to warps.  It also
times `b2md_pair_rows` on the final list with CUDA events.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2406_04210_b200 as b2
from paper_2406_04210_b200 import _lib

n = int(os.environ.get("N", 1_000_000))
steps = int(os.environ.get("STEPS", 600))
st, box = b2.init_lattice_any(n, 0.75)
b2.init_velocities(st, 1.2, 42)
sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001, force_mode=b2.TRUNCATED,
                    skin=0.3, sample_interval=100, reorder="hilbert", pair_rows=True)
sim.run(steps)
k = sim._keep
npairs = (n + 1) // 2
pc = (k["pair_counts"][:npairs].cpu().numpy() & 0xFFFF).astype(np.int64)
tiles = (pc + 3) // 4
full = npairs // 32 * 32


def warp_trips(t):
    return t[:full].reshape(-1, 32).max(1)


base = warp_trips(tiles)
print(f"pairs {npairs}  mean row {pc.mean():.2f}  mean tiles {tiles.mean():.3f}  "
      f"warp trips now {base.mean():.3f}  (global sort bound {np.sort(tiles)[:full].reshape(-1, 32).max(1).mean():.3f})")
for W in (64, 128, 256, 512, 1024, 4096):
    m = npairs // W * W
    srt = np.sort(tiles[:m].reshape(-1, W), axis=1).reshape(-1)
    trips = srt.reshape(-1, 32).max(1).mean()
    print(f"  window {W:5d}: warp trips {trips:.3f}  ({trips / base.mean():.3f} of now)")
# CTA-level imbalance: trips of the slowest warp of each 128-thread CTA
cta = base[: base.size // 4 * 4].reshape(-1, 4)
print(f"CTA (4 warps): mean of max {cta.max(1).mean():.3f}  mean {cta.mean():.3f}")

cfg = k["cfg"]
lib = _lib.load()
s = torch.cuda.current_stream().cuda_stream
rows = int(k["nbr"].shape[0])
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for rep in range(3):
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(5):
        _lib.call("b2md_pair_rows", k["nbr"].data_ptr(), k["counts"].data_ptr(), cfg.pitch, rows, n,
                  k["pair_nbr"].data_ptr(), k["pair_counts"].data_ptr(), cfg.pair_pitch,
                  cfg.pair_rows, s)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"b2md_pair_rows: {ev[0].elapsed_time(ev[1]) / 5 * 1e3:.1f} us")
sim.close()
