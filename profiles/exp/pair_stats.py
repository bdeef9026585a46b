"""Distribution of pair-row lengths and partner distances at N = 1 M (GPU box)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2406_04210_b200 as b2

n = 1_000_000
st, box = b2.init_lattice_any(n, 0.75)
b2.init_velocities(st, 1.2, 42)
sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001, force_mode=b2.TRUNCATED,
                    skin=0.3, sample_interval=100, reorder="hilbert", pair_rows=True)
sim.run(600)
k = sim._keep
pc = k["pair_counts"][: (n + 1) // 2].cpu().numpy()
c = k["counts"][:n].cpu().numpy()
print("rows: mean", c.mean(), "max", c.max(), "warp-max mean", c[: n // 32 * 32].reshape(-1, 32).max(1).mean())
print("pair rows: mean", pc.mean(), "p50", np.percentile(pc, 50), "p90", np.percentile(pc, 90),
      "p99", np.percentile(pc, 99), "max", pc.max())
m = pc[: pc.size // 32 * 32].reshape(-1, 32)
print("warp-max mean", m.max(1).mean(), "warp-mean", m.mean(1).mean(), "tiles mean", np.ceil(m.max(1) / 4).mean())
dev = sim.state.device_state()
p = dev.pos_hi[:n, :3].double().cpu().numpy()
L = box.edge_lengths[0]
d = p[0::2] - p[1::2]
d -= L * np.rint(d / L)
r = np.sqrt((d * d).sum(1))
print("partner distance: mean", r.mean(), "p50", np.percentile(r, 50), "p90", np.percentile(r, 90), "p99", np.percentile(r, 99), "max", r.max())
for lo, hi in [(0, 1), (1, 1.5), (1.5, 2), (2, 3), (3, 10)]:
    sel = (r >= lo) & (r < hi)
    print(f"  d in [{lo},{hi}): frac {sel.mean():.3f} mean union {pc[sel].mean() if sel.any() else 0:.1f}")
cell = k["cell_of"][:n].cpu().numpy()
print("same-cell partners:", (cell[0::2] == cell[1::2]).mean())
