"""What a tile redistribution inside each force-kernel warp could save: the warp runs T_cut
trips over its own rows plus ceil(overflow / 32) trips over the excess tiles of its long rows
(each about 1.6 x the cost of a normal trip: operands fetched by shuffle, partial sums returned).
    python profiles/exp/balance_stats.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2406_04210_b200 as b2

n = 1_000_000
st, box = b2.init_lattice_any(n, 0.75)
b2.init_velocities(st, 1.2, 42)
sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001, force_mode=b2.TRUNCATED, skin=0.3,
                    sample_interval=100, reorder="hilbert")
sim.run(400)
k = sim._keep; cfg = k["cfg"]
c = k["pair_counts"][:cfg.pair_pitch].cpu().numpy()
t = ((c + 3) // 4)[: (len(c) // 32) * 32].reshape(-1, 32)
t = t[t.max(axis=1) > 0]
now = t.max(axis=1).mean()
best = {}
for extra_cost in (1.3, 1.6, 2.0):
    tot = []
    for w in t[::7]:
        lo, hi = int(np.floor(w.mean())), int(w.max())
        cand = [tc + extra_cost * np.ceil(np.maximum(w - tc, 0).sum() / 32.0) for tc in range(lo, hi + 1)]
        tot.append(min(cand))
    best[extra_cost] = float(np.mean(tot))
print(json.dumps({"tiles_per_warp_now": float(now), "mean_row_tiles": float(t.mean()),
                  "std_within_warp": float(t.std(axis=1).mean()),
                  "balanced_trips_at_overflow_trip_cost": best}))
