"""N = 1 M NVE, 20 000 steps after 1000: ms per step, energy drift, rebuilds (stability check).
    python profiles/exp/long_run.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch, json
import paper_2406_04210_b200 as b2
n = 1_000_000
st, box = b2.init_lattice_any(n, 0.75)
b2.init_velocities(st, 1.2, 42)
sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001, force_mode=b2.TRUNCATED, skin=0.3,
                    sample_interval=500, sample_initial=True)
sim.run(1000); sim.samples.clear(); sim.samples.append(sim.measure())
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); sim.run(20000); b.record(); torch.cuda.synchronize()
e = np.array([s.total_energy for s in sim.samples]); p = np.array([s.total_momentum for s in sim.samples])
print(json.dumps({"n": n, "steps": 20000, "ms_per_step": a.elapsed_time(b) / 20000,
                  "drift_end_to_end": abs(e[-1] - e[0]) / abs(e[0]), "drift_max": float(np.max(np.abs(e - e[0])) / abs(e[0])),
                  "rebuilds": sim.rebuild_count, "T_end": sim.samples[-1].temperature,
                  "max_momentum_norm": float(np.max(np.linalg.norm(p, axis=1))), "overflow_events": sim.overflow_events}))
