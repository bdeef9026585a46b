"""all2all-2k-long preset (N = 2000, 20 000 steps, untruncated all pairs; reference
bench.py:153-157) through the native all-to-all loop: throughput and energy drift."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2406_04210_b200 import harness
cfg = harness.PRESETS["all2all-2k-long"]
rec, samples = harness.run_benchmark(cfg)
e = np.array([s.total_energy for s in samples])
print(json.dumps({"preset": "all2all-2k-long", "steps": cfg.steps, "steps_per_second": rec.steps_per_second,
                  "drift_end_to_end": rec.final_energy_drift_rel,
                  "drift_max_over_samples": float(np.max(np.abs(e - e[0])) / abs(e[0])),
                  "samples": len(samples), "T_end": samples[-1].temperature,
                  "max_momentum": float(np.max(np.abs([s.total_momentum for s in samples])))}))
