"""all2all-2k preset of the harness (the reference's untruncated N = 2000 benchmark,
bench.py:147-151) through the native all-to-all loop; and the operator loop beside it.
    python profiles/exp/all_pairs_preset.py"""
import dataclasses, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2406_04210_b200 as b2
from paper_2406_04210_b200 import harness

for name in ("all2all-2k", "smoke-256"):
    cfg = harness.PRESETS[name]
    rec, _ = harness.run_benchmark(cfg)
    rec, _ = harness.run_benchmark(cfg)
    print(json.dumps({"preset": name, "steps_per_second": rec.steps_per_second,
                      "us_per_step": 1e6 / rec.steps_per_second,
                      "pair_evaluations_per_s": rec.steps_per_second * cfg.n_particles ** 2,
                      "drift": rec.final_energy_drift_rel,
                      "force_time_fraction": rec.force_time_fraction}), flush=True)
