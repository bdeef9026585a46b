"""Short run of a harness preset for an ncu launch list.
    python profiles/exp/preset_launches.py trunc-10k 300"""
import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2406_04210_b200 import harness
cfg = dataclasses.replace(harness.PRESETS[sys.argv[1]], steps=int(sys.argv[2]), equilibration_steps=50)
rec, _ = harness.run_benchmark(cfg)
print(rec.steps_per_second)
