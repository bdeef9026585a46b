"""Native all-to-all loop, steps only: GPU time per step (CUDA events of the call) and host
wall time per step, NVE, no sample inside the timed call.
    python profiles/exp/all_pairs_steps.py [n ...]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2406_04210_b200 as b2

def run(n, steps):
    st, box = b2.init_lattice_any(n, 0.8)
    b2.init_velocities(st, 1.0, 42)
    sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0), 0.002, sample_interval=10 ** 9)
    sim.run(200)
    sim.reset_counters()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim.run(steps)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    out = {"n": n, "steps": steps, "wall_us_per_step": 1e6 * wall / steps,
           "gpu_us_per_step": 1e6 * sim.force_seconds / steps, "launches": sim.kernel_launches}
    sim.close()
    return out

for n in [int(x) for x in sys.argv[1:]] or [256, 2000, 8000]:
    print(json.dumps(run(n, 2000)), flush=True)
