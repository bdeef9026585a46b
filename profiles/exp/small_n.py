"""Per-step time of small systems: persistent step kernel vs one launch per step.
    python profiles/exp/small_n.py [n ...]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2406_04210_b200 as b2

def run(n, steps, persistent, interval):
    st, box = b2.init_lattice_any(n, 0.75)
    b2.init_velocities(st, 1.2, 42)
    sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001, force_mode=b2.TRUNCATED,
                        skin=0.3, sample_interval=interval, persistent_steps=persistent)
    sim.run(500)
    sim.reset_counters()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sim.run(steps)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    e = sim.measure().total_energy
    out = {"n": n, "persistent_steps": persistent, "us_per_step": round(1e6 * dt / steps, 2),
           "particle_steps_per_s": round(n * steps / dt / 1e9, 3), "rebuilds": sim.rebuild_count,
           "launches": sim.kernel_launches, "E": e}
    sim.close()
    return out

for n in [int(x) for x in sys.argv[1:]] or [4096, 16384, 65536, 131072]:
    for p in (0, 256):
        print(json.dumps(run(n, 2000, p, 100)))
