"""Where a step of a small system goes: steps only (no sample inside the timed run),
phase timers of the native loop (CUDA events), rebuild count.
    python profiles/exp/small_n_phases.py [n ...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2406_04210_b200 as b2

def run(n, steps, persistent):
    st, box = b2.init_lattice_any(n, 0.75)
    b2.init_velocities(st, 1.2, 42)
    sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001, force_mode=b2.TRUNCATED,
                        skin=0.3, sample_interval=10 ** 9, persistent_steps=persistent)
    sim.run(1000)
    sim.reset_counters()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    sim.run(steps)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    out = {"n": n, "persistent_steps": persistent, "us_per_step": 1e3 * ms / steps,
           "rebuilds": sim.rebuild_count, "launches": sim.kernel_launches,
           "force_us_per_step": 1e6 * sim.force_seconds / steps,
           "nlist_us_per_step": 1e6 * sim.nlist_seconds / steps,
           "nlist_us_per_rebuild": 1e6 * sim.nlist_seconds / max(1, sim.rebuild_count)}
    sim.close()
    return out

for n in [int(x) for x in sys.argv[1:]] or [4096, 65536]:
    for p in (0, 256):
        print(json.dumps(run(n, 4000, p)), flush=True)
