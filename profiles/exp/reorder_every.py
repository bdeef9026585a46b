"""ms per MD step at N = 1 M against the reorder cadence (Hilbert sort at every k-th rebuild)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2406_04210_b200 as b2

n = 1_000_000
for k in (1, 2, 3):
    st, box = b2.init_lattice_any(n, 0.75)
    b2.init_velocities(st, 1.2, 42)
    lj = b2.make_shifted(1.0, 1.0, 2.5)
    sim = b2.Simulation(st, box, lj, 0.001, force_mode=b2.TRUNCATED, skin=0.3, sample_interval=100,
                        reorder="hilbert", reorder_every=k)
    sim.run(400)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); r0 = sim.rebuild_count
    a.record(); sim.run(2000); b.record(); torch.cuda.synchronize()
    print(f"reorder_every={k}: {a.elapsed_time(b) / 2000:.5f} ms per step, {sim.rebuild_count - r0} rebuilds", flush=True)
    sim.close(); del sim, st
    torch.cuda.empty_cache()
