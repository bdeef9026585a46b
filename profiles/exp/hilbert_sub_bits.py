"""ms per MD step at N = 1 M against the resolution of the Hilbert key (sub-cell bits per axis)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2406_04210_b200 as b2
from paper_2406_04210_b200 import sim as simmod

n = 1_000_000
for bits in (0, 1, 2, 3, 4):
    simmod.HILBERT_SUB_BITS = bits
    st, box = b2.init_lattice_any(n, 0.75)
    b2.init_velocities(st, 1.2, 42)
    lj = b2.make_shifted(1.0, 1.0, 2.5)
    sim = b2.Simulation(st, box, lj, 0.001, force_mode=b2.TRUNCATED, skin=0.3, sample_interval=100,
                        reorder="hilbert")
    sim.run(400)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); r0 = sim.rebuild_count
    a.record(); sim.run(2000); b.record(); torch.cuda.synchronize()
    print(f"sub_bits={bits}: {a.elapsed_time(b) / 2000:.5f} ms per step, {sim.rebuild_count - r0} rebuilds", flush=True)
    sim.close(); del sim, st
    torch.cuda.empty_cache()
