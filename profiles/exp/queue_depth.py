"""ms per MD step of small systems: host-driven row kernel vs queued one-launch steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2406_04210_b200 as b2
for n in (4096, 16_384, 65_536, 131_072, 262_144):
    res = []
    for kw in (dict(pair_rows=False, advance=False), dict(pair_rows=False, advance=True, queue_depth=1),
               dict(pair_rows=False, advance=True, queue_depth=4),
               dict(pair_rows=False, advance=True, queue_depth=16)):
        st, box = b2.init_lattice_any(n, 0.75)
        b2.init_velocities(st, 1.2, 42)
        sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001, force_mode=b2.TRUNCATED,
                            skin=0.3, sample_interval=100, **kw)
        sim.run(300)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); sim.run(2000); b.record(); torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / 2000)
        sim.close()
    print(n, "rows, separate launches %.4f | one-launch steps, depth 1: %.4f, 4: %.4f, 16: %.4f ms/step" % tuple(res), flush=True)
