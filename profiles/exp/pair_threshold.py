"""ms per MD step with and without pair rows across system sizes (GPU box)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2406_04210_b200 as b2
for n in (32_768, 65_536, 131_072, 262_144, 524_288):
    out = []
    for pr in (False, True):
        st, box = b2.init_lattice_any(n, 0.75)
        b2.init_velocities(st, 1.2, 42)
        sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001, force_mode=b2.TRUNCATED,
                            skin=0.3, sample_interval=100, pair_rows=pr)
        sim.run(300)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); sim.run(1000); b.record(); torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / 1000)
        sim.close()
    print(n, "rows %.4f ms/step, pair rows %.4f ms/step" % tuple(out), flush=True)
