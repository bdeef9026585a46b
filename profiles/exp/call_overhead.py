"""Host-side cost of one Simulation.run() call of the native loop (cProfile over many short
calls at N = 1 M, pair rows: the gap between two calls is GPU idle time at 20 steps per call).
    python profiles/exp/call_overhead.py"""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2406_04210_b200 as b2

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
st, box = b2.init_lattice_any(n, 0.75)
b2.init_velocities(st, 1.2, 42)
sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001, force_mode=b2.TRUNCATED, skin=0.3,
                    sample_interval=100)
sim.run(200)
torch.cuda.synchronize()
for k in (20, 1):
    t0 = time.perf_counter()
    for _ in range(100):
        sim.run(k)
    torch.cuda.synchronize()
    print(f"run({k}): {1e3 * (time.perf_counter() - t0) / 100:.4f} ms per call")
pr = cProfile.Profile()
pr.enable()
for _ in range(300):
    sim.run(1)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
