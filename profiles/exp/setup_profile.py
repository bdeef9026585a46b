import os, sys, time, cProfile, pstats
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2406_04210_b200 as b2
n=1_000_000
st0, box = b2.init_lattice_any(n, 0.75)
b2.init_velocities(st0, 1.2, 42)
pos0 = np.array(st0.positions.acquire_read(b2.HOST)); vel0 = np.array(st0.velocities.acquire_read(b2.HOST))
lj = b2.make_shifted(1.0, 1.0, 2.5)
for rep in range(3):
    st = b2.ParticleState(pos0.copy(), velocities=vel0.copy(), copy=False)
    st.sync_to_compute(); torch.cuda.synchronize()
    pr=cProfile.Profile()
    t=time.perf_counter(); pr.enable()
    sim = b2.Simulation(st, box, lj, 0.001, force_mode=b2.TRUNCATED, skin=0.3, sample_interval=100)
    torch.cuda.synchronize(); pr.disable(); print("Simulation()", (time.perf_counter()-t)*1e3, "stride", sim.stride, "rebuilds", sim.rebuild_count)
    t=time.perf_counter(); sim.run(1); torch.cuda.synchronize(); print("run(1)", (time.perf_counter()-t)*1e3)
    if rep==2: pstats.Stats(pr).sort_stats('cumtime').print_stats(25)
    sim.close()
