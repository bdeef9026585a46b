#!/usr/bin/env python
"""Where the end-to-end call spends its time (host arrays -> run -> host arrays)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_04210_b200 as b2

n, steps = 1_000_000, int(sys.argv[1]) if len(sys.argv) > 1 else 200
st0, box = b2.init_lattice_any(n, 0.75)
b2.init_velocities(st0, 1.2, 42)
pos0 = np.array(st0.positions.acquire_read(b2.HOST)); vel0 = np.array(st0.velocities.acquire_read(b2.HOST))
host_pos = torch.from_numpy(pos0).pin_memory().numpy(); host_vel = torch.from_numpy(vel0).pin_memory().numpy()
lj = b2.make_shifted(1.0, 1.0, 2.5)
for rep in range(3):
    host_pos[...] = pos0; host_vel[...] = vel0
    torch.cuda.synchronize(); t = [time.perf_counter()]
    def lap(): torch.cuda.synchronize(); t.append(time.perf_counter())
    st = b2.ParticleState(host_pos, velocities=host_vel, copy=False); lap()
    st.sync_to_compute(); lap()
    sim = b2.Simulation(st, box, lj, 0.001, force_mode=b2.TRUNCATED, skin=0.3, sample_interval=100); lap()
    sim.run(steps); lap()
    s = sim.measure(); lap()
    p = st.positions.acquire_read(b2.HOST); v = st.velocities.acquire_read(b2.HOST); lap()
    sim.close()
    names = ["ParticleState()", "sync_to_compute (H2D+pack)", "Simulation() (alloc+first list+forces)", f"run({steps})", "measure", "download pos+vel"]
    print(f"rep {rep}: total {1e3*(t[-1]-t[0]):.1f} ms | " + " | ".join(f"{nm} {1e3*(b-a):.1f}" for nm, a, b in zip(names, t, t[1:])))
    del sim, st
