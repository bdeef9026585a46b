"""Where Simulation() spends its time at N = 1 M (runner creation, first build, first forces)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2406_04210_b200 as b2
from paper_2406_04210_b200 import sim as simmod, _lib

n = 1_000_000
st0, box = b2.init_lattice_any(n, 0.75)
b2.init_velocities(st0, 1.2, 42)
pos0 = np.array(st0.positions.acquire_read(b2.HOST)); vel0 = np.array(st0.velocities.acquire_read(b2.HOST))
lj = b2.make_shifted(1.0, 1.0, 2.5)
laps = {}
lib = _lib.load()
for name in ("b2md_runner_create", "b2md_runner_destroy"):
    orig = getattr(lib, name)
    def wrap(*a, _orig=orig, _name=name):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = _orig(*a)
        torch.cuda.synchronize(); laps[_name] = 1e3 * (time.perf_counter() - t)
        return r
    setattr(lib, name, wrap)
orig_call = simmod.Simulation._native_call
def timed_call(self, name, *a):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = orig_call(self, name, *a)
    torch.cuda.synchronize(); laps[name] = laps.get(name, 0) + 1e3 * (time.perf_counter() - t)
    return r
simmod.Simulation._native_call = timed_call
for rep in range(5):
    laps.clear()
    st = b2.ParticleState(pos0, velocities=vel0, copy=False)
    st.sync_to_compute(); torch.cuda.synchronize()
    t = time.perf_counter()
    sim = b2.Simulation(st, box, lj, 0.001, force_mode=b2.TRUNCATED, skin=0.3, sample_interval=100)
    torch.cuda.synchronize(); total = 1e3 * (time.perf_counter() - t)
    t = time.perf_counter(); sim.run(20); torch.cuda.synchronize(); run = 1e3 * (time.perf_counter() - t)
    t = time.perf_counter(); sim.close(); torch.cuda.synchronize(); close = 1e3 * (time.perf_counter() - t)
    print(f"rep {rep}: Simulation() {total:.2f} ms; run(20) {run:.2f}; close {close:.2f}; "
          + ", ".join(f"{k} {v:.2f}" for k, v in laps.items()))
    del sim, st
