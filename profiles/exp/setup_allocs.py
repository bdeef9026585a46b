"""Allocation / zero-fill share of Simulation() at N = 1 M."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2406_04210_b200 as b2

n = 1_000_000
st0, box = b2.init_lattice_any(n, 0.75)
b2.init_velocities(st0, 1.2, 42)
pos0 = np.array(st0.positions.acquire_read(b2.HOST)); vel0 = np.array(st0.velocities.acquire_read(b2.HOST))
host_pos = torch.from_numpy(pos0).pin_memory().numpy(); host_vel = torch.from_numpy(vel0).pin_memory().numpy()
lj = b2.make_shifted(1.0, 1.0, 2.5)
acc = {"zeros": 0.0, "zeros_like": 0.0, "bytes": 0}
for name in ("zeros", "zeros_like", "empty", "empty_like"):
    orig = getattr(torch, name)
    def wrap(*a, _orig=orig, _name=name, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        out = _orig(*a, **k)
        torch.cuda.synchronize(); acc[_name] = acc.get(_name, 0.0) + 1e3 * (time.perf_counter() - t)
        acc["bytes"] += out.numel() * out.element_size()
        return out
    setattr(torch, name, wrap)
for rep in range(4):
    for k in acc: acc[k] = 0
    torch.cuda.synchronize(); t0 = time.perf_counter()
    st = b2.ParticleState(host_pos, velocities=host_vel, copy=False)
    st.sync_to_compute(); torch.cuda.synchronize(); t1 = time.perf_counter()
    up = dict(acc)
    sim = b2.Simulation(st, box, lj, 0.001, force_mode=b2.TRUNCATED, skin=0.3, sample_interval=100)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"rep {rep}: upload {1e3*(t1-t0):.2f} ms (allocs {up}); Simulation() {1e3*(t2-t1):.2f} ms, "
          f"allocs+fills {({k: round(v - up.get(k, 0), 2) for k, v in acc.items()})}")
    sim.close(); del sim, st
print(torch.cuda.memory_summary(abbreviated=True)[:1500])
