"""A/B timing of force-kernel variants on the molten N = 1 M state (GPU box).
Each variant runs in its own process (the library reads its env knobs once)."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r'''
import os, sys, ctypes
sys.path.insert(0, %r)
import numpy as np, torch
import paper_2406_04210_b200 as b2
from paper_2406_04210_b200 import _lib
n = 1_000_000
st, box = b2.init_lattice_any(n, 0.75)
b2.init_velocities(st, 1.2, 42)
lj = b2.make_shifted(1.0, 1.0, 2.5)
sim = b2.Simulation(st, box, lj, 0.001, force_mode=b2.TRUNCATED, skin=0.3, sample_interval=100, reorder="hilbert", pair_rows=True)
sim.run(500)
dev = sim.state.device_state(); k = sim._keep; cfg = k["cfg"]
tab = np.ascontiguousarray(lj.table()); tp = tab.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
def launch():
    _lib.call("b2md_force_lj_pairs", dev.pos_hi.data_ptr(), n, box.c_box(), k["pair_nbr"].data_ptr(), k["pair_counts"].data_ptr(), cfg.pair_pitch,
              k["nbr"].data_ptr(), k["counts"].data_ptr(), k["pitch"], k["boundary"].data_ptr(), tp, 1, 1,
              dev.force.data_ptr(), dev.virial.data_ptr(), dev.status.data_ptr(), dev.stream)
launch(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50): launch()
b.record(); torch.cuda.synchronize()
print("RESULT", a.elapsed_time(b) / 50)
'''
for env in sys.argv[1:]:
    e = dict(os.environ)
    for kv in env.split(","):
        if "=" in kv:
            key, val = kv.split("=", 1); e[key] = val
    out = subprocess.run([sys.executable, "-c", CHILD % ROOT], env=e, capture_output=True, text=True)
    res = [l for l in out.stdout.splitlines() if l.startswith("RESULT")]
    print(env, res[0] if res else out.stderr[-800:])
