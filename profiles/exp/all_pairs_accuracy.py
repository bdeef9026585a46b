"""Error of the all-pairs kernel against the fp64 oracle (untruncated LJ, fluid-like state):
M1 (per-particle, relative to its own net force), M3 (relative to the rms force), L2.
    python profiles/exp/all_pairs_accuracy.py [n ...]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2406_04210_b200 as b2
from helpers import fluid_state, force_error_metrics, quantize_f32, scalar_rel_error
from oracle import oracle as orc

for n in [int(x) for x in sys.argv[1:]] or [2000, 12500]:
    pos, _, edge = fluid_state(n, density=0.8, seed=5)
    pos = quantize_f32(pos)
    lj = b2.make_shifted(1.0, 1.0)
    st = b2.ParticleState(pos)
    b2.compute_forces_all_to_all(st, lj, b2.SimBox.cubic(edge))
    rf, rpe, rw = orc.forces_all_pairs(pos, [edge] * 3, lj.table(), threads=orc.host_threads())
    f = np.array(st.forces.acquire_read(b2.HOST))
    m = force_error_metrics(f, rf)
    m["L2"] = float(np.linalg.norm(f - rf) / np.linalg.norm(rf))
    m["pe_rel"] = scalar_rel_error(st.per_particle_potential.acquire_read(b2.HOST), rpe)
    m["virial_rel"] = scalar_rel_error(st.virial.acquire_read(b2.HOST), rw)
    m["n"] = n
    print(json.dumps(m), flush=True)
