"""All-pairs LJ kernel (k_force_all_pairs) against the FP32 issue roofline.
    python profiles/exp/all_pairs_roofline.py [n ...]
One JSON line per N: pair evaluations per second, warp instructions per evaluation
are taken from the ncu capture named in profiles/README.md; the roofline here is the
evaluation rate a B200 reaches if every FP32 lane issues one instruction per clock."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2406_04210_b200 as b2

SM, LANES, GHZ = 148, 128, 1.965            # B200: 148 SMs x 128 FP32 lanes, max SM clock

def run(n, reps=20):
    st, box = b2.init_lattice_any(n, 0.75)
    lj = b2.make_shifted(1.0, 1.0, 2.5)
    for _ in range(3):
        b2.compute_forces_all_to_all(st, lj, box)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        b2.compute_forces_all_to_all(st, lj, box)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    evals = float(n) * n
    rate = evals / ms * 1e3
    lane_rate = SM * LANES * GHZ * 1e9
    return {"n": n, "ms_per_call": ms, "pair_evaluations_per_s": rate,
            "fp32_lane_instructions_per_s_peak": lane_rate,
            "lane_slots_per_evaluation_at_this_rate": lane_rate / rate}

for n in [int(x) for x in sys.argv[1:]] or [2000, 8192, 32768, 131072]:
    print(json.dumps(run(n)), flush=True)
