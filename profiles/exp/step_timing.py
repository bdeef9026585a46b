"""Quick A/B figure of merit on the GPU box (no CPU legs): ms per MD step of the molten
N = 1 M fluid, GPU time per rebuild (phase timers), and the step kernel timed alone.
    python profiles/exp/step_timing.py [steps] [n]"""
import os, sys, time, ctypes, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2406_04210_b200 as b2
from paper_2406_04210_b200 import _lib

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
skin = float(os.environ.get("B2MD_EXP_SKIN", "0.3"))
st, box = b2.init_lattice_any(n, 0.75)
b2.init_velocities(st, 1.2, 42)
lj = b2.make_shifted(1.0, 1.0, 2.5)
sim = b2.Simulation(st, box, lj, 0.001, force_mode=b2.TRUNCATED, skin=skin, sample_interval=100,
                    reorder="hilbert")
sim.run(400)
sim.reset_counters()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); sim.run(steps); b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / steps
out = {"ms_per_step": round(ms, 5), "particle_steps_per_s": round(n / ms * 1e3 / 1e9, 3),
       "rebuilds": sim.rebuild_count,
       "ms_per_rebuild": round(1e3 * sim.nlist_seconds / max(sim.rebuild_count, 1), 4),
       "rebuild_us_per_step": round(1e6 * sim.nlist_seconds / steps, 2),
       "other_us_per_step": round(1e6 * sim.force_seconds / steps, 2)}
if sim.pair_rows and sim.advance:
    dev = sim.state.device_state(); k = sim._keep; cfg = k["cfg"]
    tab = np.ascontiguousarray(lj.table()); tp = tab.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    scratch = {nm: getattr(dev, nm).clone() for nm in ("pos_lo", "vel", "image")}
    ref = k["ref_pos"].clone(); outp = torch.empty_like(dev.pos_hi)
    status = torch.zeros(16, dtype=torch.int32, device=dev.pos_hi.device)
    def launch():
        _lib.call("b2md_force_lj_pairs_advance", dev.pos_hi.data_ptr(), outp.data_ptr(),
                  scratch["pos_lo"].data_ptr(), scratch["vel"].data_ptr(), scratch["image"].data_ptr(),
                  n, box.c_box(), 1e-9, ref.data_ptr(), 1e30, k["pair_nbr"].data_ptr(),
                  k["pair_counts"].data_ptr(), cfg.pair_pitch, k["nbr"].data_ptr(),
                  k["counts"].data_ptr(), k["pitch"], k["boundary"].data_ptr(), tp, 1,
                  (4 if getattr(cfg, "pair_schedule", 0) and not os.environ.get("B2MD_EXP_UNSCHEDULED") else 0), 12, 14,
                  status.data_ptr(), dev.stream)
    launch(); torch.cuda.synchronize()
    a.record()
    for _ in range(50): launch()
    b.record(); torch.cuda.synchronize()
    out["advance_kernel_us"] = round(1e3 * a.elapsed_time(b) / 50, 2)
    os.environ["B2MD_EXP_NO_BOUNDARY"] = "1"       # timing only: wrong forces near the faces
    launch(); torch.cuda.synchronize()
    a.record()
    for _ in range(50): launch()
    b.record(); torch.cuda.synchronize()
    os.environ["B2MD_EXP_NO_BOUNDARY"] = "0"
    out["advance_kernel_us_without_image_shifts"] = round(1e3 * a.elapsed_time(b) / 50, 2)
    for v in (0, 8, 24, 56, 7):
        os.environ["B2MD_EXP_VARIANT"] = str(v)
        launch(); torch.cuda.synchronize()
        a.record()
        for _ in range(30): launch()
        b.record(); torch.cuda.synchronize()
        out[f"advance_kernel_us_all_warps_variant_{v}"] = round(1e3 * a.elapsed_time(b) / 30, 2)
    os.environ["B2MD_EXP_VARIANT"] = "-1"
    os.environ["B2MD_EXP_VARIANT"] = "0"
    for pct in (0, 50, 100):
        os.environ["B2MD_EXP_TILES_PCT"] = str(pct)
        launch(); torch.cuda.synchronize()
        a.record()
        for _ in range(30): launch()
        b.record(); torch.cuda.synchronize()
        out[f"v0_tiles{pct}"] = round(1e3 * a.elapsed_time(b) / 30, 2)
    os.environ["B2MD_EXP_TILES_PCT"] = "-1"
    os.environ["B2MD_EXP_UNSCHEDULED"] = "1"
    launch(); torch.cuda.synchronize()
    a.record()
    for _ in range(30): launch()
    b.record(); torch.cuda.synchronize()
    del os.environ["B2MD_EXP_UNSCHEDULED"]
    out["v0_unscheduled"] = round(1e3 * a.elapsed_time(b) / 30, 2)
    os.environ["B2MD_EXP_VARIANT"] = "-1"
    os.environ["B2MD_EXP_UNSCHEDULED"] = "1"
    launch(); torch.cuda.synchronize()
    a.record()
    for _ in range(30): launch()
    b.record(); torch.cuda.synchronize()
    del os.environ["B2MD_EXP_UNSCHEDULED"]
    out["advance_kernel_us_unscheduled"] = round(1e3 * a.elapsed_time(b) / 30, 2)
    bd = k["boundary"][:n] & 7
    out["boundary_particle_fraction"] = round(float((bd != 0).float().mean().item()), 4)
print(json.dumps(out))
