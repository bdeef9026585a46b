#!/usr/bin/env python
"""Per-kernel roofline table from one `ncu --set full` report holding every launch of a
window of MD steps (profiles/capture_all_kernels.sh):
    python profiles/kernel_roofline.py gpurun_out/allkernels.ncu-rep [hbm_peak_GBps]
For each kernel: launches in the window, mean duration, DRAM bytes per launch (read +
write), achieved DRAM GB/s and its fraction of the measured HBM peak, L2 throughput,
issue-slot and FP32 (FMA pipe) utilisation.  Durations under ncu are cold-cache and
serialised: compare shares and fractions, not absolute step times."""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

COLS = {
    "t": "gpu__time_duration.sum",
    "rd": "dram__bytes_read.sum",
    "wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "fma": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "alu": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3,
         "second": 1e6}


def peak_default():
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(path))["hbm_gbs"])
    except Exception:       # noqa: BLE001
        return 6456.5


def main():
    rep = sys.argv[1]
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else peak_default()
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {k: hdr.index(v) for k, v in COLS.items() if v in hdr}
    name_col = hdr.index("Kernel Name")
    agg = defaultdict(lambda: defaultdict(float))
    for r in rows[2:]:
        name = r[name_col]
        if "at::" in name or "elementwise" in name:
            name = "(torch fill / copy)"
        name = name.replace("void ", "").replace("b2md::", "").split("(")[0]
        a = agg[name]
        a["n"] += 1
        for k, c in idx.items():
            v = float(r[c].replace(",", "") or 0.0)
            if k in ("t", "rd", "wr"):
                v *= SCALE.get(units[c], 1.0)
            a[k] += v
    total_t = sum(a["t"] for a in agg.values())
    print(f"HBM peak used for the fractions: {peak:.1f} GB/s (MEASURED_PEAKS.json hbm_gbs)")
    print(f"{'kernel':44s} {'n':>4s} {'avg us':>8s} {'share':>6s} {'MB/launch':>10s} "
          f"{'GB/s':>7s} {'/peak':>6s} {'L2%':>5s} {'L1%':>5s} {'issue%':>6s} {'fma%':>5s} "
          f"{'alu%':>5s} {'regs':>4s}")
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        n = a["n"]
        t = a["t"] / n
        mb = (a["rd"] + a["wr"]) / n / 1e6
        gbs = mb * 1e6 / (t * 1e-6) / 1e9 if t > 0 else 0.0
        print(f"{name[:44]:44s} {int(n):4d} {t:8.1f} {100 * a['t'] / total_t:5.1f}% {mb:10.1f} "
              f"{gbs:7.0f} {gbs / peak:6.2f} {a['l2_pct'] / n:5.1f} {a['l1_pct'] / n:5.1f} "
              f"{a['issue'] / n:6.1f} {a['fma'] / n:5.1f} {a['alu'] / n:5.1f} "
              f"{int(a['regs'] / n):4d}")


if __name__ == "__main__":
    main()
