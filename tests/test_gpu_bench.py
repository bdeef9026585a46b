"""bench.py end to end on the GPU (short run): the JSON line the driver reads carries
every contract key, and every kernel the harness times through the C ABI still accepts
the arguments bench.py passes."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_line_has_the_contract_keys():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "40",
                          "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "clocks",
                "gpu_launches", "roofline", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["value"] > 1e9 and line["gpu_launches"] > 0
    roof = line["roofline"]
    assert roof["bound"] == "hbm" and 0.0 < roof["frac"] < 1.5 and roof["achieved"] > 0
    assert "ADVANCE" in roof["kernel"]
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
    cpu = line["cpu_baseline"]
    assert cpu["kind"] in ("reference", "port") and cpu["value"] > 0 and cpu["cores"] >= 1
    if cpu["kind"] == "reference":          # baseline/_ref travelled with the snapshot
        assert cpu["one_core"]["value"] > 0 and cpu["port"]["kind"] == "port"
    cfg = line["config"]
    assert cfg["particles"] == 1_000_000 and cfg["timed_repeats"] >= 3
    assert line["clocks"]["samples"] >= 2
    par = cfg["parity"]
    assert par["neighbour_rows_identical"] is True
    assert par["force_M2_vs_sum_of_pair_terms"] <= 1e-5
    assert par["particles_above_tolerance_without_such_a_pair"] == 0


def test_reference_arm_prints_the_same_workload_keys():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"]["particles"] == 1_000_000          # N is never shrunk
    assert line["config"]["workload"].startswith("3D LJ fluid N=1M")
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"],
                           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
