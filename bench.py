#!/usr/bin/env python
"""Headline benchmark: particle-steps/s of the per-step MD hot path.

    python bench.py --gpus N --steps K --warmup W [--impl b200|reference]

Workload (BASELINE.json configs[2], the one the metric is quoted on): 3-D
Lennard-Jones fluid, N = 1 000 000 particles per GPU, rho = 0.75, T0 = 1.2,
r_c = 2.5, skin 0.3, dt = 0.001, NVE velocity Verlet from the reference's fcc +
Maxwell-Boltzmann initial state (synthetic).  One "step" = one MD step over all
particles, rebuilds and sampling included as they occur (reference bench.py:344-362:
particle-steps/s = n_particles * steps / wall).  For N > 1 GPUs the box is slab-
decomposed along x with 1 M particles per rank (weak scaling).

The JSON line carries, besides the driver's contract keys:
  roofline      force kernel: algorithmic bytes per launch / CUDA-event time vs the
                measured HBM peak (MEASURED_PEAKS.json)
  cpu_baseline  the CPU oracle (port of the reference) timed on this box's cores
  e2e           the same metric through the public API from HOST arrays: upload,
                Simulation.run(K), measure, download -- all inside the timed region
`--impl reference` times the CPU oracle port alone (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

N_PER_GPU = 1_000_000
DENSITY, T0, R_CUT, SKIN, DT = 0.75, 1.2, 2.5, 0.3, 0.001
METRIC = "particle-steps/s"
WORKLOAD = ("3D LJ fluid N=1M per GPU, rho=0.75, T0=1.2, rc=2.5, skin=0.3, dt=0.001, "
            "NVE velocity-Verlet from fcc start (BASELINE.json configs[2])")


# --------------------------------------------------------------------- helpers
def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index=0):
        self.proc = None
        self.device_index = device_index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.device_index), "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def initial_state(n, seed=42):
    """The reference's generators (integrate.py:146-198): fcc + vacancies,
    Philox Maxwell-Boltzmann velocities, zero momentum, exact T."""
    import paper_2406_04210_b200 as b2
    st, box = b2.init_lattice_any(n, DENSITY)
    b2.init_velocities(st, T0, seed)
    return (np.array(st.positions.acquire_read(b2.HOST)),
            np.array(st.velocities.acquire_read(b2.HOST)), box)


# ------------------------------------------------------------ CPU oracle timing
def time_cpu_oracle(n, steps, warmup, threads):
    """Oracle port of the reference loop on `threads` host cores: returns
    (particle-steps/s, seconds) for `steps` MD steps after `warmup`."""
    from oracle import oracle as orc
    pos, edge = orc.fcc_lattice(n, DENSITY)
    vel = orc.maxwell_velocities(n, T0, 42)
    sim = orc.Sim(pos, vel, [edge] * 3, orc.pair_table(1.0, 1.0, R_CUT), DT, SKIN,
                  sample_interval=100, threads=threads)
    sim.run(warmup)
    t0 = time.perf_counter()
    sim.run(steps)
    dt = time.perf_counter() - t0
    return n * steps / dt, dt


def cpu_baseline_sample(n_full):
    """Bounded sample (about 10-30 s of CPU work) of the same workload."""
    from oracle import oracle as orc
    threads = orc.host_threads()
    steps = 10 if n_full >= 500_000 else 50
    value, secs = time_cpu_oracle(n_full, steps, 1, threads)
    return {"value": value, "unit": METRIC, "cores": threads, "kind": "port",
            "sample": f"N={n_full}, {steps} MD steps after 1 warm-up step (list prebuilt), "
                      f"{secs:.1f} s, oracle C/numpy port of the reference on {threads} threads"}


def run_reference_arm(args):
    """--impl reference: the CPU path alone, bounded so K+W steps end in minutes."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as orc
    threads = orc.host_threads()
    budget_particle_steps = 1.2e8          # ~100 s at ~1.2e6 particle-steps/s
    n = int(min(N_PER_GPU * args.gpus, max(4096, budget_particle_steps / (args.steps + args.warmup))))
    value, secs = time_cpu_oracle(n, args.steps, args.warmup, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": METRIC,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "timed_sample_particles": n},
        "cpu_baseline": {"value": value, "unit": METRIC, "cores": threads, "kind": "port",
                         "sample": f"each step = one MD step of the same state point at N={n} "
                                   f"(bounded sample of the N=1M workload), {threads} threads"},
        "e2e": {"value": value, "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))


# -------------------------------------------------------------------- GPU arm
def time_kernel(fn, iters, torch, stream):
    """Average CUDA-event time (ms) of `fn` over `iters` launches on `stream`."""
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    start.record(stream)
    for _ in range(iters):
        fn()
    stop.record(stream)
    torch.cuda.synchronize()
    return start.elapsed_time(stop) / iters


def run_gpu_arm(args):
    import torch
    import torch.distributed as dist
    import paper_2406_04210_b200 as b2

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("launch with torch.distributed.run --nproc-per-node N for --gpus N")
    torch.cuda.set_device(local_rank)

    if world > 1 or args.force_slab:
        # NCCL writes its version banner to stdout when the communicator is created (eagerly,
        # with device_id): keep fd 1 clean for the one JSON line from before the init on
        sys.stdout.flush()
        real_stdout = os.dup(1)
        os.dup2(2, 1)
        try:
            if world > 1:
                dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
            else:           # exercise the decomposed driver on one rank (validation only)
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", "29533")
                dist.init_process_group("nccl", rank=0, world_size=1,
                                        device_id=torch.device("cuda", local_rank))
            from paper_2406_04210_b200.decomp import run_slab_benchmark
            # default: weak scaling, 1 M particles per GPU; --total-particles T fixes the job
            # size instead (BASELINE.json configs[4]: T = 16 M over 2 / 4 / 8 GPUs)
            n_rank = args.particles_per_gpu or N_PER_GPU
            if args.total_particles:
                n_rank = args.total_particles // world
            line = run_slab_benchmark(args, rank, world, local_rank, n_rank, WORKLOAD, METRIC,
                                      measured_peak, ClockSampler,
                                      scaling="strong" if args.total_particles else "weak")
            dist.destroy_process_group()
        finally:
            sys.stdout.flush()
            os.dup2(real_stdout, 1)
            os.close(real_stdout)
        if line is not None:
            print(json.dumps(line))
        return

    n = N_PER_GPU
    lj = b2.make_shifted(1.0, 1.0, R_CUT)
    pos0, vel0, box = initial_state(n)
    stream = torch.cuda.current_stream()

    def fresh_sim():
        st = b2.ParticleState(pos0, velocities=vel0, device=local_rank)
        return b2.Simulation(st, box, lj, DT, force_mode=b2.TRUNCATED, skin=SKIN,
                             sample_interval=100, reorder="hilbert")

    # ---- device-resident throughput ------------------------------------------
    sim = fresh_sim()
    sim.run(args.warmup)
    sim.reset_counters()
    clocks = ClockSampler(local_rank)
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    clocks.start()
    start.record(stream)
    sim.run(args.steps)
    stop.record(stream)
    torch.cuda.synchronize()
    clock_info = clocks.stop()
    ms = start.elapsed_time(stop)
    value = n * args.steps / (ms * 1e-3)
    launches = sim.kernel_launches
    rebuilds = sim.rebuild_count
    last = sim.samples[-1] if sim.samples else sim.measure()

    # ---- per-kernel roofline (force kernel dominant) --------------------------
    dev = sim.state.device_state()
    k = sim._keep
    counts = k["counts"][:n]
    cbar = float(counts.float().mean().item())
    from paper_2406_04210_b200 import _lib
    import ctypes
    tab = np.ascontiguousarray(lj.table())
    tab_ptr = tab.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    rows = k["nbr"].shape[0]

    def launch_force_rows():
        _lib.call("b2md_force_lj", dev.pos_hi.data_ptr(), n, box.c_box(), k["nbr"].data_ptr(),
                  k["counts"].data_ptr(), k["pitch"], rows, k["boundary"].data_ptr(), tab_ptr, 1,
                  _lib.FORCE_SKIP_THERMO, dev.force.data_ptr(), dev.virial.data_ptr(), dev.status.data_ptr(), dev.stream)

    def launch_force_pairs():
        cfg = k["cfg"]
        _lib.call("b2md_force_lj_pairs", dev.pos_hi.data_ptr(), n, box.c_box(),
                  k["pair_nbr"].data_ptr(), k["pair_counts"].data_ptr(), cfg.pair_pitch,
                  k["nbr"].data_ptr(), k["counts"].data_ptr(), k["pitch"],
                  k["boundary"].data_ptr(), tab_ptr, 1, _lib.FORCE_SKIP_THERMO,
                  dev.force.data_ptr(), dev.virial.data_ptr(), dev.status.data_ptr(), dev.stream)

    # the kernel the step loop launches (pair rows for systems this large)
    force_kernel = "k_force_lj_pair" if sim.pair_rows else "k_force_lj"
    force_ms = time_kernel(launch_force_pairs if sim.pair_rows else launch_force_rows, 50, torch,
                           stream)
    pair_entries = float(k["pair_counts"].float().sum().item()) / n if sim.pair_rows else None
    extra_kernels = {}
    if sim.pair_rows:
        # for comparison: the thread-per-particle kernel on the same list, and the merge
        rows_ms = time_kernel(launch_force_rows, 20, torch, stream)
        extra_kernels["k_force_lj (thread per particle, same list)"] = {
            "launch_ms": rows_ms,
            "achieved": n * (32.0 + 4.0 * cbar) / (rows_ms * 1e-3) / 1e9}
        cfg = k["cfg"]

        def launch_merge():
            _lib.call("b2md_pair_rows", k["nbr"].data_ptr(), k["counts"].data_ptr(), k["pitch"],
                      rows, n, k["pair_nbr"].data_ptr(), k["pair_counts"].data_ptr(),
                      cfg.pair_pitch, cfg.pair_rows, dev.stream)
        extra_kernels["k_pair_rows (once per rebuild)"] = {
            "launch_ms": time_kernel(launch_merge, 10, torch, stream)}
    force_bytes = n * (32.0 + 4.0 * cbar)          # pos 16 + idx 4*c + force 16 (no-thermo variant)
    peak, peak_src = measured_peak()
    achieved = force_bytes / (force_ms * 1e-3) / 1e9

    scratch_state = {name: getattr(dev, name).clone() for name in ("pos_hi", "pos_lo", "vel", "image")}
    ref_scratch = k["ref_pos"].clone()

    def launch_integrate():
        _lib.call("b2md_vv_finalize_integrate", scratch_state["pos_hi"].data_ptr(),
                  scratch_state["pos_lo"].data_ptr(), scratch_state["vel"].data_ptr(),
                  dev.force.data_ptr(), scratch_state["image"].data_ptr(), n, box.c_box(), DT,
                  ref_scratch.data_ptr(), 1e30, dev.status.data_ptr(), dev.stream)

    integ_ms = time_kernel(launch_integrate, 50, torch, stream)
    if sim.pair_rows and sim.advance:
        # the one-launch step: force + finalize + integrate + displacement check (scratch
        # copies of everything it updates in place, its own status block)
        scratch_status = torch.zeros(16, dtype=torch.int32, device=dev.pos_hi.device)
        scratch_out = torch.empty_like(dev.pos_hi)
        cfg = k["cfg"]

        def launch_advance():
            _lib.call("b2md_force_lj_pairs_advance", dev.pos_hi.data_ptr(), scratch_out.data_ptr(),
                      scratch_state["pos_lo"].data_ptr(), scratch_state["vel"].data_ptr(),
                      scratch_state["image"].data_ptr(), n, box.c_box(), 1e-9,
                      ref_scratch.data_ptr(), 1e30, k["pair_nbr"].data_ptr(),
                      k["pair_counts"].data_ptr(), cfg.pair_pitch, k["nbr"].data_ptr(),
                      k["counts"].data_ptr(), k["pitch"], k["boundary"].data_ptr(), tab_ptr, 1, 0,
                      12, 14, scratch_status.data_ptr(), dev.stream)   # gate words of the scratch block
        adv_ms = time_kernel(launch_advance, 30, torch, stream)
        # SURVEY 8(d) rows it replaces: integrate 128 + force 32+4c (no-thermo) + finalize 48,
        # minus the 80 B per particle of force / velocity traffic that fusion makes unnecessary
        # (force written once and read twice, velocities written and re-read between the kicks)
        adv_bytes = n * (128.0 + 4.0 * cbar)
        # this is the kernel 98 % of the steps launch: it becomes the roofline entry, the
        # plain force kernel (first / last step of a call, sample steps) moves to the list
        extra_kernels["k_force_lj_pair (force only: first / last step of a call)"] = {
            "launch_ms": force_ms, "algorithmic_bytes_per_launch": force_bytes,
            "achieved": achieved, "frac": achieved / peak}
        force_kernel = "k_force_lj_pair<ADVANCE> (force + finalize + integrate: one launch per MD step)"
        force_ms, force_bytes = adv_ms, adv_bytes
        achieved = adv_bytes / (adv_ms * 1e-3) / 1e9
    integ_bytes = n * 128.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "force_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            key = "advance" if (sim.pair_rows and sim.advance) else ("pairs" if sim.pair_rows else "rows")
            traffic = tj.get(key, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    step_bytes = n * (216.0 + 4.0 * cbar)
    sim.close()
    del sim, scratch_state, ref_scratch
    torch.cuda.empty_cache()

    # ---- end to end through the public API from HOST arrays --------------------
    from paper_2406_04210_b200.core import TRANSFER_BYTES
    host_pos = torch.from_numpy(pos0).pin_memory().numpy()
    host_vel = torch.from_numpy(vel0).pin_memory().numpy()
    e2e_reps = 3
    e2e_ms = []
    h2d = d2h = 0
    for rep in range(e2e_reps + 1):
        # HOST side = the caller's page-locked arrays (copy=False): H2D / D2H go straight
        # from / to pinned memory; each repetition restarts from the same initial arrays
        host_pos[...] = pos0
        host_vel[...] = vel0
        moved0 = dict(TRANSFER_BYTES)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = b2.ParticleState(host_pos, velocities=host_vel, device=local_rank, copy=False)
        s = b2.Simulation(st, box, lj, DT, force_mode=b2.TRUNCATED, skin=SKIN,
                          sample_interval=100, reorder="hilbert")
        s.run(args.steps)
        sample = s.measure()
        out_pos = st.positions.acquire_read(b2.HOST)
        out_vel = st.velocities.acquire_read(b2.HOST)
        torch.cuda.synchronize()
        if rep > 0:       # first repetition warms allocator and page tables
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        h2d = TRANSFER_BYTES["h2d"] - moved0["h2d"]
        d2h = TRANSFER_BYTES["d2h"] - moved0["d2h"] + 64      # + the 8 reduced doubles
        s.close()
        del s, st
    e2e_best = min(e2e_ms)
    e2e_value = n * args.steps / (e2e_best * 1e-3)

    cpu = cpu_baseline_sample(n)

    line = {
        "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 pair arithmetic, double-single positions, f64 reductions",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "particles": n, "l2": "inputs larger than L2: the "
                   f"neighbour list streamed every step is {rows * k['pitch'] * 4 / 1e6:.0f} MB "
                   "(L2 126 MB), state 80 MB",
                   "mean_listed_neighbours": cbar, "pair_row_entries_per_particle": pair_entries,
                   "rebuilds_in_timed_region": rebuilds,
                   "reorder": "hilbert", "sample_interval": 100,
                   "step_algorithmic_bytes": step_bytes,
                   "step_hbm_fraction": step_bytes * value / n / 1e9 / peak,
                   "final_energy_per_particle": last.total_energy / n,
                   "final_temperature": last.temperature},
        "clocks": clock_info,
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": force_kernel, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": force_bytes,
                     "launch_ms": force_ms,
                     "other_kernels": {**extra_kernels, "k_integrate<2>": {
                         "achieved": integ_bytes / (integ_ms * 1e-3) / 1e9, "launch_ms": integ_ms,
                         "algorithmic_bytes_per_launch": integ_bytes,
                         "frac": integ_bytes / (integ_ms * 1e-3) / 1e9 / peak}}},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": METRIC,
                "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
                "call": f"ParticleState(host arrays) -> Simulation(...) -> run({args.steps}) -> "
                        "measure() -> positions/velocities read back; host<->device copies, "
                        "buffer allocation and the initial list build inside the timed region; "
                        f"best of {e2e_reps}", "ms_per_call": e2e_best,
                "h2d_bytes_per_call": h2d, "d2h_bytes_per_call": d2h},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--particles-per-gpu", type=int, default=0,
                    help="slab arm (--gpus > 1 or --force-slab): particles per rank (default 1 M)")
    ap.add_argument("--total-particles", type=int, default=0,
                    help="slab arm: fixed job size split over the ranks (strong scaling)")
    ap.add_argument("--force-slab", action="store_true",
                    help="run the slab-decomposed driver even on one rank (validation)")
    args = ap.parse_args()
    if args.steps < 1 or args.warmup < 0:
        raise SystemExit("--steps must be >= 1 and --warmup >= 0")
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
