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

Timed region: `Simulation.run(K)` repeated back to back on the same (evolving) system
until at least MIN_TIMED_SECONDS of GPU time and MIN_REPEATS repeats have been collected;
`value` = all particle-steps of those repeats / their total CUDA-event time (what a long
run delivers: rebuilds occur at their natural rate), `ms_per_step` the matching mean;
median / best repeat are in `config`.  The driver's short runs (K = 20) are therefore no
longer a 4 ms window.

The JSON line carries, besides the driver's contract keys:
  roofline      step kernel: algorithmic bytes per launch / CUDA-event time vs the
                measured HBM peak (MEASURED_PEAKS.json)
  cpu_baseline  the reference itself (unmodified `mdbench` from baseline/_ref, numba
                parallel backend on all host cores, plus its 1-core sequential figure) on a
                bounded sample of the same workload; the C/OpenMP oracle port beside it
  e2e           the same metric through the public API from HOST arrays: upload,
                Simulation(...), run(K), measure, download -- all inside the timed region
  config.parity forces of the production kernel at this N vs the fp64 oracle (checker,
                after all timing)
`--impl reference` times the reference's own CPU path alone (rank 0 only): same N, fewer
steps when K + W would not end within minutes -- N is never shrunk.
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
MIN_TIMED_SECONDS = 1.0      # GPU time collected per measurement (repeats of K steps)
MIN_REPEATS = 3
MAX_REPEATS = 400
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
        self.extra = []

    def sample_now(self):
        """One synchronous query (the background poll may not fire inside a short region)."""
        try:
            out = subprocess.run(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.device_index)], capture_output=True, text=True, timeout=10).stdout
            self.extra.extend(out.strip().splitlines())
        except Exception:
            pass

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
        for line in out.strip().splitlines() + self.extra:
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


# ------------------------------------------------------- CPU baselines (checkers)
def workload_config(n_total, n_per_gpu):
    """Keys both arms print identically: what is being simulated."""
    return {"workload": WORKLOAD, "particles": int(n_total), "particles_per_gpu": int(n_per_gpu),
            "density": DENSITY, "t0": T0, "r_cut": R_CUT, "skin": SKIN, "dt": DT,
            "sample_interval": 100}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def import_reference():
    """The UNMODIFIED reference package (`mdbench` 0.1.0), installed by
    `pip install --no-index --no-deps --target baseline/_ref /root/reference/pkg` in the
    build container; git-ignored, travels with the snapshot.  Returns the
    module or None (not installed / numba missing on this box)."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "mdbench")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/b2md_numba_cache")
    sys.dont_write_bytecode = True
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    try:
        import mdbench
        return mdbench
    except Exception as err:            # pragma: no cover - depends on the box
        print(f"bench.py: reference not importable ({err!r}); timing the oracle port", file=sys.stderr)
        return None


def time_reference(ref, n, steps, warmup, workers):
    """The reference's own step loop (mdbench.Simulation, reference bench.py:288-352) on
    `workers` host threads (1 -> its sequential backend).  Returns (particle-steps/s,
    seconds of the timed `steps`)."""
    kind = "parallel" if workers > 1 else "sequential"
    # JIT warm-up on a small system (numba compiles per signature, not per size)
    st, box = ref.init_lattice_any(500, DENSITY)
    ref.init_velocities(st, T0, 42)
    warm = ref.Simulation(st, box, ref.make_shifted(1.0, 1.0, R_CUT), dt=DT,
                          backend=ref.BackendSelector(kind, workers), force_mode="truncated",
                          skin=SKIN, sample_interval=100)
    warm.run(2)
    st, box = ref.init_lattice_any(n, DENSITY)
    ref.init_velocities(st, T0, 42)
    sim = ref.Simulation(st, box, ref.make_shifted(1.0, 1.0, R_CUT), dt=DT,
                         backend=ref.BackendSelector(kind, workers), force_mode="truncated",
                         skin=SKIN, sample_interval=100)
    sim.run(warmup)
    t0 = time.perf_counter()
    sim.run(steps)
    secs = time.perf_counter() - t0
    return n * steps / secs, secs


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
    """Bounded sample (about 20-30 s of CPU work) of the same workload: the reference on
    all cores and on one core, and the oracle port on all cores."""
    from oracle import oracle as orc
    cores = host_cores()
    port_steps = 10 if n_full >= 500_000 else 50
    port_value, port_secs = time_cpu_oracle(n_full, port_steps, 1, orc.host_threads())
    port = {"value": port_value, "unit": METRIC, "cores": orc.host_threads(), "kind": "port",
            "sample": f"N={n_full}, {port_steps} MD steps after 1 warm-up step, {port_secs:.1f} s, "
                      "oracle C/OpenMP port of the reference"}
    ref = import_reference()
    if ref is None:
        return port
    steps = 5 if n_full >= 500_000 else 50
    value, secs = time_reference(ref, n_full, steps, 1, cores)
    one_steps = 2 if n_full >= 500_000 else 20
    one_value, one_secs = time_reference(ref, n_full, one_steps, 0, 1)
    return {"value": value, "unit": METRIC, "cores": cores, "kind": "reference",
            "sample": f"N={n_full}, {steps} MD steps after 1 warm-up step (list prebuilt, numba "
                      f"JIT warm), {secs:.1f} s: unmodified mdbench {ref.__version__} from "
                      f"baseline/_ref, parallel backend with {cores} workers",
            "one_core": {"value": one_value, "unit": METRIC, "cores": 1,
                         "sample": f"N={n_full}, {one_steps} MD steps, {one_secs:.1f} s, sequential "
                                   "backend"},
            "port": port}


def run_reference_arm(args):
    """--impl reference: the reference's CPU path alone, on this arm's own workload.  N is
    never reduced; when K + W steps would not end within minutes fewer steps are timed and
    the line says so."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_per_gpu = args.particles_per_gpu or N_PER_GPU
    n = args.total_particles or n_per_gpu * args.gpus
    cores = host_cores()
    ref = import_reference()
    # ~0.7 us per particle-step on 8 cores: keep the timed part near 90 s
    per_step_s = n * 0.7e-6 * (8.0 / max(cores, 1)) ** 0.7
    steps = int(max(1, min(args.steps, 90.0 / per_step_s)))
    warmup = int(max(1, min(args.warmup, 15.0 / per_step_s)))
    if ref is not None:
        value, secs = time_reference(ref, n, steps, warmup, cores)
        kind, used = "reference", cores
        what = (f"unmodified mdbench {ref.__version__} (baseline/_ref), numba parallel backend, "
                f"{cores} workers")
    else:
        from oracle import oracle as orc
        used = orc.host_threads()
        value, secs = time_cpu_oracle(n, steps, warmup, used)
        kind, what = "port", f"oracle C/OpenMP port of the reference, {used} threads"
    note = "" if steps == args.steps else (f"; {steps} of the requested {args.steps} steps timed "
                                           f"(bounded sample of the same N)")
    cfg = workload_config(n, n // max(args.gpus, 1))
    cfg["timed_steps"] = steps
    cfg["timed_warmup"] = warmup
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": METRIC,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / steps, "higher_is_better": True,
        "scaling": "strong" if args.total_particles else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": METRIC, "cores": used, "kind": kind,
                         "sample": f"N={n}: {what}{note}"},
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
                                      scaling="strong" if args.total_particles else "weak",
                                      cpu_baseline_fn=cpu_baseline_sample,
                                      workload_config_fn=workload_config,
                                      min_timed_seconds=MIN_TIMED_SECONDS,
                                      min_repeats=MIN_REPEATS, max_repeats=MAX_REPEATS)
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
    # run(K) repeated back to back on the same evolving system, each repeat bracketed by
    # CUDA events, until MIN_TIMED_SECONDS of GPU time and MIN_REPEATS repeats are in
    sim = fresh_sim()
    sim.run(max(args.warmup, 3))
    sim.reset_counters()
    clocks = ClockSampler(local_rank)
    torch.cuda.synchronize()
    clocks.sample_now()
    clocks.start()
    rep_ms = []
    while (len(rep_ms) < MIN_REPEATS or sum(rep_ms) < 1e3 * MIN_TIMED_SECONDS) \
            and len(rep_ms) < MAX_REPEATS:
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        sim.run(args.steps)
        stop.record(stream)
        torch.cuda.synchronize()
        rep_ms.append(start.elapsed_time(stop))
    clocks.sample_now()
    clock_info = clocks.stop()
    repeats = len(rep_ms)
    ms = sum(rep_ms) / repeats                       # mean time of one repeat of K steps
    value = n * args.steps / (ms * 1e-3)
    launches = sim.kernel_launches
    rebuilds = sim.rebuild_count
    phase = {"force_seconds": sim.force_seconds, "nlist_seconds": sim.nlist_seconds}
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
    # kernels timed alone follow the runner's block schedule, as inside a step
    sched = _lib.FORCE_SCHEDULED if (sim.pair_rows and k["cfg"].pair_schedule) else 0

    def launch_force_rows():
        _lib.call("b2md_force_lj", dev.pos_hi.data_ptr(), n, box.c_box(), k["nbr"].data_ptr(),
                  k["counts"].data_ptr(), k["pitch"], rows, k["boundary"].data_ptr(), tab_ptr, 1,
                  _lib.FORCE_SKIP_THERMO, dev.force.data_ptr(), dev.virial.data_ptr(), dev.status.data_ptr(), dev.stream)

    def launch_force_pairs():
        cfg = k["cfg"]
        _lib.call("b2md_force_lj_pairs", dev.pos_hi.data_ptr(), n, box.c_box(),
                  k["pair_nbr"].data_ptr(), k["pair_counts"].data_ptr(), cfg.pair_pitch,
                  k["nbr"].data_ptr(), k["counts"].data_ptr(), k["pitch"],
                  k["boundary"].data_ptr(), tab_ptr, 1, _lib.FORCE_SKIP_THERMO | sched,
                  dev.force.data_ptr(), dev.virial.data_ptr(), dev.status.data_ptr(), dev.stream)

    extra_kernels = {}
    if sim.pair_rows:
        # The step loop's list build (b2md_build_pair_list) writes plain rows only for the pairs
        # that straddle two cells.  The per-kernel timings below want the complete per-particle
        # list next to the pair rows made from it: bin and build both here, on the positions the
        # timed run ended on -- the two-stage path the fused build replaces, timed beside it.
        cfg = k["cfg"]
        r_list = R_CUT + SKIN
        grid = _lib.Grid()
        _lib.call("b2md_grid_shape", box.c_box(), r_list, ctypes.byref(grid))
        pair_rows_alt = torch.zeros_like(k["pair_nbr"])
        pair_counts_alt = torch.zeros_like(k["pair_counts"])

        def rebin():
            _lib.call("b2md_status_reset_list", dev.status.data_ptr(), dev.stream)
            _lib.call("b2md_bin", dev.pos_hi.data_ptr(), dev.pos_lo.data_ptr(), n,
                      ctypes.byref(grid), k["cell_of"].data_ptr(), k["cell_start"].data_ptr(),
                      k["cell_particles"].data_ptr(), k["bin_scratch"].data_ptr(), dev.stream)

        def launch_list_plain():
            _lib.call("b2md_build_nlist_ex", dev.pos_hi.data_ptr(), dev.pos_lo.data_ptr(), n,
                      box.c_box(), ctypes.byref(grid), k["cell_of"].data_ptr(),
                      k["cell_start"].data_ptr(), k["cell_particles"].data_ptr(), r_list,
                      cfg.stride, k["pitch"], k["nbr"].data_ptr(), k["counts"].data_ptr(),
                      k["boundary"].data_ptr(), r_list + SKIN, n, 1, dev.status.data_ptr(),
                      dev.stream)

        def launch_list_fused():
            _lib.call("b2md_build_pair_list", dev.pos_hi.data_ptr(), dev.pos_lo.data_ptr(), n,
                      box.c_box(), ctypes.byref(grid), k["cell_of"].data_ptr(),
                      k["cell_start"].data_ptr(), k["cell_particles"].data_ptr(), r_list,
                      cfg.stride, k["pitch"], k["nbr"].data_ptr(), k["counts"].data_ptr(),
                      k["boundary"].data_ptr(), r_list + SKIN, n, 1, rows,
                      pair_rows_alt.data_ptr(), pair_counts_alt.data_ptr(), cfg.pair_pitch,
                      cfg.pair_rows, dev.status.data_ptr(), dev.stream)

        def launch_merge():
            _lib.call("b2md_pair_rows", k["nbr"].data_ptr(), k["counts"].data_ptr(), k["pitch"],
                      rows, n, k["pair_nbr"].data_ptr(), k["pair_counts"].data_ptr(),
                      cfg.pair_pitch, cfg.pair_rows, dev.stream)

        rebin()
        launch_list_fused()                       # into pair_rows_alt (fresh, zero-filled)
        k["nbr"].zero_()                          # the row kernel below reads padding entries
        launch_list_plain()                       # leaves complete per-particle rows
        pair_rows_ref = torch.zeros_like(k["pair_nbr"])
        pair_counts_ref = torch.zeros_like(k["pair_counts"])
        _lib.call("b2md_pair_rows", k["nbr"].data_ptr(), k["counts"].data_ptr(), k["pitch"],
                  rows, n, pair_rows_ref.data_ptr(), pair_counts_ref.data_ptr(),
                  cfg.pair_pitch, cfg.pair_rows, dev.stream)
        merge_ms = time_kernel(launch_merge, 5, torch, stream)       # (into the live buffers)
        if cfg.pair_schedule:
            _lib.call("b2md_pair_schedule", k["boundary"].data_ptr(), n,
                      k["pair_counts"].data_ptr(), cfg.pair_pitch, dev.stream)
        torch.cuda.synchronize()
        same_pairs = bool(torch.equal(pair_rows_alt, pair_rows_ref) and
                          torch.equal(pair_counts_alt[:cfg.pair_pitch],
                                      pair_counts_ref[:cfg.pair_pitch]))
        cbar = float(k["counts"][:n].float().mean().item())
        # the rebuild as the step loop ran it (CUDA-event phase timer of the timed region:
        # Hilbert keys, sort, gather, bin, list + pair rows, snapshot, block schedule)
        rebuild_ms = 1e3 * sim.nlist_seconds / max(rebuilds, 1)
        extra_kernels["rebuild sequence inside the timed region (reorder, bin, "
                      "b2md_build_pair_list = k_list_cells_ballot<PAIRS> + k_pair_fixup, "
                      "snapshot, schedule)"] = {
            "launch_ms": rebuild_ms, "rebuilds": rebuilds,
            "algorithmic_bytes_per_launch": n * (32.0 + 4.0 * cbar),
            "pair_rows_identical_to_two_stage_build_on_the_end_state": same_pairs}
        extra_kernels["k_pair_rows (the merge the fused list build replaces)"] = {
            "launch_ms": merge_ms}
        del pair_rows_alt, pair_counts_alt, pair_rows_ref, pair_counts_ref

    # the kernel the step loop launches (pair rows for systems this large)
    force_kernel = "k_force_lj_pair" if sim.pair_rows else "k_force_lj"
    force_ms = time_kernel(launch_force_pairs if sim.pair_rows else launch_force_rows, 50, torch,
                           stream)
    pair_entries = (float(k["pair_counts"][:k["cfg"].pair_pitch].float().sum().item()) / n
                    if sim.pair_rows else None)

    if sim.pair_rows:
        # for comparison: the thread-per-particle kernel on the same list
        rows_ms = time_kernel(launch_force_rows, 20, torch, stream)
        extra_kernels["k_force_lj (thread per particle, same list)"] = {
            "launch_ms": rows_ms,
            "achieved": n * (32.0 + 4.0 * cbar) / (rows_ms * 1e-3) / 1e9}
    force_bytes = n * (32.0 + 4.0 * cbar)          # pos 16 + idx 4*c + force 16 (no-thermo variant)
    peak, peak_src = measured_peak()
    achieved = force_bytes / (force_ms * 1e-3) / 1e9

    # scratch copies of everything the integrate / step kernels update in place; three sets
    # used in rotation (3 x 80 MB of state + 3 x 16 MB of forces > the 126 MB L2) so that the
    # integrate kernel is timed on data that comes from HBM, as it does inside a step
    scratch_sets = [{name: getattr(dev, name).clone()
                     for name in ("pos_hi", "pos_lo", "vel", "image", "force")}
                    for _ in range(3)]
    ref_sets = [k["ref_pos"].clone() for _ in range(3)]
    scratch_state, ref_scratch = scratch_sets[0], ref_sets[0]
    turn = [0]

    def launch_integrate():
        t = turn[0] = (turn[0] + 1) % 3
        sc = scratch_sets[t]
        _lib.call("b2md_vv_finalize_integrate", sc["pos_hi"].data_ptr(),
                  sc["pos_lo"].data_ptr(), sc["vel"].data_ptr(),
                  sc["force"].data_ptr(), sc["image"].data_ptr(), n, box.c_box(), DT,
                  ref_sets[t].data_ptr(), 1e30, dev.status.data_ptr(), dev.stream)

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
                      k["counts"].data_ptr(), k["pitch"], k["boundary"].data_ptr(), tab_ptr, 1,
                      sched, 12, 14, scratch_status.data_ptr(), dev.stream)   # gate words of the scratch block
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
    # DRAM bytes per launch of the same kernel from this round's `ncu --set full` capture
    # (profiles/capture.sh -> profiles/force_traffic.json names the .txt summary it was read
    # from); null when no capture of the kernel this run launches is on file
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "force_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            key = "advance" if (sim.pair_rows and sim.advance) else ("pairs" if sim.pair_rows else "rows")
            traffic = tj.get(key, {}).get("dram_bytes_per_launch")
            traffic_src = tj.get(key, {}).get("source")
        except Exception:
            traffic = None
    step_bytes = n * (216.0 + 4.0 * cbar)
    final_pos = np.array(sim.state.positions.acquire_read(b2.HOST))
    sim.close()
    del sim, scratch_state, ref_scratch, scratch_sets, ref_sets
    torch.cuda.empty_cache()

    # ---- end to end through the public API from HOST arrays --------------------
    from paper_2406_04210_b200.core import TRANSFER_BYTES
    host_pos = torch.from_numpy(pos0).pin_memory().numpy()
    host_vel = torch.from_numpy(vel0).pin_memory().numpy()
    e2e_ms = []
    h2d = d2h = 0
    rep = 0
    while rep == 0 or ((len(e2e_ms) < MIN_REPEATS or sum(e2e_ms) < 1e3 * MIN_TIMED_SECONDS)
                       and len(e2e_ms) < MAX_REPEATS):
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
        rep += 1
    e2e_med = statistics.median(e2e_ms)
    e2e_value = n * args.steps / (e2e_med * 1e-3)

    # ---- checkers, after all timing: CPU baselines and parity at this size -----
    cpu = cpu_baseline_sample(n)
    parity = parity_probe(b2, final_pos, box, lj, local_rank)

    cfg = workload_config(n, n)
    cfg.update({
        "l2": "inputs larger than L2: the neighbour list streamed every step is "
              f"{rows * k['pitch'] * 4 / 1e6:.0f} MB (L2 126 MB), state 80 MB",
        "timed_region": f"{repeats} back-to-back repeats of run({args.steps}) on the same evolving "
                        f"system, {sum(rep_ms) / 1e3:.2f} s of GPU time; value = all particle-steps "
                        "/ total CUDA-event time",
        "timed_repeats": repeats,
        "ms_per_step_median_repeat": statistics.median(rep_ms) / args.steps,
        "ms_per_step_best_repeat": min(rep_ms) / args.steps,
        "mean_listed_neighbours": cbar, "pair_row_entries_per_particle": pair_entries,
        "rebuilds_in_timed_region": rebuilds,
        "phase_gpu_seconds": phase,
        "reorder": "hilbert",
        "step_algorithmic_bytes": step_bytes,
        "step_hbm_fraction": step_bytes * value / n / 1e9 / peak,
        "final_energy_per_particle": last.total_energy / n,
        "final_temperature": last.temperature,
        "parity": parity})
    line = {
        "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 pair arithmetic, double-single positions, f64 reductions",
        "data": "synthetic",
        "config": cfg,
        "clocks": clock_info,
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": force_kernel, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": force_bytes,
                     "launch_ms": force_ms,
                     "other_kernels": {**extra_kernels, "k_integrate<2> (three state sets in "
                                       "rotation: working set > L2)": {
                         "achieved": integ_bytes / (integ_ms * 1e-3) / 1e9, "launch_ms": integ_ms,
                         "algorithmic_bytes_per_launch": integ_bytes,
                         "frac": integ_bytes / (integ_ms * 1e-3) / 1e9 / peak}}},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": METRIC,
                "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
                "call": f"ParticleState(host arrays) -> Simulation(...) -> run({args.steps}) -> "
                        "measure() -> positions/velocities read back; host<->device copies, "
                        "buffer allocation and the initial list build inside the timed region; "
                        f"median of {len(e2e_ms)} calls", "ms_per_call": e2e_med,
                "ms_per_call_best": min(e2e_ms),
                "h2d_bytes_per_call": h2d, "d2h_bytes_per_call": d2h},
    }
    print(json.dumps(line))


def parity_probe(b2, positions, box, lj, device):
    """Forces of the production kernel (pair rows, packed fp32x2) at the benchmark's N on
    the system the timed run ended in, against the fp64 oracle on identical inputs
    (positions rounded to the device's fp32 high words): list rows compared bit for bit,
    force error as M1 / M2 / M3 of SURVEY.md section 7.3.  Checker only -- runs after all timing."""
    from oracle import oracle as orc
    try:
        edge = [float(e) for e in box.edge_lengths]
        pos = np.asarray(positions, dtype=np.float64).astype(np.float32).astype(np.float64)
        pos = np.where(pos >= np.array(edge), 0.0, pos)
        n = pos.shape[0]
        r_list = R_CUT + SKIN
        th = orc.host_threads()
        st = b2.ParticleState(pos, device=device)
        grid = b2.bin_particles(st, box, r_list)
        nl = b2.build_neighbor_list(st, grid, r_list, 96, r_cut=R_CUT)
        b2.compute_forces_truncated(st, lj, box, nl, pair_rows=True)
        f = np.array(st.forces.acquire_read(b2.HOST))
        og = orc.bin_particles(pos, edge, r_list)
        onl = orc.build_neighbor_list(pos, np.zeros((n, 3), np.int64), og, r_list, 96,
                                      r_cut=R_CUT, threads=th)
        cnt = nl.counts
        same = bool(np.array_equal(cnt, onl.counts))
        if same:
            mask = np.arange(onl.indices.shape[1])[None, :] < cnt[:, None]
            same = bool(np.array_equal(np.where(mask, nl.indices[:, :onl.indices.shape[1]], 0),
                                       np.where(mask, onl.indices, 0)))
        rf, _, _ = orc.forces_truncated(pos, edge, lj.table(), onl, threads=th)
        fs, _, _ = orc.pair_scales(pos, edge, lj.table(), onl, threads=th)
        err = np.max(np.abs(f - rf), axis=1)
        # The truncated LJ force is discontinuous at r_c (|F(r_c)| = 0.039): a pair whose fp64
        # r^2 lies within a few fp32 roundings of r_c^2 may be cut on the other side than in
        # the reference (about 15 such pairs per 10^6 particles).  Particles above tolerance
        # must all own such a pair; they are counted and set aside.
        rc2 = R_CUT * R_CUT
        banded = []
        for i in np.nonzero(err > 0.5e-5 * fs)[0]:
            j = onl.indices[i, :onl.counts[i]]
            d = pos[i] - pos[j]
            d -= np.array(edge) * np.rint(d / np.array(edge))
            if np.any(np.abs((d * d).sum(axis=1) - rc2) <= 1e-6 * rc2):
                banded.append(int(i))
        keep = np.ones(n, dtype=bool)
        keep[banded] = False
        unexplained = int(np.count_nonzero(err[keep] > 0.5e-5 * fs[keep]))
        finf = np.max(np.abs(rf), axis=1)
        ek, fk = err[keep], finf[keep]
        return {"particles": int(n), "state": "molten (end of the timed run), fp32-representable",
                "neighbour_rows_identical": same,
                "force_M1_vs_net_force": float(np.max(ek / np.maximum(fk, 1e-3 * fk.max()))),
                "force_M2_vs_sum_of_pair_terms": float(np.max(ek / np.maximum(fs[keep], 1e-300))),
                "force_M3_vs_rms_force": float(ek.max() / np.sqrt(np.mean(rf * rf))),
                "force_L2_relative_all_particles": float(np.linalg.norm(f - rf) / np.linalg.norm(rf)),
                "particles_with_a_pair_in_the_cutoff_guard_band": len(banded),
                "max_force_error_of_those": float(err[banded].max()) if banded else 0.0,
                "particles_above_tolerance_without_such_a_pair": unexplained,
                "stated_tolerance": 1e-5}
    except Exception as err:            # the benchmark line must not die on its checker
        return {"error": repr(err)}


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
