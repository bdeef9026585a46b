"""Simulation assembly on the B200 -- counterpart of reference sim.py.

Same constructor arguments, attributes and policies as the reference
``Simulation`` (sim.py:35-186): initial force evaluation at construction,
``integrate -> force -> finalize -> sample`` per step, rebuild when any particle
moved more than skin/2, stride growth on overflow (at most
``STRIDE_GROWTH_LIMIT`` times), ``measure()``, ``reset_counters()``.

Two drivers produce bit-identical trajectories:

* ``native=True`` (default for truncated forces): the C++ step loop of libb2md
  (csrc/runtime.cu) -- one or two kernel launches per step, the rebuild test read
  back asynchronously while the force kernel runs.  With an Andersen thermostat the
  loop launches integrate / force / finalize / thermostat per step (the thermostat is
  the reference's second finalize slot, sim.py:86-87,100-102).
* ``native=False``: the reference's signal/slot loop calling the operator
  functions one by one (same kernels, one Python call each) -- what the parity
  tests exercise operator by operator.

Extensions: ``reorder`` ("hilbert" | "cell" | None) re-sorts the device rows at
rebuild time for gather locality (logical particle order on the HOST side is
unaffected); ``lj`` may be a :class:`PairTable` (Kob-Andersen etc.).
"""
from __future__ import annotations

import ctypes
import os
import time

import numpy as np

from . import _lib
from .backend import BackendSelector
from .core import COMPUTE, DeviceState, ParticleState, SignalEngine, SimBox
from .errors import ConfigError, NeighborOverflowError, SingularPairError
from .forces import (_table_ptr, compute_forces_all_to_all, compute_forces_truncated,
                     use_pair_rows)
from .integrate import IntegratorParams, andersen_thermostat, vv_finalize, vv_integrate
from .neighbor import (HILBERT_SUB_BITS, NeighborList, _round_up, bin_particles,
                       build_neighbor_list, grid_shape, needs_rebuild, reorder_hilbert)
from .observables import DETERMINISTIC, FAST, Sample, thermo
from .potential import LJParams

ALL_TO_ALL = "all_to_all"
TRUNCATED = "truncated"
FORCE_MODES = (ALL_TO_ALL, TRUNCATED)

DEFAULT_STRIDE = 64
DEFAULT_SKIN = 0.5
STRIDE_GROWTH_LIMIT = 10

#: below this size the thread-per-particle kernel also advances the particles it has
#: evaluated (one launch per step); from PAIR_ROWS_MIN_PARTICLES up the pair kernel does
ADVANCE_ROWS_MAX_PARTICLES = 60_000
#: ... and up to this size (148 SMs x 1024 resident threads, one lane per particle) the
#: intermediate steps run in batches inside one cooperative launch (b2md_steps_persistent)
PERSISTENT_MAX_PARTICLES = 148 * 1024

_REORDER_MODES = {None: 0, "none": 0, "hilbert": 1, "cell": 2}


def _torch():
    import torch
    return torch


class Simulation:
    def __init__(self, state: ParticleState, box: SimBox, lj, dt: float,
                 backend: BackendSelector | None = None, force_mode: str = ALL_TO_ALL,
                 skin: float = DEFAULT_SKIN, stride: int | None = None, thermostat=None,
                 sample_interval: int = 100, deterministic: bool = True,
                 sample_initial: bool = False, reorder: str | None = "hilbert",
                 reorder_every: int = 1, native: bool | None = None,
                 stride_policy: str = "fit", graph: int | bool = False,
                 pair_rows: bool | None = None, advance: bool | None = None,
                 queue_depth: int | None = None, persistent_steps: int | None = None,
                 prune_delta: float | None = None):
        if force_mode not in FORCE_MODES:
            raise ConfigError(f"unknown force_mode {force_mode!r}")
        if force_mode == TRUNCATED and not lj.truncated:
            raise ConfigError("truncated force mode needs a finite r_cut")
        if skin < 0.0:
            raise ConfigError("skin must be non-negative")
        thermostatted = thermostat is not None and getattr(thermostat, "rate", 0.0) > 0.0
        if reorder not in _REORDER_MODES:
            raise ConfigError(f"unknown reorder mode {reorder!r}")
        if stride_policy not in ("fit", "double", "tight"):
            raise ConfigError("stride_policy must be 'fit', 'double' or 'tight'")

        self.state = state
        self.box = box
        self.lj = lj
        self.integrator = IntegratorParams(dt)
        self.backend = backend if backend is not None else BackendSelector()
        self.force_mode = force_mode
        self.skin = float(skin)
        self.thermostat = thermostat
        self.reduction_mode = DETERMINISTIC if deterministic else FAST
        self.reorder = reorder if force_mode == TRUNCATED else None
        self.reorder_every = max(int(reorder_every), 1)
        self.stride_policy = stride_policy
        self.graph = int(graph)          # MD steps per captured CUDA graph (0 = host-driven)
        # force kernel: one thread per particle pair over merged rows (None = by size)
        self.pair_rows = use_pair_rows(state.n, pair_rows)
        # one-launch intermediate steps (needs pair rows; B2MD_ADVANCE=0 turns them off)
        # (measured, profiles/exp/queue_depth.py: a clear gain with pair rows and for small
        # systems, a loss for the sub-warp row kernel between 65 k and 200 k particles)
        if advance is None:
            env = os.environ.get("B2MD_ADVANCE")
            advance = (env != "0") if env in ("0", "1") else \
                (self.pair_rows or state.n < PERSISTENT_MAX_PARTICLES)
        self.advance = bool(advance) and not thermostatted
        # one-launch steps queued per status read-back (small systems: a step is shorter
        # than a host round trip)
        self.queue_depth = int(os.environ.get("B2MD_QUEUE_DEPTH", "1")) if queue_depth is None \
            else int(queue_depth)
        # systems without pair rows: MD steps per launch of the persistent step kernel
        # (b2md_steps_persistent; 0 = one gated launch per step).  Bit-identical trajectories.
        self.persistent_steps = int(os.environ.get("B2MD_PERSISTENT_STEPS", "256")) \
            if persistent_steps is None else int(persistent_steps)
        # Pruned pair rows for the one-launch steps: rows cut to r_cut + prune_delta, re-pruned
        # from the full list rows whenever a particle has moved prune_delta / 2 (the full rows
        # keep the reference's rebuild schedule, neighbor.py:243-254; dropped entries would
        # have contributed exact zeros, so trajectories are bit-identical).  Off by default
        # (None / 0): measured at N = 1 M, skin 0.3, delta 0.1, a step over the inner rows takes
        # 97 us instead of 109, but each of the three prune launches per list costs 209 us (the
        # per-entry compaction doubles the instructions of the issue-bound loop) -- 0.1418 against
        # 0.1425 ms per step, inside the noise (profiles/README.md).
        if prune_delta is None:
            env = os.environ.get("B2MD_PRUNE_DELTA")
            prune_delta = float(env) if env not in (None, "") else 0.0
        # (legal prunes need every particle within (skin - delta) / 2 <= 0.125 of the snapshot)
        self.prune_delta = float(prune_delta) if (0.0 < prune_delta < self.skin and
                                                  0.5 * (self.skin - prune_delta) <= 0.125) else 0.0
        self.graph_steps = 0
        # (a thermostatted native loop launches integrate / force / finalize / thermostat
        # separately: the thermostat is the reference's second finalize slot, sim.py:86-87)
        # all-to-all forces (the reference's default force mode) have their own native loop,
        # b2md_run_all_pairs: no list, nothing to decide between steps, so a call is enqueued
        # whole.  native=False keeps the operator-by-operator loop (one ctypes call and one
        # status read-back per operator: ~90 us per step of host time at N = 2000).
        self.native_all_pairs = force_mode == ALL_TO_ALL and (native is None or bool(native))
        self.native = (force_mode == TRUNCATED) if native is None else \
            (bool(native) and force_mode == TRUNCATED)
        self._thermostatted = thermostatted
        if not self.native and self.reorder == "cell":
            raise ConfigError("reorder='cell' is implemented by the native step loop only")

        # Row capacity of the first build.  The reference starts at DEFAULT_STRIDE = 64 and
        # doubles on overflow (sim.py:30,141-149); a dense fluid overflows that at once, and
        # on the device a second 1 ms build plus a re-allocation of the list is most of a
        # short call.  None (default) sizes the first build from the mean density instead:
        # 1.25 x the ideal-gas count inside r_list + 16 (an fcc start lists 78 where the
        # fluid lists 67; Kob-Andersen 134 / 110), never below the reference's 64.  Overflow
        # keeps its semantics either way: flagged, never truncated, grow and rebuild.
        if stride is None:
            stride = DEFAULT_STRIDE
            if force_mode == TRUNCATED:
                r_list = lj.max_r_cut + float(skin)
                expected = state.n / box.volume * (4.0 / 3.0) * np.pi * r_list ** 3
                stride = max(DEFAULT_STRIDE, _round_up(int(1.25 * expected) + 16, 8))
                stride = min(stride, max(_round_up(state.n, 8), DEFAULT_STRIDE))
        self._stride = int(stride)
        self._nlist: NeighborList | None = None
        self.overflow_events = 0
        self.force_seconds = 0.0
        self.nlist_seconds = 0.0
        self._rebuild_base = 0
        self._rebuild_total = 0
        self.samples: list[Sample] = []
        self.sampling_enabled = True
        self.kernel_launches = 0
        self.wasted_force_launches = 0
        self.reorders = 0

        self.engine = SignalEngine(sample_interval=sample_interval,
                                   sample_initial=sample_initial)
        self.engine.connect("integrate", self._integrate_slot)
        self.engine.connect("force", self._force_slot)
        self.engine.connect("finalize", self._finalize_slot)
        if thermostatted:
            self.engine.connect("finalize", self._thermostat_slot)     # sim.py:86-87
        self.engine.connect("sample", self._sample_slot)

        self._runner = None
        self._keep = {}
        if self.native:
            self._native_setup()
        else:
            self._compute_forces()

    # ------------------------------------------------------------------ slots
    def _integrate_slot(self):
        vv_integrate(self.state, self.integrator, self.box)

    def _finalize_slot(self):
        vv_finalize(self.state, self.integrator)

    def _thermostat_slot(self):
        andersen_thermostat(self.state, self.thermostat, self.integrator.dt,
                            self.engine.step_count)                    # sim.py:100-102

    def _force_slot(self):
        self._compute_forces()

    def _sample_slot(self):
        if self.sampling_enabled:
            self.samples.append(self.measure())

    # ---------------------------------------------- operator-by-operator path
    def _compute_forces(self):
        if self.force_mode == ALL_TO_ALL:
            t0 = time.perf_counter()
            compute_forces_all_to_all(self.state, self.lj, self.box, self.backend)
            self.force_seconds += time.perf_counter() - t0
            return
        t0 = time.perf_counter()
        if self._nlist is None or needs_rebuild(self.state, self.box, self._nlist):
            self._rebuild()
        self.nlist_seconds += time.perf_counter() - t0
        t0 = time.perf_counter()
        compute_forces_truncated(self.state, self.lj, self.box, self._nlist, self.backend,
                                 pair_rows=self.pair_rows)
        self.force_seconds += time.perf_counter() - t0

    def _grow_stride(self, max_count: int):
        if self.stride_policy == "double":
            self._stride *= 2                       # sim.py:149
        elif self.stride_policy == "tight":         # exactly what the fullest row wanted
            self._stride = max(self._stride + 1, int(max_count))
        else:
            self._stride = max(self._stride + 1, _round_up(int(max_count * 1.125) + 1, 8))

    def _rebuild(self):
        """bin -> (reorder) -> build, growing the stride on overflow (sim.py:131-149)."""
        r_list = self.lj.max_r_cut + self.skin
        if self.reorder == "hilbert" and self._rebuild_total % self.reorder_every == 0:
            reorder_hilbert(self.state, self.box, r_list, HILBERT_SUB_BITS, internal=True)
            self.reorders += 1
        growths = 0
        while True:
            grid = bin_particles(self.state, self.box, r_list)
            nlist = build_neighbor_list(self.state, grid, r_list, self._stride,
                                        r_cut=self.lj.max_r_cut, prev=self._nlist,
                                        backend=self.backend, _recycle=True)
            self._nlist = nlist
            self._rebuild_total += 1
            if not nlist.overflow:
                return
            self.overflow_events += 1
            growths += 1
            if growths > STRIDE_GROWTH_LIMIT:
                raise NeighborOverflowError(
                    f"neighbor list still overflows after {growths - 1} "
                    f"stride growths (stride {self._stride})")
            self._grow_stride(nlist.max_count)

    # ------------------------------------------------------- native step loop
    def _alloc_list(self, dev: DeviceState):
        torch = _torch()
        pitch = _round_up(dev.n, 32)
        # (64-row granules let the persistent step kernel of small systems put 16 lanes on a
        # particle: a trip of it reads 4 x 16 entries of a row)
        rows = _round_up(self._stride, self._row_multiple())
        # zero-filled: padding entries must stay valid row indices for the row kernels.  With
        # pair rows the step loop never reads a padding entry of this buffer (it is the list
        # build's scratch, b2md_build_pair_list): no fill -- 65 us of HBM writes at N = 1 M
        make = torch.empty if self.pair_rows else torch.zeros
        return make((rows, pitch), dtype=torch.int32, device=dev.device), pitch

    def _row_multiple(self) -> int:
        return 64 if self.state.n < 200_000 else 16

    def _alloc_pair_list(self, dev: DeviceState):
        """Pair-row buffer: 2 * rows entries per pair, so a merge never overflows."""
        torch = _torch()
        rows = _round_up(self._stride, self._row_multiple())
        pair_pitch = _round_up((dev.n + 1) // 2, 32)
        # (no fill: every tile a launch reads -- up to the longest row of its warp -- is written
        # by the list build first)
        return (torch.empty((2 * rows // 4, pair_pitch, 4), dtype=torch.int32,
                            device=dev.device), pair_pitch, 2 * rows)

    def _upload_state(self, k):
        """Make every buffer valid on the device.  Velocities that still have to cross PCIe go
        last and on a side stream: the first list build needs positions only, so the runner
        is told to wait for them behind it (b2md_runner_config::vel_ready_event) and the
        upload overlaps the build.  Returns the event, or None."""
        torch = _torch()
        st = self.state
        vel = st.velocities
        dev = st.device_state()
        if vel.valid_on in (COMPUTE, "both") or self.graph:
            st.sync_to_compute()
            return None
        for name, buf in st.buffers().items():
            if name != "velocities":
                buf.acquire_read(COMPUTE)
        main = torch.cuda.current_stream(dev.device)
        side = k["copy_stream"]
        side.wait_stream(main)                  # (the device rows exist and hold their defaults)
        with torch.cuda.stream(side):
            vel.acquire_read(COMPUTE)
        k["vel_ready"] = torch.cuda.Event()
        k["vel_ready"].record(side)
        return k["vel_ready"]

    def _native_setup(self):
        torch = _torch()
        k = self._keep
        dev0 = self.state.device_state()
        k["run_stream"] = torch.cuda.Stream(device=dev0.device)
        k["copy_stream"] = torch.cuda.Stream(device=dev0.device)
        vel_ready = self._upload_state(k)
        dev = self.state.device_state()
        n = dev.n
        r_list = self.lj.max_r_cut + self.skin
        g = grid_shape(self.box, r_list)
        d = dict(device=dev.device)
        lib = _lib.load()
        k = self._keep
        k["sets"] = [
            {name: getattr(dev, name) for name in DeviceState.ROW16 + ("virial",)},
            {name: torch.zeros_like(getattr(dev, name)) for name in DeviceState.ROW16 + ("virial",)},
        ]
        k["sets"][1]["vel"][:, 3] = 1.0
        k["current"] = 0
        k["nbr"], pitch = self._alloc_list(dev)
        k["pitch"] = pitch
        # (buffers below that every rebuild writes in full before anything reads them are not
        # zero-filled: Simulation() is inside the timed end-to-end call)
        k["counts"] = torch.zeros(pitch, dtype=torch.int32, **d)
        k["boundary"] = torch.zeros(pitch, dtype=torch.uint8, **d)
        k["ref_pos"] = torch.empty((pitch, 4), dtype=torch.float32, **d)
        k["at_build"] = torch.empty((n, 3), dtype=torch.float64, **d)
        k["cell_of"] = torch.empty(n, dtype=torch.int32, **d)
        k["cell_start"] = torch.zeros(int(g.n_cells) + 1, dtype=torch.int32, **d)
        k["cell_particles"] = torch.empty(n, dtype=torch.int32, **d)
        k["bin_scratch"] = torch.zeros(int(lib.b2md_bin_scratch_bytes(n, g.n_cells)),
                                       dtype=torch.uint8, **d)
        k["keys"] = torch.empty(n, dtype=torch.int64, **d)
        k["keys_tmp"] = torch.empty(n, dtype=torch.int64, **d)
        k["perm"] = torch.empty(n, dtype=torch.int32, **d)
        k["perm_tmp"] = torch.empty(n, dtype=torch.int32, **d)
        k["sort_scratch"] = torch.zeros(int(lib.b2md_sort_scratch_bytes(n)), dtype=torch.uint8, **d)
        k["table"] = np.ascontiguousarray(self.lj.table(), dtype=np.float64)
        if self.lj.ntypes > 1:
            sp = self.state.species.acquire_read("host")
            if sp.min() < 0 or sp.max() >= self.lj.ntypes:
                raise ValueError("species out of range for the pair table")

        cfg = _lib.RunnerConfig()
        cfg.n, cfg.capacity = n, dev.capacity
        cfg.box = _lib.make_box(self.box.edge_lengths)
        cfg.dt, cfg.r_cut, cfg.skin = self.integrator.dt, self.lj.max_r_cut, self.skin
        cfg.ntypes = self.lj.ntypes
        cfg.reorder_mode = _REORDER_MODES[self.reorder]
        cfg.reorder_every = self.reorder_every
        cfg.hilbert_bits = HILBERT_SUB_BITS
        cfg.table = k["table"].ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        for name in DeviceState.ROW16 + ("virial",):
            arr = getattr(cfg, name)
            arr[0] = k["sets"][0][name].data_ptr()
            arr[1] = k["sets"][1][name].data_ptr()
        cfg.current = 0
        cfg.stride = self._stride
        cfg.nbr, cfg.pitch = k["nbr"].data_ptr(), pitch
        for name in ("counts", "boundary", "ref_pos", "at_build", "cell_of", "cell_start",
                     "cell_particles", "bin_scratch", "keys", "keys_tmp", "perm", "perm_tmp",
                     "sort_scratch"):
            setattr(cfg, name, k[name].data_ptr())
        cfg.status = dev.status.data_ptr()
        cfg.stream = dev.stream
        cfg.use_graph = self.graph
        if self.advance and not self.graph:
            # second buffer for the position high words: intermediate steps then run as one
            # launch each (force + finalize + integrate, b2md_force_lj[_pairs]_advance)
            k["pos_hi_alt"] = torch.empty_like(dev.pos_hi)
            cfg.pos_hi_alt = k["pos_hi_alt"].data_ptr()
            cfg.queue_depth = max(self.queue_depth, 1)
        cfg.list_row_multiple = self._row_multiple()
        if self.advance and not self.graph and not self.pair_rows and self.persistent_steps > 0:
            # small systems: intermediate steps in batches inside one cooperative launch
            k["barrier"] = torch.zeros(1024, dtype=torch.int32, **d)      # B2MD_BARRIER_BYTES
            cfg.barrier = k["barrier"].data_ptr()
            cfg.persistent_steps = self.persistent_steps
        if self.pair_rows:
            k["pair_nbr"], cfg.pair_pitch, cfg.pair_rows = self._alloc_pair_list(dev)
            # pair counts, then the block schedule of the pair kernel (b2md_pair_schedule)
            k["pair_counts"] = torch.zeros(
                cfg.pair_pitch + int(lib.b2md_pair_schedule_len(n)), dtype=torch.int32, **d)
            # bit 0: block schedule, bit 1: lane order (b2md_pair_order), bit 2: its face key,
            # bits 8-13: its unit
            cfg.pair_schedule = int(os.environ.get("B2MD_PAIR_SCHEDULE", "1"))
            cfg.pair_nbr = k["pair_nbr"].data_ptr()
            cfg.pair_counts = k["pair_counts"].data_ptr()
            if self.prune_delta > 0.0 and self.advance and not self.graph and \
                    max(self.queue_depth, 1) == 1:
                # pruned ("inner") pair rows for the one-launch steps
                k["pair_nbr_inner"] = torch.empty_like(k["pair_nbr"])
                k["pair_counts_inner"] = torch.zeros(cfg.pair_pitch, dtype=torch.int32, **d)
                cfg.pair_nbr_inner = k["pair_nbr_inner"].data_ptr()
                cfg.pair_counts_inner = k["pair_counts_inner"].data_ptr()
                cfg.prune_delta = self.prune_delta
        # page-locked status mirror and the runner's two streams come from torch's caching
        # host allocator / stream pool: creating them per runner costs 1-7 ms of driver calls
        k["h_status"] = torch.empty(16, dtype=torch.int32).pin_memory()
        cfg.h_status = k["h_status"].data_ptr()
        if vel_ready is not None:
            cfg.vel_ready_event = vel_ready.cuda_event
        cfg.run_stream = k["run_stream"].cuda_stream
        cfg.copy_stream = k["copy_stream"].cuda_stream
        k["cfg"] = cfg
        dev.reset_status()
        handle = lib.b2md_runner_create(ctypes.byref(cfg))
        if not handle:
            raise _lib.B2mdError("b2md_runner_create failed: "
                                 + lib.b2md_last_error_string().decode())
        self._runner = ctypes.c_void_p(handle)
        if self._thermostatted:
            _lib.call("b2md_runner_set_thermostat", self._runner,
                      float(self.thermostat.redraw_probability(self.integrator.dt)),
                      float(self.thermostat.temperature), int(self.thermostat.seed) % (1 << 64))
        self._native_call("b2md_runner_prepare")
        if vel_ready is not None:
            # anything the caller enqueues on its own stream from here on sees the velocities
            torch.cuda.current_stream(dev.device).wait_stream(k["copy_stream"])

    def _native_call(self, name, *args):
        """Invoke the runner, handling overflow (grow + resume) and singular pairs."""
        dev = self.state.device_state()
        done = 0
        growths = 0
        while True:
            rep = _lib.RunReport()
            t0 = time.perf_counter()
            if name == "b2md_runner_run":
                n_steps, finalize = args
                # the thermostat stream is indexed by SignalEngine.step_count (sim.py:100-102)
                _lib.call("b2md_runner_set_step", self._runner, self.engine.step_count + done)
                _lib.call(name, self._runner, n_steps - done, finalize, ctypes.byref(rep))
            else:
                _lib.call(name, self._runner, ctypes.byref(rep))
            # phase timers from CUDA events on the runner's stream (sim.py:114-129): rebuild
            # sequences -> nlist_seconds, everything else the call enqueued -> force_seconds;
            # host time the GPU did not cover (launch latency of short steps) goes to neither
            wall = time.perf_counter() - t0
            self.nlist_seconds += 1e-3 * rep.rebuild_gpu_ms
            self.force_seconds += max(min(1e-3 * rep.gpu_ms, wall) - 1e-3 * rep.rebuild_gpu_ms, 0.0)
            done += rep.steps_done
            self._absorb(rep, dev)
            if rep.reason == _lib.RUN_SINGULAR:
                i, j = rep.singular >> 32, rep.singular & 0xFFFFFFFF
                ids = dev.particle_ids()
                i, j = sorted((int(ids[i]), int(ids[j])))
                raise SingularPairError(i, j)
            if rep.reason == _lib.RUN_OVERFLOW:
                self.overflow_events += 1
                growths += 1
                if growths > STRIDE_GROWTH_LIMIT:
                    raise NeighborOverflowError(
                        f"neighbor list still overflows after {growths - 1} "
                        f"stride growths (stride {self._stride})")
                self._grow_stride(rep.max_count)
                self._keep["nbr"], _ = self._alloc_list(dev)
                _lib.call("b2md_runner_set_list", self._runner, self._keep["nbr"].data_ptr(),
                          self._stride)
                if self.pair_rows:
                    self._keep["pair_nbr"], _, rows2 = self._alloc_pair_list(dev)
                    _lib.call("b2md_runner_set_pair_list", self._runner,
                              self._keep["pair_nbr"].data_ptr(), rows2)
                    self._keep["cfg"].pair_rows = rows2
                    if "pair_nbr_inner" in self._keep:
                        self._keep["pair_nbr_inner"] = _torch().empty_like(self._keep["pair_nbr"])
                        _lib.call("b2md_runner_set_inner_pair_list", self._runner,
                                  self._keep["pair_nbr_inner"].data_ptr())
                continue
            return

    def _absorb(self, rep, dev: DeviceState):
        """Fold a run report into the Python-side bookkeeping."""
        k = self._keep
        self._rebuild_total += rep.rebuilds
        self.reorders += rep.reorders
        self.kernel_launches += rep.kernel_launches
        self.wasted_force_launches += rep.wasted_force_launches
        self.graph_steps += rep.graph_steps
        if rep.reorders:
            dev.identity_order = False
        if rep.current != k["current"]:
            k["current"] = rep.current
            for name, t in k["sets"][rep.current].items():
                setattr(dev, name, t)
        self._max_count = rep.max_count
        self._n_boundary = rep.n_boundary
        # the kernels rewrote these buffers in HBM
        self.state.mark_compute_written("positions", "images", "velocities", "forces",
                                        "per_particle_potential", "virial")

    def _run_native(self, n_steps: int):
        eng = self.engine
        eng._check_ready(n_steps)
        if n_steps == 0:
            return
        # make sure host-side edits since the last call reach the device
        self.state.sync_to_compute()
        eng.emit_initial_sample()
        left = n_steps
        while left > 0:
            to_sample = eng.sample_interval - (eng.step_count % eng.sample_interval)
            chunk = min(left, to_sample)
            self._native_call("b2md_runner_run", chunk, 1)
            eng.step_count += chunk
            left -= chunk
            if eng.step_count % eng.sample_interval == 0:
                eng.emit("sample")

    # ------------------------------------------------------------ observation
    @property
    def rebuild_count(self) -> int:
        """Rebuilds since the last counter reset."""
        return self._rebuild_total - self._rebuild_base

    @property
    def stride(self) -> int:
        return self._stride

    def measure(self) -> Sample:
        """Observe the system now: one device reduction pass, 8 doubles read back."""
        t = thermo(self.state)
        return Sample(
            step=self.engine.step_count,
            time=self.engine.step_count * self.integrator.dt,
            potential_energy=t.potential_energy,
            kinetic_energy=t.kinetic_energy,
            total_energy=t.potential_energy + t.kinetic_energy,
            temperature=t.temperature,
            total_momentum=t.momentum,
            rebuild_count=self.rebuild_count,
            virial=t.virial,
            pressure=t.pressure(self.box.volume),
            com_velocity=t.com_velocity,
        )

    def prune_stats(self):
        """(prune launches, one-launch steps that walked the full rows) of the native loop."""
        if not self.native or not getattr(self, "_runner", None):
            return 0, 0
        outer = ctypes.c_int64(0)
        prunes = _lib.load().b2md_runner_prune_count(self._runner, ctypes.byref(outer))
        return int(prunes), int(outer.value)

    def reset_counters(self):
        """Zero phase timers, overflow events and the rebuild baseline."""
        self.force_seconds = 0.0
        self.nlist_seconds = 0.0
        self.overflow_events = 0
        self.kernel_launches = 0
        self.wasted_force_launches = 0
        self._rebuild_base = self._rebuild_total

    def _run_native_all_pairs(self, n_steps: int):
        """Simulation.run for force_mode = "all_to_all" through b2md_run_all_pairs: the steps
        between two samples are one call (bit-identical to the operator loop)."""
        eng = self.engine
        eng._check_ready(n_steps)
        if n_steps == 0:
            return
        torch = _torch()
        st = self.state
        st.sync_to_compute()
        eng.emit_initial_sample()
        dev = st.device_state()
        tab, tab_ptr, nt = _table_ptr(self.lj, st)
        if "h_status" not in self._keep:
            self._keep["h_status"] = torch.empty(64, dtype=torch.uint8).pin_memory()
        # second buffer for the position high words: intermediate steps are one launch each
        alt = self._keep.get("pos_alt")
        if alt is None or alt.shape != dev.pos_hi.shape or alt.device != dev.pos_hi.device:
            alt = self._keep["pos_alt"] = torch.empty_like(dev.pos_hi)
        p = self.thermostat.redraw_probability(self.integrator.dt) if self._thermostatted else 0.0
        temperature = float(self.thermostat.temperature) if self._thermostatted else 1.0
        seed = int(self.thermostat.seed) % (1 << 64) if self._thermostatted else 0
        left = n_steps
        while left > 0:
            to_sample = eng.sample_interval - (eng.step_count % eng.sample_interval)
            chunk = min(left, to_sample)
            rep = _lib.RunReport()
            t0 = time.perf_counter()
            _lib.call("b2md_run_all_pairs", dev.pos_hi.data_ptr(), dev.pos_lo.data_ptr(),
                      dev.vel.data_ptr(), dev.force.data_ptr(), dev.image.data_ptr(),
                      dev.virial.data_ptr(), dev.n, self.box.c_box(), tab_ptr, nt,
                      float(self.integrator.dt), chunk, float(p), temperature, seed,
                      eng.step_count, alt.data_ptr(), dev.status.data_ptr(),
                      self._keep["h_status"].data_ptr(),
                      dev.stream, ctypes.byref(rep))
            wall = time.perf_counter() - t0
            self.force_seconds += min(1e-3 * rep.gpu_ms, wall)
            self.kernel_launches += rep.kernel_launches
            st.mark_compute_written("positions", "images", "velocities", "forces",
                                    "per_particle_potential", "virial")
            if rep.reason == _lib.RUN_SINGULAR:
                i, j = rep.singular >> 32, rep.singular & 0xFFFFFFFF
                if not dev.identity_order:
                    ids = dev.particle_ids()
                    i, j = sorted((int(ids[i]), int(ids[j])))
                raise SingularPairError(int(i), int(j))
            eng.step_count += chunk
            left -= chunk
            if eng.step_count % eng.sample_interval == 0:
                eng.emit("sample")

    def run(self, n_steps: int):
        if getattr(self, "_closed", False):
            raise RuntimeError("this Simulation was closed")
        if self.native_all_pairs:
            self._run_native_all_pairs(n_steps)
        elif self.native:
            self._run_native(n_steps)
        else:
            self.engine.run_steps(n_steps)

    def close(self):
        """Destroy the native runner and hand the simulation's device buffers (lists, pair
        rows, sort scratch, the spare state set: 1 GB at N = 1 M) back to the allocator now,
        not when the cycle collector gets round to it (slots are bound methods: a Simulation
        and its SignalEngine reference each other).  The ParticleState stays usable."""
        if self._runner is not None:
            _lib.load().b2md_runner_destroy(self._runner)
            self._runner = None
            k = self._keep
            if k:
                # the state keeps whichever set is live; everything else goes
                dev = self.state.device_state()
                live = k["sets"][k.get("current", 0)]
                for name, t in live.items():
                    setattr(dev, name, t)
            self._keep = {}
        elif self.native_all_pairs:
            self._keep = {}          # pinned status block, second position buffer
        self._nlist = None
        self._closed = True
        for slots in self.engine._slots.values():
            slots.clear()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass
