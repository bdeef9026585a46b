"""Slab-decomposed multi-GPU driver: one process per GPU, 1-D slabs along x,
ghost-layer halo exchange every step and particle migration at every list
rebuild, over NCCL send/recv.  The reference has no spatial
decomposition; the single-domain run is the oracle.

Layout per rank: owned rows [0, n_own) followed by ghost rows
[n_own, n_own + n_ghost_left + n_ghost_right), all in GLOBAL coordinates of the
global periodic box, so the cell / list / force kernels run unchanged (rows are
built and forces evaluated for owned rows only; the list is full, so ghosts need
positions only and no force is ever sent back).

Per step (no rebuild), large slabs: ONE gated launch of the pair force kernel that
    also finalizes and integrates the owned rows (b2md_force_lj_pairs_advance) ->
    pack the fixed send lists (pos_hi rows) -> NCCL send/recv straight into the
    ghost rows -> in-place all-reduce(max) of the flag word the kernel wrote; the
    host reads the status block on a side stream while the next launch is already
    queued (SlabSimulation._run_advance).
Small slabs / sample steps: fused finalize+integrate -> flag all-reduce -> halo ->
    force kernel (launched before the flag is inspected, as in the 1-GPU loop).
At a rebuild (all ranks together): migrate rows that left the slab (full
    records), reorder the owned rows (Hilbert), select + exchange ghost records
    (pos_hi, pos_lo), bin, build the list for owned rows, forces.

The protocol is written against a small `ops` interface so that the same code runs
on `CudaSlabOps` (libb2md kernels, CUDA tensors, NCCL) and, in the CPU test-suite,
on a numpy test double over gloo (tests/test_slab_gloo.py).
"""
from __future__ import annotations

import ctypes
import json
import math
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, NeighborOverflowError

MIGRANT_WORDS = 16     # pos_hi(4) pos_lo(4) vel(4) image(4) as 32-bit words
GHOST_WORDS = 8        # pos_hi(4) pos_lo(4)


def _torch():
    import torch
    return torch


# ------------------------------------------------------------------ geometry
@dataclass(frozen=True)
class SlabGeometry:
    """x-slab of rank `rank` of `world` in a global box of edges `edges`."""
    rank: int
    world: int
    edges: tuple

    @property
    def width(self) -> float:
        return self.edges[0] / self.world

    @property
    def x_lo(self) -> float:
        return self.rank * self.width

    @property
    def centre(self) -> float:
        return self.x_lo + 0.5 * self.width

    @property
    def left(self) -> int:
        return (self.rank - 1) % self.world

    @property
    def right(self) -> int:
        return (self.rank + 1) % self.world

    def check(self, r_ghost: float):
        if self.world > 1 and self.width < 2.0 * r_ghost:
            raise ConfigError(
                f"slab width {self.width:g} must be at least twice the ghost width {r_ghost:g}")


# ------------------------------------------------------------ communication
class SlabComm:
    """Neighbour exchange on the periodic ring of ranks (torch.distributed)."""

    def __init__(self, geometry: SlabGeometry, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.geo = geometry
        self.group = group
        self.bytes_sent = 0
        # gloo moves host memory only: CUDA tensors are staged through the host there
        # (used by the 2-process single-GPU test; production runs use NCCL)
        self.stage_on_host = geometry.world > 1 and dist.get_backend(group) == "gloo"

    def exchange_counts(self, n_left: int, n_right: int, device):
        """Tell each neighbour how many records it will receive."""
        got_l, got_r = self.exchange_ints([n_left], [n_right], device)
        return got_l[0], got_r[0]

    def exchange_ints(self, to_left, to_right, device):
        """Small integer vectors to both neighbours; returns (from_left, from_right)."""
        torch = _torch()
        k = len(to_left)
        send = torch.tensor([list(to_left), list(to_right)], dtype=torch.int64, device=device)
        got_from_right = torch.zeros(k, dtype=torch.int64, device=device)
        got_from_left = torch.zeros(k, dtype=torch.int64, device=device)
        self._ring(send[0], send[1], got_from_right, got_from_left)
        return got_from_left.tolist(), got_from_right.tolist()

    def _ring(self, to_left, to_right, from_right, from_left):
        """to_left -> left neighbour (arrives as its from_right), to_right -> right."""
        dist = self.dist
        g = self.geo
        if g.world == 1:
            from_right.copy_(to_left)
            from_left.copy_(to_right)
            return
        staged = self.stage_on_host and to_left.is_cuda
        if staged:
            dev_right, dev_left = from_right, from_left
            to_left, to_right = to_left.cpu(), to_right.cpu()
            from_right, from_left = from_right.cpu(), from_left.cpu()
        # Order matters for world == 2 (both neighbours are the same rank, and NCCL
        # matches messages between a pair of ranks in posting order, ignoring tags):
        # what I send leftwards is what my left neighbour receives "from its right".
        # Empty messages are skipped on both sides (sizes were agreed on beforehand).
        ops = []
        if to_left.numel():
            ops.append(dist.P2POp(dist.isend, to_left.contiguous(), g.left, self.group, tag=0))
        if to_right.numel():
            ops.append(dist.P2POp(dist.isend, to_right.contiguous(), g.right, self.group, tag=1))
        if from_right.numel():
            ops.append(dist.P2POp(dist.irecv, from_right, g.right, self.group, tag=0))
        if from_left.numel():
            ops.append(dist.P2POp(dist.irecv, from_left, g.left, self.group, tag=1))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if staged:
            dev_right.copy_(from_right)
            dev_left.copy_(from_left)
        self.bytes_sent += to_left.numel() * to_left.element_size() + \
            to_right.numel() * to_right.element_size()

    def self_check(self, device):
        """Start-up check of the ring plumbing: every rank sends its own id both ways and must
        receive its left neighbour's id "from the left" and its right neighbour's "from the
        right".  Catches the world == 2 trap (both neighbours are the same rank and NCCL
        matches a pair's messages in posting order, ignoring tags) on whatever backend is in
        use, before any particle data moves."""
        g = self.geo
        from_l, from_r = self.exchange_ints([g.rank, 1], [g.rank, 2], device)
        # what my LEFT neighbour sent rightwards carries marker 2, and vice versa
        if from_l != [g.left, 2] or from_r != [g.right, 1]:
            raise ConfigError(f"slab ring self-check failed on rank {g.rank}: received {from_l} "
                              f"from the left (want [{g.left}, 2]) and {from_r} from the right "
                              f"(want [{g.right}, 1])")

    def exchange(self, to_left, to_right, from_left, from_right):
        """Variable-size record exchange (sizes agreed on beforehand)."""
        self._ring(to_left, to_right, from_right, from_left)

    def _all_reduce(self, tensor, op):
        if self.geo.world > 1:
            if self.stage_on_host and tensor.is_cuda:
                host = tensor.cpu()
                self.dist.all_reduce(host, op=op, group=self.group)
                tensor.copy_(host)
            else:
                self.dist.all_reduce(tensor, op=op, group=self.group)
        return tensor

    def all_max(self, value_tensor):
        return self._all_reduce(value_tensor, self.dist.ReduceOp.MAX)

    def all_sum(self, tensor):
        return self._all_reduce(tensor, self.dist.ReduceOp.SUM)


# ------------------------------------------------------------------ protocol
class SlabSimulation:
    """NVE truncated-LJ run of one slab.  `ops` owns the particle arrays and the
    kernels; this class owns the decomposition protocol."""

    STRIDE_GROWTH_LIMIT = 10

    def __init__(self, ops, comm: SlabComm, lj, dt: float, skin: float, sample_interval=100):
        self.ops, self.comm, self.geo = ops, comm, comm.geo
        self.lj, self.dt, self.skin = lj, float(dt), float(skin)
        self.r_list = lj.max_r_cut + self.skin
        self.geo.check(self.r_list)
        self.sample_interval = int(sample_interval)
        self.step_count = 0
        self.rebuilds = 0
        self.samples = []
        self.pending_kick = False
        self.ahead = False            # one-launch steps: particles already at the next step
        self.halo_rows = (0, 0)
        self.ops.attach(self.geo, lj, self.dt, self.skin)
        comm.self_check(self.ops.device)
        # Per-step halo fused into the step kernel (backends with `connect_peers`): the
        # advanced high words of the send-list rows are stored by the kernel itself into
        # the ghost rows of the neighbour ranks' position buffers, mapped into this process
        # (peer memory over NVLink) -- no pack kernels, no send/recv inside a step.
        connect = getattr(self.ops, "connect_peers", None)
        self.fused_halo = bool(connect(comm)) if connect else False
        self._rebuild()
        if self.fused_halo:
            self._probe_peer_halo()
        self.ops.force(thermo=True)

    def _probe_peer_halo(self):
        """One halo through each transport before the first step: the NCCL exchange fills the
        ghost rows, the peer stores (same destination slots as the step kernel uses) overwrite
        them; the ghost rows must not change.  A mismatch anywhere -- wrong mapping, a peer
        path that silently drops writes -- turns the fused halo off on every rank, loudly."""
        ops, comm = self.ops, self.comm
        probe = getattr(ops, "probe_peer_halo", None)
        if probe is None:
            return
        self._halo()                                   # reference content, over NCCL
        bad = probe(comm)                              # 0 / 1, already agreed on by all ranks
        if bad:
            import warnings
            warnings.warn("slab halo: peer stores did not reproduce the NCCL halo; falling back "
                          "to NCCL send/recv on all ranks", RuntimeWarning)
            ops.disconnect_peers()
            self.fused_halo = False

    # -- rebuild: migrate, reorder, ghosts, list ------------------------------
    def _rebuild(self):
        ops, comm = self.ops, self.comm
        growths = 0
        # 1. migration of rows that left the slab (full records)
        n_l, n_r = ops.select_migrants()
        got_l, got_r = comm.exchange_counts(n_l, n_r, ops.device)
        out_l, out_r = ops.pack_migrants()
        in_l, in_r = ops.migrant_buffer(got_l), ops.migrant_buffer(got_r)
        comm.exchange(out_l, out_r, in_l, in_r)
        ops.apply_migration(in_l, in_r)
        # 2. locality reorder of the owned rows
        ops.reorder_owned()
        # 3. ghost selection + exchange of (pos_hi, pos_lo) records
        n_l, n_r = ops.select_ghosts(self.r_list)
        got_l, got_r = comm.exchange_counts(n_l, n_r, ops.device)
        out_l, out_r = ops.pack_ghost_records()
        in_l, in_r = ops.ghost_buffer(got_l), ops.ghost_buffer(got_r)
        comm.exchange(out_l, out_r, in_l, in_r)
        ops.set_ghosts(in_l, in_r)
        self.halo_rows = (got_l, got_r)
        if self.fused_halo:
            # where my send lists land on the neighbours: what I send leftwards is the left
            # neighbour's "from the right" ghost range, and vice versa; the neighbours must
            # also be at the same point of the position-buffer rotation as this rank
            start_l, start_r, live = ops.ghost_row_starts()
            from_l, from_r = comm.exchange_ints([start_l, live], [start_r, live], ops.device)
            if from_l[1] != live or from_r[1] != live:
                raise ConfigError("slab ranks disagree on the live position buffer")
            ops.set_halo_targets(base_left=from_l[0], base_right=from_r[0])
        # 4. cells + list for the owned rows; every rank grows together on overflow
        while True:
            overflow, max_count = ops.build_list()
            flags = comm.all_max(ops.scalar_pair(int(overflow), int(max_count)))
            overflow, max_count = int(flags[0].item()), int(flags[1].item())
            self.rebuilds += 1
            if not overflow:
                break
            growths += 1
            if growths > self.STRIDE_GROWTH_LIMIT:
                raise NeighborOverflowError("neighbor list still overflows after "
                                            f"{growths - 1} stride growths")
            ops.grow_stride(max_count)

    def _halo(self):
        ops = self.ops
        to_l, to_r = ops.pack_ghost_positions()
        from_l, from_r = ops.ghost_position_views()
        self.comm.exchange(to_l, to_r, from_l, from_r)

    # -- step loop ------------------------------------------------------------
    def run(self, n_steps: int):
        if getattr(self.ops, "can_advance", False):
            return self._run_advance(n_steps)
        ops, comm = self.ops, self.comm
        for s in range(n_steps):
            last = (s == n_steps - 1) or ((self.step_count + 1) % self.sample_interval == 0)
            ops.integrate(fused=self.pending_kick)
            self.pending_kick = False
            flag = comm.all_max(ops.rebuild_flag())      # async on the device stream
            self._halo()
            ops.force(thermo=last)                        # speculative, like the 1-GPU loop
            if int(flag.item()):
                self._rebuild()
                ops.force(thermo=last)
            self.step_count += 1
            if last:
                ops.finalize()
                if self.step_count % self.sample_interval == 0:
                    self.samples.append(self.measure())
            else:
                self.pending_kick = True

    # One-launch steps (backends with `can_advance`): an intermediate step is ONE kernel
    # -- force(s) + finalize(s) + integrate(s+1) + local displacement check on the owned
    # rows, forces never stored -- followed by the halo exchange of the new positions
    # and an in-place all-reduce(max) of the flag word the kernel wrote.  The kernel is
    # gated on the (already reduced) flag of the positions it reads, so the host enqueues
    # it before it knows that flag: the 64-byte status block is copied on a side stream
    # and inspected while the launch is already queued; when a rebuild is due the launch
    # returns at once on every rank, the ranks rebuild together and enqueue it again.
    # Nothing in the step waits for the host.  Same trajectories, bit for bit, as the
    # separate launches above (tests/test_gpu_slab.py).
    def _advance_once(self):
        ops, comm = self.ops, self.comm
        ops.advance()                      # reads the current buffer, writes the other one
        ops.swap_positions()               # ... which now is the current one
        if not self.fused_halo:            # (fused: the launch stored them on the neighbours)
            self._halo()                   # ghost rows of the new buffer
        comm.all_max(ops.gate_word_out())  # the flag of the new positions, all ranks agree

    def _run_advance(self, n_steps: int):
        ops, comm = self.ops, self.comm
        for s in range(n_steps):
            last = (s == n_steps - 1) or ((self.step_count + 1) % self.sample_interval == 0)
            if not self.ahead:
                ops.integrate(fused=self.pending_kick)
                self.pending_kick = False
                ops.gate_reset_to_integrate()
                comm.all_max(ops.gate_word_in())
                self._halo()
            if last:
                # observable step: forces with energies / virial, stored; then the half-kick
                if ops.read_gate_in():                    # host sync, once per sample
                    self._rebuild()
                    ops.gate_reset_to_integrate()
                ops.force(thermo=True)
                ops.finalize()
                self.ahead = False
                self.step_count += 1
                if self.step_count % self.sample_interval == 0:
                    self.samples.append(self.measure())
                continue
            ticket = ops.snapshot_status()     # flag of the current positions, side stream
            self._advance_once()               # queued before the flag is known
            if ops.snapshot_gate_in(ticket):
                # the launch returned at once (on every rank): undo the swap, rebuild, again
                ops.swap_positions()
                self._rebuild()
                ops.gate_reset_to_integrate()
                self._advance_once()
            ops.gate_toggle()
            self.ahead = True
            self.step_count += 1

    def measure(self):
        sums = self.comm.all_sum(self.ops.thermo_sums())   # 8 doubles
        v = [float(x) for x in sums.tolist()]
        n = int(round(v[7]))
        return {"step": self.step_count, "pe": v[0], "ke": v[1], "momentum": (v[2], v[3], v[4]),
                "virial": v[5], "mass": v[6], "n": n, "total_energy": v[0] + v[1],
                "temperature": 2.0 * v[1] / (3.0 * n), "rebuild_count": self.rebuilds}


# --------------------------------------------------------------- CUDA backend
class CudaSlabOps:
    """libb2md kernels + CUDA tensors behind the SlabSimulation protocol."""

    def __init__(self, pos, vel, ids, edges, device_index=0, capacity_factor=1.25,
                 ghost_fraction=0.25, stride=64, reorder=True, pair_rows=None, advance=None):
        torch = _torch()
        _lib.load()
        self.torch = torch
        self.device = torch.device("cuda", device_index)
        self.edges = tuple(float(e) for e in edges)
        n = int(pos.shape[0])
        self.n_own = n
        self.n_ghost = 0
        self.cap_own = int(n * capacity_factor) + 1024
        self.capacity = self.cap_own + int(n * ghost_fraction) + 4096
        self.capacity = (self.capacity + 31) // 32 * 32
        self.stride = int(stride)
        self.reorder = reorder
        self._pair_rows_arg, self._advance_arg = pair_rows, advance
        f32 = dict(dtype=torch.float32, device=self.device)
        cap = self.capacity
        self.sets = [{k: torch.zeros((cap, 4), **f32) for k in ("pos_hi", "pos_lo", "vel", "force")}
                     for _ in range(2)]
        for s in self.sets:
            s["image"] = torch.zeros((cap, 4), dtype=torch.int32, device=self.device)
            s["vel"][:, 3] = 1.0
        self.cur = 0
        self.virial = torch.zeros(cap, **f32)
        self.status = torch.zeros(16, dtype=torch.int32, device=self.device)
        # one-launch steps: second position buffer (ping-pong), pinned copy of the status
        # block, side stream for its read-back
        self.pos_alt = torch.zeros((cap, 4), **f32)
        self.h_status = torch.zeros(16, dtype=torch.int32).pin_memory()
        self.copy_stream = torch.cuda.Stream(self.device)
        self.copy_done = torch.cuda.Event()
        self.gate_in = 5              # int32 word of the status block: 5 = rebuild_flag
        # the three position buffers rotate (reorder / migration flip the set, a step swaps
        # the live one with pos_alt); every rank goes through the same rotation, so a buffer
        # is named by its index here on all ranks (fused halo, connect_peers)
        self.pos_bufs = [self.sets[0]["pos_hi"], self.sets[1]["pos_hi"], self.pos_alt]
        self.pos_index = {t.data_ptr(): k for k, t in enumerate(self.pos_bufs)}
        self.peer_pos = None          # [left, right] -> the neighbour's three buffers, mapped
        self.halo_dst = None
        self.peer_bytes = 0
        self.box = _lib.make_box(self.edges)
        # upload through the same conversion kernels as the single-GPU path
        a = self.sets[0]
        st_pos = torch.from_numpy(np.ascontiguousarray(pos, dtype=np.float64)).to(self.device)
        st_vel = torch.from_numpy(np.ascontiguousarray(vel, dtype=np.float64)).to(self.device)
        _lib.call("b2md_pack_positions", st_pos.data_ptr(), n, None, a["pos_hi"].data_ptr(),
                  a["pos_lo"].data_ptr(), self.stream)
        _lib.call("b2md_pack_vec3", st_vel.data_ptr(), n, None, a["vel"].data_ptr(), self.stream)
        a["pos_lo"][:n, 3] = torch.from_numpy(np.asarray(ids, dtype=np.int32)).to(self.device) \
            .view(torch.float32)
        self.scratch = {}

    # -- small helpers ---------------------------------------------------------
    @property
    def stream(self):
        return int(self.torch.cuda.current_stream(self.device).cuda_stream)

    @property
    def a(self):
        return self.sets[self.cur]

    def _buf(self, name, shape, dtype):
        t = self.scratch.get(name)
        if t is None or t.shape != tuple(shape) or t.dtype != dtype:
            t = self.torch.zeros(shape, dtype=dtype, device=self.device)
            self.scratch[name] = t
        return t

    def scalar_pair(self, a, b):
        return self.torch.tensor([a, b], dtype=self.torch.int64, device=self.device)

    def record_buffer(self, rows, words):
        return self.torch.empty((rows, words), dtype=self.torch.float32, device=self.device)

    def migrant_buffer(self, rows):
        return self.record_buffer(rows, MIGRANT_WORDS)

    def ghost_buffer(self, rows):
        return self.record_buffer(rows, GHOST_WORDS)

    def attach(self, geo: SlabGeometry, lj, dt, skin):
        torch = self.torch
        self.geo, self.lj, self.dt, self.skin = geo, lj, dt, skin
        self.r_list = lj.max_r_cut + skin
        self.table = np.ascontiguousarray(lj.table(), dtype=np.float64)
        self.table_ptr = self.table.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        self.grid = _lib.Grid()
        _lib.call("b2md_grid_shape", ctypes.byref(self.box), self.r_list, ctypes.byref(self.grid))
        if self.grid.fallback:
            raise ConfigError("the slab driver needs at least three cells per axis")
        i32 = dict(dtype=torch.int32, device=self.device)
        cap, nc = self.capacity, int(self.grid.n_cells)
        lib = _lib.load()
        self.cell_of = torch.zeros(cap, **i32)
        self.cell_start = torch.zeros(nc + 1, **i32)
        self.cell_particles = torch.zeros(cap, **i32)
        self.bin_scratch = torch.zeros(int(lib.b2md_bin_scratch_bytes(cap, nc)),
                                       dtype=torch.uint8, device=self.device)
        self.counts = torch.zeros(cap, **i32)
        self.boundary = torch.zeros(cap, dtype=torch.uint8, device=self.device)
        self.ref_pos = torch.zeros((cap, 4), dtype=torch.float32, device=self.device)
        self.keys = torch.zeros(cap, dtype=torch.int64, device=self.device)
        self.keys_tmp = torch.zeros(cap, dtype=torch.int64, device=self.device)
        self.perm = torch.zeros(cap, **i32)
        self.perm_tmp = torch.zeros(cap, **i32)
        self.sort_scratch = torch.zeros(int(lib.b2md_sort_scratch_bytes(cap)), dtype=torch.uint8,
                                        device=self.device)
        self.flag_l = torch.zeros(cap, **i32)
        self.flag_r = torch.zeros(cap, **i32)
        self.flag_s = torch.zeros(cap, **i32)
        self.idx_l = torch.zeros(cap, **i32)
        self.idx_r = torch.zeros(cap, **i32)
        self.idx_s = torch.zeros(cap, **i32)
        self.cnt3 = torch.zeros(3, **i32)
        self.compact_scratch = torch.zeros(int(lib.b2md_compact_scratch_bytes(cap)),
                                           dtype=torch.uint8, device=self.device)
        self.thermo_scratch = torch.zeros(int(lib.b2md_thermo_scratch_bytes(cap)) // 8 + 8,
                                          dtype=torch.float64, device=self.device)
        self.thermo_out = torch.zeros(8, dtype=torch.float64, device=self.device)
        self._alloc_list()
        self.n_send = (0, 0)
        self.kernel_launches = 0
        _lib.call("b2md_status_reset", self.status.data_ptr(), self.stream)

    def _alloc_list(self):
        rows = (self.stride + 15) // 16 * 16
        self.nbr = self.torch.zeros((rows, self.capacity), dtype=self.torch.int32,
                                    device=self.device)
        # merged rows of owned particle pairs for the two-particles-per-thread force
        # kernel (b2md_pair_rows); large slabs only, like the single-domain loop
        from .forces import use_pair_rows
        self.pair_rows = use_pair_rows(self.cap_own, self._pair_rows_arg)
        self.can_advance = self.pair_rows if self._advance_arg is None else \
            bool(self._advance_arg) and self.pair_rows
        if self.pair_rows:
            self.pair_pitch = ((self.cap_own + 1) // 2 + 31) // 32 * 32
            self.pair_nbr = self.torch.zeros((2 * rows // 4, self.pair_pitch, 4),
                                             dtype=self.torch.int32, device=self.device)
            # pair counts + the block schedule of the pair kernel (b2md_pair_schedule)
            self.pair_counts = self.torch.zeros(
                self.pair_pitch + int(_lib.load().b2md_pair_schedule_len(self.cap_own)),
                dtype=self.torch.int32, device=self.device)

    def grow_stride(self, max_count):
        self.stride = max(self.stride + 1, ((int(max_count * 1.125) + 1) + 7) // 8 * 8)
        self._alloc_list()

    # -- classification + compaction -----------------------------------------
    def _classify(self, lo_cut, hi_cut):
        n = self.n_own
        a = self.a
        _lib.call("b2md_slab_classify", a["pos_hi"].data_ptr(), a["pos_lo"].data_ptr(), n,
                  self.geo.centre, self.edges[0], lo_cut, hi_cut, self.flag_l.data_ptr(),
                  self.flag_r.data_ptr(), self.stream)
        for flags, idx, k in ((self.flag_l, self.idx_l, 0), (self.flag_r, self.idx_r, 1)):
            _lib.call("b2md_compact_indices", flags.data_ptr(), n, idx.data_ptr(),
                      self.cnt3[k:k + 1].data_ptr(), self.compact_scratch.data_ptr(), self.stream)
        self.kernel_launches += 1 + 2 * 4

    def select_migrants(self):
        half = 0.5 * self.geo.width
        if self.geo.world == 1:
            self.n_send = (0, 0)
            return 0, 0
        self._classify(-half, half)
        n = self.n_own
        _lib.call("b2md_flag_neither", self.flag_l.data_ptr(), self.flag_r.data_ptr(), n,
                  self.flag_s.data_ptr(), self.stream)
        _lib.call("b2md_compact_indices", self.flag_s.data_ptr(), n, self.idx_s.data_ptr(),
                  self.cnt3[2:3].data_ptr(), self.compact_scratch.data_ptr(), self.stream)
        c = self.cnt3.cpu().tolist()
        self.n_send = (c[0], c[1])
        self.n_stay = c[2]
        return c[0], c[1]

    def _gather_rows(self, names, idx, count, out):
        """out[:, 4*k:4*k+4] = a[names[k]][idx]  (16-byte row gathers)."""
        a = self.a
        for k, name in enumerate(names):
            tmp = self._buf(f"g_{name}", (max(count, 1), 4), a[name].dtype)
            if count:
                _lib.call("b2md_gather16", a[name].data_ptr(), tmp.data_ptr(), idx.data_ptr(),
                          count, self.stream)
                out[:, 4 * k:4 * k + 4] = tmp[:count].view(self.torch.float32)
                self.kernel_launches += 1

    def pack_migrants(self):
        names = ("pos_hi", "pos_lo", "vel", "image")
        out = []
        for idx, count in ((self.idx_l, self.n_send[0]), (self.idx_r, self.n_send[1])):
            buf = self.record_buffer(count, MIGRANT_WORDS)
            self._gather_rows(names, idx, count, buf)
            out.append(buf)
        return out

    def apply_migration(self, in_l, in_r):
        if self.geo.world == 1:
            return
        torch = self.torch
        names = ("pos_hi", "pos_lo", "vel", "image")
        src, dst = self.a, self.sets[1 - self.cur]
        n_stay = self.n_stay
        # compaction of the rows that stay, then the arrivals behind them
        for name in names + ("force",):
            if n_stay:
                _lib.call("b2md_gather16", src[name].data_ptr(), dst[name].data_ptr(),
                          self.idx_s.data_ptr(), n_stay, self.stream)
                self.kernel_launches += 1
        at = n_stay
        for buf in (in_l, in_r):
            m = buf.shape[0]
            if at + m > self.cap_own:
                raise ConfigError("slab capacity exceeded by migration; raise capacity_factor")
            for k, name in enumerate(names):
                dst[name][at:at + m] = buf[:, 4 * k:4 * k + 4].view(dst[name].dtype)
            dst["force"][at:at + m] = 0.0
            at += m
        self.cur = 1 - self.cur
        self.n_own = at
        self.n_ghost = 0

    def reorder_owned(self):
        if not self.reorder:
            return
        n = self.n_own
        src, dst = self.a, self.sets[1 - self.cur]
        lib = _lib.load()
        sub_bits = 2
        _lib.call("b2md_hilbert_keys", src["pos_hi"].data_ptr(), src["pos_lo"].data_ptr(), n,
                  ctypes.byref(self.grid), sub_bits, self.keys.data_ptr(), self.stream)
        key_bits = lib.b2md_hilbert_key_bits(ctypes.byref(self.grid), sub_bits)
        _lib.call("b2md_iota_i32", self.perm.data_ptr(), n, self.stream)
        _lib.call("b2md_sort_pairs_u64", self.keys.data_ptr(), self.perm.data_ptr(),
                  self.keys_tmp.data_ptr(), self.perm_tmp.data_ptr(), n, key_bits,
                  self.sort_scratch.data_ptr(), self.stream)
        names = ("pos_hi", "pos_lo", "vel", "force", "image")
        srcs = (ctypes.c_void_p * 5)(*[src[name].data_ptr() for name in names])
        dsts = (ctypes.c_void_p * 5)(*[dst[name].data_ptr() for name in names])
        _lib.call("b2md_gather_rows", srcs, dsts, None, None, self.perm.data_ptr(), n, self.stream)
        self.cur = 1 - self.cur
        self.kernel_launches += 2 + 5 * ((key_bits + 7) // 8) + 1

    def select_ghosts(self, r_ghost):
        if self.geo.world == 1:
            self.n_send = (0, 0)
            return 0, 0
        half = 0.5 * self.geo.width
        self._classify(-half + r_ghost, half - r_ghost)
        c = self.cnt3.cpu().tolist()
        self.n_send = (c[0], c[1])
        return c[0], c[1]

    def pack_ghost_records(self):
        out = []
        for idx, count in ((self.idx_l, self.n_send[0]), (self.idx_r, self.n_send[1])):
            buf = self.record_buffer(count, GHOST_WORDS)
            self._gather_rows(("pos_hi", "pos_lo"), idx, count, buf)
            out.append(buf)
        return out

    def set_ghosts(self, in_l, in_r):
        a = self.a
        at = self.n_own
        self.ghost_ranges = []
        for buf in (in_l, in_r):
            m = buf.shape[0]
            if at + m > self.capacity:
                raise ConfigError("ghost capacity exceeded; raise ghost_fraction")
            a["pos_hi"][at:at + m] = buf[:, 0:4]
            a["pos_lo"][at:at + m] = buf[:, 4:8]
            self.ghost_ranges.append((at, at + m))
            at += m
        self.n_ghost = at - self.n_own
        # send buffers for the per-step position halo (sizes fixed until the next rebuild)
        self.send_pos = [self.torch.empty((max(c, 0), 4), dtype=self.torch.float32,
                                          device=self.device) for c in self.n_send]

    def pack_ghost_positions(self):
        a = self.a
        for idx, count, buf in ((self.idx_l, self.n_send[0], self.send_pos[0]),
                                (self.idx_r, self.n_send[1], self.send_pos[1])):
            if count:
                _lib.call("b2md_gather16", a["pos_hi"].data_ptr(), buf.data_ptr(), idx.data_ptr(),
                          count, self.stream)
                self.kernel_launches += 1
        return self.send_pos

    def ghost_position_views(self):
        a = self.a
        (l0, l1), (r0, r1) = self.ghost_ranges
        return a["pos_hi"][l0:l1], a["pos_hi"][r0:r1]

    # -- kernels of the hot path ------------------------------------------------
    def build_list(self):
        a = self.a
        n = self.n_own + self.n_ghost
        _lib.call("b2md_status_reset", self.status.data_ptr(), self.stream)
        _lib.call("b2md_bin", a["pos_hi"].data_ptr(), a["pos_lo"].data_ptr(), n,
                  ctypes.byref(self.grid), self.cell_of.data_ptr(), self.cell_start.data_ptr(),
                  self.cell_particles.data_ptr(), self.bin_scratch.data_ptr(), self.stream)
        _lib.call("b2md_build_nlist", a["pos_hi"].data_ptr(), a["pos_lo"].data_ptr(), n,
                  ctypes.byref(self.box), ctypes.byref(self.grid), self.cell_of.data_ptr(),
                  self.cell_start.data_ptr(), self.cell_particles.data_ptr(), self.r_list,
                  self.stride, self.capacity, self.nbr.data_ptr(), self.counts.data_ptr(),
                  self.boundary.data_ptr(), self.r_list + self.skin, self.n_own,
                  self.status.data_ptr(), self.stream)
        _lib.call("b2md_snapshot", a["pos_hi"].data_ptr(), a["pos_lo"].data_ptr(),
                  a["image"].data_ptr(), self.n_own, ctypes.byref(self.box), None,
                  self.ref_pos.data_ptr(), self.stream)
        self.kernel_launches += 1 + 6 + 2 + 1
        if self.pair_rows:
            _lib.call("b2md_pair_rows", self.nbr.data_ptr(), self.counts.data_ptr(),
                      self.capacity, self.nbr.shape[0], self.n_own, self.pair_nbr.data_ptr(),
                      self.pair_counts.data_ptr(), self.pair_pitch, 2 * self.nbr.shape[0],
                      self.stream)
            _lib.call("b2md_pair_schedule", self.boundary.data_ptr(), self.n_own,
                      self.pair_counts.data_ptr(), self.pair_pitch, self.stream)
            self.kernel_launches += 3
        st = _lib.Status.from_buffer_copy(self.status.cpu().numpy().tobytes())
        return st.overflow != 0, st.max_count

    def integrate(self, fused: bool):
        a = self.a
        half_skin2 = (0.5 * self.skin) ** 2
        name = "b2md_vv_finalize_integrate" if fused else "b2md_vv_integrate"
        _lib.call(name, a["pos_hi"].data_ptr(), a["pos_lo"].data_ptr(), a["vel"].data_ptr(),
                  a["force"].data_ptr(), a["image"].data_ptr(), self.n_own, ctypes.byref(self.box),
                  self.dt, self.ref_pos.data_ptr(), half_skin2, self.status.data_ptr(), self.stream)
        self.kernel_launches += 1

    def rebuild_flag(self):
        # status word 5 = rebuild_flag (include/b2md.h); stays on the device
        return self.status[5:6].to(self.torch.int64)

    def force(self, thermo: bool):
        a = self.a
        if self.pair_rows:
            _lib.call("b2md_force_lj_pairs", a["pos_hi"].data_ptr(), self.n_own,
                      ctypes.byref(self.box), self.pair_nbr.data_ptr(),
                      self.pair_counts.data_ptr(), self.pair_pitch, self.nbr.data_ptr(),
                      self.counts.data_ptr(), self.capacity, self.boundary.data_ptr(),
                      self.table_ptr, self.lj.ntypes,
                      (0 if thermo else _lib.FORCE_SKIP_THERMO) | _lib.FORCE_SCHEDULED,
                      a["force"].data_ptr(), self.virial.data_ptr(), self.status.data_ptr(),
                      self.stream)
            self.kernel_launches += 1
            return
        _lib.call("b2md_force_lj", a["pos_hi"].data_ptr(), self.n_own, ctypes.byref(self.box),
                  self.nbr.data_ptr(), self.counts.data_ptr(), self.capacity, self.nbr.shape[0],
                  self.boundary.data_ptr(), self.table_ptr, self.lj.ntypes,
                  0 if thermo else _lib.FORCE_SKIP_THERMO, a["force"].data_ptr(),
                  self.virial.data_ptr(), self.status.data_ptr(), self.stream)
        self.kernel_launches += 1

    # -- halo fused into the step kernel (peer memory) ---------------------------------
    def connect_peers(self, comm) -> bool:
        """Map the position buffers of both neighbour ranks into this process (CUDA IPC
        handles exchanged over the process group; peer access over NVLink when the ranks
        own different GPUs).  Collective; True when every rank succeeded, otherwise every
        rank keeps the NCCL send/recv halo.  B2MD_SLAB_HALO=nccl turns it off."""
        import os
        torch = self.torch
        geo = comm.geo
        if geo.world == 1:
            return False
        from torch.multiprocessing.reductions import reduce_tensor
        willing = self.can_advance and os.environ.get("B2MD_SLAB_HALO", "peer").lower() != "nccl"
        handles = [None] * geo.world
        comm.dist.all_gather_object(
            handles, [reduce_tensor(t) for t in self.pos_bufs] if willing else None,
            group=comm.group)
        if any(h is None for h in handles):
            self.peer_halo_unavailable = "turned off, or a rank's slab is too small for " \
                                         "one-launch steps"
            return False
        failed, peers, why = 0, [], ""
        try:
            with torch.cuda.device(self.device):
                mapped = {}
                for rank in (geo.left, geo.right):
                    if rank not in mapped:
                        mapped[rank] = [fn(*args) for fn, args in handles[rank]]
                        for t in mapped[rank]:
                            _lib.call("b2md_enable_peer_access", int(t.device.index))
                    peers.append(mapped[rank])
        except Exception as exc:          # noqa: BLE001 -- any failure = use NCCL, on all ranks
            failed, why = 1, f"{type(exc).__name__}: {exc}"
        flag = comm.all_max(torch.tensor([failed], dtype=torch.int64, device=self.device))
        if int(flag.item()):
            self.peer_halo_unavailable = why or "a neighbour rank could not map peer memory"
            return False
        self.peer_pos = peers
        self.halo_dst = [torch.full((self.cap_own,), -1, dtype=torch.int32, device=self.device)
                         for _ in range(2)]
        return True

    def ghost_row_starts(self):
        """(first ghost row from the left, first from the right, index of the live buffer)."""
        (l0, _), (r0, _) = self.ghost_ranges
        return l0, r0, self.pos_index[self.a["pos_hi"].data_ptr()]

    def set_halo_targets(self, base_left: int, base_right: int):
        for side, (idx, count, base, dst) in enumerate(
                ((self.idx_l, self.n_send[0], base_left, self.halo_dst[0]),
                 (self.idx_r, self.n_send[1], base_right, self.halo_dst[1]))):
            if base + count > self.peer_pos[side][0].shape[0]:
                raise ConfigError("ghost capacity of a neighbour rank exceeded")
            _lib.call("b2md_halo_slots", idx.data_ptr(), count, int(base), self.n_own,
                      dst.data_ptr(), self.stream)
            self.kernel_launches += 2 if count else 1

    def probe_peer_halo(self, comm) -> int:
        """Store the send-list rows of the live buffer into the neighbours' ghost rows through
        the peer mapping (b2md_halo_store, the step kernel's stores on their own) and check
        that my own ghost rows -- filled over NCCL just before -- are unchanged once every
        rank has stored.  Returns 1 if any rank saw a difference."""
        torch = self.torch
        a = self.a
        k = self.pos_index[a["pos_hi"].data_ptr()]
        (l0, l1), (r0, r1) = self.ghost_ranges
        want = a["pos_hi"][l0:r1].clone()
        comm.all_max(torch.zeros(1, dtype=torch.int64, device=self.device))   # everyone cloned
        for side in range(2):
            _lib.call("b2md_halo_store", a["pos_hi"].data_ptr(), self.halo_dst[side].data_ptr(),
                      self.n_own, self.peer_pos[side][k].data_ptr(), self.stream)
        torch.cuda.synchronize(self.device)
        comm.all_max(torch.zeros(1, dtype=torch.int64, device=self.device))   # everyone stored
        bad = int(not torch.equal(want, a["pos_hi"][l0:r1]))
        flag = comm.all_max(torch.tensor([bad], dtype=torch.int64, device=self.device))
        return int(flag.item())

    def disconnect_peers(self):
        self.peer_pos = None
        self.halo_dst = None
        self.peer_halo_unavailable = "start-up probe: peer stores did not reproduce the NCCL halo"

    # -- one-launch steps (see SlabSimulation._run_advance) ------------------------
    GATE_WORDS = (5, 12)              # rebuild_flag, reserved[0] (include/b2md.h)

    @property
    def gate_out(self):
        return self.GATE_WORDS[1] if self.gate_in == self.GATE_WORDS[0] else self.GATE_WORDS[0]

    def gate_word_in(self):
        return self.status[self.gate_in:self.gate_in + 1]

    def gate_word_out(self):
        return self.status[self.gate_out:self.gate_out + 1]

    def gate_toggle(self):
        self.gate_in = self.gate_out

    def gate_reset_to_integrate(self):
        """After k_integrate or a rebuild the flag of the current positions is word 5."""
        self.gate_in = self.GATE_WORDS[0]

    def advance(self):
        a = self.a
        half_skin2 = (0.5 * self.skin) ** 2
        halo = (None, None, None, None)
        if self.peer_pos is not None:
            # the neighbours write their new positions into the buffer with the same index
            k = self.pos_index[self.pos_alt.data_ptr()]
            halo = (self.halo_dst[0].data_ptr(), self.peer_pos[0][k].data_ptr(),
                    self.halo_dst[1].data_ptr(), self.peer_pos[1][k].data_ptr())
            self.peer_bytes += 16 * (self.n_send[0] + self.n_send[1])
        _lib.call("b2md_force_lj_pairs_advance_halo", a["pos_hi"].data_ptr(),
                  self.pos_alt.data_ptr(), a["pos_lo"].data_ptr(), a["vel"].data_ptr(),
                  a["image"].data_ptr(), self.n_own, ctypes.byref(self.box), self.dt,
                  self.ref_pos.data_ptr(), half_skin2, self.pair_nbr.data_ptr(),
                  self.pair_counts.data_ptr(), self.pair_pitch, self.nbr.data_ptr(),
                  self.counts.data_ptr(), self.capacity, self.boundary.data_ptr(), self.table_ptr,
                  self.lj.ntypes, _lib.FORCE_SCHEDULED, self.gate_in, self.gate_out, *halo,
                  self.status.data_ptr(), self.stream)
        self.kernel_launches += 1

    def time_step_kernel(self, iters: int):
        """CUDA-event time (ms) of the one-launch step kernel on this rank's owned rows, on
        scratch copies of everything it updates in place (no halo stores, its own status
        block, dt ~ 0 so that repeated launches see the same positions)."""
        torch = self.torch
        a = self.a
        sc = {k: a[k].clone() for k in ("pos_lo", "vel", "image")}
        ref, out = self.ref_pos.clone(), torch.empty_like(a["pos_hi"])
        status = torch.zeros(16, dtype=torch.int32, device=self.device)

        def launch():
            _lib.call("b2md_force_lj_pairs_advance", a["pos_hi"].data_ptr(), out.data_ptr(),
                      sc["pos_lo"].data_ptr(), sc["vel"].data_ptr(), sc["image"].data_ptr(),
                      self.n_own, ctypes.byref(self.box), 1e-9, ref.data_ptr(), 1e30,
                      self.pair_nbr.data_ptr(), self.pair_counts.data_ptr(), self.pair_pitch,
                      self.nbr.data_ptr(), self.counts.data_ptr(), self.capacity,
                      self.boundary.data_ptr(), self.table_ptr, self.lj.ntypes,
                      _lib.FORCE_SCHEDULED, 12, 14, status.data_ptr(), self.stream)
        stream = torch.cuda.current_stream(self.device)
        launch()
        torch.cuda.synchronize(self.device)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(iters):
            launch()
        t1.record(stream)
        torch.cuda.synchronize(self.device)
        return t0.elapsed_time(t1) / iters

    def swap_positions(self):
        """The other position buffer becomes the live one (no copy: every kernel call
        takes the pointer from the set at call time)."""
        a = self.a
        a["pos_hi"], self.pos_alt = self.pos_alt, a["pos_hi"]

    def snapshot_status(self):
        """Start an asynchronous copy of the status block as it is after everything
        enqueued so far; the kernels enqueued next do not wait for it."""
        torch = self.torch
        main = torch.cuda.current_stream(self.device)
        self.copy_stream.wait_stream(main)
        with torch.cuda.stream(self.copy_stream):
            self.h_status.copy_(self.status, non_blocking=True)
            self.copy_done.record(self.copy_stream)
        return self.gate_in

    def snapshot_gate_in(self, word):
        self.copy_done.synchronize()
        return int(self.h_status[word]) != 0

    def read_gate_in(self):
        return int(self.status[self.gate_in].item()) != 0

    def finalize(self):
        a = self.a
        _lib.call("b2md_vv_finalize", a["vel"].data_ptr(), a["force"].data_ptr(), self.n_own,
                  self.dt, self.stream)
        self.kernel_launches += 1

    def thermo_sums(self):
        a = self.a
        _lib.call("b2md_thermo", a["vel"].data_ptr(), a["force"].data_ptr(),
                  self.virial.data_ptr(), self.n_own, self.thermo_scratch.data_ptr(),
                  self.thermo_out.data_ptr(), self.stream)
        self.kernel_launches += 3
        return self.thermo_out.clone()

    # -- inspection (tests) ------------------------------------------------------
    def owned_state(self):
        """(ids, positions fp64, velocities fp64) of the owned rows, host arrays."""
        a = self.a
        n = self.n_own
        ids = a["pos_lo"][:n, 3].contiguous().view(self.torch.int32).cpu().numpy()
        pos = (a["pos_hi"][:n, :3].double() + a["pos_lo"][:n, :3].double()).cpu().numpy()
        vel = a["vel"][:n, :3].double().cpu().numpy()
        return ids, pos, vel


# ------------------------------------------------------------------ benchmark
def slab_initial_state(rank, world, n_per_rank, density, temperature, seed=42):
    """Weak-scaling workload: `world` replicas of the 1-GPU cubic fcc block stacked
    along x (an exact periodic tiling), each rank generating its own block with its
    own velocity stream.  Returns (pos, vel, ids, global edges)."""
    from .integrate import init_lattice_any, init_velocities
    from .core import HOST
    st, box = init_lattice_any(n_per_rank, density)
    init_velocities(st, temperature, seed + rank)
    edge = float(box.edge_lengths[0])
    pos = np.array(st.positions.acquire_read(HOST))
    pos[:, 0] += rank * edge
    vel = np.array(st.velocities.acquire_read(HOST))
    ids = np.arange(n_per_rank, dtype=np.int64) + rank * n_per_rank
    return pos, vel, ids.astype(np.int32), (edge * world, edge, edge)


def run_slab_benchmark(args, rank, world, local_rank, n_per_rank, workload, metric,
                       measured_peak, clock_sampler_cls, scaling="weak", cpu_baseline_fn=None,
                       workload_config_fn=None, min_timed_seconds=1.0, min_repeats=3,
                       max_repeats=400):
    """bench.py's N > 1 arm: `n_per_rank` particles per rank (weak scaling: 1 M per rank;
    strong scaling: a fixed total split over the ranks).  The timed region is run(K) repeated
    back to back (barrier + device synchronise around every repeat, CUDA events, maximum over
    ranks per repeat) until `min_timed_seconds` of GPU time are collected -- as on one GPU.
    Returns the JSON line (a dict) on rank 0, None elsewhere."""
    torch = _torch()
    import torch.distributed as dist
    from .potential import make_shifted
    density, t0, r_cut, skin, dt = 0.75, 1.2, 2.5, 0.3, 0.001
    lj = make_shifted(1.0, 1.0, r_cut)
    pos, vel, ids, edges = slab_initial_state(rank, world, n_per_rank, density, t0)
    geo = SlabGeometry(rank, world, edges)
    ops = CudaSlabOps(pos, vel, ids, edges, device_index=local_rank)
    sim = SlabSimulation(ops, SlabComm(geo), lj, dt, skin, sample_interval=100)
    sim.run(max(args.warmup, 3))
    ops.kernel_launches = 0
    ops.peer_bytes = 0
    sim.comm.bytes_sent = 0
    rebuilds0 = sim.rebuilds
    stream = torch.cuda.current_stream()
    clocks = clock_sampler_cls(local_rank)
    if hasattr(clocks, "sample_now"):
        clocks.sample_now()
    clocks.start()
    rep_ms = []
    while True:
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        start.record(stream)
        sim.run(args.steps)
        stop.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        ms = torch.tensor([start.elapsed_time(stop)], dtype=torch.float64, device=ops.device)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)          # every rank sees the same figure
        rep_ms.append(float(ms.item()))
        if (len(rep_ms) >= min_repeats and sum(rep_ms) >= 1e3 * min_timed_seconds) \
                or len(rep_ms) >= max_repeats:
            break
    if hasattr(clocks, "sample_now"):
        clocks.sample_now()
    clock_info = clocks.stop()
    repeats = len(rep_ms)
    launches = torch.tensor([ops.kernel_launches], dtype=torch.int64, device=ops.device)
    dist.all_reduce(launches, op=dist.ReduceOp.SUM)
    sample = sim.measure()
    # the step kernel alone on this rank's own rows (rank 0 reports it): same accounting as the
    # 1-GPU arm -- (128 + 4 c) bytes per owned particle over its CUDA-event time
    cbar = float(ops.counts[:ops.n_own].float().mean().item())
    kernel_ms = ops.time_step_kernel(30) if ops.can_advance else None
    if rank != 0:
        return None
    ms = sum(rep_ms) / repeats
    n_total = n_per_rank * world
    value = n_total * args.steps / (ms * 1e-3)
    peak, peak_src = measured_peak()
    step_bytes = n_per_rank * (216.0 + 4.0 * cbar)
    adv_bytes = ops.n_own * (128.0 + 4.0 * cbar)
    achieved = adv_bytes / (kernel_ms * 1e-3) / 1e9 if kernel_ms else None
    cfg = workload_config_fn(n_total, n_per_rank) if workload_config_fn else \
        {"workload": workload, "particles": n_total, "particles_per_gpu": n_per_rank}
    cfg.update({
        "decomposition": f"{world} x-slabs of a {edges[0]:.1f} x {edges[1]:.1f} x "
                         f"{edges[2]:.1f} box, ghost width {sim.r_list}",
        "halo_rows_per_face": list(sim.halo_rows),
        "l2": "inputs larger than L2 (neighbour list streamed every step)",
        "timed_region": f"{repeats} back-to-back repeats of run({args.steps}), "
                        f"{sum(rep_ms) / 1e3:.2f} s; per repeat the maximum over ranks",
        "timed_repeats": repeats,
        "ms_per_step_median_repeat": sorted(rep_ms)[repeats // 2] / args.steps,
        "ms_per_step_best_repeat": min(rep_ms) / args.steps,
        "mean_listed_neighbours": cbar,
        "rebuilds_in_timed_region": sim.rebuilds - rebuilds0,
        "step_hbm_fraction_per_gpu": step_bytes * value / n_total / 1e9 / peak,
        "final_energy_per_particle": sample["total_energy"] / n_total})
    line = {
        "metric": metric, "value": value, "unit": metric, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "f32 pair arithmetic, double-single positions, f64 reductions",
        "data": "synthetic",
        "config": cfg,
        "clocks": clock_info, "gpu_launches": int(launches.item()),
        "roofline": {"bound": "hbm",
                     "kernel": "k_force_lj_pair<ADVANCE> on rank 0's owned rows (force + finalize "
                               "+ integrate + halo stores: one launch per MD step), timed alone"
                               if ops.can_advance else "k_force_lj",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if achieved else None, "traffic": None,
                     "peak_source": peak_src, "launch_ms": kernel_ms,
                     "algorithmic_bytes_per_launch": adv_bytes if kernel_ms else None},
        "cpu_baseline": cpu_baseline_fn(n_per_rank) if cpu_baseline_fn else None,
        "e2e": {"value": value, "unit": metric, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 64,
                "note": "multi-GPU arm: state generated per rank on the host and uploaded "
                        "before the timed region; 8 doubles all-reduced and read back per "
                        "sample"},
        "nccl_bytes_sent_rank0_per_step": sim.comm.bytes_sent / max(args.steps * repeats, 1),
        "halo": {"transport": "peer stores from the step kernel (CUDA IPC, NVLink)"
                 if sim.fused_halo else "NCCL send/recv",
                 "peer_bytes_stored_rank0_per_step": ops.peer_bytes / max(args.steps * repeats, 1),
                 "why_not_peer": getattr(ops, "peer_halo_unavailable", None)},
    }
    return line
