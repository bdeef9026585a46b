"""Cell binning, Verlet neighbour lists, the rebuild criterion and spatial
reordering on the B200 -- operator-for-operator counterpart of reference
neighbor.py (same function names, argument meaning and error behaviour).

    bin_particles(state, box, r_list)            neighbor.py:57-91
    build_neighbor_list(state, grid, r_list, stride, r_cut, prev, backend)
                                                 neighbor.py:185-240
    needs_rebuild(state, box, nlist)             neighbor.py:243-254
    reorder_by_cell(state, grid)                 neighbor.py:257-270
    reorder_hilbert(state, box)                  (extension: Hilbert-curve order)

All integer-valued results (cell of particle, CSR arrays, neighbour sets,
permutations, the rebuild decision) are bit-exact with the reference for
positions representable as double-single.  Results live in HBM; the numpy views
the reference exposes (``grid.cell_of_particle``, ``nlist.indices`` ...) are
decoded lazily on access.
"""
from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .backend import BackendSelector
from .core import COMPUTE, DeviceState, ParticleState, SimBox
from .errors import ConfigError


def _torch():
    import torch
    return torch


# ------------------------------------------------------------------- grid
class CellGrid:
    """CSR cell occupancy of one configuration (reference neighbor.py:33-54),
    arrays resident on the device."""

    def __init__(self, cgrid: _lib.Grid, box_edges, dev: DeviceState, d_cell_of, d_cell_start,
                 d_cell_particles):
        self._c = cgrid
        self.cells_per_axis = np.array(list(cgrid.ncell), dtype=np.int64)
        self.cell_edge = np.array(list(cgrid.cell_edge), dtype=np.float64)
        self.box_edges = np.array(box_edges, dtype=np.float64)
        self.fallback = bool(cgrid.fallback)
        self._dev = dev
        self.d_cell_of = d_cell_of
        self.d_cell_start = d_cell_start
        self.d_cell_particles = d_cell_particles

    @property
    def n_cells(self) -> int:
        return int(self._c.n_cells)

    def c_grid(self):
        return ctypes.byref(self._c)

    @property
    def cell_of_particle(self) -> np.ndarray:
        return self.d_cell_of.cpu().numpy().astype(np.int64)

    @property
    def cell_start(self) -> np.ndarray:
        return self.d_cell_start.cpu().numpy().astype(np.int64)

    @property
    def cell_particles(self) -> np.ndarray:
        return self.d_cell_particles.cpu().numpy().astype(np.int64)

    def occupancy_counts(self):
        return np.diff(self.cell_start)

    def occupants(self, flat_cell: int):
        start = self.cell_start
        return self.cell_particles[start[flat_cell]:start[flat_cell + 1]]


def grid_shape(box: SimBox, r_list: float) -> _lib.Grid:
    """Cells per axis / cell edge in host fp64 (neighbor.py:64-71,90)."""
    if not (r_list > 0.0 and np.isfinite(r_list)):
        raise ValueError("r_list must be positive and finite")
    edges = box.edge_lengths
    if np.any(edges < r_list):
        raise ConfigError(
            f"every box edge must be >= r_list ({r_list:g}); box is {edges}")
    g = _lib.Grid()
    _lib.call("b2md_grid_shape", box.c_box(), float(r_list), ctypes.byref(g))
    return g


def bin_particles(state: ParticleState, box: SimBox, r_list: float) -> CellGrid:
    """Bin particles into cells at least r_list wide (neighbor.py:57-91)."""
    g = grid_shape(box, r_list)
    torch = _torch()
    state.positions.acquire_read(COMPUTE)
    dev = state.device_state()
    n = dev.n
    i32 = dict(dtype=torch.int32, device=dev.device)
    d_cell_of = torch.empty(n, **i32)
    d_cell_start = torch.empty(int(g.n_cells) + 1, **i32)
    d_cell_particles = torch.empty(n, **i32)
    scratch = torch.empty(int(_lib.load().b2md_bin_scratch_bytes(n, g.n_cells)),
                          dtype=torch.uint8, device=dev.device)
    _lib.call("b2md_bin", dev.pos_hi.data_ptr(), dev.pos_lo.data_ptr(), n, ctypes.byref(g),
              d_cell_of.data_ptr(), d_cell_start.data_ptr(), d_cell_particles.data_ptr(),
              scratch.data_ptr(), dev.stream)
    return CellGrid(g, box.edge_lengths, dev, d_cell_of, d_cell_start, d_cell_particles)


# ------------------------------------------------------------------- list
def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


class NeighborList:
    """Fixed-stride full neighbour list plus its rebuild bookkeeping
    (reference neighbor.py:94-109).  Device layout: column-major, padded --
    entry k of particle i at ``d_nbr[k, i]`` with row pitch ``pitch``."""

    def __init__(self, dev, d_nbr, d_counts, d_boundary, d_at_build, d_ref_pos, stride, pitch,
                 overflow, max_count, r_list, r_cut, rebuild_count):
        self._dev = dev
        self.d_nbr, self.d_counts, self.d_boundary = d_nbr, d_counts, d_boundary
        self.d_at_build, self.d_ref_pos = d_at_build, d_ref_pos
        self.stride = int(stride)
        self.pitch = int(pitch)
        self.overflow = bool(overflow)
        self.max_count = int(max_count)
        self.r_list = float(r_list)
        self.r_cut = float(r_cut)
        self.rebuild_count = int(rebuild_count)
        self._pair = None          # (d_pair_nbr, d_pair_counts, pair_pitch), built on demand
        self._consumed = False     # buffers recycled by a later build (internal rebuilds only)

    def _live(self):
        if self._consumed:
            raise RuntimeError("this NeighborList's buffers were recycled by a later rebuild")

    def pair_rows(self):
        """Merged rows of particles (2t, 2t+1) for the two-particles-per-thread force
        kernel (``b2md_pair_rows``): returns ``(d_pair_nbr, d_pair_counts, pair_pitch)``
        with ``d_pair_nbr`` of shape (tiles, pair_pitch, 4) int32, entry
        ``j << 2 | listed_for_2t | listed_for_2t+1 << 1``.  Derived from this list
        on first use and cached (the list is immutable once built)."""
        self._live()
        if self._pair is None:
            torch = _torch()
            dev = self._dev
            n = dev.n
            rows = int(self.d_nbr.shape[0])
            pair_pitch = _round_up((n + 1) // 2, 32)
            buf = self._pair_buf
            if buf is None or buf[0].shape != (2 * rows // 4, pair_pitch, 4):
                buf = (torch.zeros((2 * rows // 4, pair_pitch, 4), dtype=torch.int32,
                                   device=dev.device),
                       torch.zeros(pair_pitch, dtype=torch.int32, device=dev.device))
            _lib.call("b2md_pair_rows", self.d_nbr.data_ptr(), self.d_counts.data_ptr(),
                      self.pitch, rows, n, buf[0].data_ptr(), buf[1].data_ptr(), pair_pitch,
                      2 * rows, dev.stream)
            self._pair = (buf[0], buf[1], pair_pitch)
        return self._pair

    _pair_buf = None               # buffers handed over by the list this one replaced

    @property
    def skin(self) -> float:
        return self.r_list - self.r_cut

    @property
    def counts(self) -> np.ndarray:
        """(n,) int32 valid entries per row, logical particle order."""
        self._live()
        return self.d_counts[:self._dev.n].cpu().numpy()

    @property
    def indices(self) -> np.ndarray:
        """(n, stride) int32 row-major copy in the reference's layout (physical
        row indices; identical to logical ids unless rows were reordered)."""
        self._live()
        n = self._dev.n
        return np.ascontiguousarray(self.d_nbr[:self.stride, :n].t().cpu().numpy())

    @property
    def positions_at_build(self) -> np.ndarray:
        self._live()
        return self.d_at_build.cpu().numpy()

    def pair_set(self):
        """Unordered logical-id pairs listed (test helper)."""
        ids = self._dev.particle_ids().astype(np.int64)
        idx, cnt = self.indices, self.counts
        out = set()
        for r in range(cnt.size):
            a = int(ids[r])
            for j in idx[r, :cnt[r]]:
                b = int(ids[int(j)])
                out.add((a, b) if a < b else (b, a))
        return out


def build_neighbor_list(state: ParticleState, grid: CellGrid, r_list: float, stride: int,
                        r_cut: float | None = None, prev: NeighborList | None = None,
                        backend: BackendSelector | None = None,
                        _recycle: bool = False) -> NeighborList:
    """Build a full neighbour list from a cell grid (neighbor.py:185-240).

    Rows that would exceed ``stride`` raise the overflow flag instead of being
    truncated silently; the caller grows the stride and rebuilds.  Grids with
    fewer than three cells on an axis use the all-pairs scan (``grid.fallback``).
    Reading ``overflow`` synchronises with the device once per build.

    ``prev`` only supplies the lineage counter (neighbor.py:239): every list owns its
    buffers, as in the reference.  ``_recycle=True`` (internal: ``Simulation._rebuild``,
    which drops the old list) builds into ``prev``'s device buffers instead and marks
    ``prev`` consumed -- its accessors then raise.
    """
    if int(stride) < 1:
        raise ConfigError("stride must be >= 1")
    stride = int(stride)
    if r_cut is None:
        r_cut = r_list
    if not (0.0 < r_cut <= r_list):
        raise ValueError("need 0 < r_cut <= r_list")
    torch = _torch()
    state.positions.acquire_read(COMPUTE)
    state.images.acquire_read(COMPUTE)
    dev = state.device_state()
    n = dev.n
    pitch = _round_up(n, 32)
    # small systems: 64-row granules, so that the row kernels may put 16 lanes on a particle
    rows = _round_up(stride, 64 if n < 200_000 else 16)
    reuse = (_recycle and prev is not None and not prev._consumed and
             prev.d_nbr.shape == (rows, pitch) and prev._dev is dev)
    if reuse:
        d_nbr, d_counts, d_boundary = prev.d_nbr, prev.d_counts, prev.d_boundary
        d_at_build, d_ref_pos = prev.d_at_build, prev.d_ref_pos
    else:
        # zero-filled so that padding entries are always valid row indices
        d_nbr = torch.zeros((rows, pitch), dtype=torch.int32, device=dev.device)
        d_counts = torch.zeros(pitch, dtype=torch.int32, device=dev.device)
        d_boundary = torch.zeros(pitch, dtype=torch.uint8, device=dev.device)
        d_at_build = torch.empty((n, 3), dtype=torch.float64, device=dev.device)
        d_ref_pos = torch.empty((pitch, 4), dtype=torch.float32, device=dev.device)
    box = SimBox(grid.box_edges)
    skin = float(r_list) - float(r_cut)
    dev.reset_status()
    _lib.call("b2md_build_nlist", dev.pos_hi.data_ptr(), dev.pos_lo.data_ptr(), n, box.c_box(),
              grid.c_grid(), grid.d_cell_of.data_ptr(), grid.d_cell_start.data_ptr(),
              grid.d_cell_particles.data_ptr(), float(r_list), stride, pitch,
              d_nbr.data_ptr(), d_counts.data_ptr(), d_boundary.data_ptr(),
              float(r_list) + skin, n, dev.status.data_ptr(), dev.stream)
    _lib.call("b2md_snapshot", dev.pos_hi.data_ptr(), dev.pos_lo.data_ptr(),
              dev.image.data_ptr(), n, box.c_box(), d_at_build.data_ptr(), d_ref_pos.data_ptr(),
              dev.stream)
    st = dev.read_status()
    out = NeighborList(dev, d_nbr, d_counts, d_boundary, d_at_build, d_ref_pos, stride, pitch,
                       overflow=st.overflow != 0, max_count=st.max_count, r_list=r_list,
                       r_cut=r_cut,
                       rebuild_count=(prev.rebuild_count if prev is not None else 0) + 1)
    if reuse:
        if prev._pair is not None:
            out._pair_buf = prev._pair[:2]     # same shapes: merge into the old buffers
            prev._pair = None
        prev._consumed = True                  # its buffers now hold the new list
    return out


def max_displacement_sq(state: ParticleState, box: SimBox, nlist: NeighborList) -> float:
    """max_i |unwrapped_i - at_build_i|^2 in exact fp64 (neighbor.py:251-253)."""
    state.positions.acquire_read(COMPUTE)
    state.images.acquire_read(COMPUTE)
    dev = state.device_state()
    dev.reset_status()
    _lib.call("b2md_max_displacement", dev.pos_hi.data_ptr(), dev.pos_lo.data_ptr(),
              dev.image.data_ptr(), dev.n, box.c_box(), nlist.d_at_build.data_ptr(),
              dev.status.data_ptr(), dev.stream)
    bits = dev.read_status().max_disp2_f64_bits
    return struct.unpack("<d", struct.pack("<Q", bits))[0]


def needs_rebuild(state: ParticleState, box: SimBox, nlist: NeighborList) -> bool:
    """True once any particle moved more than skin/2 since the list was built
    (strictly greater; unwrapped coordinates; neighbor.py:243-254)."""
    half_skin = 0.5 * nlist.skin
    return max_displacement_sq(state, box, nlist) > half_skin * half_skin


# ---------------------------------------------------------------- reorder
def _sort_permutation(dev: DeviceState, d_keys, key_bits: int):
    """Stable radix sort of 64-bit keys; returns the device permutation
    (new row k = old row perm[k])."""
    torch = _torch()
    n = dev.n
    d_perm = torch.empty(n, dtype=torch.int32, device=dev.device)
    _lib.call("b2md_iota_i32", d_perm.data_ptr(), n, dev.stream)
    keys_tmp = torch.empty_like(d_keys)
    perm_tmp = torch.empty_like(d_perm)
    scratch = torch.empty(int(_lib.load().b2md_sort_scratch_bytes(n)), dtype=torch.uint8,
                          device=dev.device)
    _lib.call("b2md_sort_pairs_u64", d_keys.data_ptr(), d_perm.data_ptr(), keys_tmp.data_ptr(),
              perm_tmp.data_ptr(), n, int(key_bits), scratch.data_ptr(), dev.stream)
    return d_perm


def apply_permutation(dev: DeviceState, d_perm):
    """Gather every packed array through ``d_perm`` (values moved bit-for-bit)."""
    torch = _torch()
    n = dev.n
    for name in DeviceState.ROW16:
        src = getattr(dev, name)
        dst = torch.empty_like(src)
        _lib.call("b2md_gather16", src.data_ptr(), dst.data_ptr(), d_perm.data_ptr(), n,
                  dev.stream)
        if dev.capacity > n:
            dst[n:] = src[n:]
        setattr(dev, name, dst)
    dst = torch.empty_like(dev.virial)
    _lib.call("b2md_gather4", dev.virial.data_ptr(), dst.data_ptr(), d_perm.data_ptr(), n,
              dev.stream)
    if dev.capacity > n:
        dst[n:] = dev.virial[n:]
    dev.virial = dst


def _bits_for(value: int) -> int:
    return max(1, int(value).bit_length())


def reorder_by_cell(state: ParticleState, grid: CellGrid) -> np.ndarray:
    """Permute all per-particle arrays into cell order, stable by old index
    (neighbor.py:257-270).  Returns the permutation applied: new row k holds old
    row perm[k].  The logical particle order changes, exactly as in the
    reference; the grid is stale afterwards."""
    torch = _torch()
    dev = state.sync_to_compute()
    if not dev.identity_order:
        raise ConfigError("reorder_by_cell needs rows in logical order; "
                          "the engine already reordered this state internally")
    d_keys = torch.empty(dev.n, dtype=torch.int64, device=dev.device)
    _lib.call("b2md_cell_keys", grid.d_cell_of.data_ptr(), dev.n, d_keys.data_ptr(), dev.stream)
    d_perm = _sort_permutation(dev, d_keys, _bits_for(grid.n_cells - 1))
    apply_permutation(dev, d_perm)
    _lib.call("b2md_set_ids", dev.pos_lo.data_ptr(), dev.capacity, dev.stream)
    for buf in state.buffers().values():
        buf.acquire_write(COMPUTE)
    return d_perm.cpu().numpy().astype(np.int64)


HILBERT_SUB_BITS = 2


def hilbert_keys(state: ParticleState, box: SimBox, r_list: float,
                 sub_bits: int = HILBERT_SUB_BITS):
    """Device tensor of cell-aligned Hilbert keys of the current positions: the
    Hilbert index of (cell << sub_bits | sub-cell coordinate) per axis, cells as
    in :func:`bin_particles` for ``r_list``.  Sorting by it makes every cell's
    particles contiguous, cells following the curve."""
    torch = _torch()
    g = grid_shape(box, r_list)
    state.positions.acquire_read(COMPUTE)
    dev = state.device_state()
    d_keys = torch.empty(dev.n, dtype=torch.int64, device=dev.device)
    _lib.call("b2md_hilbert_keys", dev.pos_hi.data_ptr(), dev.pos_lo.data_ptr(), dev.n,
              ctypes.byref(g), int(sub_bits), d_keys.data_ptr(), dev.stream)
    key_bits = _lib.load().b2md_hilbert_key_bits(ctypes.byref(g), int(sub_bits))
    return d_keys, key_bits


def reorder_hilbert(state: ParticleState, box: SimBox, r_list: float,
                    sub_bits: int = HILBERT_SUB_BITS, internal: bool = True) -> np.ndarray:
    """Sort device rows along a 3-D Hilbert curve (64-bit keys, stable radix
    sort).  With ``internal=True`` (what ``Simulation`` uses) only the physical
    row order changes: ids travel with the rows and the HOST side keeps its
    logical order.  With ``internal=False`` the logical order changes like
    :func:`reorder_by_cell`.  Returns perm (new row k = old row perm[k])."""
    dev = state.sync_to_compute()
    d_keys, key_bits = hilbert_keys(state, box, r_list, sub_bits)
    d_perm = _sort_permutation(dev, d_keys, key_bits)
    apply_permutation(dev, d_perm)
    if internal:
        dev.identity_order = False
    else:
        if not dev.identity_order:
            raise ConfigError("logical reorder needs rows in logical order")
        _lib.call("b2md_set_ids", dev.pos_lo.data_ptr(), dev.capacity, dev.stream)
        for buf in state.buffers().values():
            buf.acquire_write(COMPUTE)
    return d_perm.cpu().numpy().astype(np.int64)
