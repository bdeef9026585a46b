"""Pair-force evaluation on the B200: counterparts of reference forces.py.

    compute_forces_truncated(state, params, box, nlist, backend)   forces.py:141-159
    compute_forces_all_to_all(state, params, box, backend)         forces.py:129-138

Both overwrite ``state.forces`` and ``state.per_particle_potential`` (half of
every pair energy per partner) and, as an extension, ``state.virial``
(half of every pair's r.f).  ``params`` is an :class:`LJParams` or a
:class:`PairTable` (per-species-pair parameters, species taken from
``state.species``).  Pair arithmetic is fp32 (stated tolerance: 1e-5 relative on
per-particle forces/energies against the fp64 reference); a coincident pair
raises :class:`SingularPairError` naming the lowest i and its first partner j
(forces.py:113-116); an overflowed list is refused (forces.py:149-151).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .backend import BackendSelector
from .core import COMPUTE, HOST, ParticleState, SimBox
from .errors import NeighborOverflowError, SingularPairError
from .neighbor import NeighborList

_NO_SINGULAR = 0xFFFFFFFFFFFFFFFF


def _table_ptr(params, state: ParticleState):
    tab = np.ascontiguousarray(params.table(), dtype=np.float64)
    nt = int(params.ntypes)
    if nt > 1:
        sp = state.species.acquire_read(HOST)
        if sp.min() < 0 or sp.max() >= nt:
            raise ValueError(f"species must lie in [0, {nt - 1}] for this pair table")
    return tab, tab.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), nt


def raise_if_singular(state: ParticleState, status: _lib.Status):
    """Map the device status word to SingularPairError(i, j) in logical ids."""
    if status.singular != _NO_SINGULAR:
        i, j = status.singular >> 32, status.singular & 0xFFFFFFFF
        dev = state.device_state()
        if not dev.identity_order:
            # rows were permuted internally: report logical ids, lowest first
            ids = dev.particle_ids()
            i, j = sorted((int(ids[i]), int(ids[j])))
        raise SingularPairError(i, j)


#: systems at least this large use the two-particles-per-thread kernel over pair
#: rows; smaller ones are latency-bound and want more threads (sub-warp per particle)
PAIR_ROWS_MIN_PARTICLES = 200_000


def use_pair_rows(n: int, pair_rows: bool | None = None) -> bool:
    """Kernel choice: explicit argument, else B2MD_PAIR_ROWS=0/1, else by size."""
    if pair_rows is not None:
        return bool(pair_rows)
    env = os.environ.get("B2MD_PAIR_ROWS")
    if env in ("0", "1"):
        return env == "1"
    return n >= PAIR_ROWS_MIN_PARTICLES


def compute_forces_truncated(state: ParticleState, params, box: SimBox, nlist: NeighborList,
                             backend: BackendSelector | None = None, check: bool = True,
                             pair_rows: bool | None = None):
    """Fill forces / per-particle potential / virial scanning listed neighbours.

    ``check=False`` skips the synchronising status read (the step loop polls the
    status block itself at sample time).  ``pair_rows`` selects the kernel (None =
    by system size): one thread per particle over the list itself, or one thread
    per particle pair over the merged rows; per-particle results are bit-identical."""
    if nlist.overflow:
        raise NeighborOverflowError(
            "neighbor list overflowed its stride; rebuild with a larger one")
    tab, tab_ptr, nt = _table_ptr(params, state)
    state.positions.acquire_read(COMPUTE)
    if nt > 1:
        state.species.acquire_read(COMPUTE)
    dev = state.device_state()
    if check:
        dev.reset_status()
    if use_pair_rows(dev.n, pair_rows):
        d_pair_nbr, d_pair_counts, pair_pitch = nlist.pair_rows()
        _lib.call("b2md_force_lj_pairs", dev.pos_hi.data_ptr(), dev.n, box.c_box(),
                  d_pair_nbr.data_ptr(), d_pair_counts.data_ptr(), pair_pitch,
                  nlist.d_nbr.data_ptr(), nlist.d_counts.data_ptr(), nlist.pitch,
                  nlist.d_boundary.data_ptr(), tab_ptr, nt, 0, dev.force.data_ptr(),
                  dev.virial.data_ptr(), dev.status.data_ptr(), dev.stream)
    else:
        _lib.call("b2md_force_lj", dev.pos_hi.data_ptr(), dev.n, box.c_box(),
                  nlist.d_nbr.data_ptr(), nlist.d_counts.data_ptr(), nlist.pitch,
                  nlist.d_nbr.shape[0], nlist.d_boundary.data_ptr(), tab_ptr, nt, 0,
                  dev.force.data_ptr(), dev.virial.data_ptr(), dev.status.data_ptr(), dev.stream)
    state.mark_compute_written("forces", "per_particle_potential", "virial")
    if check:
        raise_if_singular(state, dev.read_status())


def compute_forces_all_to_all(state: ParticleState, params, box: SimBox,
                              backend: BackendSelector | None = None):
    """Fill forces / per-particle potential / virial scanning every pair."""
    tab, tab_ptr, nt = _table_ptr(params, state)
    state.positions.acquire_read(COMPUTE)
    if nt > 1:
        state.species.acquire_read(COMPUTE)
    dev = state.device_state()
    dev.reset_status()
    _lib.call("b2md_force_lj_all_pairs", dev.pos_hi.data_ptr(), dev.n, box.c_box(), tab_ptr, nt,
              dev.force.data_ptr(), dev.virial.data_ptr(), dev.status.data_ptr(), dev.stream)
    state.mark_compute_written("forces", "per_particle_potential", "virial")
    raise_if_singular(state, dev.read_status())
