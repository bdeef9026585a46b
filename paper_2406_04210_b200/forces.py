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


def compute_forces_truncated(state: ParticleState, params, box: SimBox, nlist: NeighborList,
                             backend: BackendSelector | None = None, check: bool = True):
    """Fill forces / per-particle potential / virial scanning listed neighbours.

    ``check=False`` skips the synchronising status read (the step loop polls the
    status block itself at sample time)."""
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
