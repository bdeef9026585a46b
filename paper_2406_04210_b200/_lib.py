"""ctypes binding of libb2md.so (declarations mirror include/b2md.h).

There is no CPU fallback: if the library is missing or a call fails, the
operator raises.  PyTorch is used only to own device memory and to provide the
CUDA stream the kernels are enqueued on.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char_p, c_double, c_float, c_int32, c_int64,
                    c_uint8, c_uint32, c_uint64, c_void_p)

from .build import LIB_PATH


class B2mdError(RuntimeError):
    """A libb2md call returned a non-zero code."""


class Status(Structure):
    _fields_ = [
        ("overflow", c_int32),
        ("max_count", c_int32),
        ("singular", c_uint64),
        ("max_disp2_bits", c_uint32),
        ("rebuild_flag", c_int32),
        ("max_disp2_f64_bits", c_uint64),
        ("n_boundary", c_int32),
        ("graph_steps", c_int32),
        ("graph_rebuilds", c_int32),
        ("frozen", c_int32),
        ("reserved", c_int32 * 4),
    ]


class Box(Structure):
    _fields_ = [("edge", c_double * 3)]


class Grid(Structure):
    _fields_ = [
        ("ncell", c_int32 * 3),
        ("fallback", c_int32),
        ("cell_edge", c_double * 3),
        ("n_cells", c_int64),
    ]


assert ctypes.sizeof(Status) == 64


class RunnerConfig(Structure):
    _fields_ = [
        ("n", c_int64), ("capacity", c_int64), ("box", Box),
        ("dt", c_double), ("r_cut", c_double), ("skin", c_double),
        ("ntypes", c_int32), ("reorder_mode", c_int32), ("reorder_every", c_int32),
        ("hilbert_bits", c_int32),
        ("table", POINTER(c_double)),
        ("pos_hi", c_void_p * 2), ("pos_lo", c_void_p * 2), ("vel", c_void_p * 2),
        ("force", c_void_p * 2), ("image", c_void_p * 2), ("virial", c_void_p * 2),
        ("current", c_int32), ("stride", c_int32),
        ("nbr", c_void_p), ("pitch", c_int64), ("counts", c_void_p), ("boundary", c_void_p),
        ("ref_pos", c_void_p), ("at_build", c_void_p),
        ("cell_of", c_void_p), ("cell_start", c_void_p), ("cell_particles", c_void_p),
        ("bin_scratch", c_void_p),
        ("keys", c_void_p), ("keys_tmp", c_void_p), ("perm", c_void_p), ("perm_tmp", c_void_p),
        ("sort_scratch", c_void_p),
        ("status", c_void_p), ("stream", c_void_p),
        ("use_graph", c_int32), ("pair_rows", c_int32),
        ("pair_nbr", c_void_p), ("pair_counts", c_void_p), ("pair_pitch", c_int64),
        ("pos_hi_alt", c_void_p), ("queue_depth", c_int32), ("pair_schedule", c_int32),
        ("persistent_steps", c_int32), ("list_row_multiple", c_int32), ("barrier", c_void_p),
        ("h_status", c_void_p), ("run_stream", c_void_p), ("copy_stream", c_void_p),
        ("pair_nbr_inner", c_void_p), ("pair_counts_inner", c_void_p), ("prune_delta", c_double),
        ("vel_ready_event", c_void_p),
    ]


class RunReport(Structure):
    _fields_ = [
        ("steps_done", c_int64), ("reason", c_int32), ("rebuilds", c_int32),
        ("reorders", c_int32), ("current", c_int32), ("max_count", c_int32),
        ("wasted_force_launches", c_int32), ("kernel_launches", c_int64),
        ("list_valid", c_int32), ("n_boundary", c_int32), ("max_disp2", c_double),
        ("singular", c_uint64), ("graph_steps", c_int64),
        ("gpu_ms", c_double), ("rebuild_gpu_ms", c_double),
    ]


RUN_DONE, RUN_OVERFLOW, RUN_SINGULAR = 0, 1, 2
FORCE_SKIP_THERMO = 1
FORCE_SCHEDULED = 4

_P = c_void_p
_SIGNATURES = {
    # name: (restype, argtypes)
    "b2md_version": (c_int32, []),
    "b2md_last_error_string": (c_char_p, []),
    "b2md_status_reset": (c_int32, [_P, _P]),
    "b2md_status_reset_list": (c_int32, [_P, _P]),
    "b2md_pack_positions": (c_int32, [_P, c_int64, _P, _P, _P, _P]),
    "b2md_unpack_positions": (c_int32, [_P, _P, c_int64, _P, _P, _P]),
    "b2md_pack_vec3": (c_int32, [_P, c_int64, _P, _P, _P]),
    "b2md_unpack_vec3": (c_int32, [_P, c_int64, _P, _P, _P]),
    "b2md_pack_w_f64": (c_int32, [_P, c_int64, _P, _P, _P]),
    "b2md_unpack_w_f64": (c_int32, [_P, c_int64, _P, _P, _P]),
    "b2md_pack_w_i32": (c_int32, [_P, c_int64, _P, _P, _P]),
    "b2md_unpack_w_i32": (c_int32, [_P, c_int64, _P, _P, _P]),
    "b2md_pack_images": (c_int32, [_P, c_int64, _P, _P, _P]),
    "b2md_unpack_images": (c_int32, [_P, c_int64, _P, _P, _P]),
    "b2md_pack_scalar_f32": (c_int32, [_P, c_int64, _P, _P, _P]),
    "b2md_unpack_scalar_f32": (c_int32, [_P, c_int64, _P, _P, _P]),
    "b2md_set_ids": (c_int32, [_P, c_int64, _P]),
    "b2md_get_ids": (c_int32, [_P, c_int64, _P, _P]),
    "b2md_grid_shape": (c_int32, [POINTER(Box), c_double, POINTER(Grid)]),
    "b2md_bin_scratch_bytes": (c_int64, [c_int64, c_int64]),
    "b2md_bin": (c_int32, [_P, _P, c_int64, POINTER(Grid), _P, _P, _P, _P, _P]),
    "b2md_build_nlist": (c_int32, [_P, _P, c_int64, POINTER(Box), POINTER(Grid), _P, _P, _P,
                                   c_double, c_int32, c_int64, _P, _P, _P, c_double, c_int64,
                                   _P, _P]),
    "b2md_build_nlist_ex": (c_int32, [_P, _P, c_int64, POINTER(Box), POINTER(Grid), _P, _P, _P,
                                      c_double, c_int32, c_int64, _P, _P, _P, c_double, c_int64,
                                      c_int32, _P, _P]),
    "b2md_build_pair_list": (c_int32, [_P, _P, c_int64, POINTER(Box), POINTER(Grid), _P, _P, _P,
                                       c_double, c_int32, c_int64, _P, _P, _P, c_double, c_int64,
                                       c_int32, c_int32, _P, _P, c_int64, c_int32, _P, _P]),
    "b2md_slab_classify": (c_int32, [_P, _P, c_int64, c_double, c_double, c_double, c_double,
                                     _P, _P, _P]),
    "b2md_compact_scratch_bytes": (c_int64, [c_int64]),
    "b2md_compact_indices": (c_int32, [_P, c_int64, _P, _P, _P, _P]),
    "b2md_gather_rows": (c_int32, [_P, _P, _P, _P, _P, c_int64, _P]),
    "b2md_halo_slots": (c_int32, [_P, c_int64, c_int32, c_int64, _P, _P]),
    "b2md_halo_store": (c_int32, [_P, _P, c_int64, _P, _P]),
    "b2md_enable_peer_access": (c_int32, [c_int32]),
    "b2md_flag_neither": (c_int32, [_P, _P, c_int64, _P, _P]),
    "b2md_snapshot": (c_int32, [_P, _P, _P, c_int64, POINTER(Box), _P, _P, _P]),
    "b2md_max_displacement": (c_int32, [_P, _P, _P, c_int64, POINTER(Box), _P, _P, _P]),
    "b2md_force_lj": (c_int32, [_P, c_int64, POINTER(Box), _P, _P, c_int64, c_int32, _P,
                                POINTER(c_double), c_int32, c_int32, _P, _P, _P, _P]),
    "b2md_pair_rows": (c_int32, [_P, _P, c_int64, c_int32, c_int64, _P, _P, c_int64, c_int32, _P]),
    "b2md_steps_persistent_lanes": (c_int32, [c_int64, c_int32, c_int32]),
    "b2md_steps_persistent": (c_int32, [_P, _P, _P, _P, _P, c_int64, POINTER(Box), c_double, _P,
                                        c_double, _P, _P, c_int64, c_int32, _P, POINTER(c_double),
                                        c_int32, c_int32, c_int32, c_int32, _P, _P, _P]),
    "b2md_pair_schedule_len": (c_int64, [c_int64]),
    "b2md_pair_schedule": (c_int32, [_P, c_int64, _P, c_int64, _P]),
    "b2md_pair_order": (c_int32, [_P, c_int64, _P, _P, c_int64, c_int32, c_int32, c_int32, _P]),
    "b2md_force_lj_pairs": (c_int32, [_P, c_int64, POINTER(Box), _P, _P, c_int64, _P, _P, c_int64,
                                      _P, POINTER(c_double), c_int32, c_int32, _P, _P, _P, _P]),
    "b2md_force_lj_advance": (c_int32, [_P, _P, _P, _P, _P, c_int64, POINTER(Box), c_double, _P,
                                        c_double, _P, _P, c_int64, c_int32, _P, POINTER(c_double),
                                        c_int32, c_int32, c_int32, c_int32, _P, _P]),
    "b2md_force_lj_pairs_advance": (c_int32, [_P, _P, _P, _P, _P, c_int64, POINTER(Box), c_double,
                                              _P, c_double, _P, _P, c_int64, _P, _P, c_int64, _P,
                                              POINTER(c_double), c_int32, c_int32, c_int32,
                                              c_int32, _P, _P]),
    "b2md_force_lj_pairs_advance_pruned": (c_int32, [_P, _P, _P, _P, _P, c_int64, POINTER(Box),
                                                     c_double, _P, c_double, _P, _P, c_int64, _P,
                                                     _P, c_int64, _P, POINTER(c_double), c_int32,
                                                     c_int32, c_int32, c_int32, c_int32, c_int32,
                                                     _P, _P, c_int32, c_double, c_double,
                                                     c_double, _P, _P]),
    "b2md_force_lj_pairs_advance_halo": (c_int32, [_P, _P, _P, _P, _P, c_int64, POINTER(Box),
                                                   c_double, _P, c_double, _P, _P, c_int64, _P, _P,
                                                   c_int64, _P, POINTER(c_double), c_int32,
                                                   c_int32, c_int32, c_int32, _P, _P, _P, _P, _P,
                                                   _P]),
    "b2md_force_lj_all_pairs": (c_int32, [_P, c_int64, POINTER(Box), POINTER(c_double), c_int32,
                                          _P, _P, _P, _P]),
    "b2md_vv_integrate": (c_int32, [_P, _P, _P, _P, _P, c_int64, POINTER(Box), c_double, _P,
                                    c_double, _P, _P]),
    "b2md_vv_integrate_gated": (c_int32, [_P, _P, _P, _P, _P, c_int64, POINTER(Box), c_double,
                                          _P, c_double, _P, c_int32, _P]),
    "b2md_vv_finalize": (c_int32, [_P, _P, c_int64, c_double, _P]),
    "b2md_vv_finalize_integrate": (c_int32, [_P, _P, _P, _P, _P, c_int64, POINTER(Box), c_double,
                                             _P, c_double, _P, _P]),
    "b2md_andersen": (c_int32, [_P, _P, c_int64, c_uint64, c_uint64, c_double, c_double, _P, _P]),
    "b2md_stream_words": (c_int32, [c_uint64, c_uint64, c_uint64, c_int64, c_int64, _P, _P, _P,
                                    _P]),
    "b2md_reduce_scratch_bytes": (c_int64, [c_int64]),
    "b2md_reduce_sum_f64": (c_int32, [_P, c_int64, _P, _P, _P]),
    "b2md_thermo_scratch_bytes": (c_int64, [c_int64]),
    "b2md_thermo": (c_int32, [_P, _P, _P, c_int64, _P, _P, _P]),
    "b2md_hilbert_key_bits": (c_int32, [POINTER(Grid), c_int32]),
    "b2md_hilbert_keys": (c_int32, [_P, _P, c_int64, POINTER(Grid), c_int32, _P, _P]),
    "b2md_cell_keys": (c_int32, [_P, c_int64, _P, _P]),
    "b2md_iota_i32": (c_int32, [_P, c_int64, _P]),
    "b2md_sort_scratch_bytes": (c_int64, [c_int64]),
    "b2md_sort_pairs_u64": (c_int32, [_P, _P, _P, _P, c_int64, c_int32, _P, _P]),
    "b2md_gather16": (c_int32, [_P, _P, _P, c_int64, _P]),
    "b2md_gather4": (c_int32, [_P, _P, _P, c_int64, _P]),
    "b2md_runner_create": (c_void_p, [POINTER(RunnerConfig)]),
    "b2md_runner_destroy": (None, [c_void_p]),
    "b2md_runner_set_list": (c_int32, [c_void_p, _P, c_int32]),
    "b2md_runner_set_pair_list": (c_int32, [c_void_p, _P, c_int32]),
    "b2md_runner_prepare": (c_int32, [c_void_p, POINTER(RunReport)]),
    "b2md_runner_run": (c_int32, [c_void_p, c_int64, c_int32, POINTER(RunReport)]),
    "b2md_runner_set_inner_pair_list": (c_int32, [c_void_p, _P]),
    "b2md_runner_prune_count": (c_int64, [c_void_p, POINTER(c_int64)]),
    "b2md_runner_set_thermostat": (c_int32, [c_void_p, c_double, c_double, c_uint64]),
    "b2md_runner_set_step": (c_int32, [c_void_p, c_int64]),
    "b2md_vv_finalize_andersen": (c_int32, [_P, _P, _P, _P, _P, c_int64, _P, c_double, c_uint64,
                                            c_uint64, c_double, c_double, c_int32, _P, c_double,
                                            _P, _P]),
    "b2md_run_all_pairs": (c_int32, [_P, _P, _P, _P, _P, _P, c_int64, _P, _P, c_int32, c_double,
                                     c_int64, c_double, c_double, c_uint64, c_int64, _P, _P, _P,
                                     _P, _P]),
    "b2md_force_lj_all_pairs_advance": (c_int32, [_P, _P, _P, _P, _P, c_int64, _P, _P, c_int32,
                                                  c_double, _P, _P]),
}

#: entry points that report errors through their int return value
_CHECKED = {name for name, (res, _) in _SIGNATURES.items()
            if res is c_int32 and name not in ("b2md_version", "b2md_hilbert_key_bits",
                                             "b2md_steps_persistent_lanes")}

_lib = None


def exported_symbols():
    """Names include/b2md.h declares (used by the symbol-export test)."""
    return sorted(_SIGNATURES)


def load():
    """Load libb2md.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise B2mdError(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a).  This package has no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)     # AttributeError if the symbol is not exported
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def call(name, *args):
    """Invoke a checked entry point and raise B2mdError on failure."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if name in _CHECKED and rc != 0:
        msg = lib.b2md_last_error_string().decode("utf-8", "replace")
        raise B2mdError(f"{name} failed (code {rc}): {msg}")
    return rc


def make_box(edge_lengths) -> Box:
    b = Box()
    for a in range(3):
        b.edge[a] = float(edge_lengths[a])
    return b
