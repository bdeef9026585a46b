"""CPU oracle for the MD hot path -- TEST INFRASTRUCTURE, not product code.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product package
``paper_2406_04210_b200`` never imports it and has no CPU fallback.

What it is: a numpy + C (``md_oracle.c``, built by ``oracle/Makefile`` into
``oracle/libmdoracle.so``) restatement of the reference package ``mdbench`` 0.1.0
(``/root/reference/pkg/src/mdbench``), operating on plain arrays in the
reference's own formats (fp64 positions (n,3), int64 images, ...).  Each function
cites the reference lines it follows.  Parity status:

* PINNED by golden vectors generated from the real reference in the build
  container (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``, checked
  bit-for-bit by ``tests/test_oracle_golden.py``): cell binning, neighbour lists
  (cell path, brute path, overflow), reorder permutation, truncated and
  all-pairs forces + per-particle energies, velocity-Verlet integrate/finalize
  with wrap, deterministic reductions, KE/T/momentum, rebuild criterion, and a
  whole NVE trajectory's sample series.
* PARITY UNPINNED (no counterpart in the reference): Hilbert
  keys, per-particle virial, centre-of-mass velocity, per-pair-type tables,
  slab decomposition helpers.  They extend the reference's conventions and are
  checked by construction (ntypes=1 tables reproduce the pinned single-type
  result bit-for-bit; virial is checked against a finite-difference /
  brute-force identity; Hilbert keys against the curve's adjacency property).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libmdoracle.so")
_lib = None

_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def build_library(force: bool = False) -> str:
    """Compile md_oracle.c (gcc, no FMA contraction, OpenMP) if needed."""
    src = os.path.join(_HERE, "md_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        import subprocess
        subprocess.check_call(["make", "-s", "-C", _HERE, "libmdoracle.so"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build_library()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_tree_sum.restype = ctypes.c_double
        L.orc_tree_sum.argtypes = [_f64p, ctypes.c_int64]
        L.orc_max_disp2.restype = ctypes.c_double
        _lib = L
    return _lib


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _p(a, t):
    return a.ctypes.data_as(t)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# --------------------------------------------------------------------------
# geometry (core.py:60-93)
# --------------------------------------------------------------------------

def minimum_image(dr, edges):
    """core.py:60-69: dr - L * rint(dr * (1/L)), half-even ties."""
    dr = np.asarray(dr, dtype=np.float64)
    edges = np.asarray(edges, dtype=np.float64)
    return dr - edges * np.rint(dr * (1.0 / edges))


def wrap_position(r, image, edges):
    """core.py:72-93: floor + nudge; returns (wrapped, image + k)."""
    r = np.asarray(r, dtype=np.float64)
    image = np.asarray(image, dtype=np.int64)
    edges = np.asarray(edges, dtype=np.float64)
    k = np.floor(r * (1.0 / edges))
    w = r - k * edges
    below = w < 0.0
    w = np.where(below, w + edges, w)
    k = np.where(below, k - 1.0, k)
    above = w >= edges
    w = np.where(above, w - edges, w)
    k = np.where(above, k + 1.0, k)
    return w, image + k.astype(np.int64)


# --------------------------------------------------------------------------
# potential (potential.py:47-66)
# --------------------------------------------------------------------------

def lj_shift(epsilon: float, sigma: float, r_cut: float) -> float:
    """potential.py:47-50,61-66: -4 eps (s6*s6 - s6), s2 = sigma^2 / rc^2."""
    if math.isinf(r_cut):
        return 0.0
    s2 = (sigma * sigma) / (r_cut * r_cut)
    s6 = s2 * s2 * s2
    return -(4.0 * epsilon * (s6 * s6 - s6))


def pair_table(epsilon, sigma, r_cut, shifted: bool = True):
    """(ntypes*ntypes, 4) rows = eps, sigma^2, rc^2, shift.  Scalars give the
    single-type table whose row is exactly forces.py:119-126's scalar pack."""
    eps = np.atleast_2d(np.asarray(epsilon, dtype=np.float64))
    sig = np.atleast_2d(np.asarray(sigma, dtype=np.float64))
    rc = np.atleast_2d(np.asarray(r_cut, dtype=np.float64))
    nt = eps.shape[0]
    tab = np.zeros((nt * nt, 4), dtype=np.float64)
    for a in range(nt):
        for b in range(nt):
            e, s, r = float(eps[a, b]), float(sig[a, b]), float(rc[a, b])
            tab[a * nt + b] = (e, s * s, r * r,
                               lj_shift(e, s, r) if shifted else 0.0)
    return tab


# --------------------------------------------------------------------------
# cells and lists (neighbor.py:57-270)
# --------------------------------------------------------------------------

@dataclass
class Grid:
    cells_per_axis: np.ndarray
    cell_edge: np.ndarray
    box_edges: np.ndarray
    cell_of_particle: np.ndarray
    cell_start: np.ndarray
    cell_particles: np.ndarray
    fallback: bool


def grid_shape(edges, r_list):
    """neighbor.py:67-71: cells per axis, cell edge."""
    edges = np.asarray(edges, dtype=np.float64)
    if not (r_list > 0.0 and np.isfinite(r_list)):
        raise ValueError("r_list must be positive and finite")
    if np.any(edges < r_list):
        raise ValueError("every box edge must be >= r_list")
    ncells = np.maximum(np.floor(edges / r_list).astype(np.int64), 1)
    return ncells, edges / ncells


def bin_particles(pos, edges, r_list) -> Grid:
    """neighbor.py:57-91."""
    edges = np.asarray(edges, dtype=np.float64)
    ncells, cell_edge = grid_shape(edges, r_list)
    pos = np.asarray(pos, dtype=np.float64)
    idx = np.floor(pos / cell_edge).astype(np.int64)
    idx = np.minimum(np.maximum(idx, 0), ncells - 1)
    flat = (idx[:, 0] * ncells[1] + idx[:, 1]) * ncells[2] + idx[:, 2]
    order = np.argsort(flat, kind="stable").astype(np.int64)
    occ = np.bincount(flat, minlength=int(np.prod(ncells)))
    start = np.zeros(occ.size + 1, dtype=np.int64)
    start[1:] = np.cumsum(occ)
    return Grid(ncells, cell_edge, edges.copy(), flat, start, order,
                bool(np.any(ncells < 3)))


@dataclass
class NList:
    indices: np.ndarray       # (n, stride) int32 row-major, rows ascending
    counts: np.ndarray        # (n,) int32
    stride: int
    overflow: bool
    row_overflow: np.ndarray  # (n,) uint8
    r_list: float
    r_cut: float
    positions_at_build: np.ndarray


def build_neighbor_list(pos, images, grid: Grid, r_list, stride, r_cut=None,
                        threads: int = 1) -> NList:
    """neighbor.py:185-240 (+ kernels 112-182 in md_oracle.c)."""
    pos = _c(pos, np.float64)
    n = pos.shape[0]
    stride = int(stride)
    if stride < 1:
        raise ValueError("stride must be >= 1")
    if r_cut is None:
        r_cut = r_list
    if not (0.0 < r_cut <= r_list):
        raise ValueError("need 0 < r_cut <= r_list")
    edges = _c(grid.box_edges, np.float64)
    rl2 = float(r_list) * float(r_list)
    nbr = np.zeros((n, stride), dtype=np.int32)
    counts = np.zeros(n, dtype=np.int32)
    over = np.zeros(n, dtype=np.uint8)
    L = lib()
    if grid.fallback:
        L.orc_list_brute(ctypes.c_int64(n), _p(pos, _f64p), _p(edges, _f64p),
                         ctypes.c_double(rl2), ctypes.c_int64(stride),
                         _p(nbr, _i32p), _p(counts, _i32p), _p(over, _u8p),
                         ctypes.c_int(threads))
    else:
        nc = _c(grid.cells_per_axis, np.int64)
        cof = _c(grid.cell_of_particle, np.int64)
        cst = _c(grid.cell_start, np.int64)
        cpa = _c(grid.cell_particles, np.int64)
        L.orc_list_cells(ctypes.c_int64(n), _p(pos, _f64p), _p(edges, _f64p),
                         _p(nc, _i64p), _p(cof, _i64p), _p(cst, _i64p),
                         _p(cpa, _i64p), ctypes.c_double(rl2),
                         ctypes.c_int64(stride), _p(nbr, _i32p),
                         _p(counts, _i32p), _p(over, _u8p),
                         ctypes.c_int(threads))
    images = np.asarray(images, dtype=np.int64)
    return NList(nbr, counts, stride, bool(over.any()), over, float(r_list),
                 float(r_cut), pos + images * edges)


def max_displacement_sq(pos, images, edges, at_build) -> float:
    """neighbor.py:251-253."""
    pos = _c(pos, np.float64)
    images = _c(images, np.int64)
    edges = _c(edges, np.float64)
    at_build = _c(at_build, np.float64)
    return float(lib().orc_max_disp2(ctypes.c_int64(pos.shape[0]),
                                     _p(pos, _f64p), _p(images, _i64p),
                                     _p(edges, _f64p), _p(at_build, _f64p)))


def needs_rebuild(pos, images, edges, nlist: NList) -> bool:
    """neighbor.py:243-254: strict > (skin/2)^2."""
    half = 0.5 * (nlist.r_list - nlist.r_cut)
    return max_displacement_sq(pos, images, edges,
                               nlist.positions_at_build) > half * half


def reorder_permutation(cell_of_particle) -> np.ndarray:
    """neighbor.py:266: stable argsort; new row k = old row perm[k]."""
    return np.argsort(np.asarray(cell_of_particle), kind="stable")


def pair_set(nlist_indices, counts):
    """Unordered pair set of a row-major list (test helper)."""
    out = set()
    for i in range(len(counts)):
        for j in nlist_indices[i, :counts[i]]:
            j = int(j)
            out.add((i, j) if i < j else (j, i))
    return out


def pairs_within(pos, edges, radius):
    """bruteforce.py:27-34 (O(n^2) numpy; small n only)."""
    pos = np.asarray(pos, dtype=np.float64)
    d = pos[:, None, :] - pos[None, :, :]
    d = minimum_image(d, edges)
    r2 = (d * d).sum(axis=-1)
    n = pos.shape[0]
    mask = (r2 < radius * radius) & ~np.eye(n, dtype=bool)
    ii, jj = np.nonzero(np.triu(mask, k=1))
    return {(int(a), int(b)) for a, b in zip(ii, jj)}


# --------------------------------------------------------------------------
# forces (forces.py:72-159; extensions: virial, pair tables)
# --------------------------------------------------------------------------

class SingularPair(RuntimeError):
    def __init__(self, i, j):
        self.i, self.j = int(i), int(j)
        super().__init__(f"particles {i} and {j} coincide")


def _first_singular(bad_j):
    """forces.py:113-116: lowest i with a flagged partner."""
    if bad_j.max() >= 0:
        i = int(np.argmax(bad_j >= 0))
        raise SingularPair(i, bad_j[i])


def forces_truncated(pos, edges, table, nlist: NList, species=None,
                     threads: int = 1):
    """forces.py:141-159 -> (forces (n,3), pe (n,), virial (n,))."""
    if nlist.overflow:
        raise RuntimeError("neighbor list overflowed its stride")
    pos = _c(pos, np.float64)
    n = pos.shape[0]
    edges = _c(edges, np.float64)
    table = _c(table, np.float64)
    ntypes = int(round(math.sqrt(table.shape[0])))
    sp = None if species is None else _c(species, np.int32)
    f = np.zeros((n, 3), dtype=np.float64)
    pe = np.zeros(n, dtype=np.float64)
    w = np.zeros(n, dtype=np.float64)
    bad = np.full(n, -1, dtype=np.int64)
    lib().orc_force_truncated(
        ctypes.c_int64(n), _p(pos, _f64p), _p(edges, _f64p),
        _p(sp, _i32p) if sp is not None else None, ctypes.c_int(ntypes),
        _p(table, _f64p), ctypes.c_int64(nlist.stride),
        _p(nlist.indices, _i32p), _p(nlist.counts, _i32p), _p(f, _f64p),
        _p(pe, _f64p), _p(w, _f64p), _p(bad, _i64p), ctypes.c_int(threads))
    _first_singular(bad)
    return f, pe, w


def pair_scales(pos, edges, table, nlist: NList, species=None, threads: int = 1):
    """Per-particle sums of absolute pair contributions (|f|, |u|/2, |w|/2) --
    the denominators of the backward-error metrics used for the fp32 kernels."""
    pos = _c(pos, np.float64)
    n = pos.shape[0]
    edges = _c(edges, np.float64)
    table = _c(table, np.float64)
    ntypes = int(round(math.sqrt(table.shape[0])))
    sp = None if species is None else _c(species, np.int32)
    fs, us, ws = (np.zeros(n) for _ in range(3))
    lib().orc_pair_scales(
        ctypes.c_int64(n), _p(pos, _f64p), _p(edges, _f64p),
        _p(sp, _i32p) if sp is not None else None, ctypes.c_int(ntypes), _p(table, _f64p),
        ctypes.c_int64(nlist.stride), _p(nlist.indices, _i32p), _p(nlist.counts, _i32p),
        _p(fs, _f64p), _p(us, _f64p), _p(ws, _f64p), ctypes.c_int(threads))
    return fs, us, ws


def forces_all_pairs(pos, edges, table, species=None, threads: int = 1):
    """forces.py:129-138 -> (forces, pe, virial)."""
    pos = _c(pos, np.float64)
    n = pos.shape[0]
    edges = _c(edges, np.float64)
    table = _c(table, np.float64)
    ntypes = int(round(math.sqrt(table.shape[0])))
    sp = None if species is None else _c(species, np.int32)
    f = np.zeros((n, 3), dtype=np.float64)
    pe = np.zeros(n, dtype=np.float64)
    w = np.zeros(n, dtype=np.float64)
    bad = np.full(n, -1, dtype=np.int64)
    lib().orc_force_all_pairs(
        ctypes.c_int64(n), _p(pos, _f64p), _p(edges, _f64p),
        _p(sp, _i32p) if sp is not None else None, ctypes.c_int(ntypes),
        _p(table, _f64p), _p(f, _f64p), _p(pe, _f64p), _p(w, _f64p),
        _p(bad, _i64p), ctypes.c_int(threads))
    _first_singular(bad)
    return f, pe, w


def forces_bruteforce_numpy(pos, edges, table, species=None):
    """Independent expression tree (bruteforce.py:37-65) extended with the
    virial and pair tables; O(n^2) memory, small n only."""
    pos = np.asarray(pos, dtype=np.float64)
    n = pos.shape[0]
    table = np.asarray(table, dtype=np.float64)
    nt = int(round(math.sqrt(table.shape[0])))
    sp = np.zeros(n, dtype=np.int64) if species is None else np.asarray(species, dtype=np.int64)
    pair_type = sp[:, None] * nt + sp[None, :]
    eps, sig2, rc2, shift = (table[pair_type, c] for c in range(4))
    d = minimum_image(pos[:, None, :] - pos[None, :, :], edges)
    r2 = d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1] + d[..., 2] * d[..., 2]
    np.fill_diagonal(r2, np.inf)
    inside = r2 < rc2
    sr2 = np.where(inside, sig2 / r2, 0.0)
    sr6 = sr2 ** 3
    sr12 = sr6 ** 2
    e_pair = np.where(inside, 4.0 * eps * (sr12 - sr6) + shift, 0.0)
    fr = np.where(inside, (48.0 * eps * sr12 - 24.0 * eps * sr6) / r2, 0.0)
    forces = (fr[..., None] * d).sum(axis=1)
    r2_safe = np.where(inside, r2, 0.0)
    return forces, 0.5 * e_pair.sum(axis=1), 0.5 * (fr * r2_safe).sum(axis=1)


# --------------------------------------------------------------------------
# integrator (integrate.py:58-79)
# --------------------------------------------------------------------------

def vv_integrate(pos, images, vel, forces, masses, edges, dt):
    """integrate.py:58-70, numpy statement order preserved; returns new
    (pos, images, vel)."""
    vel = np.array(vel, dtype=np.float64)
    pos = np.array(pos, dtype=np.float64)
    forces = np.asarray(forces, dtype=np.float64)
    masses = np.asarray(masses, dtype=np.float64)
    vel += (forces / masses[:, None]) * (0.5 * dt)
    pos += vel * dt
    pos, images = wrap_position(pos, images, edges)
    return pos, images, vel


def vv_finalize(vel, forces, masses, dt):
    """integrate.py:73-79."""
    vel = np.array(vel, dtype=np.float64)
    vel += (np.asarray(forces, dtype=np.float64)
            / np.asarray(masses, dtype=np.float64)[:, None]) * (0.5 * dt)
    return vel


# --------------------------------------------------------------------------
# random streams + Andersen thermostat (rng.py:40-66, integrate.py:82-107)
# --------------------------------------------------------------------------

def stream_raw(seed, stream, step, count):
    """rng.py:40-53: numpy Philox keyed (seed, 0) at counter (0, 0, stream, step)."""
    two64 = 1 << 64
    gen = np.random.Philox(counter=np.array([0, 0, stream % two64, step % two64], dtype=np.uint64),
                           key=np.array([seed % two64, 0], dtype=np.uint64))
    return gen.random_raw(count) if count else np.empty(0, dtype=np.uint64)


def stream_uniforms(seed, stream, step, count, word_offset=0):
    """rng.py:56-60."""
    words = stream_raw(seed, stream, step, word_offset + count)[word_offset:]
    return ((words >> np.uint64(11)).astype(np.float64) + 0.5) * np.float64(2.0 ** -53)


def stream_normals(seed, stream, step, count, word_offset=0):
    """rng.py:63-66 (scipy.special.ndtri = Cephes ndtri)."""
    from scipy.special import ndtri
    return ndtri(stream_uniforms(seed, stream, step, count, word_offset))


def andersen_thermostat(vel, masses, temperature, rate, seed, dt, step):
    """integrate.py:82-107 -> (new velocities, redraw mask)."""
    vel = np.array(vel, dtype=np.float64)
    n = vel.shape[0]
    p = min(rate * dt, 1.0)
    if p <= 0.0:
        return vel, np.zeros(n, dtype=bool)
    redraw = stream_uniforms(seed, 0, step, n) < p
    if redraw.any():
        z = stream_normals(seed, 0, step, 3 * n, word_offset=n).reshape(n, 3)
        scale = np.sqrt(temperature / np.asarray(masses, dtype=np.float64))
        vel[redraw] = z[redraw] * scale[redraw, None]
    return vel, redraw


# --------------------------------------------------------------------------
# observables (observables.py:28-98)
# --------------------------------------------------------------------------

def reduce_sum(values, deterministic: bool = True) -> float:
    """observables.py:43-74."""
    a = np.ascontiguousarray(values, dtype=np.float64).ravel()
    if a.size == 0:
        return 0.0
    if not deterministic:
        return float(np.sum(a))
    return float(lib().orc_tree_sum(_p(a, _f64p), ctypes.c_int64(a.size)))


def per_particle_kinetic(vel, masses):
    """observables.py:82 with the row product summed left to right."""
    v = np.asarray(vel, dtype=np.float64)
    m = np.asarray(masses, dtype=np.float64)
    return 0.5 * m * ((v[:, 0] * v[:, 0] + v[:, 1] * v[:, 1]) + v[:, 2] * v[:, 2])


def thermo(vel, masses, pe, virial=None, deterministic: bool = True):
    """observables.py:77-98 + extensions (virial sum, centre-of-mass velocity).
    Returns dict(pe, ke, temperature, momentum(3), virial, com_velocity(3))."""
    v = np.asarray(vel, dtype=np.float64)
    m = np.asarray(masses, dtype=np.float64)
    n = v.shape[0]
    ke = reduce_sum(per_particle_kinetic(v, m), deterministic)
    mom = np.array([reduce_sum(m * v[:, c], deterministic) for c in range(3)])
    out = {
        "pe": reduce_sum(pe, deterministic),
        "ke": ke,
        "temperature": 2.0 * ke / (3.0 * n),
        "momentum": mom,
        "mass": reduce_sum(m, deterministic),
    }
    out["com_velocity"] = mom / out["mass"]
    if virial is not None:
        out["virial"] = reduce_sum(virial, deterministic)
    return out


# --------------------------------------------------------------------------
# Hilbert keys (extension; north_star subsystem 2)
# --------------------------------------------------------------------------

HILBERT_SUB_BITS = 2


def hilbert_cell_coords(pos, edges, r_list, sub_bits: int = HILBERT_SUB_BITS):
    """Cell-aligned integer coordinates q = (cell << sub_bits) | sub, with
    cell = bin_particles' cell coordinate (fp64 division + clip) and
    sub = clip(floor(fp32((pos - cell*edge)) * fp32(1/edge) * 2^sub_bits)).
    Returns (q (n,3) uint64, bits per axis)."""
    pos = np.asarray(pos, dtype=np.float64)
    ncells, cell_edge = grid_shape(edges, r_list)
    cell = np.floor(pos / cell_edge).astype(np.int64)
    cell = np.minimum(np.maximum(cell, 0), ncells - 1)
    frac = (pos - cell * cell_edge).astype(np.float32) * (1.0 / cell_edge).astype(np.float32)
    sub = np.floor(frac * np.float32(1 << sub_bits)).astype(np.int64)
    sub = np.minimum(np.maximum(sub, 0), (1 << sub_bits) - 1)
    cell_bits = 1
    while (1 << cell_bits) < int(ncells.max()):
        cell_bits += 1
    q = (cell << sub_bits) | sub
    return q.astype(np.uint64), cell_bits + sub_bits


def hilbert_keys(q, bits: int):
    """3-D Hilbert index (Skilling 2004 transpose form) of integer coords
    q (n,3) with `bits` bits per axis -> uint64 keys of 3*bits bits.  The key
    interleaves the transposed words MSB first as x,y,z."""
    X = [np.array(q[:, c], dtype=np.uint64) for c in range(3)]
    one = np.uint64(1)
    M = one << np.uint64(bits - 1)
    # inverse undo excess work
    Q = M
    while Q > one:
        P = Q - one
        for i in range(3):
            hit = (X[i] & Q) != 0
            X[0] = np.where(hit, X[0] ^ P, X[0])
            t = (X[0] ^ X[i]) & P
            t = np.where(hit, np.uint64(0), t)
            X[0] = X[0] ^ t
            X[i] = X[i] ^ t
        Q >>= one
    # Gray encode
    for i in range(1, 3):
        X[i] = X[i] ^ X[i - 1]
    t = np.zeros_like(X[0])
    Q = M
    while Q > one:
        t = np.where((X[2] & Q) != 0, t ^ (Q - one), t)
        Q >>= one
    for i in range(3):
        X[i] = X[i] ^ t
    key = np.zeros_like(X[0])
    for b in range(bits - 1, -1, -1):
        for i in range(3):
            key = (key << one) | ((X[i] >> np.uint64(b)) & one)
    return key


def hilbert_permutation(pos, edges, r_list, sub_bits: int = HILBERT_SUB_BITS):
    q, bits = hilbert_cell_coords(pos, edges, r_list, sub_bits)
    keys = hilbert_keys(q, bits)
    return np.argsort(keys, kind="stable"), keys


# --------------------------------------------------------------------------
# whole-step loop (sim.py:114-174, core.py:262-279) for the CPU baseline and
# for trajectory parity
# --------------------------------------------------------------------------

class Sim:
    """NVE truncated-LJ simulation with the reference's rebuild policy
    (sim.py:131-149: stride doubling, at most 10 growths)."""

    DEFAULT_STRIDE = 64
    GROWTH_LIMIT = 10

    def __init__(self, pos, vel, edges, table, dt, skin, species=None,
                 masses=None, images=None, stride=DEFAULT_STRIDE,
                 sample_interval=100, threads=1, deterministic=True):
        self.pos = np.array(pos, dtype=np.float64)
        n = self.pos.shape[0]
        self.vel = np.zeros((n, 3)) if vel is None else np.array(vel, dtype=np.float64)
        self.images = np.zeros((n, 3), dtype=np.int64) if images is None \
            else np.array(images, dtype=np.int64)
        self.masses = np.ones(n) if masses is None else np.array(masses, dtype=np.float64)
        self.species = None if species is None else np.array(species, dtype=np.int32)
        self.edges = np.array(edges, dtype=np.float64)
        self.table = np.array(table, dtype=np.float64)
        self.r_cut = float(np.sqrt(self.table[:, 2].max()))
        self.dt = float(dt)
        self.skin = float(skin)
        self.stride = int(stride)
        self.sample_interval = int(sample_interval)
        self.threads = int(threads)
        self.deterministic = deterministic
        self.nlist = None
        self.rebuilds = 0
        self.step_count = 0
        self.samples = []
        self.forces = np.zeros((n, 3))
        self.pe = np.zeros(n)
        self.virial = np.zeros(n)
        self._compute_forces()

    def _rebuild(self):
        r_list = self.r_cut + self.skin
        growths = 0
        while True:
            grid = bin_particles(self.pos, self.edges, r_list)
            nl = build_neighbor_list(self.pos, self.images, grid, r_list,
                                     self.stride, r_cut=self.r_cut,
                                     threads=self.threads)
            self.nlist = nl
            self.rebuilds += 1
            if not nl.overflow:
                return
            growths += 1
            if growths > self.GROWTH_LIMIT:
                raise RuntimeError("neighbor list still overflows")
            self.stride *= 2

    def _compute_forces(self):
        if self.nlist is None or needs_rebuild(self.pos, self.images,
                                               self.edges, self.nlist):
            self._rebuild()
        self.forces, self.pe, self.virial = forces_truncated(
            self.pos, self.edges, self.table, self.nlist, self.species,
            threads=self.threads)

    def measure(self):
        t = thermo(self.vel, self.masses, self.pe, self.virial,
                   self.deterministic)
        t["step"] = self.step_count
        t["total_energy"] = t["pe"] + t["ke"]
        t["rebuild_count"] = self.rebuilds
        return t

    def run(self, n_steps: int):
        for _ in range(n_steps):
            self.pos, self.images, self.vel = vv_integrate(
                self.pos, self.images, self.vel, self.forces, self.masses,
                self.edges, self.dt)
            self._compute_forces()
            self.vel = vv_finalize(self.vel, self.forces, self.masses, self.dt)
            self.step_count += 1
            if self.step_count % self.sample_interval == 0:
                self.samples.append(self.measure())


# --------------------------------------------------------------------------
# synthetic inputs: fcc lattice (integrate.py:110-171).  Velocities: the
# reference draws Philox normals (rng.py) -- out of the hot path; the bench and
# tests use numpy's default_rng normals with the same COM removal and exact
# rescale (integrate.py:193-198).
# --------------------------------------------------------------------------

def fcc_lattice(n: int, density: float):
    """integrate.py:146-171: smallest enclosing fcc block, evenly spread
    vacancies (site floor(i*M/n)); returns (positions (n,3), cubic edge)."""
    k = 1
    while 4 * k ** 3 < n:
        k += 1
    m_sites = 4 * k ** 3
    edge = (n / density) ** (1.0 / 3.0)
    base = np.array([[0.0, 0.0, 0.0], [0.0, 0.5, 0.5],
                     [0.5, 0.0, 0.5], [0.5, 0.5, 0.0]])
    ax = np.arange(k)
    cells = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), axis=-1).reshape(-1, 3)
    sites = (cells[:, None, :] + base[None, :, :]).reshape(-1, 3) * (edge / k)
    if m_sites != n:
        keep = (np.arange(n, dtype=np.int64) * m_sites) // n
        sites = sites[keep]
    return sites, edge


def maxwell_velocities(n: int, temperature: float, seed: int, masses=None):
    """integrate.py:191-198 with numpy normals: zero COM, exact T."""
    m = np.ones(n) if masses is None else np.asarray(masses, dtype=np.float64)
    z = np.random.default_rng(seed).standard_normal((n, 3))
    v = z * np.sqrt(temperature / m)[:, None]
    v -= (m[:, None] * v).sum(axis=0) / m.sum()
    t_now = (m[:, None] * v * v).sum() / (3.0 * n)
    v *= math.sqrt(temperature / t_now)
    return v
