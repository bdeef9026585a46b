"""Shared helpers for the parity tests: input quantisation to the device
formats and the stated fp32 error metrics (hard part 3)."""
import numpy as np


def quantize_ds(x):
    """Nearest double-single (fp32 hi + fp32 lo) value of each fp64 entry --
    the set of positions the device can hold exactly."""
    x = np.asarray(x, dtype=np.float64)
    hi = x.astype(np.float32)
    lo = (x - hi.astype(np.float64)).astype(np.float32)
    return hi.astype(np.float64) + lo.astype(np.float64)


def quantize_f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def force_error_metrics(got, ref, pair_scale=None):
    """errinf_i = max_c |got - ref|.
    M1: errinf_i / max(Finf_i, 1e-3 max_j Finf_j)   (per-particle norm)
    M3: errinf_i / rms(F)
    M2: errinf_i / sum_j |f_ij|  when pair_scale (the per-particle sum of pair
        force magnitudes) is given."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.max(np.abs(got - ref), axis=1)
    finf = np.max(np.abs(ref), axis=1)
    m1 = float(np.max(err / np.maximum(finf, 1e-3 * finf.max())))
    m3 = float(np.max(err) / np.sqrt(np.mean(ref * ref)))
    out = {"M1": m1, "M3": m3}
    if pair_scale is not None:
        out["M2"] = float(np.max(err / np.maximum(pair_scale, 1e-300)))
    return out


def scalar_rel_error(got, ref, floor_fraction=1e-3):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    denom = np.maximum(np.abs(ref), floor_fraction * np.max(np.abs(ref)))
    return float(np.max(np.abs(got - ref) / np.maximum(denom, np.finfo(np.float64).tiny)))


def pair_force_scale(pos, edges, table, nlist_indices, counts, species=None):
    """sum_j |f_ij| per particle in fp64 (denominator of metric M2)."""
    pos = np.asarray(pos, dtype=np.float64)
    edges = np.asarray(edges, dtype=np.float64)
    n = pos.shape[0]
    nt = int(round(np.sqrt(table.shape[0])))
    out = np.zeros(n)
    for i in range(n):
        js = nlist_indices[i, :counts[i]].astype(np.int64)
        d = pos[i] - pos[js]
        d -= edges * np.rint(d / edges)
        r2 = (d * d).sum(axis=1)
        t = (0 if species is None else species[i]) * nt + (0 if species is None else species[js])
        eps, sig2, rc2 = table[t, 0], table[t, 1], table[t, 2]
        inside = r2 < rc2
        s6 = (sig2 / r2) ** 3
        fr = np.where(inside, 24.0 * eps * (2.0 * s6 * s6 - s6) / r2, 0.0)
        out[i] = np.sum(np.abs(fr) * np.sqrt(r2))
    return out


def fluid_state(n, density=0.75, temperature=1.2, seed=42, jitter=0.08):
    """fcc + vacancies (the reference's generator) with a small random
    displacement so the configuration is not degenerate; velocities Maxwell."""
    from oracle import oracle as orc
    pos, edge = orc.fcc_lattice(n, density)
    gen = np.random.default_rng(seed)
    pos = pos + gen.normal(scale=jitter, size=pos.shape)
    pos -= np.floor(pos / edge) * edge
    pos = np.where(pos >= edge, pos - edge, pos)
    vel = orc.maxwell_velocities(n, temperature, seed + 1)
    return pos, vel, edge
