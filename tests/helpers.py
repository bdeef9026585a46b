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


def backward_error(got, ref, scale):
    """max_i |got_i - ref_i| / scale_i (vector rows use the max component)."""
    err = np.abs(np.asarray(got, dtype=np.float64) - np.asarray(ref, dtype=np.float64))
    if err.ndim == 2:
        err = err.max(axis=1)
    return float(np.max(err / np.maximum(scale, 1e-300)))


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
