"""Lennard-Jones parameters (reference potential.py:23-91) plus per-pair-type
tables for mixtures (Kob-Andersen), which the reference lacks.

    u(r) = 4 eps [(sigma/r)^12 - (sigma/r)^6] + energy_shift    r <  r_cut
    u(r) = 0                                                    r >= r_cut

Forces are not shifted.  Parameters stay on the host in fp64; the force kernels
receive {eps, sigma^2, r_cut^2, shift} rows (forces.py:119-126) and narrow them.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class LJParams:
    epsilon: float
    sigma: float
    r_cut: float
    energy_shift: float

    def __post_init__(self):
        if not (self.epsilon > 0.0 and math.isfinite(self.epsilon)):
            raise ValueError("epsilon must be positive and finite")
        if not (self.sigma > 0.0 and math.isfinite(self.sigma)):
            raise ValueError("sigma must be positive and finite")
        if math.isfinite(self.r_cut) and self.r_cut <= self.sigma:
            raise ValueError("finite r_cut must exceed sigma")

    @property
    def truncated(self) -> bool:
        return math.isfinite(self.r_cut)

    @property
    def r_cut_sq(self) -> float:
        return self.r_cut * self.r_cut

    # -- uniform access used by the force operators -----------------------
    @property
    def ntypes(self) -> int:
        return 1

    @property
    def max_r_cut(self) -> float:
        return self.r_cut

    def table(self) -> np.ndarray:
        """(1, 4) row: eps, sigma^2, r_cut^2, shift (forces.py:123-126)."""
        return np.array([[self.epsilon, self.sigma * self.sigma, self.r_cut_sq,
                          self.energy_shift]], dtype=np.float64)


def _bare_energy(r_squared, epsilon, sigma):
    s2 = (sigma * sigma) / r_squared
    s6 = s2 * s2 * s2
    return 4.0 * epsilon * (s6 * s6 - s6)


def make_shifted(epsilon: float, sigma: float, r_cut: float = math.inf) -> LJParams:
    """LJ parameters whose shift zeroes u exactly at r_cut (potential.py:53-66)."""
    if math.isinf(r_cut):
        shift = 0.0
    else:
        probe = LJParams(epsilon, sigma, r_cut, 0.0)   # validates
        shift = -_bare_energy(probe.r_cut_sq, epsilon, sigma)
    return LJParams(epsilon, sigma, r_cut, shift)


def lj_eval(r_squared, params: LJParams):
    """(energy, force_over_r) at squared separations (potential.py:69-91)."""
    r2 = np.asarray(r_squared, dtype=np.float64)
    if np.any(r2 <= 0.0):
        raise ValueError("r_squared must be strictly positive")
    s2 = (params.sigma * params.sigma) / r2
    s6 = s2 * s2 * s2
    s12 = s6 * s6
    inside = r2 < params.r_cut_sq
    energy = np.where(inside, 4.0 * params.epsilon * (s12 - s6) + params.energy_shift, 0.0)
    force_over_r = np.where(inside, 24.0 * params.epsilon * (2.0 * s12 - s6) / r2, 0.0)
    if energy.ndim == 0:
        return float(energy), float(force_over_r)
    return energy, force_over_r


class PairTable:
    """Per-pair-type LJ parameters: symmetric (ntypes, ntypes) matrices of
    epsilon, sigma and r_cut; every pair gets its own energy shift through
    :func:`make_shifted`.  ``species`` values index the rows."""

    MAX_TYPES = 8

    def __init__(self, epsilon, sigma, r_cut):
        eps = np.array(epsilon, dtype=np.float64)
        sig = np.array(sigma, dtype=np.float64)
        rc = np.array(r_cut, dtype=np.float64)
        if eps.ndim != 2 or eps.shape[0] != eps.shape[1] or sig.shape != eps.shape \
                or rc.shape != eps.shape:
            raise ValueError("epsilon, sigma, r_cut must be square matrices of one shape")
        if eps.shape[0] > self.MAX_TYPES:
            raise ValueError(f"at most {self.MAX_TYPES} species are supported")
        for m in (eps, sig, rc):
            if not np.array_equal(m, m.T):
                raise ValueError("pair parameter matrices must be symmetric")
        if not np.all(np.isfinite(rc)):
            raise ValueError("tabulated potentials need finite cutoffs")
        self.epsilon, self.sigma, self.r_cut = eps, sig, rc
        self.pairs = [[make_shifted(float(eps[a, b]), float(sig[a, b]), float(rc[a, b]))
                       for b in range(eps.shape[0])] for a in range(eps.shape[0])]

    @classmethod
    def kob_andersen(cls, r_cut_factor: float = 2.5) -> "PairTable":
        """80:20 binary mixture of Kob & Andersen (PRE 51, 4626): eps AA/AB/BB =
        1/1.5/0.5, sigma = 1/0.8/0.88, r_cut = 2.5 sigma_ab."""
        eps = np.array([[1.0, 1.5], [1.5, 0.5]])
        sig = np.array([[1.0, 0.8], [0.8, 0.88]])
        return cls(eps, sig, r_cut_factor * sig)

    @property
    def ntypes(self) -> int:
        return self.epsilon.shape[0]

    @property
    def truncated(self) -> bool:
        return True

    @property
    def max_r_cut(self) -> float:
        return float(self.r_cut.max())

    @property
    def r_cut_value(self) -> float:
        return self.max_r_cut

    def table(self) -> np.ndarray:
        nt = self.ntypes
        out = np.zeros((nt * nt, 4), dtype=np.float64)
        for a in range(nt):
            for b in range(nt):
                p = self.pairs[a][b]
                out[a * nt + b] = (p.epsilon, p.sigma * p.sigma, p.r_cut_sq, p.energy_shift)
        return out
