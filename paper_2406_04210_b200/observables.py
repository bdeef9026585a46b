"""Scalar observables reduced on the device with the reference's fixed summation
tree (reference observables.py:28-112).

The reference reads the HOST side of velocities / masses / per-particle energies
on every sample, forcing a compute->host copy (observables.py:80-96).  Here the
sums are formed in HBM in one pass (`b2md_thermo`): fp64 accumulation of the
fp32 state in exactly the reference's grouping (4096-value blocks, adjacent-pair
trees), so only 8 doubles cross the bus.  Added observables: virial sum,
pressure, centre-of-mass velocity.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import COMPUTE, ParticleState

DETERMINISTIC = "deterministic"
FAST = "fast"


def _torch():
    import torch
    return torch


def reduce_sum(values, mode: str = DETERMINISTIC, backend=None, device: int = 0) -> float:
    """Sum a float array on the device; empty input sums to exactly 0.0.

    Both modes use the reference's deterministic tree (it is also the fastest
    single-pass order on the GPU), so results are bit-identical to
    ``mdbench.reduce_sum(values, "deterministic")`` for fp64 input."""
    if mode not in (DETERMINISTIC, FAST):
        raise ValueError(f"unknown reduction mode {mode!r}")
    torch = _torch()
    a = np.ascontiguousarray(values, dtype=np.float64).ravel()
    if a.size == 0:
        return 0.0
    lib = _lib.load()
    dev = torch.device("cuda", device)
    d_in = torch.from_numpy(a).to(dev)
    scratch = torch.empty(int(lib.b2md_reduce_scratch_bytes(a.size)) // 8 + 1,
                          dtype=torch.float64, device=dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    stream = int(torch.cuda.current_stream(dev).cuda_stream)
    _lib.call("b2md_reduce_sum_f64", d_in.data_ptr(), a.size, scratch.data_ptr(),
              out.data_ptr(), stream)
    return float(out.cpu()[0])


@dataclass(frozen=True)
class Thermo:
    """One pass of device reductions."""
    potential_energy: float
    kinetic_energy: float
    momentum: tuple
    virial: float
    mass: float
    n: int

    @property
    def temperature(self) -> float:
        return 2.0 * self.kinetic_energy / (3.0 * self.n)   # observables.py:84

    @property
    def com_velocity(self) -> tuple:
        return tuple(p / self.mass for p in self.momentum)

    def pressure(self, volume: float) -> float:
        """Virial pressure (2 KE + W) / (3 V), W = sum over pairs of r.f."""
        return (2.0 * self.kinetic_energy + self.virial) / (3.0 * volume)


def thermo(state: ParticleState) -> Thermo:
    """All of measure()'s sums in one kernel pass (sim.py:159-174)."""
    torch = _torch()
    lib = _lib.load()
    for name in ("velocities", "masses", "per_particle_potential", "virial"):
        getattr(state, name).acquire_read(COMPUTE)
    dev = state.device_state()
    scratch = torch.empty(int(lib.b2md_thermo_scratch_bytes(dev.n)) // 8 + 8,
                          dtype=torch.float64, device=dev.device)
    out = torch.empty(8, dtype=torch.float64, device=dev.device)
    _lib.call("b2md_thermo", dev.vel.data_ptr(), dev.force.data_ptr(), dev.virial.data_ptr(),
              dev.n, scratch.data_ptr(), out.data_ptr(), dev.stream)
    v = out.cpu().numpy()
    return Thermo(float(v[0]), float(v[1]), (float(v[2]), float(v[3]), float(v[4])),
                  float(v[5]), float(v[6]), int(v[7]))


def kinetic_energy_and_temperature(state: ParticleState, mode: str = DETERMINISTIC):
    """Total kinetic energy and 2 KE / (3 n) (observables.py:77-84)."""
    t = thermo(state)
    return t.kinetic_energy, t.temperature


def potential_energy_total(state: ParticleState, mode: str = DETERMINISTIC) -> float:
    """Sum of the per-particle half-shares (observables.py:87-90)."""
    return thermo(state).potential_energy


def total_momentum(state: ParticleState, mode: str = DETERMINISTIC):
    """Componentwise sum of m v (observables.py:93-98)."""
    return np.array(thermo(state).momentum)


def virial_total(state: ParticleState) -> float:
    return thermo(state).virial


def com_velocity(state: ParticleState):
    return np.array(thermo(state).com_velocity)


@dataclass(frozen=True)
class Sample:
    """One observation of the running system (observables.py:101-112) plus the
    virial sum and the centre-of-mass velocity."""

    step: int
    time: float
    potential_energy: float
    kinetic_energy: float
    total_energy: float
    temperature: float
    total_momentum: tuple
    rebuild_count: int
    virial: float = 0.0
    pressure: float = 0.0
    com_velocity: tuple = (0.0, 0.0, 0.0)
