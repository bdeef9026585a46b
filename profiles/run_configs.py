#!/usr/bin/env python
"""BASELINE.json configs 1, 2, 4 and a single-GPU data point of config 5 on the
B200 path: energy conservation, rebuild cadence and throughput.  One JSON line
per config (CUDA-event timing of the production loop, sampling included)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2406_04210_b200 as b2


def run(name, n, density, lj, steps, every, t0=1.2, dt=0.001, skin=0.3, species=None, seed=42,
        warmup=0):
    st, box = b2.init_lattice_any(n, density)
    if species is not None:
        st = b2.ParticleState(st.positions.acquire_read(b2.HOST), species=species)
    b2.init_velocities(st, t0, seed)
    sim = b2.Simulation(st, box, lj, dt, force_mode=b2.TRUNCATED, skin=skin,
                        sample_interval=every, sample_initial=True)
    if warmup:
        sim.run(warmup)
        sim.samples.clear()
        sim.samples.append(sim.measure())
        sim.reset_counters()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record()
    sim.run(steps)
    stop.record()
    torch.cuda.synchronize()
    ms = start.elapsed_time(stop)
    e = np.array([s.total_energy for s in sim.samples])
    half = len(e) // 2
    t = np.arange(len(e) - half)
    slope = np.polyfit(t, e[half:], 1)[0] * (len(e) - half) / abs(e[0]) if len(e) - half > 2 else 0.0
    p = np.array([s.total_momentum for s in sim.samples])
    out = {
        "config": name, "n": n, "steps": steps, "ms_per_step": ms / steps,
        "particle_steps_per_s": n * steps / ms * 1e3,
        "drift_end_to_end": abs(e[-1] - e[0]) / abs(e[0]),
        "drift_max_over_samples": float(np.max(np.abs(e - e[0])) / abs(e[0])),
        "second_half_max_dev": float(np.max(np.abs(e[half:] - e[half])) / abs(e[0])),
        "second_half_slope_rel": float(slope),
        "max_momentum_norm": float(np.max(np.linalg.norm(p, axis=1))),
        "T_end": sim.samples[-1].temperature, "pressure_end": sim.samples[-1].pressure,
        "e_pot_per_particle_end": sim.samples[-1].potential_energy / n,
        "rebuilds": sim.rebuild_count, "stride": sim.stride,
        "overflow_events": sim.overflow_events, "kernel_launches": sim.kernel_launches,
    }
    sim.close()
    print(json.dumps(out), flush=True)
    del sim, st
    torch.cuda.empty_cache()


ap = argparse.ArgumentParser()
ap.add_argument("--which", default="1,2,4,5")
args = ap.parse_args()
which = set(args.which.split(","))
lj = b2.make_shifted(1.0, 1.0, 2.5)
if "1" in which:
    run("1: LJ N=4096 1000 steps", 4096, 0.75, lj, 1000, 100)
if "2" in which:
    run("2: LJ N=65536 1e4 steps, skin 0.3, Hilbert reordering", 65536, 0.75, lj, 10_000, 100)
if "3" in which:
    run("3: LJ N=1M 2000 steps after 200 warm-up", 1_000_000, 0.75, lj, 2000, 100, warmup=200)
if "4" in which:
    n = 262_144
    species = (np.random.default_rng(42).permutation(n) < n // 5).astype(np.int32)
    run("4: Kob-Andersen N=262144 rho=1.2 NVE 2000 steps", n, 1.2, b2.PairTable.kob_andersen(),
        2000, 100, t0=1.0, species=species)
if "A" in which:
    # the paper's primary benchmark: untruncated all-pairs, N=2000
    rec, samples = b2.run_benchmark(b2.preset_config("all2all-2k"))
    print(json.dumps({"config": "A: all2all-2k preset (N=2000, 5000 steps, all pairs)",
                      "steps_per_second": rec.steps_per_second, "wall_time_s": rec.wall_time_s,
                      "pair_evaluations_per_s": 2000 * 1999 * rec.steps_per_second,
                      "drift": rec.final_energy_drift_rel}), flush=True)
    rec, samples = b2.run_benchmark(b2.preset_config("trunc-10k"))
    print(json.dumps({"config": "B: trunc-10k preset (N=10000, 5000 steps, thermostat 5.0)",
                      "steps_per_second": rec.steps_per_second, "wall_time_s": rec.wall_time_s,
                      "rebuilds": rec.rebuild_count,
                      "T_mean": float(np.mean([s.temperature for s in samples]))}), flush=True)
if "5" in which:
    run("5 (single GPU): LJ N=16M 100 steps", 16_000_000, 0.75, lj, 100, 50)
