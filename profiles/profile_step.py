#!/usr/bin/env python
"""Workload for ncu captures: the N=1M bench state, `--steps` MD steps through the
native loop (no CPU baseline, no end-to-end leg).  Usage on the GPU box:

  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
      --log-file gpurun_out/launches.csv python profiles/profile_step.py --steps 60
  ncu --set full --clock-control none --import-source on -k regex:k_force_lj -s 20 -c 2 \
      -o gpurun_out/force python profiles/profile_step.py --steps 30
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2406_04210_b200 as b2

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--steps", type=int, default=60)
ap.add_argument("--melt", type=int, default=0, help="untimed steps before (to leave the lattice)")
ap.add_argument("--reorder", default="hilbert")
ap.add_argument("--density", type=float, default=0.75)
ap.add_argument("--reorder-every", type=int, default=1)
ap.add_argument("--graph", type=int, default=0)
ap.add_argument("--profiler-range", action="store_true",
                help="cudaProfilerStart/Stop around the timed steps (ncu --profile-from-start off)")
args = ap.parse_args()

st, box = b2.init_lattice_any(args.n, args.density)
b2.init_velocities(st, 1.2, 42)
sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001, force_mode=b2.TRUNCATED,
                    skin=0.3, sample_interval=100,
                    reorder=None if args.reorder == "none" else args.reorder,
                    reorder_every=args.reorder_every, graph=args.graph)
if args.melt:
    sim.run(args.melt)
torch.cuda.synchronize()
start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if args.profiler_range:
    torch.cuda.profiler.start()
start.record()
sim.run(args.steps)
stop.record()
torch.cuda.synchronize()
if args.profiler_range:
    torch.cuda.profiler.stop()
ms = start.elapsed_time(stop)
print(f"n={args.n} steps={args.steps} ms/step={ms / args.steps:.4f} "
      f"particle-steps/s={args.n * args.steps / ms * 1e3:.3e} rebuilds={sim.rebuild_count} "
      f"launches={sim.kernel_launches} wasted={sim.wasted_force_launches} stride={sim.stride} "
      f"boundary={getattr(sim, '_n_boundary', None)} graph_steps={sim.graph_steps}")
sim.close()
