#!/bin/bash
# Every kernel of a window of MD steps under `ncu --set full` (molten N = 1 M state: 300
# untimed steps, then 70 profiled steps = ~2 rebuilds with Hilbert reorder, one sample step):
# the per-kernel roofline table of BASELINE.json configs[2] (force, neighbour build, sort,
# integrate, reductions).  Run on the GPU box through gpurun.
set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --profile-from-start off -c 400 \
    -o gpurun_out/allkernels -f python profiles/profile_step.py --melt 330 --steps 70 \
    --profiler-range > gpurun_out/prof_allkernels.log 2>&1
tail -2 gpurun_out/prof_allkernels.log
python profiles/kernel_roofline.py gpurun_out/allkernels.ncu-rep > gpurun_out/kernel_roofline.txt 2>&1
cat gpurun_out/kernel_roofline.txt
# the reports themselves exceed what gpurun copies back (64 MiB): keep the summaries
rm -f gpurun_out/*.ncu-rep
