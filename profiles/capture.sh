#!/bin/bash
# Round-1 profiling recipe (run on the GPU box through gpurun; outputs under gpurun_out/).
#   1. the bench line (timed with CUDA events, NOT under a profiler)
#   2. ncu launch list of the same bench command (cold-cache, serialised: shares only)
#   3. ncu --set full captures of the force, integrate and list-build kernels
set -x
mkdir -p gpurun_out
python bench.py --steps 2000 --warmup 200 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 2000 --warmup 200 > gpurun_out/bench_reference.json 2>> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches_bench.csv python bench.py --steps 100 --warmup 20 > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_force_lj_pair -s 450 -c 1 \
    -o gpurun_out/force python profiles/profile_step.py --steps 500 > gpurun_out/prof_force.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_integrate -s 30 -c 1 \
    -o gpurun_out/integrate python profiles/profile_step.py --steps 40 > gpurun_out/prof_integrate.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_list_cells -s 12 -c 1 \
    -o gpurun_out/nlist python profiles/profile_step.py --steps 400 > gpurun_out/prof_nlist.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pair_rows -s 12 -c 1 \
    -o gpurun_out/pairrows python profiles/profile_step.py --steps 400 > gpurun_out/prof_pairrows.log 2>&1
for k in force integrate nlist pairrows; do python profiles/ncu_summary.py gpurun_out/$k.ncu-rep > gpurun_out/ncu_$k.txt 2>&1; done
python profiles/launch_table.py gpurun_out/launches_bench.csv 30 > gpurun_out/launch_table_bench.txt 2>&1
tail -c 2500 gpurun_out/bench.json; cat gpurun_out/bench_reference.json
# the reports themselves exceed what gpurun copies back (64 MiB): keep the summaries
rm -f gpurun_out/*.ncu-rep
