#!/bin/bash
# Round-2 evidence (run on the GPU box through gpurun; outputs under gpurun_out/r02/, copied to
# profiles/r02/ afterwards):
#   gpurun --timeout 3000 -- 'bash profiles/capture_r02.sh'
#   1. bench lines (CUDA events, NOT under a profiler): the driver's step count and 2000 steps,
#      and the reference arm
#   2. ncu launch list of the bench command (cold-cache, serialised: shares only)
#   3. ncu --set full captures of the one-launch step kernel, the list kernel that emits pair
#      rows and the fix-up merge, with per-source-line instruction counts of the list kernel
#   4. every kernel of a window of MD steps under ncu --set full -> per-kernel roofline table
set -x
o=gpurun_out/r02; mkdir -p $o
python bench.py --steps 20 --warmup 5 > $o/bench_1gpu_steps20.json 2> $o/bench.err
python bench.py --steps 2000 --warmup 200 > $o/bench_1gpu_steps2000.json 2>> $o/bench.err
python bench.py --impl reference --steps 20 --warmup 5 > $o/bench_reference_steps20.json 2>> $o/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $o/launches_bench.csv python bench.py --steps 100 --warmup 20 > $o/bench_under_ncu.log 2>&1
python profiles/launch_table.py $o/launches_bench.csv 30 > $o/launch_table_bench.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_force_lj_pair -s 450 -c 1 \
    -o $o/force python profiles/profile_step.py --steps 500 > $o/prof_force.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_list_cells -s 12 -c 1 \
    -o $o/nlist python profiles/profile_step.py --steps 400 > $o/prof_nlist.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pair_fixup -s 12 -c 1 \
    -o $o/fixup python profiles/profile_step.py --steps 400 > $o/prof_fixup.log 2>&1
python profiles/ncu_summary.py $o/force.ncu-rep > $o/ncu_force_advance.txt 2>&1
python profiles/ncu_summary.py $o/nlist.ncu-rep > $o/ncu_list_pairs.txt 2>&1
python profiles/ncu_summary.py $o/fixup.ncu-rep > $o/ncu_pair_fixup.txt 2>&1
python profiles/source_lines.py $o/nlist.ncu-rep paper_2406_04210_b200/lib/obj/nlist.o k_list_cells_ballotILi8ELb1 60 \
    > $o/list_pairs_source_lines.txt 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -c 400 \
    -o $o/allkernels -f python profiles/profile_step.py --melt 330 --steps 70 \
    --profiler-range > $o/prof_allkernels.log 2>&1
python profiles/kernel_roofline.py $o/allkernels.ncu-rep > $o/kernel_roofline.txt 2>&1
# the all-pairs kernel of the paper's N = 2000 benchmark (warp-split shape, fixed-point min-image)
# and of a large system (one thread per particle), and the config table
ncu --set full --clock-control none --import-source on -k regex:k_force_all_pairs -s 20 -c 1 \
    -o $o/allpairs2k python profiles/exp/all_pairs_steps.py 2000 > $o/prof_allpairs2k.log 2>&1
python profiles/ncu_summary.py $o/allpairs2k.ncu-rep > $o/ncu_all_pairs_n2000.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_force_all_pairs -s 2 -c 1 \
    -o $o/allpairs131k python profiles/exp/all_pairs_roofline.py 131072 > $o/prof_allpairs131k.log 2>&1
python profiles/ncu_summary.py $o/allpairs131k.ncu-rep > $o/ncu_all_pairs_n131072.txt 2>&1
python profiles/run_configs.py --which 1,2,3,4,A,5 > $o/configs.jsonl 2> $o/configs.err
python profiles/exp/all_pairs_preset.py > $o/all_pairs_preset.jsonl 2>&1
python profiles/exp/all_pairs_steps.py 256 2000 4096 8000 > $o/all_pairs_steps.jsonl 2>&1
python profiles/exp/all_pairs_roofline.py 16384 32768 131072 > $o/all_pairs_roofline.jsonl 2>&1
# the reports themselves exceed what gpurun copies back (64 MiB): keep the summaries
rm -f $o/*.ncu-rep
tail -c 1500 $o/bench_1gpu_steps20.json; cat $o/kernel_roofline.txt | tail -40
