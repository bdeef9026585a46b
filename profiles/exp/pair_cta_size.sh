# CTA size of k_force_lj_pair (B2MD_PAIR_THREADS, 1024 threads per SM): rebuilds the library on the
# GPU box per variant, prints variant, ms per step, ms per one-launch step kernel.
for t in ${SIZES:-256 512 1024 64 128}; do
  B2MD_NVCC_EXTRA=-DB2MD_PAIR_THREADS=$t python -m paper_2406_04210_b200.build > /dev/null 2>&1
  python bench.py --steps 1000 --warmup 100 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('threads $t', round(d['ms_per_step'],5), round(d['roofline']['launch_ms'],5), round(d['roofline']['other_kernels']['k_force_lj_pair (force only: first / last step of a call)']['launch_ms'],5))"
done
