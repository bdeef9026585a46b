# compute-sanitizer over the hot path (SURVEY.md section 5 "race detection"):
#   gpurun --timeout 3000 -- 'bash profiles/sanitize.sh'
# Summaries land in gpurun_out/sanitize_*.txt (copied to profiles/r02/ by hand).
out=gpurun_out
mkdir -p $out
for tool in memcheck racecheck initcheck synccheck; do
  extra=""
  SAN_STEPS=${SAN_STEPS:-120} timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 \
      --log-file $out/sanitize_${tool}_workload.log python profiles/sanitize_workload.py \
      > $out/sanitize_${tool}_workload.out 2>&1
  echo "== $tool workload: exit $? ==" > $out/sanitize_${tool}.txt
  tail -3 $out/sanitize_${tool}_workload.out >> $out/sanitize_${tool}.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Uninitialized|hazard|Race reported" $out/sanitize_${tool}_workload.log | sort | uniq -c | sort -rn | head -40 >> $out/sanitize_${tool}.txt
  grep -E "at b2md|at .*k_[a-z_]+" $out/sanitize_${tool}_workload.log | sed 's/ *=* *//' | sort | uniq -c | sort -rn | head -30 >> $out/sanitize_${tool}.txt
done
# CUDA-graph steps (conditional IF nodes; off by default in the product) on their own
for tool in memcheck synccheck; do
  SAN_GRAPH=1 SAN_STEPS=60 timeout 900 compute-sanitizer --tool $tool --print-limit 10 \
      --log-file $out/sanitize_${tool}_graph.log python profiles/sanitize_workload.py \
      > $out/sanitize_${tool}_graph.out 2>&1
  echo "== $tool, CUDA-graph steps: exit $? ==" > $out/sanitize_${tool}_graph.txt
  tail -2 $out/sanitize_${tool}_graph.out >> $out/sanitize_${tool}_graph.txt
  grep -E "ERROR SUMMARY|Invalid|Barrier error" $out/sanitize_${tool}_graph.log | sort | uniq -c | sort -rn | head -10 >> $out/sanitize_${tool}_graph.txt
  grep -E "at b2md" $out/sanitize_${tool}_graph.log | sed 's/ *=* *//' | sort | uniq -c | sort -rn | head -10 >> $out/sanitize_${tool}_graph.txt
done
# the 2-rank slab path (two processes on one GPU, gloo control plane, peer stores through CUDA IPC)
timeout 1200 compute-sanitizer --tool memcheck --target-processes all --print-limit 30 \
    --log-file $out/sanitize_memcheck_slab.%p.log \
    python -m pytest tests/test_gpu_slab.py -q -x -k "halo_stored_by_the_step_kernel" > $out/sanitize_memcheck_slab.out 2>&1
echo "== memcheck slab (2 ranks): exit $? ==" > $out/sanitize_memcheck_slab.txt
tail -3 $out/sanitize_memcheck_slab.out >> $out/sanitize_memcheck_slab.txt
cat $out/sanitize_memcheck_slab.*.log 2>/dev/null | grep -E "ERROR SUMMARY|Invalid" | sort | uniq -c | sort -rn | head -20 >> $out/sanitize_memcheck_slab.txt
cat $out/sanitize_*.txt
