# Compile-time variants of the pair kernel (same arithmetic, different code shape): ptxas'
# register assignment inside the 64-register loop decides +-5 % (profiles/README.md).
#   gpurun --timeout 4000 -- 'bash profiles/exp/lottery.sh'      -> gpurun_out/lottery.txt
out=gpurun_out/lottery.txt; : > $out
for m in ${LOTTERY_MIN_BLOCKS:-8}; do for o in 0 1 2 3; do for t in 0 1; do for h in 0 1; do for f in 0 1; do
  v="-DB2MD_PAIR_OUTLINE=$o -DB2MD_PAIR_TILE_ROTATE=$t -DB2MD_PAIR_HALF_TILE=$h -DB2MD_PAIR_MIN_BLOCKS=$m -DB2MD_PAIR_INTERIOR_FACE=$f"
  B2MD_NVCC_EXTRA="$v" python -c "from paper_2406_04210_b200 import build as b; b.build_library(force=True)" > /dev/null 2>&1 || echo "build failed: $v" >> $out
  echo "variant [$v] $(timeout 120 python profiles/exp/step_timing.py 600 2>&1 | tail -1 | cut -c1-330)" >> $out
done; done; done; done; done
