# A/B of compile-time variants on the GPU box: each argument is one set of nvcc -D flags
# ("base" = none); force.cu is rebuilt there per variant, then step_timing.py runs.
#   gpurun -- 'bash profiles/exp/variant_ab.sh base "-DB2MD_PAIR_OUTLINE=2"'
for v in "$@"; do
  if [ "$v" = "base" ]; then extra=""; else extra="$v"; fi
  B2MD_NVCC_EXTRA="$extra" python -c "from paper_2406_04210_b200 import build as b; b.build_library(force=True)" > /dev/null 2>&1 || echo "build failed: $v"
  echo "variant [$v] $(timeout 120 python profiles/exp/step_timing.py ${STEPS:-400} 2>&1 | tail -1)"
done
B2MD_NVCC_EXTRA="" python -c "from paper_2406_04210_b200 import build as b; b.build_library(force=True)" > /dev/null 2>&1
