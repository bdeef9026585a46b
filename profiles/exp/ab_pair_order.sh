#!/bin/bash
# A/B of the lane order of the pair kernel (B2MD_PAIR_SCHEDULE bits: 1 block schedule, 2 lane
# order, 4 face key, unit << 8) on the molten N = 1 M fluid: ms per step over 2000 steps.
out=gpurun_out/ab_pair_order.txt
: > $out
for round in 1 2; do
  for mode in ${MODES:-1 3 7 515 519}; do
    echo -n "mode=$mode " >> $out
    B2MD_PAIR_SCHEDULE=$mode python profiles/profile_step.py --melt 600 --steps 2000 2>&1 | tail -1 >> $out
  done
done
cat $out
