#!/bin/bash
OUT=gpurun_out/r02o; mkdir -p $OUT; rm -f $OUT/dim2.txt
for r in 1 2; do
for cfg in "64 2" "48 2" "32 2" "80 2" "48 3" "32 3" "32 4"; do
  set -- $cfg
  echo -n "ring $1 KB, $2 CTA/SM: " >> $OUT/dim2.txt
  COOT_DIM_RING_KB=$1 COOT_TMA_CTAS=$2 timeout 300 python tools/sweep.py --reps 20 --only f32_dim1 2>&1 | tail -n +2 >> $OUT/dim2.txt
done
done
cat $OUT/dim2.txt
