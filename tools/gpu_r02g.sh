#!/bin/bash
# low-precision dev build (packed 16-bit pairs without repacking; fp8 c2 fast EXP): tests + A/B sweep
OUT=gpurun_out/r02g; mkdir -p $OUT
LP=$PWD/paper_2508_11385_b200/libcoot_lp.so
COOT_LIB_PATH=$LP timeout 1200 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_half.py tests/test_gpu_views_narrow.py -q -x > $OUT/pytest_lp.log 2>&1; echo "pytest lp rc=$?"; tail -3 $OUT/pytest_lp.log
L=e4m3_c2_2p32,e4m3_c2_eval_2p31,bf16_c2_2p31,f16_c2_2p31
for r in 1; do
  echo "== main r$r" >> $OUT/sweep.txt; timeout 600 python tools/sweep.py --reps 10 --only $L 2>&1 | tail -n +2 >> $OUT/sweep.txt
  echo "== lp r$r" >> $OUT/sweep.txt; COOT_LIB_PATH=$LP timeout 600 python tools/sweep.py --reps 10 --only $L 2>&1 | tail -n +2 >> $OUT/sweep.txt
done
cat $OUT/sweep.txt
