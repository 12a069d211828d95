#!/bin/bash
OUT=gpurun_out/r02y; mkdir -p $OUT; rm -f $OUT/sweep.txt
LP=$PWD/paper_2508_11385_b200/libcoot_lp.so
COOT_LIB_PATH=$LP timeout 1200 python -m pytest tests/test_gpu_half.py tests/test_gpu_fp8.py tests/test_gpu_stats.py tests/test_gpu_range.py tests/test_gpu_views_narrow.py -q -k "bf16 or f16 or e4m3 or e5m2" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
L=bf16_var_2p31,f16_var_2p31,e4m3_var_2p32
for r in 1 2; do
  echo "== main r$r" >> $OUT/sweep.txt; timeout 600 python tools/sweep.py --reps 10 --only $L 2>&1 | tail -n +2 >> $OUT/sweep.txt
  echo "== lp r$r" >> $OUT/sweep.txt; COOT_LIB_PATH=$LP timeout 600 python tools/sweep.py --reps 10 --only $L 2>&1 | tail -n +2 >> $OUT/sweep.txt
done
cat $OUT/sweep.txt
