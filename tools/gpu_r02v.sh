#!/bin/bash
OUT=gpurun_out/r02v; mkdir -p $OUT; rm -f $OUT/sweep.txt
X=$PWD/paper_2508_11385_b200/libcoot_x2.so
COOT_LIB_PATH=$X timeout 1200 python -m pytest tests/test_gpu_fused.py tests/test_gpu_fp8.py tests/test_gpu_configs.py -q -x -k "f32 or e4m3 or e5m2 or c2 or headline or c1" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
L=c2_eval_accu,c2_reduce,c2_interp,axpy_accu_2p30,poly_interp_2p30,e4m3_c2_2p32,e4m3_c2_eval_2p31,e5m2_axpy_eval_2p31,hl_c2_2p30
for r in 1 2; do
  echo "== main r$r" >> $OUT/sweep.txt; timeout 600 python tools/sweep.py --reps 10 --only $L 2>&1 | tail -n +2 >> $OUT/sweep.txt
  echo "== x2 r$r" >> $OUT/sweep.txt; COOT_LIB_PATH=$X timeout 600 python tools/sweep.py --reps 10 --only $L 2>&1 | tail -n +2 >> $OUT/sweep.txt
done
cat $OUT/sweep.txt
