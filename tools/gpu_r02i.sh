#!/bin/bash
OUT=gpurun_out/r02i; mkdir -p $OUT
IB=$PWD/paper_2508_11385_b200/libcoot_ib.so
COOT_LIB_PATH=$IB timeout 1200 python -m pytest tests/test_gpu_fused.py -q -x -k "f32" > $OUT/pytest_ib.log 2>&1; echo "pytest ib rc=$?"; tail -2 $OUT/pytest_ib.log
L=c2_interp,axpy_interp_2p30,poly_interp_2p30,f32_log_interp_2p30,c2_eval_accu
for r in 1 2; do
  echo "== main r$r" >> $OUT/sweep.txt; timeout 600 python tools/sweep.py --reps 20 --only $L 2>&1 | tail -n +2 >> $OUT/sweep.txt
  echo "== ib r$r" >> $OUT/sweep.txt; COOT_LIB_PATH=$IB timeout 600 python tools/sweep.py --reps 20 --only $L 2>&1 | tail -n +2 >> $OUT/sweep.txt
done
cat $OUT/sweep.txt
