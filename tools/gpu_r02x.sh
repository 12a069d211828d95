#!/bin/bash
OUT=gpurun_out/r02x; mkdir -p $OUT; rm -f $OUT/sweep.txt
L=c2_interp,poly_interp_2p30,f32_log_interp_2p30,axpy_interp_2p30
for r in 1 2; do for v in ig4 ig8 ig16; do
  echo "== $v r$r" >> $OUT/sweep.txt; COOT_LIB_PATH=$PWD/paper_2508_11385_b200/libcoot_$v.so timeout 600 python tools/sweep.py --reps 10 --only $L 2>&1 | tail -n +2 >> $OUT/sweep.txt
done; done
COOT_LIB_PATH=$PWD/paper_2508_11385_b200/libcoot_ig8.so timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_transcendental.py -q -x -k f32 > $OUT/pytest8.log 2>&1; echo "pytest ig8 rc=$?"; tail -1 $OUT/pytest8.log
cat $OUT/sweep.txt
