#!/bin/bash
OUT=gpurun_out/r02m; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_views.py tests/test_gpu_views_narrow.py -q -x > $OUT/pytest_views.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_views.log
timeout 600 python tools/sweep.py --reps 20 --only submat_axpy,dot_2p30,diag_add_1e4,axpy_accu_2p30 > $OUT/sweep.txt 2>&1; cat $OUT/sweep.txt
