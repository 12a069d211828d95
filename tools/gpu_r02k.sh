#!/bin/bash
# exchange tests (sequential emulation, records + sum(X,1) vectors), comm, dist; bench N=2 shared dry run
OUT=gpurun_out/r02k; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_comm.py tests/test_gpu_dist.py tests/test_gpu_dim.py -q -x > $OUT/pytest_x.log 2>&1; echo "pytest rc=$?"; tail -15 $OUT/pytest_x.log
COOT_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 50 --warmup 5 --no-other-configs > $OUT/bench_dry2.json 2> $OUT/bench_dry2.err; echo "dry2 rc=$?"; head -c 400 $OUT/bench_dry2.json; echo; tail -5 $OUT/bench_dry2.err
