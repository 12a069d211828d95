#!/bin/bash
# round-2 check: GPU tests (incl. full-size parity), bench, N=2 dry run, r1-vs-now A/B, ncu of narrow-type c2 and K2
set -u
OUT=gpurun_out/r02f; mkdir -p $OUT
nproc > $OUT/host.txt; free -g >> $OUT/host.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
for r in 1 2; do
  (cd _ab/r1 && COOT_LIB_PATH=$PWD/paper_2508_11385_b200/libcoot.so TUNE_ROUNDS=1 timeout 300 python tools/tma_tune.py 0,0,2 2>&1 | tail -1 | sed 's/^/r1  /') >> $OUT/ab.txt
  TUNE_ROUNDS=1 timeout 300 python tools/tma_tune.py 0,0,2 2>&1 | tail -1 | sed 's/^/now /' >> $OUT/ab.txt
done
cat $OUT/ab.txt
COOT_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 50 --warmup 5 --no-other-configs > $OUT/bench_dry2.json 2> $OUT/bench_dry2.err; echo "dry2 rc=$?"; head -c 600 $OUT/bench_dry2.json; echo
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 $OUT/pytest_gpu.log
SKIP_SANITIZE=1 bash tools/profile_all.sh r02f c2ro_bf16 c2ro_e4m3 c2i
