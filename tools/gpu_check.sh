#!/bin/bash
# One gpurun call: smoke, GPU tests, bench, ncu launch list + full capture.
# usage (from the repo root on the GPU box): bash tools/gpu_check.sh TAG [skip-tests]
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/nvidia_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
tail -1 $OUT/smoke.log
if [ "${2:-}" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -3 $OUT/pytest_gpu.log
fi
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
head -c 4000 $OUT/bench.json; echo
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $OUT/launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_tma_kernel -s 1 -c 1 \
   -o $OUT/c2_full python tools/profile_step.py c2 3 > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -1 $OUT/ncu_full.log
