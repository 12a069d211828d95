#!/bin/bash
# ncu --set full captures of the top kernel of every BASELINE workload, plus
# compute-sanitizer runs.  Reports are exported to CSV on the box (raw + source
# pages) and the .ncu-rep files dropped to stay under gpurun's 64 MiB limit.
# usage (GPU box, repo root): bash tools/profile_all.sh TAG [workloads...]
set -u
TAG=${1:-r01}
shift || true
WL=${@:-c2ro axpy c3d0 c3d1 c4u c4s dot norm2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for w in $WL; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'fused|dim' -s 1 -c 1 \
     -o /tmp/prof_$w python tools/profile_step.py $w 2 > $OUT/ncu_$w.log 2>&1
  echo "ncu $w rc=$?"
  ncu -i /tmp/prof_$w.ncu-rep --page raw --csv > $OUT/raw_$w.csv 2>/dev/null
  ncu -i /tmp/prof_$w.ncu-rep --page source --csv --print-source sass > $OUT/src_$w.csv 2>/dev/null
  gzip -f $OUT/src_$w.csv
  rm -f /tmp/prof_$w.ncu-rep
done
if [ -z "${SKIP_SANITIZE:-}" ]; then
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_driver.py > $OUT/sanitize_$tool.log 2>&1
  echo "sanitizer $tool rc=$? $(grep -E 'SUMMARY|sanitize driver ok' $OUT/sanitize_$tool.log | tr '\n' ' ')"
done
fi
du -sh $OUT
