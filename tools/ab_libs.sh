#!/bin/bash
# Interleaved A/B of side-by-side library builds (libcoot_<v>.so) on the TMA
# tuner's workloads (c2 eval+accu / reduce, axpy, dot, accu), default geometry.
# usage: bash tools/ab_libs.sh OUTDIR ROUNDS v1 v2 ...   ("main" = libcoot.so)
OUT=gpurun_out/$1; ROUNDS=$2; shift 2
mkdir -p $OUT
for r in $(seq $ROUNDS); do
  for v in "$@"; do
    lib=$PWD/paper_2508_11385_b200/libcoot_$v.so; [ "$v" = main ] && lib=$PWD/paper_2508_11385_b200/libcoot.so
    echo -n "$v r$r " >> $OUT/ab.txt
    COOT_LIB_PATH=$lib TUNE_ROUNDS=1 timeout 300 python tools/tma_tune.py ${GEOM:-0,0,2} 2>&1 | tail -1 >> $OUT/ab.txt
  done
done
cat $OUT/ab.txt
