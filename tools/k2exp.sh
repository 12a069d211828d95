# A/B of experimental f32 dev builds (libcoot_<v>.so): tools/sweep.py per variant
# usage: bash tools/k2exp.sh OUTDIR variant[:ENV=VAL] ...
OUT=gpurun_out/$1
mkdir -p $OUT
shift
for spec in "$@"; do
  v=${spec%%:*}; envs=""; [ "$spec" != "$v" ] && envs=${spec#*:}
  echo "== $spec" >> $OUT/sweep.txt
  env $envs COOT_LIB_PATH=$PWD/paper_2508_11385_b200/libcoot_$v.so timeout 300 python tools/sweep.py --reps 10 --only ${ONLY:-c2_eval_accu,c2_reduce,hl_c2_2p30,c2_interp,axpy_interp_2p30,poly_interp_2p30,f32_log_interp_2p30} 2>&1 | tail -n +2 >> $OUT/sweep.txt
done
cat $OUT/sweep.txt
