OUT=gpurun_out/hint3; mkdir -p $OUT
W=c2_eval_accu,c2_reduce,c2_interp,poly_interp_2p30,bf16_c2_2p31,f16_c2_2p31,e4m3_c2_2p32,bf16_interp_c2,accu_2p30,dot_2p30,var_2p30,bf16_var_2p31,submat_axpy,e5m2_axpy_eval_2p31,hl_c2_2p30,axpy_accu_2p30
for r in 1 2; do
COOT_PRODUCER_SLEEP=0 python tools/sweep.py --only $W > $OUT/poll$r.txt 2>&1
python tools/sweep.py --only $W > $OUT/policy$r.txt 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
