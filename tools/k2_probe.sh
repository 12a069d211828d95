OUT=gpurun_out/pdl3; mkdir -p $OUT
W=var_2p30,imin_2p30,mean_2p30,norm2_2p30,accu_2p30,c2_eval_accu,c2_reduce,dot_2p30,c3_dim1,c4_u32,axpy_accu_2p30
COOT_PDL=0 python tools/sweep.py --only $W > $OUT/nopdl.txt 2>&1
COOT_PDL=1 python tools/sweep.py --only $W > $OUT/pdl.txt 2>&1
python tools/latency_parts.py > $OUT/parts.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
