OUT=gpurun_out/k2c; mkdir -p $OUT
W=c2_interp,axpy_interp_2p30,poly_interp_2p30,f64_c2_interp_2p29,bf16_interp_c2
L=$(ls $PWD/paper_2508_11385_b200/libcoot_*.so | head -1); N=$(basename $L .so)
COOT_LIB_PATH=$L COOT_TMA_CTAS=3 python tools/sweep.py --only $W > $OUT/${N}_c3.txt 2>&1
COOT_LIB_PATH=$L python tools/sweep.py --only $W > $OUT/${N}_c2.txt 2>&1
