OUT=gpurun_out/fhab; mkdir -p $OUT
W=bf16_dim1,e4m3_dim1,bf16_dim0,e4m3_dim0,bf16_dot_2p31,e4m3_dot_2p32
L=$(ls $PWD/paper_2508_11385_b200/libcoot*.so | head -1); N=$(basename $L .so)
for r in 1 2; do COOT_LIB_PATH=$L python tools/sweep.py --only $W > $OUT/${N}_$r.txt 2>&1; done
