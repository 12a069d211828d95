OUT=gpurun_out/dim2; mkdir -p $OUT
W=bf16_dim1,e4m3_dim1,c3_dim1,f32_dim1,bf16_dim0,e4m3_dim0,c3_dim0
for b in 2 3 4 6; do COOT_DIM_BLOCKS_PER_SM=$b python tools/sweep.py --only $W > $OUT/b$b.txt 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -x -k "dim or sum" > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
