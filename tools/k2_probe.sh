OUT=gpurun_out/d2; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "dim or fp8 or half or narrow" > $OUT/pytest.txt 2>&1; tail -2 $OUT/pytest.txt
python tools/sweep.py > $OUT/sweep.txt 2>&1
