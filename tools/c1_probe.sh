mkdir -p gpurun_out/c1
python tools/latency_parts.py > gpurun_out/c1/parts2.txt 2>&1
python tools/small_n.py > gpurun_out/c1/small_n2.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/c1/pytest.txt 2>&1; tail -3 gpurun_out/c1/pytest.txt
