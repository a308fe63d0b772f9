mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/ger_dot_sweep.py > gpurun_out/gd_sweep.jsonl 2>&1
timeout 600 python tools/odd_shapes.py > gpurun_out/odd.jsonl 2>&1
timeout 300 python tools/b2b.py R1 D2 > gpurun_out/tune22.jsonl 2>&1
