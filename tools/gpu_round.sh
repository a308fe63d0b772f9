mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bounds.py tests/test_gpu_modes.py -m gpu -q -p no:cacheprovider -k "row_major or guard or modes" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/cm_sweep.py > gpurun_out/cm_sweep.jsonl 2>&1
