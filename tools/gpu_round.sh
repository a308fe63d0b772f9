mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bounds.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
