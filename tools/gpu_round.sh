mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_capi.py -m "gpu or not gpu" -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
