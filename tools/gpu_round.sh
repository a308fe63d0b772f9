mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cpp_dropin.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
LD_LIBRARY_PATH=paper_2108_02025_b200 ./tests/cpp/mgpu_example > gpurun_out/mgpu.log 2>&1; echo "rc=$?" >> gpurun_out/mgpu.log
