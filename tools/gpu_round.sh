mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cpp_dropin.py -m gpu -q --timeout 800 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
(cd tests/cpp && ./mgpu_example > ../../gpurun_out/mgpu.log 2>&1; echo "rc=$?" >> ../../gpurun_out/mgpu.log)
