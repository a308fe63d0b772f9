mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_modes.py -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_modes.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_modes.log
timeout 900 python bench.py --no-suite > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
