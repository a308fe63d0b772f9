mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -p no:cacheprovider -k "dot" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/tune.py D2 D1 > gpurun_out/tune13.jsonl 2>&1
CABL_DOT_CHUNKED=0 timeout 300 python tools/tune.py D2 >> gpurun_out/tune13.jsonl 2>&1
