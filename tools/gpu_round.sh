mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "dot or determin" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2; do
python tools/tune.py D1 > gpurun_out/tune8.jsonl 2>&1
CABL_DOT_FINISH=0 python tools/tune.py D1 >> gpurun_out/tune8.jsonl 2>&1
CABL_DOT_CFG=512,2,2 python tools/tune.py D1 >> gpurun_out/tune8.jsonl 2>&1
CABL_DOT_CFG=512,2,2 CABL_DOT_FINISH=0 python tools/tune.py D1 >> gpurun_out/tune8.jsonl 2>&1
done
