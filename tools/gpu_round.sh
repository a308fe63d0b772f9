mkdir -p gpurun_out
rm -f gpurun_out/tune12.jsonl
for cfg in 6,32 12,16 4,48 3,64 24,8; do
CABL_BULK=$cfg timeout 120 python tools/tune.py G3 >> gpurun_out/tune12.jsonl 2>&1
done
CABL_BULK=12,16 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 100 -p no:cacheprovider -k "col_major" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
