mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 800 -p no:cacheprovider -k "row_major or 65536" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/tune22.jsonl
timeout 300 python tools/b2b.py G1 G4 >> gpurun_out/tune22.jsonl 2>&1
CABL_GEMV_RM_ORDER=reference timeout 300 python tools/b2b.py G1 G4 | sed "s/^/ref /" >> gpurun_out/tune22.jsonl 2>&1
