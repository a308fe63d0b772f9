mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/tune.py G1 G2 G4 R1 > gpurun_out/tune10.jsonl 2>&1
CABL_GEMV_DYN=0 python tools/tune.py G1 G2 G4 >> gpurun_out/tune10.jsonl 2>&1
