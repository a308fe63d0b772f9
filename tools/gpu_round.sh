mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bounds.py -q -x -k "row_major or gemv_guard" --timeout 600 -p no:cacheprovider > gpurun_out/pytest_rm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_rm.log
python tools/rm_few.py > gpurun_out/rm_few_default.jsonl 2>&1
