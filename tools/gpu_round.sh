mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bounds.py -q -x -k "col_major or gemv_guard" --timeout 600 -p no:cacheprovider > gpurun_out/pytest_cm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cm.log
python tools/cm_realign.py > gpurun_out/cm_realign_after.jsonl 2>&1
