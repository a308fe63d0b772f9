mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bounds.py -q -x -k "row_major or gemv_guard" --timeout 600 -p no:cacheprovider > gpurun_out/pytest_rm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_rm.log
CABL_RM_REALIGN=0 python tools/rm_realign.py > gpurun_out/rm_realign_before.jsonl 2>&1
for c in 4,2,2 2,4,2 2,8,1 8,1,2 4,4,1 2,2,3; do CABL_RM_REALIGN_CFG=$c python tools/rm_realign.py > gpurun_out/rm_realign_c$c.jsonl 2>&1; done
