mkdir -p gpurun_out
python tools/rm_mid.py > gpurun_out/rm_mid_new.jsonl 2>&1
CABL_RM_FEW_GROUPS=0 python tools/rm_mid.py > gpurun_out/rm_mid_old.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/b2b.py G1 G4 > gpurun_out/b2b_g.jsonl 2>&1
