mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bounds.py -q -x -k "ger" --timeout 600 -p no:cacheprovider > gpurun_out/pytest_ger.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ger.log
for c in 1,8,0,2 0,8,0,2 1,4,1,2 0,4,1,2 1,4,0,2 0,4,0,2 1,4,1,4 0,4,1,4 1,8,0,3; do CABL_GER_ANY_CFG=$c python tools/ger_odd.py > gpurun_out/ger_odd_c$c.jsonl 2>&1; done
