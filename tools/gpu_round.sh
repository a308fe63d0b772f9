mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "col_major or guard or modes or baseline or smoke" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
CM_MS=150000,200000,260000 timeout 900 python tools/cm_awk.py > gpurun_out/cm_awk.jsonl 2>&1
timeout 300 python tools/b2b.py G2 > gpurun_out/tune22.jsonl 2>&1
