mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "col_major or guard or baseline" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/cm_sweep.py > gpurun_out/cm_sweep.jsonl 2>&1
timeout 300 python tools/b2b.py G2 > gpurun_out/tune22.jsonl 2>&1
