mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "col_major or guard or modes" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/cm_awk.py > gpurun_out/cm_awk.jsonl 2>&1
timeout 900 python tools/cm_mid.py > gpurun_out/cm_mid.jsonl 2>&1
timeout 600 python tools/odd_shapes.py > gpurun_out/odd.jsonl 2>&1
