mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "row_major or guard or modes" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
RM_NS=16,64,65,128,256,1024,1025,2048 timeout 900 python tools/rm_ragged.py > gpurun_out/rm_ragged.jsonl 2>&1
timeout 300 python tools/b2b.py G1 > gpurun_out/tune22.jsonl 2>&1
