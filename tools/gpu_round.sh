mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "row_major or guard or modes" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/rm_ragged.jsonl
timeout 900 python tools/rm_ragged.py > gpurun_out/rm_ragged.jsonl 2>&1
RM_NS=16384,32768,32776,50000,65536,65544 timeout 900 python tools/rm_ragged.py >> gpurun_out/rm_ragged.jsonl 2>&1
timeout 300 python tools/b2b.py G1 G4 > gpurun_out/tune22.jsonl 2>&1
