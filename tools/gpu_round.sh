mkdir -p gpurun_out
timeout 300 python tools/b2b.py G2 > gpurun_out/tune22.jsonl 2>&1
