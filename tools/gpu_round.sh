mkdir -p gpurun_out
timeout 600 python tools/odd_shapes.py > gpurun_out/odd.jsonl 2>&1
