mkdir -p gpurun_out
timeout 600 python tools/e2e_depth.py > gpurun_out/e2e_depth.jsonl 2>&1
timeout 600 python tools/e2e_depth.py --distinct >> gpurun_out/e2e_depth.jsonl 2>&1
