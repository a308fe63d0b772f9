mkdir -p gpurun_out
timeout 1200 python tools/shape_sweep.py > gpurun_out/shape_sweep.md 2> gpurun_out/shape_sweep.err
timeout 600 python tools/odd_shapes.py > gpurun_out/odd.jsonl 2>&1
