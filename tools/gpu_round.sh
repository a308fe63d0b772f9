#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_benchcli.py -m gpu -q > gpurun_out/pytest_fix.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fix.log
timeout 600 python tools/e2e_depth.py > gpurun_out/e2e_depth.jsonl 2>&1
timeout 600 python tools/e2e_depth.py --distinct >> gpurun_out/e2e_depth.jsonl 2>&1
timeout 300 python tools/host_paths.py > gpurun_out/host_paths.jsonl 2>&1
python bench.py --gpus 2 --steps 3 > gpurun_out/gpus2.out 2> gpurun_out/gpus2.err; echo "rc=$?" >> gpurun_out/gpus2.err
