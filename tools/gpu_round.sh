#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/ncu_runner.py --config CM4096 --reps 2 > gpurun_out/plain_CM4096.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_cm_fullcol -s 2 -c 2 -o gpurun_out/prof_CM4096 -f python tools/ncu_runner.py --config CM4096 --reps 2 > gpurun_out/ncu_CM4096.log 2>&1
python tools/shape_sweep.py > gpurun_out/shape_sweep.md 2> gpurun_out/shape_sweep.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
