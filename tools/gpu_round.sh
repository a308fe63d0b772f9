#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/cmlab.py > gpurun_out/cmlab2.jsonl 2> gpurun_out/cmlab2.err
python tools/ncu_runner.py --config D1 --reps 20 > gpurun_out/plain_D1s.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.max,dram__bytes_read.sum --clock-control none -k regex:dot_kernel --csv --log-file gpurun_out/ncu_D1_series.csv python tools/ncu_runner.py --config D1 --reps 20 > gpurun_out/ncu_D1s.log 2>&1
