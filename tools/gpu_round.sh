#!/bin/bash
mkdir -p gpurun_out
( time timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err ) 2> gpurun_out/bench_time.txt
( time timeout 2400 python -m pytest tests -m gpu -q --durations=25 -p no:cacheprovider > gpurun_out/pytest_durations.log 2>&1 ) 2> gpurun_out/pytest_time.txt
