mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py tests/test_benchcli.py -m gpu -q --timeout 600 -p no:cacheprovider -k "col_major or modes or cli" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/tune.py G2 G3 > gpurun_out/tune15.jsonl 2>&1
timeout 600 python -m paper_2108_02025_b200.benchcli --kernel gemv-col --sizes 1024:16384:2 --rect 65536x1024,1024x65536 --dtype f64 --reps 5 --csv gpurun_out/sweep_cm.csv > gpurun_out/sweep.log 2>&1; echo "rc=$?" >> gpurun_out/sweep.log
