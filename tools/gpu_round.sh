mkdir -p gpurun_out
timeout 900 python -m paper_2108_02025_b200.benchcli --kernel gemv-col --sizes 2048:16384:2 --dtype f32 --reps 5 --csv gpurun_out/sweep_cm32.csv > gpurun_out/sweep.log 2>&1; echo "rc=$?" >> gpurun_out/sweep.log
timeout 900 python -m paper_2108_02025_b200.benchcli --kernel gemv-col --sizes 2048:16384:2 --dtype f64 --reps 5 --csv gpurun_out/sweep_cm64.csv >> gpurun_out/sweep.log 2>&1; echo "rc=$?" >> gpurun_out/sweep.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -p no:cacheprovider -k "col_major" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
