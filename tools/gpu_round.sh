mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bounds.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -x --timeout 120 -k "col_major or cm or fuzz" > gpurun_out/pytest_cm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cm.log
rm -f gpurun_out/ab.jsonl
timeout 300 python tools/ab_shapes.py --tag product --op gemv-col --n 6500,8193,14001,16383 --dtypes f32 >> gpurun_out/ab.jsonl 2>&1
