mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -m gpu -q -x -p no:cacheprovider -k "dot" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/tune22.jsonl
for cfg in 512,2,2 512,4,2 256,4,4 1024,4,1 256,8,1 256,2,8 1024,2,1; do
  CABL_DOT_CFG=$cfg timeout 300 python tools/b2b.py D1 | sed "s/^/$cfg /" >> gpurun_out/tune22.jsonl 2>&1
done
