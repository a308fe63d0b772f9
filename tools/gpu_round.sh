mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bounds.py -m gpu -q -x -p no:cacheprovider -k "ger" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/tune22.jsonl
for pf in 0 1 0 1; do
  CABL_PDL_PREFETCH=$pf timeout 300 python tools/b2b.py R1 | sed "s/^/pf$pf /" >> gpurun_out/tune22.jsonl 2>&1
done
