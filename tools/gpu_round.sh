mkdir -p gpurun_out
export CABL_GEMV_RM_ORDER=reference
CABL_ORD_CFG=tma timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "row_major_matches or 65536" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/tune22.jsonl
for cfg in tma 1024,3,1; do
  CABL_ORD_CFG=$cfg timeout 300 python tools/b2b.py G1 G4 | sed "s/^/$cfg /" >> gpurun_out/tune22.jsonl 2>&1
done
