mkdir -p gpurun_out
export CABL_GEMV_RM_ORDER=reference
rm -f gpurun_out/tune22.jsonl
for cfg in 1024,3,1 1024,3,2 1024,3,4 512,5,2; do
  CABL_ORD_CFG=$cfg timeout 300 python tools/b2b.py G1 G4 | sed "s/^/$cfg /" >> gpurun_out/tune22.jsonl 2>&1
done
CABL_ORD_CFG=1024,3,2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "row_major_matches" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
