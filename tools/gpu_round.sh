mkdir -p gpurun_out
export CABL_GEMV_RM_ORDER=reference
rm -f gpurun_out/tune22.jsonl
for cfg in 1024,3,1 1024,2,1; do
  CABL_ORD_CFG=$cfg timeout 300 python tools/b2b.py G1 G4 | sed "s/^/$cfg /" >> gpurun_out/tune22.jsonl 2>&1
done
