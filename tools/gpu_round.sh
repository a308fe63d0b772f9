#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ord2.jsonl
for cfg in "1024,3,1" "2048,3,1,1w" "2048,3,2,1w"; do
  echo "cfg=$cfg" >> gpurun_out/ord2.jsonl
  CABL_TUNING=1 CABL_GEMV_RM_ORDER=reference CABL_ORD_CFG=$cfg timeout 300 python tools/b2b.py G1 G4 >> gpurun_out/ord2.jsonl 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "reference_order_mode" > gpurun_out/pytest_ord.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ord.log
