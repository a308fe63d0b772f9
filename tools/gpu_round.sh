#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ord3.jsonl
for cfg in "1024,3,1" "512,5,1" "1024,3,2" "tma"; do
  echo "cfg=$cfg" >> gpurun_out/ord3.jsonl
  CABL_TUNING=1 CABL_GEMV_RM_ORDER=reference CABL_ORD_CFG=$cfg timeout 300 python tools/b2b.py G1 G4 >> gpurun_out/ord3.jsonl 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "reference_order_mode" > gpurun_out/pytest_ord.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ord.log
