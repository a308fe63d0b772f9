#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "col_major or fuzz or cm or modes or bounds" > gpurun_out/pytest_cm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cm.log
timeout 600 python tools/cm_mid2.py --tag fullcol > gpurun_out/cm_mid4.jsonl 2>gpurun_out/cm_mid4.err
CABL_CM_FULLCOL=0 timeout 600 python tools/cm_mid2.py --tag split >> gpurun_out/cm_mid4.jsonl 2>>gpurun_out/cm_mid4.err
