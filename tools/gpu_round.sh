mkdir -p gpurun_out
for u in 2,2 2,4 4,2; do CABL_RM_UNIT=$u python tools/rm_few.py > gpurun_out/rm_unit_$u.jsonl 2>&1; done
