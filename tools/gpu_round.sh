mkdir -p gpurun_out
rm -f gpurun_out/rm_ragged.jsonl
export RM_NS=68,132,260,516,1028,2052,4100,8196,16388
timeout 900 python tools/rm_ragged.py | sed "s/^/h16 /" >> gpurun_out/rm_ragged.jsonl 2>&1
CABL_RM_H16=0 timeout 900 python tools/rm_ragged.py | sed "s/^/scalar /" >> gpurun_out/rm_ragged.jsonl 2>&1
