mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x --timeout 120 -k "fullcol or col_major_matches" > gpurun_out/pytest_cm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cm.log
rm -f gpurun_out/cm_ab.jsonl
for i in 1 2; do
CABL_LIB=$PWD/tools/ab/libcabl_head.so timeout 300 python tools/cm_mid2.py --tag head >> gpurun_out/cm_ab.jsonl 2>&1
timeout 300 python tools/cm_mid2.py --tag stream2 >> gpurun_out/cm_ab.jsonl 2>&1
CABL_TUNING=1 CABL_CM_FULLCOL2=1 timeout 300 python tools/cm_mid2.py --tag fc2stream2 >> gpurun_out/cm_ab.jsonl 2>&1
done
