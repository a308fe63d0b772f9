mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "fullcol" > gpurun_out/pytest_cm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cm.log
rm -f gpurun_out/cm_ab.jsonl
CABL_LIB=$PWD/tools/ab/libcabl_head.so timeout 600 python tools/cm_mid2.py --tag head >> gpurun_out/cm_ab.jsonl 2>&1
CABL_CM_FC_MODE=0 timeout 600 python tools/cm_mid2.py --tag mode0 >> gpurun_out/cm_ab.jsonl 2>&1
CABL_CM_FC_P=64 timeout 600 python tools/cm_mid2.py --tag p64 >> gpurun_out/cm_ab.jsonl 2>&1
CABL_CM_FC_P=128 timeout 600 python tools/cm_mid2.py --tag p128 >> gpurun_out/cm_ab.jsonl 2>&1
CABL_CM_FC_P=32 timeout 600 python tools/cm_mid2.py --tag p32 >> gpurun_out/cm_ab.jsonl 2>&1
CABL_CM_FC_P=296 timeout 600 python tools/cm_mid2.py --tag p296 >> gpurun_out/cm_ab.jsonl 2>&1
CABL_CM_FC_FENCE=1 timeout 600 python tools/cm_mid2.py --tag fence >> gpurun_out/cm_ab.jsonl 2>&1
