mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_bounds.py -m gpu -q -p no:cacheprovider -x --timeout 120 -k "col_major or fullcol or host or concurrent or fuzz or cm" > gpurun_out/pytest_cm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cm.log
rm -f gpurun_out/cm_ab.jsonl
CABL_LIB=$PWD/tools/ab/libcabl_head.so timeout 300 python tools/cm_mid2.py --tag round_start >> gpurun_out/cm_ab.jsonl 2>&1
timeout 300 python tools/cm_mid2.py --tag product >> gpurun_out/cm_ab.jsonl 2>&1
python tools/ncu_runner.py --cm 16384x4096 --reps 2 > gpurun_out/plain_cm.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_cm -s 2 -c 2 -o gpurun_out/prof_cm16384_product -f python tools/ncu_runner.py --cm 16384x4096 --reps 2 > gpurun_out/ncu_cm.log 2>&1
