mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize_driver.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/san_plain.log
timeout 900 $CS --tool memcheck --leak-check no python tools/sanitize_driver.py > gpurun_out/san_mem.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_mem.log
CABL_GEMV_RM_ORDER=reference timeout 900 $CS --tool memcheck python tools/sanitize_driver.py > gpurun_out/san_mem_ord.log 2>&1; echo "memcheck ord rc=$?" >> gpurun_out/san_mem_ord.log
CABL_GEMV_RM_ORDER=reference CABL_ORD_CFG=tma timeout 900 $CS --tool memcheck python tools/sanitize_driver.py > gpurun_out/san_mem_tma.log 2>&1; echo "memcheck tma rc=$?" >> gpurun_out/san_mem_tma.log
CABL_GEMV_RM_ORDER=reference timeout 900 $CS --tool racecheck python tools/sanitize_driver.py > gpurun_out/san_race_ord.log 2>&1; echo "racecheck ord rc=$?" >> gpurun_out/san_race_ord.log
