mkdir -p gpurun_out
python tools/sanitize_driver.py > gpurun_out/san_plain.log 2>&1; echo "rc=$?" >> gpurun_out/san_plain.log
CABL_GEMV_RM_ORDER=reference python tools/sanitize_driver.py >> gpurun_out/san_plain.log 2>&1; echo "rc=$?" >> gpurun_out/san_plain.log
