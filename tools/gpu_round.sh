mkdir -p gpurun_out
LD_LIBRARY_PATH=paper_2108_02025_b200 ./tests/cpp/mgpu_example > gpurun_out/mgpu.log 2>&1; echo "rc=$?" >> gpurun_out/mgpu.log
