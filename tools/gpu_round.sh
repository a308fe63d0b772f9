mkdir -p gpurun_out
./tests/cpp/mgpu_example > gpurun_out/mgpu_example.log 2>&1; echo "rc=$?" >> gpurun_out/mgpu_example.log
