mkdir -p gpurun_out machines
python -m paper_2108_02025_b200.benchcli --describe --dtype f32 > gpurun_out/b200.json 2> gpurun_out/describe.err; echo "describe rc=$?"
cp gpurun_out/b200.json machines/b200.json
timeout 600 python -m pytest tests/test_machine.py tests/test_smoke.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
LD_LIBRARY_PATH=paper_2108_02025_b200 ./tests/cpp/device_example > gpurun_out/devex.log 2>&1; echo "devex rc=$?" >> gpurun_out/devex.log
timeout 600 python bench.py --steps 200 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
