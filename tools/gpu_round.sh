mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/tune18.jsonl
python tools/b2b.py G1 D1 R1 G2 G3 >> gpurun_out/tune18.jsonl 2>&1
CABL_PDL=0 python tools/b2b.py G1 D1 R1 G2 G3 | sed "s/^/nopdl /" >> gpurun_out/tune18.jsonl 2>&1
