mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "fullcol or col_major_matches" > gpurun_out/pytest_cm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cm.log
rm -f gpurun_out/cm_ab.jsonl
for i in 1 2; do
CABL_LIB=$PWD/tools/ab/libcabl_head.so timeout 600 python tools/cm_mid2.py --tag head >> gpurun_out/cm_ab.jsonl 2>&1
timeout 600 python tools/cm_mid2.py --tag batchtree >> gpurun_out/cm_ab.jsonl 2>&1
done
for i in 1 2 3; do timeout 300 python bench.py --steps 20 --warmup 5 --no-suite > gpurun_out/bench_k20_$i.json 2>gpurun_out/bench_k20_$i.err; done
