mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 250 -p no:cacheprovider -k "col_major" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/tune21.jsonl
for k in 2 4 6 12; do CABL_CM_CHUNKS_PER_CTA=$k timeout 200 python tools/b2b.py G3 | sed "s/^/per_cta=$k /" >> gpurun_out/tune21.jsonl 2>&1; done
CABL_CM_SPLIT=1 timeout 200 python tools/b2b.py G3 | sed "s/^/static /" >> gpurun_out/tune21.jsonl 2>&1
