mkdir -p gpurun_out
for f in 0 1; do CABL_GATHER_FENCE=$f python tools/peer_cost.py 2>&1 | grep gemv > gpurun_out/peer_cost_f$f.jsonl; done
timeout 900 python -m pytest tests/test_gpu_peer_gemv.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_pgemv.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pgemv.log
