mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_peer.py tests/test_gpu_peer_gemv.py -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_peer.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_peer.log
