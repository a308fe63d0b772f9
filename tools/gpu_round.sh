mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_peer.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_peer.log
