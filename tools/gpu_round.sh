mkdir -p gpurun_out
python tools/nccl_vs_peer.py > gpurun_out/nccl_vs_peer.jsonl 2>&1
