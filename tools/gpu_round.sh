mkdir -p gpurun_out
timeout 120 python tools/pcie_duplex.py pipe > gpurun_out/pcie_pipe.jsonl 2>&1
