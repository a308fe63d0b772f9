mkdir -p gpurun_out
cat > /tmp/h2d.py <<'PY'
import torch, time, json
n = 256 << 20
h = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d = torch.empty(n // 4, dtype=torch.float32, device='cuda')
for chunks in (1, 2, 4, 8):
    ss = [torch.cuda.Stream() for _ in range(chunks)]
    step = (n // 4) // chunks
    def go():
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i*step:(i+1)*step].copy_(h[i*step:(i+1)*step], non_blocking=True)
        torch.cuda.synchronize()
    for _ in range(3): go()
    t = time.perf_counter()
    for _ in range(10): go()
    dt = (time.perf_counter() - t) / 10
    print(json.dumps({"chunks": chunks, "ms": round(dt*1e3, 3), "GBs": round(n/dt/1e9, 1)}))
PY
python /tmp/h2d.py > gpurun_out/h2d.jsonl 2>&1
nvidia-smi -q | grep -i -A3 "PCIe Generation" > gpurun_out/pcie.txt 2>&1
nvidia-smi -q | grep -i -A2 "Link Width" >> gpurun_out/pcie.txt 2>&1
