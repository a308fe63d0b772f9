#!/usr/bin/env python
"""Col-major GEMV, short-wide / mid m at 256 MiB (exploration of the final combine)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
import paper_2108_02025_b200 as cb
dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
pol = cb.default_policy(1)
flush = bench.L2Flush(dev)
def timeit(fn, reps=7):
    for _ in range(2): fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts)//2] * 1e3
for dt in (torch.float32, torch.float64):
    s = torch.tensor([], dtype=dt).element_size()
    for m in (256, 512, 1024, 1536, 2040, 2047, 4096, 8192):
        n = (1 << 28) // (m * s)
        A = cb.fill_uniform(torch.empty(m * n, dtype=dt, device=dev), 1, 3)
        x = cb.fill_uniform(torch.empty(n, dtype=dt, device=dev), 1, 1)
        c = torch.zeros(m, dtype=dt, device=dev)
        M = cb.DenseMatrix.wrap(A, m, n, cb.Layout.ColMajor)
        us = timeit(lambda: cb.gemv_col_major(M, x, c, pol))
        print(json.dumps({"dtype": str(dt)[6:], "m": m, "n": n, "us": round(us, 1),
                          "gbs": round(m * n * s / us / 1e3, 1)}), flush=True)
        del A, M
