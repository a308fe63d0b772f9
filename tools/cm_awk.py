#!/usr/bin/env python
"""Col-major GEMV at awkward heights (aligned, multiple of 8 rows), 256 MiB
fp32 (exploration)."""
import json, os, sys
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
import os
MS = [int(v) for v in os.environ.get('CM_MS', '520,1000,5000,20000,50000,100000,200000,300000,303104,400000,1000000').split(',')]
for m in MS:
    n = (1 << 26) // m
    A = cb.fill_uniform(torch.empty(m * n, device=dev), 1, 3)
    x = cb.fill_uniform(torch.empty(n, device=dev), 1, 1)
    c = torch.zeros(m, device=dev)
    M = cb.DenseMatrix.wrap(A, m, n, cb.Layout.ColMajor)
    us = timeit(lambda: cb.gemv_col_major(M, x, c, pol))
    print(json.dumps({"m": m, "n": n, "ctas": cb.last_exec().threads_used, "us": round(us, 1),
                      "gbs": round((m * n + 2 * m + n) * 4 / us / 1e3, 1)}), flush=True)
    del A, M
