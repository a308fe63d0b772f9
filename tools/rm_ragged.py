#!/usr/bin/env python
"""Row-major GEMV at awkward widths (aligned, multiple of 8 floats) — how much
the sweep's ragged last pass costs (exploration)."""
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
import os
NS = [int(v) for v in os.environ.get('RM_NS', '2048,2056,3000,4096,4104,5000,6144,8192,8200,10000,12288,16392').split(',')]
for n in NS:
    m = (1 << 26) // n
    A = cb.fill_uniform(torch.empty(m * n, device=dev), 1, 3)
    x = cb.fill_uniform(torch.empty(n, device=dev), 1, 1)
    c = torch.zeros(m, device=dev)
    M = cb.DenseMatrix.wrap(A, m, n, cb.Layout.RowMajor)
    us = timeit(lambda: cb.gemv_row_major(M, x, c, pol))
    print(json.dumps({"m": m, "n": n, "us": round(us, 1), "gbs": round(m * n * 4 / us / 1e3, 1)}), flush=True)
    del A, M
