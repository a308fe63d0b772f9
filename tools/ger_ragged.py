#!/usr/bin/env python
"""GER at awkward widths (aligned, multiple of 8 floats) — ragged column
blocks of the tile kernel (exploration)."""
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
NS = [int(v) for v in os.environ.get("GER_NS", "1024,1032,2048,2056,3000,4096,4104,8192,8200,10000").split(",")]
for n in NS:
    m = (1 << 26) // n
    C = cb.fill_uniform(torch.empty(m * n, device=dev), 1, 5)
    x = cb.fill_uniform(torch.empty(m, device=dev), 1, 1)
    y = cb.fill_uniform(torch.empty(n, device=dev), 1, 2)
    M = cb.DenseMatrix.wrap(C, m, n, cb.Layout.RowMajor)
    us = timeit(lambda: cb.ger(x, y, M, pol))
    print(json.dumps({"m": m, "n": n, "ctas": cb.last_exec().threads_used, "us": round(us, 1),
                      "gbs": round(2 * m * n * 4 / us / 1e3, 1)}), flush=True)
    del C, M
