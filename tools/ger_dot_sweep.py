#!/usr/bin/env python
"""GER across aspect ratios at 256 MiB of C (fp32), both layouts, and DOT
across lengths — looking for cliffs (exploration)."""
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
dt = torch.float32; s = 4
total = 1 << 26
for lm in [0, 2, 4, 6, 8, 10, 13, 16, 20, 24, 26]:
    m = 1 << lm; n = total // m
    C = cb.fill_uniform(torch.empty(m * n, dtype=dt, device=dev), 1, 5)
    x = cb.fill_uniform(torch.empty(m, dtype=dt, device=dev), 1, 1)
    y = cb.fill_uniform(torch.empty(n, dtype=dt, device=dev), 1, 2)
    for lay in (cb.Layout.RowMajor, cb.Layout.ColMajor):
        M = cb.DenseMatrix.wrap(C, m, n, lay)
        us = timeit(lambda: cb.ger(x, y, M, pol))
        print(json.dumps({"op": "ger", "layout": "cm" if lay else "rm", "m": m, "n": n,
                          "ctas": cb.last_exec().threads_used, "us": round(us, 1),
                          "gbs": round(2 * m * n * s / us / 1e3, 1)}), flush=True)
    del C
for ln in [10, 13, 14, 16, 18, 20, 22, 24, 26]:
    n = 1 << ln
    x = cb.fill_uniform(torch.empty(n, dtype=dt, device=dev), 1, 1)
    y = cb.fill_uniform(torch.empty(n, dtype=dt, device=dev), 1, 2)
    out = torch.empty(1, device=dev)
    us = timeit(lambda: cb.dot_into(x, y, 0.0, out, pol))
    print(json.dumps({"op": "dot", "n": n, "ctas": cb.last_exec().threads_used, "us": round(us, 2),
                      "gbs": round(2 * n * s / us / 1e3, 1)}), flush=True)
