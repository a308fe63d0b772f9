#!/usr/bin/env python
"""Col-major GEMV across m at a fixed 256 MiB (fp32) / 512 MiB (fp64) of A —
which kernel each shape takes and how close it gets (exploration)."""
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
    total = (1 << 26)  # elements
    for lm in [0, 2, 4] + list(range(6, 26, 2)):
        m = 1 << lm; n = total // m
        A = cb.fill_uniform(torch.empty(m * n, dtype=dt, device=dev), 1, 3)
        x = cb.fill_uniform(torch.empty(n, dtype=dt, device=dev), 1, 1)
        c = torch.zeros(m, dtype=dt, device=dev)
        for lay, f in ((cb.Layout.ColMajor, cb.gemv_col_major), (cb.Layout.RowMajor, cb.gemv_row_major)):
            M = cb.DenseMatrix.wrap(A, m, n, lay)
            us = timeit(lambda: f(M, x, c, pol))
            print(json.dumps({"dtype": str(dt)[6:], "layout": "cm" if lay else "rm", "m": m, "n": n,
                              "ctas": cb.last_exec().threads_used, "us": round(us, 1),
                              "gbs": round(m * n * s / us / 1e3, 1)}), flush=True)
        del A
