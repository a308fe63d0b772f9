#!/usr/bin/env python
"""Row-major GEMV with short rows at ~256 MiB of A (exploration of the lane
threshold: run under CABL_RM_LANE_MAX=<bytes>)."""
import os as _os
_os.environ.setdefault("CABL_TUNING", "1")  # exploration script: honour CABL_* knobs
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
lim = os.environ.get("CABL_RM_LANE_MAX", "default")
for dt in (torch.float32, torch.float64):
    s = torch.tensor([], dtype=dt).element_size()
    for n in (1, 4, 5, 16, 64, 128, 256, 512, 1024):
        m = (1 << 28) // (n * s)
        A = cb.fill_uniform(torch.empty(m * n, dtype=dt, device=dev), 1, 3)
        x = cb.fill_uniform(torch.empty(n, dtype=dt, device=dev), 1, 1)
        c = torch.zeros(m, dtype=dt, device=dev)
        M = cb.DenseMatrix.wrap(A, m, n, cb.Layout.RowMajor)
        us = timeit(lambda: cb.gemv_row_major(M, x, c, pol))
        print(json.dumps({"lane_max": lim, "dtype": str(dt)[6:], "n": n, "row_bytes": n * s, "m": m,
                          "us": round(us, 1), "gbs": round((m * n * s + 2 * m * s) / us / 1e3, 1)}), flush=True)
        del A, M
        torch.cuda.empty_cache()
