#!/usr/bin/env python
"""Host-container calls (cabl_host_*) with pinned vs pageable buffers, G1 /
D1 / R1 shapes (exploration)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2108_02025_b200 as cb
pol = cb.default_policy(1)
torch.cuda.init()
def t(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return sorted(ts)[len(ts)//2]
m = n = 8192
for pinned in (True, False):
    mk = (lambda a: torch.from_numpy(a).pin_memory()) if pinned else (lambda a: torch.from_numpy(a))
    A = mk(np.random.rand(m * n).astype(np.float32)); x = mk(np.random.rand(n).astype(np.float32))
    c = mk(np.random.rand(m).astype(np.float32))
    M = cb.DenseMatrix.wrap(A, m, n, cb.Layout.RowMajor)
    s = t(lambda: cb.gemv_row_major(M, x, c, pol))
    print(json.dumps({"op": "gemv G1", "pinned": pinned, "ms": round(s * 1e3, 2), "gbs": round((m*n*4) / s / 1e9, 1)}), flush=True)
    xx = mk(np.random.rand(1 << 24).astype(np.float32)); yy = mk(np.random.rand(1 << 24).astype(np.float32))
    s = t(lambda: cb.dot(xx, yy, 0.0, pol))
    print(json.dumps({"op": "dot D1", "pinned": pinned, "ms": round(s * 1e3, 2), "gbs": round((2 << 26) / s / 1e9, 1)}), flush=True)
    C = cb.DenseMatrix.wrap(A, m, n, cb.Layout.RowMajor)
    s = t(lambda: cb.ger(x, c, C, pol))
    print(json.dumps({"op": "ger R1", "pinned": pinned, "ms": round(s * 1e3, 2), "gbs": round((2*m*n*4) / s / 1e9, 1)}), flush=True)
