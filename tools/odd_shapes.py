#!/usr/bin/env python
"""Performance on shapes / alignments that miss the vector fast paths (odd
lengths, misaligned operands), next to their aligned neighbours — looking for
cliffs.  L2 flushed between reps; GB/s of algorithmic bytes."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
import paper_2108_02025_b200 as cb

dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
pol = cb.default_policy(1)
flush = bench.L2Flush(dev)


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2] * 1e3


def buf(n, off=0, dt=torch.float32):
    t = torch.empty(n + off, dtype=dt, device=dev)
    cb.fill_uniform(t, 1, 3)
    return t[off:]


def report(name, us, nbytes):
    print(json.dumps({"case": name, "us": round(us, 2), "gbs": round(nbytes / us / 1e3, 1)}), flush=True)


s = 4
for n, off in ((1 << 24, 0), ((1 << 24) + 3, 0), (1 << 24, 1)):
    x, y = buf(n, off), buf(n, off)
    out = torch.empty(1, device=dev)
    report(f"dot n={n} off={off}", timeit(lambda: cb.dot_into(x, y, 0.0, out, pol)), 2 * n * s)
for m, n, off in ((8192, 8192, 0), (8192, 8193, 0), (8192, 8192, 1), (8192, 8196, 0)):
    A, x, c = buf(m * n, off), buf(n, off), buf(m, off)
    M = cb.DenseMatrix.wrap(A, m, n, cb.Layout.RowMajor)
    report(f"gemv_rm {m}x{n} off={off}", timeit(lambda: cb.gemv_row_major(M, x, c, pol)), m * n * s)
for m, n, off in ((8192, 8192, 0), (8193, 8192, 0), (8192, 8192, 1), (256, 1 << 20, 0), (257, 1 << 20, 0)):
    A, x, c = buf(m * n, off), buf(n, off), buf(m, off)
    M = cb.DenseMatrix.wrap(A, m, n, cb.Layout.ColMajor)
    report(f"gemv_cm {m}x{n} off={off}", timeit(lambda: cb.gemv_col_major(M, x, c, pol)), m * n * s)
for m, n, off in ((8192, 8192, 0), (8192, 8193, 0), (8192, 8192, 1), (8192, 8196, 0), (8192, 8192, 4)):
    C, x, y = buf(m * n, off), buf(m, off), buf(n, off)
    M = cb.DenseMatrix.wrap(C, m, n, cb.Layout.RowMajor)
    report(f"ger_rm {m}x{n} off={off}", timeit(lambda: cb.ger(x, y, M, pol)), 2 * m * n * s)
