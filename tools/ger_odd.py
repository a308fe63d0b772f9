#!/usr/bin/env python
"""GER on odd / misaligned rows (the flat 32-byte sweep, ger_flat_any_kernel)
against the aligned 8192^2 tile kernel, L2 flushed per rep.  Run twice, with
CABL_GER_ANY=0 (the previous scalar flat sweep) and 1, for the before/after."""
import os as _os
_os.environ.setdefault("CABL_TUNING", "1")  # exploration script: honour CABL_* knobs
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2108_02025_b200 as cb  # noqa: E402

dev = torch.device("cuda:0")
pol = cb.default_policy(1)
flush = bench.L2Flush(dev)


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2] * 1e3


def buf(n, off, dt):
    t = torch.empty(n + off, dtype=dt, device=dev)
    cb.fill_uniform(t, 1, 3)
    return t[off:]


def main():
    for dt in (torch.float32, torch.float64):
        s = torch.tensor([], dtype=dt).element_size()
        for m, n, off in ((8192, 8192, 0), (8192, 8193, 0), (8192, 8192, 1), (8192, 8196, 0),
                          (8192, 8192, 4), (4096, 16383, 0), (65536, 1001, 0), (1001, 65536, 3),
                          (262144, 255, 0), (2_000_000, 33, 0)):
            if dt == torch.float64:
                m //= 2
            x, y, C = buf(m, off, dt), buf(n, off, dt), buf(m * n, off, dt)
            Cm = cb.DenseMatrix.wrap(C, m, n, cb.Layout.RowMajor)
            us = timeit(lambda: cb.ger(x, y, Cm, pol))
            nbytes = (2 * m * n + m + n) * s
            print(json.dumps({"dtype": str(dt)[6:], "m": m, "n": n, "off": off, "us": round(us, 2),
                              "gbs": round(nbytes / us / 1e3, 1)}), flush=True)
            del x, y, C, Cm


if __name__ == "__main__":
    main()
