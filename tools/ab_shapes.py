#!/usr/bin/env python
"""A/B timing of GEMV/GER shapes at ~256 MiB (fp32) / 512 MiB (fp64): flushed
(mean of 30 single launches, L2 flushed before each) and back to back (mean
of 30).  One JSON line per shape, tagged; run once per variant (CABL_* knobs
are read once per process; CABL_TUNING=1 is set here).

    CABL_RM_GVEC_STRIDE=1 python tools/ab_shapes.py --tag stride --op gemv-row --n 1024,512,256
"""
from __future__ import annotations

import os as _os
_os.environ.setdefault("CABL_TUNING", "1")
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    import paper_2108_02025_b200 as cb
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="default")
    ap.add_argument("--op", default="gemv-row", choices=["gemv-row", "gemv-col", "ger-row", "ger-col"])
    ap.add_argument("--n", default="1024", help="row lengths (gemv-row/ger-row) or column counts")
    ap.add_argument("--dtypes", default="f32,f64")
    ap.add_argument("--bytes", type=int, default=1 << 28, help="fp32 matrix bytes (fp64: twice)")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    pol = cb.default_policy(1)
    flush = bench.L2Flush(dev)
    for dts in args.dtypes.split(","):
        dt = torch.float64 if dts == "f64" else torch.float32
        s = 8 if dts == "f64" else 4
        for nn in (int(v) for v in args.n.split(",")):
            total = args.bytes // 4  # elements (fp64 matrices are twice the bytes)
            if args.op in ("gemv-row", "ger-row"):
                n, m = nn, max(1, total // nn)
            else:
                m, n = nn, max(1, total // nn)
            lay = cb.Layout.RowMajor if args.op.endswith("row") else cb.Layout.ColMajor
            A = cb.fill_uniform(torch.empty(m * n, dtype=dt, device=dev), 42, 3)
            M = cb.DenseMatrix.wrap(A, m, n, lay)
            if args.op.startswith("gemv"):
                x = cb.fill_uniform(torch.empty(n, dtype=dt, device=dev), 42, 1)
                c = cb.fill_uniform(torch.empty(m, dtype=dt, device=dev), 42, 4)
                f = cb.gemv_row_major if lay == cb.Layout.RowMajor else cb.gemv_col_major
                fn = lambda: f(M, x, c, pol)  # noqa: E731
                alg = m * n * s + n * s + 2 * m * s
            else:
                x = cb.fill_uniform(torch.empty(m, dtype=dt, device=dev), 42, 1)
                y = cb.fill_uniform(torch.empty(n, dtype=dt, device=dev), 42, 2)
                fn = lambda: cb.ger(x, y, M, pol)  # noqa: E731
                alg = 2 * m * n * s + m * s + n * s
            fn()
            ctas = cb.last_exec().threads_used
            for _ in range(3):
                flush.zero_()
                fn()
            ts = []
            for _ in range(30):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            torch.cuda._sleep(1_000_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(30):
                fn()
            b.record()
            torch.cuda.synchronize()
            b2b = a.elapsed_time(b) * 1e3 / 30
            us = sum(ts) / len(ts)
            print(json.dumps({"tag": args.tag, "op": args.op, "dtype": "float64" if s == 8 else "float32",
                              "m": m, "n": n, "ctas": ctas,
                              "flushed_us": round(us, 2), "flushed_gbs": round(alg / us / 1e3, 1),
                              "b2b_us": round(b2b, 2), "b2b_gbs": round(alg / b2b / 1e3, 1)}), flush=True)
            del A, M
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
