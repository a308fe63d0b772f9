#!/usr/bin/env python
"""Col-major GEMV, mid-size row counts (round 2): flushed time per launch of
every aligned shape between the bulk-ring range (m < 512) and the tall kernel,
at 256 MiB fp32 / 512 MiB fp64, under the tile variant given by CABL_CM_TILE
(run once per variant: the knob is read once per process).  One JSON line per
shape with the kernel's CTAs (probe) and the flushed GB/s.

    CABL_CM_TILE=512,256 python tools/cm_mid2.py --tag single512_tile256
"""
from __future__ import annotations

import os as _os
_os.environ.setdefault("CABL_TUNING", "1")  # exploration script: honour CABL_* knobs
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    import paper_2108_02025_b200 as cb
    tag = sys.argv[sys.argv.index("--tag") + 1] if "--tag" in sys.argv else "default"
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    pol = cb.default_policy(1)
    flush = bench.L2Flush(dev)
    shapes = [(512, 131072), (1024, 65536), (2048, 32768), (4096, 16384), (8192, 8192),
              (16384, 4096), (32768, 2048), (65536, 1024), (3000, 22368), (12000, 5592)]
    for dt in (torch.float32, torch.float64):
        s = torch.tensor([], dtype=dt).element_size()
        for m, n in shapes:
            A = cb.fill_uniform(torch.empty(m * n, dtype=dt, device=dev), 42, 3)
            x = cb.fill_uniform(torch.empty(n, dtype=dt, device=dev), 42, 1)
            c = cb.fill_uniform(torch.empty(m, dtype=dt, device=dev), 42, 4)
            M = cb.DenseMatrix.wrap(A, m, n, cb.Layout.ColMajor)
            fn = lambda: cb.gemv_col_major(M, x, c, pol)  # noqa: E731
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
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(30):
                fn()
            b.record()
            torch.cuda.synchronize()
            b2b = a.elapsed_time(b) * 1e3 / 30
            us = sum(ts) / len(ts)
            alg = m * n * s + n * s + 2 * m * s
            print(json.dumps({"tag": tag, "dtype": str(dt)[6:], "m": m, "n": n, "ctas": ctas,
                              "flushed_us": round(us, 2), "flushed_gbs": round(alg / us / 1e3, 1),
                              "b2b_us": round(b2b, 2), "b2b_gbs": round(alg / b2b / 1e3, 1),
                              "env": os.environ.get("CABL_CM_TILE", "")}), flush=True)
            del A, M
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
