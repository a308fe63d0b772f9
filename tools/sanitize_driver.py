#!/usr/bin/env python
"""Drive every kernel path of libcabl_cuda.so once at small-to-moderate
shapes, for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py

Paths: DOT small / main / chunked (forced) / unaligned; GEMV row-major
(with CABL_GEMV_RM_ORDER=reference also the reference-order kernel)
ordered / segment / sweep (static and queue) / scalar; col-major ordered /
tall vec (static and queue) / tall scalar / 2-D split vec / 2-D split scalar /
bulk-copy split; GER tile queue / static / generic; the fills and the
partial combine.  Exits non-zero if any result is non-finite.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200 import _lib
    dev = torch.device("cuda:0")
    pol = cb.default_policy(1)
    f = lambda n, dt, st: cb.fill_uniform(torch.empty(n, dtype=dt, device=dev), 7, st)  # noqa: E731
    ok = True
    for dt in (torch.float32, torch.float64):
        V = 8 if dt == torch.float32 else 4
        # DOT
        for n in (0, 5, 8192, 100_003, 1 << 20):
            x, y = f(n + 3, dt, 1), f(n + 3, dt, 2)
            ok &= bool(torch.isfinite(torch.tensor(cb.dot(x[:n], y[:n], 0.5, pol))))
            ok &= bool(torch.isfinite(torch.tensor(cb.dot(x[1:n + 1], y[2:n + 2], 0.5, pol))))
        # GEMV row-major: ordered, segment, sweep, scalar
        for m, n in ((3, 5), (40, 1024), (2, 65536), (7200, 256), (3000, 999), (5000, 1028),
                     (20000, 16), (20000, 256), (20000, 33), (20001, 5), (9000, 8200)):
            A = cb.DenseMatrix.wrap(f(m * n, dt, 3), m, n, cb.Layout.RowMajor)
            c = f(m, dt, 4)
            cb.gemv_row_major(A, f(n, dt, 1), c, pol)
            ok &= bool(torch.isfinite(c).all())
        # GEMV col-major: ordered, 2-D split vec/scalar, bulk, tall vec, tall scalar
        for m, n in ((3, 5), (256, 4096), (4096, 300), (2000 + V, 77), (1001, 300),
                     (148 * 256 * V, 4), (148 * 1024 + 1, 3), (1, 100000), (257, 20000),
                     (74 * 256 * V, 20), (300000 // V * V, 9), (8193, 300)):
            A = cb.DenseMatrix.wrap(f(m * n, dt, 3), m, n, cb.Layout.ColMajor)
            c = f(m, dt, 4)
            cb.gemv_col_major(A, f(n, dt, 1), c, pol)
            ok &= bool(torch.isfinite(c).all())
        # GER: generic, tile queue, both layouts
        for m, n in ((3, 5), (37, 1000), (300, 2048), (1000, 4096), (20000, 64), (3000, 4100),
                     (50000, 5)):
            for lay in (cb.Layout.RowMajor, cb.Layout.ColMajor):
                C = cb.DenseMatrix.wrap(f(m * n, dt, 5), m, n, lay)
                cb.ger(f(m, dt, 1), f(n, dt, 2), C, pol)
                ok &= bool(torch.isfinite(C.data).all())
        # rank-ordered combine
        p = f(8, dt, 9)
        out = torch.empty(1, dtype=dt, device=dev)
        _lib.call(f"cabl_cuda_combine_partials_{'f32' if dt == torch.float32 else 'f64'}",
                  p.data_ptr(), 8, 1.0, out.data_ptr(), None)
        normal = cb.fill_normal(torch.empty(1000, dtype=torch.float64, device=dev), 1, 2)
        ok &= bool(torch.isfinite(normal).all())
    torch.cuda.synchronize()
    print("sanitize driver:", "ok" if ok else "NON-FINITE RESULT", "env:",
          {k: v for k, v in os.environ.items() if k.startswith("CABL_")})
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
