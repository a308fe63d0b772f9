#!/usr/bin/env python
"""Drive every kernel path of libcabl_cuda.so once at small-to-moderate
shapes, for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py

Paths: DOT small / main / chunked (forced) / unaligned; GEMV row-major
(with CABL_GEMV_RM_ORDER=reference also the reference-order kernel)
ordered / segment / sweep (static and queue) / scalar; col-major ordered /
tall vec (static and queue) / tall scalar / 2-D split vec / 2-D split scalar /
bulk-copy split / realigning split; GER tile queue / static / generic /
flat any-width / one-element rows; row-major few long rows; the peer-memory
DOT, gathering GEMV and row combine at world 1; the fills and the partial
combine.  Exits non-zero if any result is non-finite.
"""
from __future__ import annotations

import os as _os
_os.environ.setdefault("CABL_TUNING", "1")  # exploration script: honour CABL_* knobs
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
        # this round's paths: few long rows (chunked RM), realigning CM split
        # (odd m and an offset A), flat any-width GER, one-element-row GER
        for m, n, lay, off in ((3, 300_000, cb.Layout.RowMajor, 0), (1, 1 << 18, cb.Layout.RowMajor, 0),
                               (8193, 300, cb.Layout.ColMajor, 0), (4096, 100, cb.Layout.ColMajor, 1),
                               (1025, 777, cb.Layout.ColMajor, 3)):
            A = cb.DenseMatrix.wrap(f(m * n + off, dt, 3)[off:], m, n, lay)
            c = f(m, dt, 4)
            (cb.gemv_row_major if lay == cb.Layout.RowMajor else cb.gemv_col_major)(A, f(n, dt, 1), c, pol)
            ok &= bool(torch.isfinite(c).all())
        for m, n, off in ((777, 1001, 0), (1000, 4096, 1), (400_003, 1, 0), (1, 400_003, 1)):
            for lay in (cb.Layout.RowMajor, cb.Layout.ColMajor):
                C = cb.DenseMatrix.wrap(f(m * n + off, dt, 5)[off:], m, n, lay)
                cb.ger(f(m + off, dt, 1)[off:], f(n + off, dt, 2)[off:], C, pol)
                ok &= bool(torch.isfinite(C.data).all())
        # peer-memory paths at world 1 (DOT, gathering GEMV, row combine)
        import ctypes as C_
        sfx = "f32" if dt == torch.float32 else "f64"
        s = torch.tensor([], dtype=dt).element_size()
        mb, buf, slots = C_.c_void_p(), C_.c_void_p(), C_.c_void_p()
        _lib.call("cabl_peer_mailbox_create", C_.byref(mb))
        x, y = f(100_003, dt, 1), f(100_003, dt, 2)
        out = torch.empty(1, dtype=dt, device=dev)
        _lib.call(f"cabl_cuda_dot_peer_{sfx}", x.data_ptr(), y.data_ptr(), 100_003, 0.5,
                  out.data_ptr(), (C_.c_void_p * 1)(mb.value), 1, 0, 8192, None, None)
        ok &= bool(torch.isfinite(out).all())
        m, n = 3000, 16384 if dt == torch.float32 else 8192
        gmb = C_.c_void_p()
        _lib.call("cabl_peer_mailbox_create", C_.byref(gmb))
        _lib.call("cabl_peer_alloc", 2 * m * s, C_.byref(buf))
        A, xv, c = f(m * n, dt, 3), f(n, dt, 1), f(m, dt, 4)
        _lib.call(f"cabl_cuda_gemv_rm_gather_{sfx}", A.data_ptr(), m, n, xv.data_ptr(), c.data_ptr(),
                  0, m, (C_.c_void_p * 1)(buf.value), (C_.c_void_p * 1)(gmb.value), 1, 0, None, None)
        ok &= bool(torch.isfinite(c).all())
        rmb = C_.c_void_p()
        _lib.call("cabl_peer_mailbox_create", C_.byref(rmb))
        _lib.call("cabl_peer_alloc", 2 * 8 * 256 * s, C_.byref(slots))
        part, cc = f(256, dt, 6), f(256, dt, 7)
        _lib.call(f"cabl_cuda_combine_rows_peer_{sfx}", part.data_ptr(), 256, cc.data_ptr(),
                  (C_.c_void_p * 1)(slots.value), (C_.c_void_p * 1)(rmb.value), 1, 0, None)
        ok &= bool(torch.isfinite(cc).all())
        torch.cuda.synchronize()
        for p_ in (mb, gmb, rmb):
            _lib.call("cabl_peer_mailbox_destroy", p_)
        for p_ in (buf, slots):
            _lib.call("cabl_peer_free", p_)
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
