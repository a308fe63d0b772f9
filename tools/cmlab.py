#!/usr/bin/env python
"""Col-major GEMV lab driver (exploration only): tools/cmlab.cu's full-column
variant against the product's path on mid-size fp32 shapes (256 MiB), flushed
per launch and back to back; results checked against the product within the
GEMV tolerance.  One JSON line per (shape, variant)."""
from __future__ import annotations

import ctypes as C
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
SO = ROOT / "tools" / "libcmlab.so"


def main():
    import torch

    import bench
    import paper_2108_02025_b200 as cb
    if not SO.exists() or "--build" in sys.argv:
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                        "-O3", "-lineinfo", "-shared", "-Xcompiler", "-fPIC", "-o", str(SO),
                        str(ROOT / "tools" / "cmlab.cu")], check=True)
    L = C.CDLL(str(SO))
    L.cmlab_run.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                            C.c_void_p, C.c_int, C.c_int, C.c_void_p]
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    pol = cb.default_policy(1)
    flush = bench.L2Flush(dev)
    s = torch.cuda.current_stream().cuda_stream
    partials = torch.zeros(600 * 16384, device=dev)
    pdyn = torch.zeros(64 << 20, device=dev)
    queue = torch.zeros(4, dtype=torch.int32, device=dev)

    def timed(fn, reps=30):
        for _ in range(3):
            flush.zero_()
            fn()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return sum(ts) / len(ts), a.elapsed_time(b) * 1e3 / reps

    if "--ncu" in sys.argv:  # one flushed launch of each kernel under study, m = 4096
        m, n = 4096, 16384
        for dt in (torch.float32, torch.float64):
            A = cb.fill_uniform(torch.empty(m * n, dtype=dt, device=dev), 42, 3)
            x = cb.fill_uniform(torch.empty(n, dtype=dt, device=dev), 42, 1)
            c = cb.fill_uniform(torch.empty(m, dtype=dt, device=dev), 42, 4)
            M = cb.DenseMatrix.wrap(A, m, n, cb.Layout.ColMajor)
            flush.zero_()
            cb.gemv_col_major(M, x, c, pol)
            if dt == torch.float32:
                flush.zero_()
                L.cmlab_run(4, A.data_ptr(), x.data_ptr(), c.data_ptr(), m, n, partials.data_ptr(),
                            148, 1, s)
            del A, M
        torch.cuda.synchronize()
        print("ncu pass ok")
        return
    for m in (1024, 2048, 4096, 8192, 16384):
        n = (1 << 26) // m
        A = cb.fill_uniform(torch.empty(m * n, device=dev), 42, 3)
        x = cb.fill_uniform(torch.empty(n, device=dev), 42, 1)
        c0 = cb.fill_uniform(torch.empty(m, device=dev), 42, 4)
        M = cb.DenseMatrix.wrap(A, m, n, cb.Layout.ColMajor)
        alg = m * n * 4 + n * 4 + 8 * m
        want = c0.clone()
        cb.gemv_col_major(M, x, want, pol)
        rowabs = (A.view(n, m).abs().t().double() @ x.abs().double())
        c = c0.clone()
        f, b = timed(lambda: cb.gemv_col_major(M, x, c, pol))
        print(json.dumps({"m": m, "n": n, "variant": "product", "flushed_us": round(f, 2),
                          "flushed_gbs": round(alg / f / 1e3, 1), "b2b_us": round(b, 2),
                          "b2b_gbs": round(alg / b / 1e3, 1)}), flush=True)
        L.cmlab_sk.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_int,
                               C.c_void_p]
        if m <= 8192 and "--streamk" in sys.argv:
            for frac in (0.1, 0.2, 0.3):
                for cb_kb in (128, 256, 512):
                    ch = max(1, (cb_kb << 10) // (m * 4))
                    c = c0.clone()
                    fn = lambda: L.cmlab_sk(4, A.data_ptr(), x.data_ptr(), c.data_ptr(), m, n,  # noqa: E731
                                            partials.data_ptr(), pdyn.data_ptr(), queue.data_ptr(),
                                            148, frac, ch, s)
                    if fn() != 0:
                        continue
                    torch.cuda.synchronize()
                    err = float(((c.double() - want.double()).abs() / (rowabs * 1e-5 + 1e-30)).max())
                    f, b = timed(fn)
                    print(json.dumps({"m": m, "n": n, "variant": f"streamk_dyn{frac}_chunk{cb_kb}KB",
                                      "flushed_us": round(f, 2), "flushed_gbs": round(alg / f / 1e3, 1),
                                      "b2b_us": round(b, 2), "b2b_gbs": round(alg / b / 1e3, 1),
                                      "err_vs_product_1e-5rowabs": round(err, 4)}), flush=True)
        L.cmlab_gs_t.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                 C.c_uint64, C.c_void_p, C.c_int, C.c_void_p]
        for T, parts in ((1024, 148), (512, 296), (256, 592), (512, 148), (256, 296)):
            c = c0.clone()
            fn = lambda: L.cmlab_gs_t(T, A.data_ptr(), x.data_ptr(), c.data_ptr(), m, n,  # noqa: E731
                                      partials.data_ptr(), parts, s)
            if fn() != 0:
                continue
            torch.cuda.synchronize()
            err = float(((c.double() - want.double()).abs() / (rowabs * 1e-5 + 1e-30)).max())
            f, b = timed(fn)
            print(json.dumps({"m": m, "n": n, "variant": f"gs_T{T}_P{parts}",
                              "flushed_us": round(f, 2), "flushed_gbs": round(alg / f / 1e3, 1),
                              "b2b_us": round(b, 2), "b2b_gbs": round(alg / b / 1e3, 1),
                              "err_vs_product_1e-5rowabs": round(err, 4)}), flush=True)
        continue
        for U in (102,):  # U >= 100: grid-stride columns (U - 100 in flight)
            for parts in (148,):
                for pdl in (1,):
                    c = c0.clone()
                    rc = L.cmlab_run(U, A.data_ptr(), x.data_ptr(), c.data_ptr(), m, n,
                                     partials.data_ptr(), parts, pdl, s)
                    torch.cuda.synchronize()
                    if rc != 0:
                        continue
                    err = float(((c.double() - want.double()).abs() / (rowabs * 1e-5 + 1e-30)).max())
                    fn = lambda: L.cmlab_run(U, A.data_ptr(), x.data_ptr(), c.data_ptr(), m, n,  # noqa: E731
                                             partials.data_ptr(), parts, pdl, s)
                    f, b = timed(fn)
                    print(json.dumps({"m": m, "n": n, "variant": f"full_{'gs' if U >= 100 else 'contig'}_U{U % 100}_P{parts}_pdl{pdl}",
                                      "flushed_us": round(f, 2), "flushed_gbs": round(alg / f / 1e3, 1),
                                      "b2b_us": round(b, 2), "b2b_gbs": round(alg / b / 1e3, 1),
                                      "err_vs_product_1e-5rowabs": round(err, 4)}), flush=True)
        del A, M
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
