#!/usr/bin/env python
"""DOT lab driver (exploration only): time the tools/dotlab.cu variants on
D1 (fp32 n = 2^24) one launch at a time with the L2 flushed in between (the
bench's flushed mode), and back to back; check each result against an fp64
torch dot.  One JSON line per variant.

    python tools/dotlab.py [--reps 40] [--only kind,a,b,grid,block]
"""
from __future__ import annotations

import ctypes as C
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
SO = ROOT / "tools" / "libdotlab.so"

VARIANTS2 = [
    # (label, kind, a, b, grid, block) through dotlab_run2; kind 7: a = prefetch slabs,
    # b = final (0 none, 1 ticket, 2 CTA-0 poll); kind 8: contiguous, a = prefetch all
    ("pf0_nofinal", 7, 0, 0, 296, 512),
    ("pf2_nofinal", 7, 2, 0, 296, 512),
    ("pf6_nofinal", 7, 6, 0, 296, 512),
    ("pf14_nofinal", 7, 14, 0, 296, 512),
    ("pf0_ticket", 7, 0, 1, 296, 512),
    ("pf0_poll", 7, 0, 2, 296, 512),
    ("pf6_poll", 7, 6, 2, 296, 512),
    ("pf14_poll", 7, 14, 2, 296, 512),
    ("pf14_ticket", 7, 14, 1, 296, 512),
    ("contig_nopf", 8, 0, 0, 296, 512),
    ("contig_pf", 8, 1, 0, 296, 512),
]

VARIANTS = [
    # (label, kind, a, b, grid, block)
    ("empty_1x32", 0, 0, 0, 1, 32),
    ("empty_296x512", 0, 0, 0, 296, 512),
    ("ldg_nofinal_u2", 1, 2, 0, 296, 512),
    ("ldg_final_u2", 2, 2, 0, 296, 512),
    ("ldg_final_u1", 2, 1, 0, 296, 512),
    ("ldg_final_u4", 2, 4, 0, 296, 512),
    ("bulk_static_12x8k", 3, 12, 8, 148, 288),
    ("bulk_static_6x16k", 3, 6, 16, 148, 288),
    ("bulk_static_3x32k", 3, 3, 32, 148, 288),
    ("bulk_static_24x4k", 3, 24, 4, 148, 288),
    ("bulk_static_6x8k_2pSM", 3, 6, 8, 296, 288),
    ("bulk_static_3x16k_2pSM", 3, 3, 16, 296, 288),
    ("bulk_interleave_12x8k", 4, 12, 8, 148, 288),
    ("bulk_interleave_6x16k", 4, 6, 16, 148, 288),
    ("bulk_dyn_12x8k", 5, 12, 8, 148, 288),
    ("bulk_dyn_6x16k", 5, 6, 16, 148, 288),
    ("bulk_dyn_3x32k", 5, 3, 32, 148, 288),
    ("bulk_dyn_6x8k_2pSM", 5, 6, 8, 296, 288),
    ("ldg_cluster2", 6, 2, 0, 296, 512),
    ("ldg_cluster4", 6, 4, 0, 296, 512),
]


def build():
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-o",
                    str(SO), str(ROOT / "tools" / "dotlab.cu")], check=True)


def main():
    import torch

    import bench
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200 import workloads as WL
    if not SO.exists() or "--build" in sys.argv:
        build()
    L = C.CDLL(str(SO))
    L.dotlab_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64,
                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                             C.c_void_p]
    reps = 40
    if "--reps" in sys.argv:
        reps = int(sys.argv[sys.argv.index("--reps") + 1])
    variants = VARIANTS
    if "--only" in sys.argv:
        keep = sys.argv[sys.argv.index("--only") + 1].split(";")
        variants = [v for v in VARIANTS if v[0] in keep]
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    n = 1 << 24
    x = cb.fill_uniform(torch.empty(n, device=dev), WL.SEED, WL.STREAM_X)
    y = cb.fill_uniform(torch.empty(n, device=dev), WL.SEED, WL.STREAM_Y)
    truth = float(torch.dot(x.double(), y.double()))
    sumabs = float((x.double() * y.double()).abs().sum())
    partials = torch.zeros(1 << 16, device=dev)
    ticket = torch.zeros(4, dtype=torch.int32, device=dev)
    queue = torch.zeros(4, dtype=torch.int32, device=dev)
    out = torch.zeros(4, device=dev)
    flush = bench.L2Flush(dev)
    s = torch.cuda.current_stream().cuda_stream
    pol = cb.default_policy(1)
    prod_out = torch.zeros(1, device=dev)
    L.dotlab_run2.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint, C.c_void_p, C.c_int,
                              C.c_int, C.c_void_p]
    slots = torch.zeros(4096, dtype=torch.int64, device=dev)
    epoch = [0]

    def run2(kind, a, b, grid, block):
        epoch[0] += 1
        return L.dotlab_run2(kind, a, b, x.data_ptr(), y.data_ptr(), n, partials.data_ptr(),
                             ticket.data_ptr(), slots.data_ptr(), epoch[0], out.data_ptr(), grid,
                             block, s)
    def timed(fn):
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
        ts.sort()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return {"flushed_mean_us": round(sum(ts) / len(ts), 2), "flushed_med_us": round(ts[len(ts) // 2], 2),
                "flushed_min_us": round(ts[0], 2), "b2b_us": round(a.elapsed_time(b) * 1e3 / reps, 2)}

    if "--v2" in sys.argv:
        variants2 = VARIANTS2
        if "--only" in sys.argv:
            keep = sys.argv[sys.argv.index("--only") + 1].split(";")
            variants2 = [v for v in VARIANTS2 if v[0] in keep]
        if "--once" in sys.argv:
            for _ in range(int(sys.argv[sys.argv.index("--once") + 1])):
                flush.zero_()
                cb.dot_into(x, y, 0.0, prod_out, pol)
                for label, kind, a, b, grid, block in variants2:
                    flush.zero_()
                    run2(kind, a, b, grid, block)
            torch.cuda.synchronize()
            print("once: ok")
            return
        for label, kind, a, b, grid, block in variants2:
            fn = lambda: run2(kind, a, b, grid, block)  # noqa: E731
            if fn() != 0:
                print(json.dumps({"variant": label, "error": "launch"}), flush=True)
                continue
            torch.cuda.synchronize()
            r = timed(fn)
            line = {"variant": label, **r}
            if b or kind == 8:
                out.zero_()
                fn()
                torch.cuda.synchronize()
                line["rel_err"] = abs(float(out[0]) - truth) / sumabs
            print(json.dumps(line), flush=True)
        return

    alg = 2 * n * 4
    if "--once" in sys.argv:  # one flushed launch per variant (for ncu)
        flush.zero_()
        cb.dot_into(x, y, 0.0, prod_out, pol)
        for label, kind, a, b, grid, block in variants:
            flush.zero_()
            L.dotlab_run(kind, a, b, x.data_ptr(), y.data_ptr(), n, partials.data_ptr(),
                         ticket.data_ptr(), queue.data_ptr(), out.data_ptr(), grid, block, s)
        torch.cuda.synchronize()
        print("once: ok")
        return
    r = timed(lambda: cb.dot_into(x, y, 0.0, prod_out, pol))
    err = abs(float(prod_out) - truth) / sumabs
    print(json.dumps({"variant": "product_dot_kernel", **r, "rel_err": err,
                      "flushed_gbs": round(alg / r["flushed_mean_us"] / 1e3, 1)}), flush=True)
    for label, kind, a, b, grid, block in variants:
        fn = lambda: L.dotlab_run(kind, a, b, x.data_ptr(), y.data_ptr(), n, partials.data_ptr(),  # noqa: E731
                                  ticket.data_ptr(), queue.data_ptr(), out.data_ptr(), grid, block, s)
        rc = fn()
        torch.cuda.synchronize()
        if rc != 0:
            print(json.dumps({"variant": label, "error": rc}), flush=True)
            continue
        r = timed(fn)
        line = {"variant": label, **r}
        if kind in (2, 3, 4, 5, 6):
            out.zero_()
            fn()
            torch.cuda.synchronize()
            line["rel_err"] = abs(float(out[0]) - truth) / sumabs
        if kind:
            line["flushed_gbs"] = round(alg / r["flushed_mean_us"] / 1e3, 1)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
