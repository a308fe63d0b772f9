#!/usr/bin/env python
"""Bandwidth lab driver (exploration only): time streaming-read kernels of
different shapes and sizes with CUDA events, L2 flushed (write + read) in
between, and print one JSON line per point.  Also times the product kernels
(dot / gemv_rm) at the same sizes for comparison."""
from __future__ import annotations

import ctypes as C
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
SO = ROOT / "tools" / "libbwlab.so"


def build():
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-O3", "-shared", "-Xcompiler", "-fPIC", "-o", str(SO),
                    str(ROOT / "tools" / "bwlab.cu")], check=True)


def main():
    import torch

    import bench
    if not SO.exists():
        build()
    L = C.CDLL(str(SO))
    L.bwlab_run.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int,
                            C.c_int, C.c_void_p]
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    out = torch.zeros(1 << 16, device=dev)
    s = torch.cuda.current_stream().cuda_stream

    def timeit(fn, reps=20):
        ts = []
        for _ in range(3):
            flush.zero_()
            fn()
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return sum(ts) / len(ts) * 1e3  # mean us (event timer ticks are coarse)

    L.bwlab_dot.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                            C.c_int, C.c_int, C.c_void_p]
    if "--dot" in sys.argv:
        ticket = torch.zeros(1, dtype=torch.int32, device=dev)
        x = torch.ones((128 << 20) // 4, device=dev)
        nvec = (64 << 20) // 32
        for fin in (0, 1):
            for block, per_sm in [(256, 4), (256, 8), (512, 2)]:
                for unroll in (1, 2):
                    t = timeit(lambda: L.bwlab_dot(fin, unroll, x.data_ptr(), nvec, out.data_ptr(),
                                                   ticket.data_ptr(), 148 * per_sm, block, s))
                    print(json.dumps({"dot2_final": fin, "block": block, "ctas_per_sm": per_sm,
                                      "unroll": unroll, "us": round(t, 2)}), flush=True)
        t = timeit(lambda: L.bwlab_run(0, 2, x.data_ptr(), 2 * nvec, out.data_ptr(), 592, 256, s))
        print(json.dumps({"single_array_read_128MiB_us": round(t, 2)}))
        return
    print(json.dumps({"empty_kernel_us": timeit(lambda: L.bwlab_run(2, 1, None, 0, out.data_ptr(), 148, 256, s))}))
    for mb in [64, 128, 256, 512, 2048]:
        nbytes = mb << 20
        x = torch.ones(nbytes // 4, device=dev)
        nvec = nbytes // 32
        for kind in (0, 1):
            for block, per_sm in [(256, 4), (256, 8), (512, 2), (512, 4), (1024, 1), (1024, 2)]:
                for unroll in (1, 2, 4, 8):
                    grid = 148 * per_sm
                    t = timeit(lambda: L.bwlab_run(kind, unroll, x.data_ptr(), nvec, out.data_ptr(),
                                                   grid, block, s))
                    print(json.dumps({"mb": mb, "kind": ["gridstride", "chunk"][kind],
                                      "block": block, "ctas_per_sm": per_sm, "unroll": unroll,
                                      "us": round(t, 2), "gbs": round(nbytes / t / 1e3, 1)}),
                          flush=True)
        del x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
