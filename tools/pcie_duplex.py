#!/usr/bin/env python
"""PCIe on the GPU box: pinned H2D alone, D2H alone, and both at once on two
streams (256 MiB each way), median of 5 — the bound of GER's full-duplex host
pipeline."""
import json
import statistics
import time

import torch


def timed(fn, reps=5):
    ts = []
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts[1:])


def main():
    n = 256 << 20
    hs = torch.empty(n, dtype=torch.uint8).pin_memory()
    hd = torch.empty(n, dtype=torch.uint8).pin_memory()
    ds = torch.empty(n, dtype=torch.uint8, device="cuda")
    dd = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        with torch.cuda.stream(s1):
            ds.copy_(hs, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            hd.copy_(dd, non_blocking=True)

    def both():
        h2d()
        d2h()

    t_h2d, t_d2h, t_both = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({"bytes_each_way": n, "h2d_ms": round(t_h2d * 1e3, 3), "d2h_ms": round(t_d2h * 1e3, 3),
                      "both_ms": round(t_both * 1e3, 3), "h2d_gbs": round(n / t_h2d / 1e9, 1),
                      "d2h_gbs": round(n / t_d2h / 1e9, 1),
                      "duplex_gbs_each_way": round(n / t_both / 1e9, 1)}), flush=True)


def pipeline(slabs: int) -> dict:
    """The GER host pipeline's copy pattern without the kernel: H2D of slab k on
    one stream, D2H of slab k on another once slab k has landed."""
    n = 256 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    step = n // slabs

    def run():
        for k in range(slabs):
            a, b = k * step, (k + 1) * step if k < slabs - 1 else n
            with torch.cuda.stream(s1):
                d[a:b].copy_(h[a:b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s1)
            s2.wait_event(ev)
            with torch.cuda.stream(s2):
                h[a:b].copy_(d[a:b], non_blocking=True)

    t = timed(run)
    return {"pipeline_slabs": slabs, "ms": round(t * 1e3, 3)}


if __name__ == "__main__" and len(__import__("sys").argv) > 1:
    for sl in (8, 16, 32):
        print(json.dumps(pipeline(sl)), flush=True)


if __name__ == "__main__":
    main()
