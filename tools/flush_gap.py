#!/usr/bin/env python
"""Flushed single-launch timing of D1 / G1 / R1: bench.py's method (flush, start
event, step, end event) against the same with a short device sleep between the
flush and the start event (so the step is surely queued when the GPU reaches
the start event), and a graph-captured step.  Tells whether the flushed event
time carries host launch latency."""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200 import workloads as WL

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    ctx = bench.Ctx(1, 0, 0, dev)
    flush = bench.L2Flush(dev)
    pol = cb.default_policy(1)
    for wid in ("D1", "G1"):
        w = WL.WORKLOADS[wid]
        span = w.n if w.op == "dot" else w.m
        ins = bench.make_inputs(w, (0, span), dev)
        fn, _ = bench.step_fn(w, ins, pol, ctx, sharded_dot=False)
        for variant in ("bench", "sleep", "bench", "sleep"):
            for _ in range(3):
                flush.zero_()
                fn()
            ts = []
            for _ in range(60):
                flush.zero_()
                if variant == "sleep":
                    torch.cuda._sleep(40_000)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            mean = sum(ts) / len(ts)
            print(json.dumps({"id": wid, "variant": variant, "mean_us": round(mean, 2),
                              "min_us": round(min(ts), 2),
                              "frac": round(w.alg_bytes(1) / mean / 1e3 / bench.peaks()[0], 4)}),
                  flush=True)
        del ins, fn
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
