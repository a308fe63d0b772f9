#!/usr/bin/env python
"""Back-to-back timing (no flush between steps, one event pair around K steps)
vs per-step flushed timing, for configs whose inputs exceed 2x the L2."""
import os as _os
_os.environ.setdefault("CABL_TUNING", "1")  # exploration script: honour CABL_* knobs
import json, sys, statistics
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
import paper_2108_02025_b200 as cb
from paper_2108_02025_b200 import workloads as WL
dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
ctx = bench.Ctx(1, 0, 0, dev); pol = cb.default_policy(1); flush = bench.L2Flush(dev)
for wid in sys.argv[1:] or ["G1", "R1", "G2", "G3"]:
    w = WL.WORKLOADS[wid]
    span = w.n if w.op == "dot" else w.m
    ins = bench.make_inputs(w, (0, span), dev)
    fn, _ = bench.step_fn(w, ins, pol, ctx, sharded_dot=False)
    times, _ = bench.time_steps(fn, 30, 5, ctx, flush)
    for _ in range(5): fn()
    torch.cuda.synchronize()
    K = 100
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K): fn()
    b.record(); torch.cuda.synchronize()
    t = a.elapsed_time(b) / K * 1e3
    print(json.dumps({"id": wid, "flushed_us": round(statistics.mean(times) * 1e3, 2), "b2b_us": round(t, 2),
                      "b2b_gbs": round(w.alg_bytes(1) / t / 1e3, 1)}), flush=True)
    del ins, fn; torch.cuda.empty_cache()
