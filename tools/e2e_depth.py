#!/usr/bin/env python
"""Resident-operator e2e (GemvPipeline) on G1 at pipeline depth 1..6 —
exploration for bench.py's e2e pattern.  --distinct gives every in-flight
request its own copy of A (no L2 sharing between concurrent kernels)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
import paper_2108_02025_b200 as cb
from paper_2108_02025_b200 import workloads as WL
from paper_2108_02025_b200.operators import GemvPipeline, ResidentGemv
dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
w = WL.WORKLOADS["G1"]
ins = bench.make_inputs(w, (0, w.m), dev)
pol = cb.default_policy(1)
distinct = "--distinct" in sys.argv
for depth in (1, 2, 3, 4, 6):
    pipe = GemvPipeline(ins["A"], pol, depth=depth)
    if distinct:
        mats = [cb.DenseMatrix.wrap(ins["A"].data.clone(), w.m, w.n, ins["A"].layout())
                for _ in range(depth)]
        pipe.ops = [ResidentGemv(M, pol) for M in mats]
    for op in pipe.ops:
        op.x_host.copy_(ins["x"].cpu()); op.c_host.copy_(ins["c"].cpu())
    for _ in range(20): pipe.step()
    pipe.drain()
    K = 2000
    t0 = time.perf_counter()
    for _ in range(K): pipe.step()
    pipe.drain()
    t = (time.perf_counter() - t0) / K
    print(json.dumps({"distinct_A": distinct, "depth": depth, "us_per_step": round(t * 1e6, 2),
                      "gbs": round(w.alg_bytes(1) / t / 1e9, 1)}), flush=True)
    del pipe
    torch.cuda.empty_cache()
