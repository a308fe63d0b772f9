#!/usr/bin/env python
"""One rank's share of the strong-scaled BASELINE configs, timed alone on ONE GPU.

The sharded configs (R1 row blocks, G4 row blocks, D2 chunks) need
no data-path exchange for R1 and only a latency-bound one for G4 / D2, so the device
time of rank 0's shard of an N-GPU run — the single-GPU kernel on m/N rows or n/N
elements — bounds what N GPUs can reach: efficiency(N) <= T(1) / (N * T_shard(N)).
This is NOT a multi-GPU measurement (no NCCL, no second device); it shows how much of
the strong-scaling loss is the shrinking per-GPU problem (launch floor, L2-resident
shards) before any exchange cost.

Timing is bench.py's own (`time_steps`): the L2 policy `bench.l2_mode` picks for the
shard (back to back when the shard's footprint exceeds L2, else back to back over
rotating copies of the operands, `bench.time_rotating`; flushed before every launch as
the conservative number), GER charged its L2 write-back when flushed or rotating.

    python tools/shard_share.py > gpurun_out/shard_share.jsonl
"""
from __future__ import annotations

import dataclasses
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
    pol = cb.default_policy(1)
    flush = bench.L2Flush(dev)
    peak, _ = bench.peaks()
    steps, warmup = 30, 5
    for wid in ("R1", "G4", "D2"):
        w = WL.WORKLOADS[wid]
        base = {}
        for N in (1, 2, 4, 8):
            b, e = WL.Workload.shard_rows(w, 0, N)
            ins = bench.make_inputs(w, (b, e), dev)
            wl = dataclasses.replace(w, n=e - b) if w.op == "dot" else dataclasses.replace(w, m=e - b)
            fn, _ = bench.step_fn(wl, ins, pol, ctx, sharded_dot=False)
            shard_bytes = wl.alg_bytes(1)
            policy = bench.l2_mode(wl.footprint_bytes())
            modes = ("stream", "flush") if policy == "stream" else ("stream", "flush", "rotate")
            for mode in modes:
                if mode == "rotate":  # what bench.py's suite reports for footprints <= L2
                    R = bench.rotating_copies(wl.footprint_bytes())
                    rot = [fn] + [bench.step_fn(wl, bench.make_inputs(w, (b, e), dev), pol, ctx,
                                                sharded_dot=False)[0] for _ in range(R - 1)]
                    k = max(steps, 3 * R)
                    times = bench.time_rotating(rot, k, warmup, ctx, flush,
                                                charge_writeback=w.op == "ger")
                    us = sum(times) / k * 1e3
                    del rot
                    base["rotate"] = base["stream"]  # N = 1 runs back to back either way
                else:
                    times, _ = bench.time_steps(fn, steps, warmup, ctx, flush, mode=mode,
                                                charge_writeback=(w.op == "ger" and mode == "flush"))
                    us = sum(times) / steps * 1e3
                base.setdefault(mode, us if N == 1 else base.get(mode))
                print(json.dumps({
                    "config": wid, "ranks": N, "shard": [e - b, w.n] if w.op != "dot" else [e - b],
                    "shard_bytes": shard_bytes, "mode": mode,
                    "policy_mode": "rotate" if policy == "flush" else policy,
                    "us_per_step": round(us, 2),
                    "shard_gbs": round(shard_bytes / us / 1e3, 1),
                    "shard_frac_of_peak": round(shard_bytes / us / 1e3 / peak, 4),
                    "scaling_bound": round(base[mode] / (N * us), 4),
                }), flush=True)
            del ins
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
