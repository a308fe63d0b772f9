#!/usr/bin/env python
"""Time BASELINE configs with bench.py's method (per-step CUDA events, L2
flushed between steps) and print one JSON line per config.  Kernel variants
are selected through the library's CABL_* tuning environment variables, so
run one process per variant:

    CABL_GEMV_RM_MODE=1 python tools/tune.py G1 G4
"""
from __future__ import annotations

import os as _os
_os.environ.setdefault("CABL_TUNING", "1")  # exploration script: honour CABL_* knobs
import json
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200 import workloads as WL

    ids = sys.argv[1:] or list(WL.WORKLOADS)
    steps = int(os.environ.get("TUNE_STEPS", "40"))
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    ctx = bench.Ctx(1, 0, 0, dev)
    flush = bench.L2Flush(dev)
    pol = cb.default_policy(1)
    env = {k: v for k, v in os.environ.items() if k.startswith("CABL_")}
    for wid in ids:
        w = WL.WORKLOADS[wid]
        span = w.n if w.op == "dot" else w.m
        ins = bench.make_inputs(w, (0, span), dev)
        fn, _ = bench.step_fn(w, ins, pol, ctx, sharded_dot=False)
        times, _ = bench.time_steps(fn, steps, 5, ctx, flush)
        mean = statistics.mean(times) * 1e3
        med = statistics.median(times) * 1e3
        print(json.dumps({"id": wid, "env": env, "mean_us": round(mean, 2), "median_us": round(med, 2),
                          "gbs_mean": round(w.alg_bytes(1) / mean / 1e3, 1),
                          "frac": round(w.alg_bytes(1) / mean / 1e3 / bench.peaks()[0], 4),
                          "probe_ctas": cb.last_exec().threads_used}), flush=True)
        del ins, fn
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
