#!/usr/bin/env python
"""Launch one BASELINE config's kernel a few times (L2 flushed in between) —
the small, fixed command that ncu captures for profiles/.

    python tools/ncu_runner.py --config G1 --reps 3

Launch order per rep: flush write, flush read, the hot-path kernel — so with
`-k regex:<kernel>` ncu sees exactly `reps` launches of the kernel under test.
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200 import workloads as WL

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="G1")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-flush", action="store_true",
                    help="back-to-back launches (for DRAM-traffic checks without a flush)")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    w = WL.WORKLOADS[args.config]
    span = w.n if w.op == "dot" else w.m
    ins = bench.make_inputs(w, (0, span), dev)
    ctx = bench.Ctx(1, 0, 0, dev)
    fn, _ = bench.step_fn(w, ins, cb.default_policy(1), ctx, sharded_dot=False)
    flush = bench.L2Flush(dev)
    for _ in range(args.reps):
        if not args.no_flush:
            flush.zero_()
        fn()
    torch.cuda.synchronize()
    print(f"ran {args.reps} x {w.id}")


if __name__ == "__main__":
    main()
