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
    ap.add_argument("--cm", default="",
                    help="col-major GEMV of shape MxN[:f64] instead of a config (e.g. 16384x4096)")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    ctx = bench.Ctx(1, 0, 0, dev)
    pol = cb.default_policy(1)
    if args.cm:
        shape, _, dts = args.cm.partition(":")
        m, n = (int(v) for v in shape.split("x"))
        dt = torch.float64 if dts == "f64" else torch.float32
        A = cb.DenseMatrix.wrap(cb.fill_uniform(torch.empty(m * n, dtype=dt, device=dev), WL.SEED,
                                                WL.STREAM_A), m, n, cb.Layout.ColMajor)
        x = cb.fill_uniform(torch.empty(n, dtype=dt, device=dev), WL.SEED, WL.STREAM_X)
        c = cb.fill_uniform(torch.empty(m, dtype=dt, device=dev), WL.SEED, WL.STREAM_C)
        fn = lambda: cb.gemv_col_major(A, x, c, pol)  # noqa: E731

        class w:  # noqa: N801
            id = "CM" + args.cm
    elif args.config == "R1x":  # GER fp32 8192 x 8193: odd rows (ger_flat_any_kernel)
        m, n = 8192, 8193
        x = cb.fill_uniform(torch.empty(m, device=dev), WL.SEED, WL.STREAM_X)
        y = cb.fill_uniform(torch.empty(n, device=dev), WL.SEED, WL.STREAM_Y)
        C = cb.DenseMatrix.wrap(cb.fill_uniform(torch.empty(m * n, device=dev), WL.SEED,
                                                WL.STREAM_CC), m, n, cb.Layout.RowMajor)
        fn = lambda: cb.ger(x, y, C, pol)  # noqa: E731

        class w:  # noqa: N801
            id = "R1x"
    elif args.config == "CM4096":  # col-major GEMV fp32 4096 x 16384 (the 2-D split)
        m, n = 4096, 16384
        A = cb.DenseMatrix.wrap(cb.fill_uniform(torch.empty(m * n, device=dev), WL.SEED,
                                                WL.STREAM_A), m, n, cb.Layout.ColMajor)
        x = cb.fill_uniform(torch.empty(n, device=dev), WL.SEED, WL.STREAM_X)
        c = cb.fill_uniform(torch.empty(m, device=dev), WL.SEED, WL.STREAM_C)
        fn = lambda: cb.gemv_col_major(A, x, c, pol)  # noqa: E731

        class w:  # noqa: N801
            id = "CM4096"
    elif args.config in ("RM1024", "RM1001"):  # row-major GEMV fp32, 4 KiB rows: the sub-CTA
        # sweep (65536 x 1024) and its scalar variant for odd rows (67041 x 1001)
        m, n = (65536, 1024) if args.config == "RM1024" else (67041, 1001)
        A = cb.DenseMatrix.wrap(cb.fill_uniform(torch.empty(m * n, device=dev), WL.SEED,
                                                WL.STREAM_A), m, n, cb.Layout.RowMajor)
        x = cb.fill_uniform(torch.empty(n, device=dev), WL.SEED, WL.STREAM_X)
        c = cb.fill_uniform(torch.empty(m, device=dev), WL.SEED, WL.STREAM_C)
        fn = lambda: cb.gemv_row_major(A, x, c, pol)  # noqa: E731

        class w:  # noqa: N801
            id = args.config
    elif args.config == "G1g":  # G1 through the gathering GEMV at world 1 (gemv_rm_gather_kernel)
        from paper_2108_02025_b200 import shard
        w = WL.WORKLOADS["G1"]
        ins = bench.make_inputs(w, (0, w.m), dev)
        gg = shard.GatherGemv(dev, w.m, w.dtype)
        fn = lambda: gg(ins["A"], ins["x"], ins["c"], 0)  # noqa: E731
    else:
        # D1f: D1 through the fused peer-memory DOT at world 1 (dot_peer_kernel)
        fused = args.config == "D1f"
        w = WL.WORKLOADS["D1" if fused else args.config]
        span = w.n if w.op == "dot" else w.m
        ins = bench.make_inputs(w, (0, span), dev)
        fn, _ = bench.step_fn(w, ins, pol, ctx, sharded_dot=False, fused=fused)
    flush = bench.L2Flush(dev)
    for _ in range(args.reps):
        if not args.no_flush:
            flush.zero_()
        fn()
    torch.cuda.synchronize()
    print(f"ran {args.reps} x {w.id}")


if __name__ == "__main__":
    main()
