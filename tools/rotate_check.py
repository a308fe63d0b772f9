#!/usr/bin/env python
"""Back-to-back GER steps over rotating copies of an L2-sized shard (what
bench.time_rotating runs for an R1 shard at N = 8: 1024 x 8192 fp32, 32 MiB of C), for

    ncu --cache-control none --clock-control none -k regex:ger_ \\
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum ...

to show that every launch reads its C from DRAM and that the writes reach DRAM at the
same rate (no launch runs out of L2)."""
import dataclasses
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import bench
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200 import workloads as WL
    ranks = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    dev = torch.device("cuda:0")
    ctx = bench.Ctx(1, 0, 0, dev)
    pol = cb.default_policy(1)
    w = WL.WORKLOADS["R1"]
    b, e = w.shard_rows(0, ranks)
    wl = dataclasses.replace(w, m=e - b)
    R = bench.rotating_copies(wl.footprint_bytes())
    fns = [bench.step_fn(wl, bench.make_inputs(w, (b, e), dev), pol, ctx, sharded_dot=False)[0]
           for _ in range(R)]
    for k in range(4 * R):
        fns[k % R]()
    torch.cuda.synchronize()
    print(f"ranks={ranks} shard={e - b}x{w.n} copies={R}")


if __name__ == "__main__":
    main()
