#!/usr/bin/env python
"""World-1 torch.distributed (NCCL) timing of the Python multi-GPU paths,
back to back: the NCCL-collective versions against the peer-memory ones
(shard.py).  At world 1 the collectives move nothing, so the difference is the
cost of the extra launches / collective calls the fused paths remove."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2108_02025_b200 as cb  # noqa: E402
from paper_2108_02025_b200 import shard  # noqa: E402


def timed(fn, k=100, warm=10):
    for _ in range(warm):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) * 1000.0 / k, 2)


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29577")
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    pol = cb.default_policy(1)
    f = lambda k, st: cb.fill_uniform(torch.empty(k, device=dev), 1, st)  # noqa: E731
    n = 1 << 24
    x, y, out = f(n, 1), f(n, 2), torch.empty(1, device=dev)
    g = torch.empty(1, device=dev)
    mb = shard.PeerMailboxes(dev)
    print(json.dumps({"op": "DOT 2^24", "nccl_us": timed(lambda: shard.sharded_dot(x, y, 0.0, out, pol, gathered=g)),
                      "peer_us": timed(lambda: shard.sharded_dot_fused(x, y, 0.0, out, pol, mb))}), flush=True)
    for m, k in ((8192, 8192), (8192, 65536)):
        A = cb.DenseMatrix.wrap(f(m * k, 3), m, k, cb.Layout.RowMajor)
        xv, c = f(k, 1), f(m, 4)
        gg = shard.GatherGemv(dev, m, torch.float32)
        print(json.dumps({"op": f"GEMV {m}x{k} + c gather",
                          "nccl_us": timed(lambda: shard.sharded_gemv_rows(A, xv, c, pol, gather=True, m_total=m)),
                          "peer_us": timed(lambda: gg(A, xv, c, 0))}), flush=True)
        gg.close()
        del A
    m, k = 256, 1 << 20
    A = cb.DenseMatrix.wrap(f(m * k, 3), m, k, cb.Layout.ColMajor)
    xv, c = f(k, 1), f(m, 4)
    pr = shard.PeerRows(dev, m, torch.float32)
    print(json.dumps({"op": f"col-sharded GEMV {m}x{k}",
                      "nccl_us": timed(lambda: shard.sharded_gemv_cols(A, xv, c, pol)),
                      "peer_us": timed(lambda: shard.sharded_gemv_cols_fused(A, xv, c, pol, pr))}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
