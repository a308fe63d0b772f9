#!/usr/bin/env python
"""Cost of the GPU-count-invariant DOT (shard.sharded_dot_invariant: one launch per fixed
global segment + an index-ordered combine) against the plain one-launch DOT, on one GPU:
D2 (n = 2^32, also its 8-GPU shard 2^29) and D1 (2^24), back to back, device events."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200 import shard
    dev = torch.device("cuda:0")
    pol = cb.default_policy(1)

    def timed(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        torch.cuda._sleep(1_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e3 / reps

    for n in (1 << 32, 1 << 29, 1 << 24):
        x = cb.fill_uniform(torch.empty(n, dtype=torch.float32, device=dev), 42, 1)
        y = cb.fill_uniform(torch.empty(n, dtype=torch.float32, device=dev), 42, 2)
        out = torch.zeros(1, device=dev)
        reps = 10 if n >= (1 << 29) else 100
        plain = timed(lambda: cb.dot_into(x, y, 0.0, out, pol), reps)
        v_plain = float(out.item())
        row = {"n": n, "plain_us": round(plain, 2), "plain_gbs": round(8 * n / plain / 1e3, 1)}
        for seg in (1 << 26, 1 << 24, 1 << 22):
            if seg > n:
                continue
            us = timed(lambda: shard.sharded_dot_invariant(x, y, 0.0, out, pol, n_total=n,
                                                           segment=seg), reps)
            row[f"seg2^{seg.bit_length() - 1}_us"] = round(us, 2)
            row[f"seg2^{seg.bit_length() - 1}_gbs"] = round(8 * n / us / 1e3, 1)
            row[f"seg2^{seg.bit_length() - 1}_value_minus_plain"] = float(out.item()) - v_plain
        print(json.dumps(row), flush=True)
        del x, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
