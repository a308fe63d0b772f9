#!/usr/bin/env python
"""GER R1 (fp32 8192^2) through the host-buffer call on pinned memory (the
full-duplex slab pipeline, csrc/capi.cu host_ger_pipelined) under the
CABL_GER_PIPE="slabs,min_mib" variant of this process; median of 7 calls."""
import os as _os
_os.environ.setdefault("CABL_TUNING", "1")
import json
import os
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2108_02025_b200 as cb
    pol = cb.default_policy(1)
    m = n = 8192
    x = torch.rand(m).pin_memory()
    y = torch.rand(n).pin_memory()
    C = cb.DenseMatrix.wrap(torch.rand(m * n).pin_memory(), m, n, cb.Layout.RowMajor)
    cb.ger(x, y, C, pol)
    ts = []
    for _ in range(7):
        t0 = time.perf_counter()
        cb.ger(x, y, C, pol)
        ts.append(time.perf_counter() - t0)
    ms = statistics.median(ts) * 1e3
    print(json.dumps({"pipe": os.environ.get("CABL_GER_PIPE", "default"), "ms": round(ms, 3),
                      "gbs": round(2 * m * n * 4 / ms / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
