#!/usr/bin/env python
"""Col-major GEMV with few rows (m < 1024) and A off a 16-byte boundary, next
to the aligned case (flushed).  CABL_CM_BULK_ANY=0 gives the scalar 2-D split
(before)."""
import os as _os
_os.environ.setdefault("CABL_TUNING", "1")  # exploration script: honour CABL_* knobs
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch  # noqa: E402

import paper_2108_02025_b200 as cb  # noqa: E402
from ger_odd import buf, timeit  # noqa: E402

pol = cb.default_policy(1)
for dt in (torch.float32, torch.float64):
    s = torch.tensor([], dtype=dt).element_size()
    N = (256 << 20) // s
    for m, off in ((1000, 1), (1000, 0), (257, 1), (256, 1), (256, 0), (3, 1), (100, 3), (100, 0),
                   (600, 2)):
        n = N // m
        A, x, c = buf(m * n, off, dt), buf(n, 0, dt), buf(m, 0, dt)
        Am = cb.DenseMatrix.wrap(A, m, n, cb.Layout.ColMajor)
        us = timeit(lambda: cb.gemv_col_major(Am, x, c, pol))
        print(json.dumps({"dtype": str(dt)[6:], "m": m, "n": n, "off": off, "us": round(us, 2),
                          "gbs": round((m * n + n + 2 * m) * s / us / 1e3, 1)}), flush=True)
        del A, x, c, Am
