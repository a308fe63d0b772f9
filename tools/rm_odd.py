#!/usr/bin/env python
"""Row-major GEMV with rows that are not whole 32-byte vectors, or a
misaligned A, against the aligned neighbour (flushed).  CABL_RM_SCALAR_CTA=0|1
forces the G-lanes / CTA-per-row scalar kernels."""
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
    for m, n, off in ((8192, 8192, 0), (8192, 8193, 0), (8192, 8192, 1), (8192, 8196, 0),
                      (16384, 4097, 0), (65536, 1025, 0), (4096, 16385, 0), (30000, 255, 0),
                      (20000, 2052, 0), (2400, 27961, 3), (1000, 65537, 0), (300, 100001, 1),
                      (4000, 16385, 0)):
        if dt == torch.float64:
            m //= 2
        A, x, c = buf(m * n, off, dt), buf(n, 0, dt), buf(m, 0, dt)
        Am = cb.DenseMatrix.wrap(A, m, n, cb.Layout.RowMajor)
        us = timeit(lambda: cb.gemv_row_major(Am, x, c, pol))
        print(json.dumps({"dtype": str(dt)[6:], "m": m, "n": n, "off": off, "us": round(us, 2),
                          "gbs": round((m * n + n + 2 * m) * s / us / 1e3, 1)}), flush=True)
        del A, x, c, Am
