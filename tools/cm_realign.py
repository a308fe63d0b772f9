#!/usr/bin/env python
"""Col-major GEMV with misaligned columns (odd m >= 1024, or A offset from a
32-byte boundary) against the aligned neighbour, L2 flushed per rep.  Run with
CABL_CM_REALIGN=0 (the scalar 2-D split) and 1 (gemv_cm_split_realign_kernel)
for the before/after."""
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
    for m, n, off in ((8192, 8192, 0), (8193, 8192, 0), (8192, 8192, 1), (1025, 65536, 0),
                      (4097, 16384, 0), (65537, 1024, 0), (100_003, 671, 0), (2048, 32768, 3)):
        if dt == torch.float64:
            n //= 2
        A, x, c = buf(m * n, off, dt), buf(n, 0, dt), buf(m, 0, dt)
        Am = cb.DenseMatrix.wrap(A, m, n, cb.Layout.ColMajor)
        us = timeit(lambda: cb.gemv_col_major(Am, x, c, pol))
        nbytes = (m * n + n + 2 * m) * s
        print(json.dumps({"dtype": str(dt)[6:], "m": m, "n": n, "off": off, "us": round(us, 2),
                          "gbs": round(nbytes / us / 1e3, 1)}), flush=True)
        del A, x, c, Am
