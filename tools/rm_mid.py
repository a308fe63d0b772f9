#!/usr/bin/env python
"""Row-major GEMV, mid-size row counts at fixed bytes (flushed): the default
dispatch against the sweep kernel forced (CABL_GEMV_RM_MODE=2, CABL_RM_SWEEP,
CABL_GEMV_DYN) — the data behind the sweep's few-groups rule."""
import os as _os
_os.environ.setdefault("CABL_TUNING", "1")  # exploration script: honour CABL_* knobs
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch  # noqa: E402

import paper_2108_02025_b200 as cb  # noqa: E402
from ger_odd import buf, timeit  # noqa: E402

pol = cb.default_policy(1)
tag = "/".join(os.environ.get(k, "-") for k in ("CABL_GEMV_RM_MODE", "CABL_RM_SWEEP", "CABL_GEMV_DYN"))
for dt in (torch.float32, torch.float64):
    s = torch.tensor([], dtype=dt).element_size()
    for m, n in ((64, 1 << 20), (128, 1 << 19), (256, 1 << 18), (512, 1 << 17), (1024, 1 << 16),
                 (2048, 1 << 15), (4096, 1 << 14), (2048, 8192), (4096, 8192), (8192, 4096),
                 (16384, 4096), (4096, 4096)):
        if dt == torch.float64:
            n //= 2
        A, x, c = buf(m * n, 0, dt), buf(n, 0, dt), buf(m, 0, dt)
        Am = cb.DenseMatrix.wrap(A, m, n, cb.Layout.RowMajor)
        us = timeit(lambda: cb.gemv_row_major(Am, x, c, pol))
        print(json.dumps({"cfg": tag, "dtype": str(dt)[6:], "m": m, "n": n, "us": round(us, 2),
                          "gbs": round((m * n + n + 2 * m) * s / us / 1e3, 1)}), flush=True)
        del A, x, c, Am
