#!/usr/bin/env python
"""Row-major GEMV with few long rows at 256 MiB of A, L2 flushed per rep:
the default dispatch vs the chunked few-rows kernel (CABL_GEMV_RM_MODE=9),
and a bitwise run-to-run + oracle-tolerance spot check of the forced mode."""
import os as _os
_os.environ.setdefault("CABL_TUNING", "1")  # exploration script: honour CABL_* knobs
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_02025_b200 as cb  # noqa: E402
from ger_odd import buf, timeit  # noqa: E402

pol = cb.default_policy(1)
for dt in (torch.float32, torch.float64):
    s = torch.tensor([], dtype=dt).element_size()
    total = (256 << 20) // s
    for m in (1, 2, 4, 16, 64, 256, 1024, 2048, 4096):
        n = total // m
        A, x, c = buf(m * n, 0, dt), buf(n, 0, dt), buf(m, 0, dt)
        Am = cb.DenseMatrix.wrap(A, m, n, cb.Layout.RowMajor)
        c1, c2 = c.clone(), c.clone()
        cb.gemv_row_major(Am, x, c1, pol)
        cb.gemv_row_major(Am, x, c2, pol)
        ref = c.double() + (A.view(m, n).double() @ x.double())
        err = float(((c1.double() - ref).abs() / (A.view(m, n).double().abs() @ x.double().abs() + 1)).max())
        us = timeit(lambda: cb.gemv_row_major(Am, x, c, pol))
        nbytes = (m * n + n + 2 * m) * s
        print(json.dumps({"mode": os.environ.get("CABL_GEMV_RM_MODE", "default"),
                          "dtype": str(dt)[6:], "m": m, "n": n, "us": round(us, 2),
                          "gbs": round(nbytes / us / 1e3, 1), "bitwise_rerun": bool(torch.equal(c1, c2)),
                          "rel_err": err}), flush=True)
        del A, x, c, Am, c1, c2
