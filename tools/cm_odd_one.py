#!/usr/bin/env python
"""One col-major GEMV launch on 257 x 2^20 fp32 (for ncu)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2108_02025_b200 as cb
dev = torch.device("cuda:0"); torch.cuda.set_device(dev)
m, n = 257, 1 << 20
A = cb.fill_uniform(torch.empty(m * n, device=dev), 1, 3)
x = cb.fill_uniform(torch.empty(n, device=dev), 1, 1)
c = torch.zeros(m, device=dev)
M = cb.DenseMatrix.wrap(A, m, n, cb.Layout.ColMajor)
for _ in range(2):
    cb.gemv_col_major(M, x, c, cb.default_policy(1))
torch.cuda.synchronize()
print("ok")
