"""The multi-GPU Python path on the GPU: torch.distributed over NCCL at world
size 1 (this pool has one GPU per box), through paper_2108_02025_b200.shard
and through bench.py under torchrun.  World sizes 2-3 run over gloo on the
CPU (tests/test_shard_gloo.py); this checks the NCCL collectives, the device
combine and the torchrun launch contract on real hardware."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, %(root)r)
import paper_2108_02025_b200 as cb
from paper_2108_02025_b200 import shard
dev = torch.device('cuda:0'); torch.cuda.set_device(dev)
dist.init_process_group('nccl', rank=0, world_size=1, device_id=dev)
pol = cb.default_policy(1)
f = lambda n, st: cb.fill_uniform(torch.empty(n, device=dev), 3, st)
x, y = f(1_000_003, 1), f(1_000_003, 2)
out = torch.empty(1, device=dev)
shard.sharded_dot(x, y, 0.75, out, pol)
direct = cb.dot(x, y, 0.75, pol)
assert out.item() == direct, (out.item(), direct)
m, n = 5000, 3000
A = cb.DenseMatrix.wrap(f(m * n, 3), m, n, cb.Layout.RowMajor)
xv, c = f(n, 4), f(m, 5)
c2 = c.clone()
full = shard.sharded_gemv_rows(A, xv, c, pol, gather=True, m_total=m)
cb.gemv_row_major(A, xv, c2, pol)
assert torch.equal(full, c2) and torch.equal(c, c2)
# col-major by columns (world 1): c + (0 + A x) == the direct call bitwise
mc, nc = 256, 100_003
Ac = cb.DenseMatrix.wrap(f(mc * nc, 6), mc, nc, cb.Layout.ColMajor)
xc, cc = f(nc, 7), f(mc, 8)
cc2 = cc.clone()
shard.sharded_gemv_cols(Ac, xc, cc, pol)
cb.gemv_col_major(Ac, xc, cc2, pol)
assert torch.equal(cc, cc2)
# the rank-ordered row combine itself, against an ordered sum on the host
parts = f(3 * 1000, 9).view(3, 1000)
c3 = f(1000, 10)
want = c3.cpu().clone()
acc = torch.zeros(1000)
for g in range(3):
    acc = acc + parts[g].cpu()
want = want + acc
shard._device_combine_rows(parts.reshape(-1), 3, c3)
assert torch.equal(c3.cpu(), want)
dist.destroy_process_group()
print('ok')
"""


def test_nccl_world1_shard_paths(cuda):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29561")
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": str(ROOT)}], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert r.stdout.strip().endswith("ok")


def test_bench_under_torchrun_world1(cuda):
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "1", "--master-addr", "127.0.0.1", "--master-port",
                        "29562", str(ROOT / "bench.py"), "--gpus", "1", "--steps", "20",
                        "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--no-suite"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 1000 and d["gpu_launches"] == 20
