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


def test_rotating_copies_time_an_l2_sized_shard_from_hbm(cuda):
    """bench.time_rotating on the R1 shard of an 8-GPU run (1024 x 8192 fp32, 32 MiB of
    C): back to back over rotating copies it must be slower than the same steps on one
    buffer (which never leave L2) — the copies really push each other out — and the
    GER results must still be bitwise ger_ref on every copy."""
    import dataclasses

    import numpy as np
    import torch
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_2108_02025_b200 as cb
    from oracle import oracle as O
    from paper_2108_02025_b200 import workloads as WL
    dev = torch.device("cuda:0")
    ctx = bench.Ctx(1, 0, 0, dev)
    pol = cb.default_policy(1)
    flush = bench.L2Flush(dev)
    w = WL.WORKLOADS["R1"]
    b, e = w.shard_rows(0, 8)
    wl = dataclasses.replace(w, m=e - b)
    assert bench.l2_mode(wl.footprint_bytes()) == "flush"
    R = bench.rotating_copies(wl.footprint_bytes())
    assert R * wl.footprint_bytes() > 2 * bench.L2_BYTES
    ins = [bench.make_inputs(w, (b, e), dev) for _ in range(R)]
    C0 = ins[0]["C"].data.cpu().numpy().copy()
    fns = [bench.step_fn(wl, i, pol, ctx, sharded_dot=False)[0] for i in ins]
    steps = 3 * R
    rot = bench.time_rotating(fns, steps, 0, ctx, flush, charge_writeback=True)
    one, _ = bench.time_steps(fns[0], steps, 3, ctx, flush, mode="stream")
    assert len(rot) == steps and rot[0] > 0
    assert rot[0] > 1.1 * one[0], (rot[0], one[0])  # measured 12.7 vs 8.4 us
    # copy 1 took 1 warm-up turn (R calls over R copies) + steps / R = 3 timed ones
    x = ins[1]["x"].cpu().numpy()
    y = ins[1]["y"].cpu().numpy()
    want = np.ascontiguousarray(C0)
    for _ in range(4):
        O.ger_ref(x, y, want, 0)  # in place, row-major
    got = ins[1]["C"].data.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_bench_suite_watchdog_keeps_the_headline(cuda):
    """A suite that does not finish in time (at N > 1: a dead rank or a hung
    collective) must not take the headline down: the line is printed with the suite
    marked as timed out and the process exits 0."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "20", "--warmup", "3",
                        "--no-e2e", "--no-cpu-baseline", "--suite-timeout", "0.05"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["value"] > 1000 and d["roofline"]["frac"] > 0.5
    assert "watchdog" in d["suite"]["error"]


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_invariant_dot_gives_the_same_bits_for_every_gpu_count(cuda, dtype):
    """shard.sharded_dot_invariant: fixed global segments, one partial per segment,
    summed in index order.  The per-rank work of 1, 2, 3, 4 and 8 GPUs is run here in
    turn on one device (each rank's launches are independent of the others: nothing
    waits on a peer) and combined as the all-gather would deliver it: every GPU count
    gives the same bits, equal to the real call at world size 1, and within the
    contract bound of dot_ref."""
    import numpy as np
    import torch
    sys.path.insert(0, str(ROOT))
    import paper_2108_02025_b200 as cb
    from oracle import oracle as O
    from paper_2108_02025_b200 import shard
    from tests import tolerances as T
    dt = getattr(torch, dtype)
    seg = 1 << 20
    n = 11 * seg + 12_345  # 12 segments, the last one ragged
    dev = torch.device("cuda:0")
    x = cb.fill_uniform(torch.empty(n, dtype=dt, device=dev), 42, 1)
    y = cb.fill_uniform(torch.empty(n, dtype=dt, device=dev), 42, 2)
    pol = cb.default_policy(1)
    real = torch.zeros(1, dtype=dt, device=dev)
    shard.sharded_dot_invariant(x, y, 0.75, real, pol, n_total=n, segment=seg)
    for G in (1, 2, 3, 4, 8):
        pieces = []
        for g in range(G):
            b, e = shard.invariant_range(n, seg, G, g)
            kb, ke = shard.invariant_segments(n, seg, G, g)
            # a rank's shard is its own allocation (as on its own GPU), 256-byte aligned
            xs, ys = x[b:e].clone(), y[b:e].clone()
            pieces.append(shard.invariant_partials(xs, ys, seg, pol)[:ke - kb])
        out = torch.zeros(1, dtype=dt, device=dev)
        shard._device_combine(torch.cat(pieces), 0.75, out)
        assert torch.equal(out, real), G
    xn, yn = x.cpu().numpy(), y.cpu().numpy()
    truth, sumabs = O.dot_truth(xn, yn, 0.75)
    got = float(real.item())
    assert abs(got - O.dot_ref(xn, yn, 0.75)) <= T.contract_tol(n, sumabs, 0.75, xn.dtype.type)
    assert abs(got - truth) <= 4 * n * np.finfo(xn.dtype).eps * (sumabs + 0.75)
