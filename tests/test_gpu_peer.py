"""Peer-memory DOT (csrc/peer.cu): the sharded DOT with the exchange of
partials fused into the kernel.

Its contract is bitwise equality with the unfused path of shard.sharded_dot:
each rank's shard through cabl_cuda_dot(alpha0 = 0), then the rank-ordered
cabl_cuda_combine_partials (itself the reference's chunk-order sum then
+ alpha0, kernels.hpp:145-163), and the same value on every rank.

These boxes have one GPU, so ranks > 1 run through the emulation entry point:
the same kernel and mailbox protocol with every rank's grid in one cooperative
launch on this device (never separate launches that wait on each other).  The
real entry point runs at world size 1 — under torch.distributed NCCL too — and
against a mailbox table whose peer never arrives (the timeout path).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _lib():
    from paper_2108_02025_b200 import _lib as L
    return L


def _mailboxes(k):
    L = _lib()
    out = []
    for _ in range(k):
        p = C.c_void_p()
        L.call("cabl_peer_mailbox_create", C.byref(p))
        out.append(p.value)
    return out


def _destroy(ptrs):
    for p in ptrs:
        _lib().call("cabl_peer_mailbox_destroy", C.c_void_p(p))


def _state(p):
    e, f = C.c_uint64(), C.c_uint64()
    _lib().call("cabl_peer_mailbox_state", C.c_void_p(p), C.byref(e), C.byref(f))
    return e.value, f.value


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def unfused(xs, ys, alpha0, cutoff):
    """shard.sharded_dot's arithmetic on one device: per-shard DOT with alpha0 = 0,
    then the rank-ordered device combine."""
    L = _lib()
    sfx = "f32" if xs[0].dtype == torch.float32 else "f64"
    parts = torch.empty(len(xs), dtype=xs[0].dtype, device="cuda")
    for r, (x, y) in enumerate(zip(xs, ys)):
        L.call(f"cabl_cuda_dot_{sfx}", x.data_ptr() if x.numel() else None,
               y.data_ptr() if y.numel() else None, x.numel(), 0.0, parts[r:].data_ptr(), cutoff,
               None, _stream())
    out = torch.empty(1, dtype=xs[0].dtype, device="cuda")
    L.call(f"cabl_cuda_combine_partials_{sfx}", parts.data_ptr(), len(xs), float(alpha0),
           out.data_ptr(), _stream())
    return out


def emulate(xs, ys, alpha0, mboxes, cutoff):
    L = _lib()
    W = len(xs)
    sfx = "f32" if xs[0].dtype == torch.float32 else "f64"
    outs = [torch.full((1,), float("nan"), dtype=xs[0].dtype, device="cuda") for _ in range(W)]
    P = C.c_void_p * W
    xt = P(*[x.data_ptr() if x.numel() else None for x in xs])
    yt = P(*[y.data_ptr() if y.numel() else None for y in ys])
    nt = (C.c_uint64 * W)(*[x.numel() for x in xs])
    ot = P(*[o.data_ptr() for o in outs])
    mt = P(*mboxes)
    L.call(f"cabl_cuda_dot_peer_emulate_{sfx}", W, xt, yt, nt, float(alpha0), ot, mt, cutoff,
           _stream())
    return outs


def _shards(n_list, dtype, seed, misalign=0):
    import paper_2108_02025_b200 as cb
    xs, ys = [], []
    for r, n in enumerate(n_list):
        bx = torch.empty(n + misalign, dtype=dtype, device="cuda")
        by = torch.empty(n + misalign, dtype=dtype, device="cuda")
        if n + misalign:
            cb.fill_uniform(bx, seed, 2 * r + 1)
            cb.fill_uniform(by, seed, 2 * r + 2)
        xs.append(bx[misalign:])
        ys.append(by[misalign:])
    return xs, ys


CASES = [
    # (shard lengths, misaligned start)
    ([1 << 16], 0),
    ([300_001, 300_001], 0),
    ([100_000, 99_999, 1], 0),
    ([65_536, 0, 65_536, 17], 0),
    ([40_000] * 8, 0),
    ([77_777, 77_777], 3),   # x[3:], y[3:]: the peeled head path
    ([5, 9000, 12], 0),      # small shards: the 1-CTA path
]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("shards,mis", CASES)
def test_emulated_ranks_equal_unfused_bitwise(cuda, dtype, shards, mis):
    xs, ys = _shards(shards, dtype, 11, mis)
    cutoff = 8192
    want = unfused(xs, ys, 0.625, cutoff)
    mb = _mailboxes(len(shards))
    try:
        for call in range(5):  # > 2 calls: both parity slots, reused mailboxes
            outs = emulate(xs, ys, 0.625, mb, cutoff)
            torch.cuda.synchronize()
            for r, o in enumerate(outs):
                assert torch.equal(o, want), (call, r, o.item(), want.item())
        for p in mb:
            assert _state(p) == (5, 0)
    finally:
        _destroy(mb)


def test_emulated_sum_against_fp64_truth(cuda):
    xs, ys = _shards([123_457, 123_457, 123_456], torch.float32, 5)
    mb = _mailboxes(3)
    try:
        outs = emulate(xs, ys, -0.25, mb, 8192)
        torch.cuda.synchronize()
    finally:
        _destroy(mb)
    x = np.concatenate([t.cpu().numpy() for t in xs]).astype(np.float64)
    y = np.concatenate([t.cpu().numpy() for t in ys]).astype(np.float64)
    truth = -0.25 + float(x @ y)
    S = 0.25 + float(np.abs(x * y).sum())
    eps = float(np.finfo(np.float32).eps)
    for o in outs:
        assert abs(o.item() - truth) <= 64 * eps * S


def test_emulated_chunked_kernel(cuda):
    """The chunked (queue-scheduled) shard kernel + fused exchange, forced by
    CABL_DOT_CHUNKED=1 in a fresh process (the switch is read once)."""
    code = f"""
import sys, torch
sys.path.insert(0, {str(ROOT)!r}); sys.path.insert(0, {str(ROOT / 'tests')!r})
import test_gpu_peer as T
for dt in (torch.float32, torch.float64):
    xs, ys = T._shards([1 << 20, (1 << 20) + 8, 1 << 20], dt, 9)
    want = T.unfused(xs, ys, 1.5, 8192)
    mb = T._mailboxes(3)
    for _ in range(3):
        outs = T.emulate(xs, ys, 1.5, mb, 8192)
        torch.cuda.synchronize()
        assert all(torch.equal(o, want) for o in outs), ([o.item() for o in outs], want.item())
    T._destroy(mb)
print('ok')
"""
    env = dict(os.environ, CABL_TUNING="1", CABL_DOT_CHUNKED="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-3000:]


def test_emulation_rejects_what_does_not_fit_one_wave(cuda):
    xs, ys = _shards([1 << 24] * 4, torch.float32, 1)  # 4 x 296 CTAs > one wave
    mb = _mailboxes(4)
    try:
        with pytest.raises(ValueError, match="co-resident"):
            emulate(xs, ys, 0.0, mb, 8192)
    finally:
        _destroy(mb)


@pytest.mark.parametrize("n", [1_000_003, 1 << 27])  # grid-stride and chunked kernels
def test_real_entry_world1(cuda, n):
    L = _lib()
    xs, ys = _shards([n], torch.float32, 21)
    want = unfused(xs, ys, 0.5, 8192)
    mb = _mailboxes(1)
    try:
        out = torch.empty(1, device="cuda")
        p = L.Probe()
        for _ in range(3):
            L.call("cabl_cuda_dot_peer_f32", xs[0].data_ptr(), ys[0].data_ptr(), n, 0.5,
                   out.data_ptr(), (C.c_void_p * 1)(mb[0]), 1, 0, 8192, C.byref(p), _stream())
            torch.cuda.synchronize()
            assert torch.equal(out, want)
        assert p.variant == 2 and p.threads_used >= 2
        assert _state(mb[0]) == (3, 0)
    finally:
        _destroy(mb)
    del xs, ys
    torch.cuda.empty_cache()


def test_real_entry_in_a_cuda_graph(cuda):
    """The epoch lives in the mailbox, so graph replays stay in step."""
    L = _lib()
    xs, ys = _shards([2_000_000], torch.float64, 4)
    want = unfused(xs, ys, 0.0, 8192)
    mb = _mailboxes(1)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    tbl = (C.c_void_p * 1)(mb[0])
    s = torch.cuda.Stream()
    try:
        with torch.cuda.stream(s):
            L.call("cabl_cuda_dot_peer_f64", xs[0].data_ptr(), ys[0].data_ptr(), xs[0].numel(),
                   0.0, out.data_ptr(), tbl, 1, 0, 8192, None, C.c_void_p(s.cuda_stream))
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            L.call("cabl_cuda_dot_peer_f64", xs[0].data_ptr(), ys[0].data_ptr(), xs[0].numel(),
                   0.0, out.data_ptr(), tbl, 1, 0, 8192, None, C.c_void_p(s.cuda_stream))
        for _ in range(4):
            out.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(out, want)
        assert _state(mb[0]) == (5, 0)
    finally:
        _destroy(mb)


def test_absent_peer_times_out_instead_of_hanging(cuda):
    """Rank 0 of a 2-rank table whose rank 1 never calls: the kernel gives up
    after CABL_PEER_TIMEOUT_MS, writes NaN and records the epoch as a fault."""
    code = f"""
import sys, ctypes as C, math, torch
sys.path.insert(0, {str(ROOT)!r}); sys.path.insert(0, {str(ROOT / 'tests')!r})
import test_gpu_peer as T
L = T._lib()
xs, ys = T._shards([100_000], torch.float32, 2)
mb = T._mailboxes(2)
out = torch.zeros(1, device='cuda')
L.call('cabl_cuda_dot_peer_f32', xs[0].data_ptr(), ys[0].data_ptr(), 100_000, 0.0,
       out.data_ptr(), (C.c_void_p * 2)(*mb), 2, 0, 8192, None, T._stream())
torch.cuda.synchronize()
assert math.isnan(out.item()), out.item()
assert T._state(mb[0]) == (1, 1), T._state(mb[0])
assert T._state(mb[1])[0] == 0
T._destroy(mb)
print('ok')
"""
    env = dict(os.environ, CABL_PEER_TIMEOUT_MS="300")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-3000:]


def test_argument_errors(cuda):
    L = _lib()
    x = torch.ones(100, device="cuda")
    out = torch.empty(1, device="cuda")
    mb = _mailboxes(1)
    try:
        tbl = (C.c_void_p * 1)(mb[0])
        for world, rank, msg in [(0, 0, "world"), (9, 0, "world"), (1, 1, "rank")]:
            with pytest.raises(ValueError, match=msg):
                L.call("cabl_cuda_dot_peer_f32", x.data_ptr(), x.data_ptr(), 100, 0.0,
                       out.data_ptr(), tbl, world, rank, 8192, None, _stream())
        with pytest.raises(ValueError, match="null mailbox"):
            L.call("cabl_cuda_dot_peer_f32", x.data_ptr(), x.data_ptr(), 100, 0.0,
                   out.data_ptr(), (C.c_void_p * 2)(mb[0], None), 2, 0, 8192, None, _stream())
    finally:
        _destroy(mb)


NCCL_SCRIPT = r"""
import sys, torch, torch.distributed as dist
sys.path.insert(0, %(root)r)
import paper_2108_02025_b200 as cb
from paper_2108_02025_b200 import shard
dev = torch.device('cuda:0'); torch.cuda.set_device(dev)
dist.init_process_group('nccl', rank=0, world_size=1, device_id=dev)
pol = cb.default_policy(1)
mb = shard.PeerMailboxes(dev)
for dt in (torch.float32, torch.float64):
    x = cb.fill_uniform(torch.empty(3_000_017, dtype=dt, device=dev), 8, 1)
    y = cb.fill_uniform(torch.empty(3_000_017, dtype=dt, device=dev), 8, 2)
    a, b = torch.empty(1, dtype=dt, device=dev), torch.empty(1, dtype=dt, device=dev)
    shard.sharded_dot(x, y, -1.25, a, pol)
    for _ in range(3):
        shard.sharded_dot_fused(x, y, -1.25, b, pol, mb)
        torch.cuda.synchronize()
        assert torch.equal(a, b), (a.item(), b.item())
assert mb.state() == (6, 0), mb.state()
mb.close()
dist.destroy_process_group()
print('ok')
"""


def test_sharded_dot_fused_under_nccl_world1(cuda):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29563")
    r = subprocess.run([sys.executable, "-c", NCCL_SCRIPT % {"root": str(ROOT)}], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-3000:]


# ---------------------------------------------------------------------------
# Column-sharded GEMV combine over peer memory (cabl_cuda_combine_rows_peer_*)

def _unfused_rows(parts, c0):
    """The all-gather + cabl_cuda_combine_rows arithmetic on one device."""
    L = _lib()
    sfx = "f32" if c0.dtype == torch.float32 else "f64"
    c = c0.clone()
    stacked = torch.stack(parts).reshape(-1).contiguous()
    L.call(f"cabl_cuda_combine_rows_{sfx}", stacked.data_ptr(), len(parts), c.numel(),
           c.data_ptr(), _stream())
    return c


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("world,m", [(1, 256), (2, 256), (3, 1000), (8, 4097), (5, 1)])
def test_emulated_row_combine_equals_unfused_bitwise(cuda, dtype, world, m):
    import paper_2108_02025_b200 as cb
    L = _lib()
    sfx = "f32" if dtype == torch.float32 else "f64"
    s = torch.tensor([], dtype=dtype).element_size()
    parts = [cb.fill_uniform(torch.empty(m, dtype=dtype, device="cuda"), 3, 10 + r)
             for r in range(world)]
    c0 = cb.fill_uniform(torch.empty(m, dtype=dtype, device="cuda"), 3, 9)
    bufs = []
    for _ in range(world):
        p = C.c_void_p()
        L.call("cabl_peer_alloc", 2 * 8 * m * s, C.byref(p))
        bufs.append(p.value)
    mb = _mailboxes(world)
    cs = [c0.clone() for _ in range(world)]
    want = c0.clone()
    P = C.c_void_p * world
    try:
        for call in range(3):
            L.call(f"cabl_cuda_combine_rows_peer_emulate_{sfx}", world,
                   P(*[t.data_ptr() for t in parts]), m, P(*[t.data_ptr() for t in cs]),
                   P(*bufs), P(*mb), _stream())
            want = _unfused_rows(parts, want)
            torch.cuda.synchronize()
            for r in range(world):
                assert torch.equal(cs[r], want), (call, r)
        for p in mb:
            assert _state(p) == (3, 0)
    finally:
        for p in bufs:
            L.lib().cabl_peer_free(C.c_void_p(p))
        _destroy(mb)


COLS_SCRIPT = r"""
import sys, torch, torch.distributed as dist
sys.path.insert(0, %(root)r)
import paper_2108_02025_b200 as cb
from paper_2108_02025_b200 import shard
dev = torch.device('cuda:0'); torch.cuda.set_device(dev)
dist.init_process_group('nccl', rank=0, world_size=1, device_id=dev)
pol = cb.default_policy(1)
m, n = 256, 300_007
f = lambda k, st: cb.fill_uniform(torch.empty(k, dtype=torch.float64, device=dev), 6, st)
A = cb.DenseMatrix.wrap(f(m * n, 3), m, n, cb.Layout.ColMajor)
x, c = f(n, 1), f(m, 4)
c2 = c.clone()
peers = shard.PeerRows(dev, m, torch.float64)
for _ in range(3):
    shard.sharded_gemv_cols_fused(A, x, c, pol, peers)
    shard.sharded_gemv_cols(A, x, c2, pol)
    torch.cuda.synchronize()
    assert torch.equal(c, c2)
assert peers.state() == (3, 0)
peers.close()
dist.destroy_process_group()
print('ok')
"""


def test_sharded_gemv_cols_fused_under_nccl_world1(cuda):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29565")
    r = subprocess.run([sys.executable, "-c", COLS_SCRIPT % {"root": str(ROOT)}], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-3000:]


def test_emulated_protocol_stress(cuda):
    """Many back-to-back collective calls on reused mailboxes, 8 emulated
    ranks with uneven shards (ranks finish at different times): every call's
    result on every rank equals the unfused path, no fault, epochs in step."""
    xs, ys = _shards([40_000, 3, 70_000, 0, 12_345, 65_536, 1, 50_000], torch.float32, 17)
    want = unfused(xs, ys, -0.5, 8192)
    mb = _mailboxes(8)
    try:
        outs_all = []
        for _ in range(200):
            outs_all.append(emulate(xs, ys, -0.5, mb, 8192))
        torch.cuda.synchronize()
        for k, outs in enumerate(outs_all):
            for r, o in enumerate(outs):
                assert torch.equal(o, want), (k, r)
        for p in mb:
            assert _state(p) == (200, 0)
    finally:
        _destroy(mb)


@pytest.mark.parametrize("seed", range(10))
def test_random_emulated_dots(cuda, seed):
    """Random world sizes, shard lengths (incl. empty and tiny), dtypes, alpha0."""
    rng = np.random.default_rng(100 + seed)
    world = int(rng.integers(1, 9))
    dtype = torch.float32 if rng.integers(0, 2) == 0 else torch.float64
    # shards small enough that every rank's grid fits one co-resident wave
    shards = [int(rng.choice([0, rng.integers(1, 50), rng.integers(50, 20_000),
                              rng.integers(20_000, 60_000)])) for _ in range(world)]
    alpha = float(rng.uniform(-2, 2))
    xs, ys = _shards(shards, dtype, 40 + seed, int(rng.choice([0, 0, 2])))
    want = unfused(xs, ys, alpha, 8192)
    mb = _mailboxes(world)
    try:
        for _ in range(3):
            outs = emulate(xs, ys, alpha, mb, 8192)
            torch.cuda.synchronize()
            assert all(torch.equal(o, want) for o in outs), (seed, shards)
    finally:
        _destroy(mb)
