"""Row-major GEMV with the c all-gather fused into the kernel (csrc/peer_gemv.cu).

Contract: every rank's c slice gets exactly the bits of the plain
cabl_cuda_gemv_rm on its slice (same sweep body, same group shape), and after
call k every rank's gathered buffer half k & 1 holds the concatenation of all
ranks' slices, in row order.

These boxes have one GPU, so ranks > 1 run through the emulation entry point
(every rank's grid in ONE cooperative launch; mailboxes and gathered buffers
side by side on this device).  The real entry point runs at world size 1, under
torch.distributed NCCL too, and against a peer that never arrives.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _lib():
    from paper_2108_02025_b200 import _lib as L
    return L


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _alloc(nbytes):
    p = C.c_void_p()
    _lib().call("cabl_peer_alloc", nbytes, C.byref(p))
    return p.value


def _mbox():
    p = C.c_void_p()
    _lib().call("cabl_peer_mailbox_create", C.byref(p))
    return p.value


def _state(p):
    e, f = C.c_uint64(), C.c_uint64()
    _lib().call("cabl_peer_mailbox_state", C.c_void_p(p), C.byref(e), C.byref(f))
    return e.value, f.value


def _view(ptr, n, dtype):
    from paper_2108_02025_b200.shard import _CudaArray
    return torch.as_tensor(_CudaArray(ptr, n, dtype), device="cuda")


def _slices(m_total, world):
    from paper_2108_02025_b200.shard import partition
    return [partition(m_total, world, r) for r in range(world)]


def _inputs(m_total, n, dtype, seed=7):
    import paper_2108_02025_b200 as cb
    A = cb.fill_uniform(torch.empty(m_total * n, dtype=dtype, device="cuda"), seed, 3)
    x = cb.fill_uniform(torch.empty(n, dtype=dtype, device="cuda"), seed, 1)
    c = cb.fill_uniform(torch.empty(m_total, dtype=dtype, device="cuda"), seed, 4)
    return A, x, c


def _plain(A_s, x, c_s, n):
    import paper_2108_02025_b200 as cb
    m = c_s.numel()
    cb.gemv_row_major(cb.DenseMatrix.wrap(A_s, m, n, cb.Layout.RowMajor), x, c_s,
                      cb.default_policy(1))


# (world, rows per rank ~, n): slices of long aligned rows, all on the (2, 8, 1) sweep
CASES = [(1, 2000, 16384), (2, 1900, 16384), (3, 2001, 16384), (4, 1800, 10240), (8, 1780, 16384)]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("world,rows,n", CASES)
def test_emulated_gather_equals_plain_slices(cuda, dtype, world, rows, n):
    L = _lib()
    if dtype == torch.float64:
        n //= 2  # same vectors per row
    m_total = world * rows + (world > 2)  # ragged when world > 2
    A, x, c0 = _inputs(m_total, n, dtype)
    sl = _slices(m_total, world)
    s = torch.tensor([], dtype=dtype).element_size()
    sfx = "f32" if dtype == torch.float32 else "f64"
    bufs = [_alloc(2 * m_total * s) for _ in range(world)]
    mbs = [_mbox() for _ in range(world)]
    cs = [c0[b:e].clone() for b, e in sl]
    want = [c0[b:e].clone() for b, e in sl]
    P = C.c_void_p * world
    try:
        for call in range(1, 4):  # both halves, reused mailboxes
            L.call(f"cabl_cuda_gemv_rm_gather_emulate_{sfx}", world,
                   P(*[A[b * n:e * n].data_ptr() for b, e in sl]),
                   (C.c_uint64 * world)(*[e - b for b, e in sl]), n, P(*[x.data_ptr()] * world),
                   P(*[t.data_ptr() for t in cs]), (C.c_uint64 * world)(*[b for b, _ in sl]),
                   m_total, P(*bufs), P(*mbs), _stream())
            for r, (b, e) in enumerate(sl):
                _plain(A[b * n:e * n], x, want[r], n)
            torch.cuda.synchronize()
            full = torch.cat(want)
            for r in range(world):
                assert torch.equal(cs[r], want[r]), (call, r)
                half = _view(bufs[r] + (call & 1) * m_total * s, m_total, dtype)
                assert torch.equal(half, full), (call, r)
        for p in mbs:
            assert _state(p) == (3, 0)
    finally:
        for p in bufs:
            L.lib().cabl_peer_free(C.c_void_p(p))
        for p in mbs:
            L.lib().cabl_peer_mailbox_destroy(C.c_void_p(p))


def test_real_entry_world1_and_unsupported_shape(cuda):
    L = _lib()
    m, n = 3000, 16384
    A, x, c0 = _inputs(m, n, torch.float32)
    buf, mb = _alloc(2 * m * 4), _mbox()
    try:
        c, want = c0.clone(), c0.clone()
        for call in range(1, 4):
            p = L.Probe()
            L.call("cabl_cuda_gemv_rm_gather_f32", A.data_ptr(), m, n, x.data_ptr(), c.data_ptr(),
                   0, m, (C.c_void_p * 1)(buf), (C.c_void_p * 1)(mb), 1, 0, C.byref(p), _stream())
            _plain(A, x, want, n)
            torch.cuda.synchronize()
            assert torch.equal(c, want)
            assert torch.equal(_view(buf + (call & 1) * m * 4, m, torch.float32), want)
            assert p.variant == 4 and p.threads_used >= 1
        assert _state(mb) == (3, 0)
        # few rows: not the sweep kernel -> EINVAL, nothing launched
        with pytest.raises(ValueError, match="sweep"):
            L.call("cabl_cuda_gemv_rm_gather_f32", A.data_ptr(), 16, n, x.data_ptr(),
                   c.data_ptr(), 0, m, (C.c_void_p * 1)(buf), (C.c_void_p * 1)(mb), 1, 0, None,
                   _stream())
    finally:
        L.lib().cabl_peer_free(C.c_void_p(buf))
        L.lib().cabl_peer_mailbox_destroy(C.c_void_p(mb))


def test_absent_peer_times_out_instead_of_hanging(cuda):
    code = f"""
import sys, ctypes as C, torch
sys.path.insert(0, {str(ROOT)!r}); sys.path.insert(0, {str(ROOT / 'tests')!r})
import test_gpu_peer_gemv as T
L = T._lib()
m, n = 2000, 16384
A, x, c = T._inputs(2 * m, n, torch.float32)
bufs = [T._alloc(2 * 2 * m * 4) for _ in range(2)]
mbs = [T._mbox() for _ in range(2)]
L.call('cabl_cuda_gemv_rm_gather_f32', A.data_ptr(), m, n, x.data_ptr(), c.data_ptr(), 0, 2 * m,
       (C.c_void_p * 2)(*bufs), (C.c_void_p * 2)(*mbs), 2, 0, None, T._stream())
torch.cuda.synchronize()
assert T._state(mbs[0]) == (1, 1), T._state(mbs[0])
print('ok')
"""
    env = dict(os.environ, CABL_PEER_TIMEOUT_MS="300")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-3000:]


NCCL_SCRIPT = r"""
import sys, torch, torch.distributed as dist
sys.path.insert(0, %(root)r)
import paper_2108_02025_b200 as cb
from paper_2108_02025_b200 import shard
dev = torch.device('cuda:0'); torch.cuda.set_device(dev)
dist.init_process_group('nccl', rank=0, world_size=1, device_id=dev)
pol = cb.default_policy(1)
m, n = 4000, 16384
A = cb.DenseMatrix.wrap(cb.fill_uniform(torch.empty(m * n, device=dev), 5, 3), m, n, cb.Layout.RowMajor)
x = cb.fill_uniform(torch.empty(n, device=dev), 5, 1)
c = cb.fill_uniform(torch.empty(m, device=dev), 5, 4)
c2 = c.clone()
gg = shard.GatherGemv(dev, m, torch.float32)
for k in range(3):
    full = gg(A, x, c, 0)
    ref = shard.sharded_gemv_rows(A, x, c2, pol, gather=True, m_total=m)
    torch.cuda.synchronize()
    assert torch.equal(c, c2) and torch.equal(full, ref), k
assert gg.state() == (3, 0)
gg.close()
dist.destroy_process_group()
print('ok')
"""


def test_gather_gemv_under_nccl_world1(cuda):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29564")
    r = subprocess.run([sys.executable, "-c", NCCL_SCRIPT % {"root": str(ROOT)}], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-3000:]


@pytest.mark.parametrize("seed", range(6))
def test_random_emulated_gathers(cuda, seed):
    """Random world sizes, ragged slices, dtypes and offsets into the gathered
    buffer: every rank's half equals the concatenation of the plain slices."""
    import numpy as np
    L = _lib()
    rng = np.random.default_rng(seed)
    world = int(rng.integers(1, 9))
    dtype = torch.float32 if rng.integers(0, 2) == 0 else torch.float64
    n = 9216 if dtype == torch.float32 else 4608  # long rows (> 1024 vectors)
    ms = [int(v) for v in rng.integers(300, 1500, size=world)]
    m_total = sum(ms)
    offs = [sum(ms[:r]) for r in range(world)]
    A, x, c0 = _inputs(m_total, n, dtype, seed)
    s = torch.tensor([], dtype=dtype).element_size()
    sfx = "f32" if dtype == torch.float32 else "f64"
    bufs = [_alloc(2 * m_total * s) for _ in range(world)]
    mbs = [_mbox() for _ in range(world)]
    cs = [c0[o:o + m].clone() for o, m in zip(offs, ms)]
    want = [c0[o:o + m].clone() for o, m in zip(offs, ms)]
    P = C.c_void_p * world
    try:
        for call in range(1, 3):
            L.call(f"cabl_cuda_gemv_rm_gather_emulate_{sfx}", world,
                   P(*[A[o * n:(o + m) * n].data_ptr() for o, m in zip(offs, ms)]),
                   (C.c_uint64 * world)(*ms), n, P(*[x.data_ptr()] * world),
                   P(*[t.data_ptr() for t in cs]), (C.c_uint64 * world)(*offs), m_total,
                   P(*bufs), P(*mbs), _stream())
            for r, (o, m) in enumerate(zip(offs, ms)):
                _plain(A[o * n:(o + m) * n], x, want[r], n)
            torch.cuda.synchronize()
            full = torch.cat(want)
            for r in range(world):
                assert torch.equal(cs[r], want[r]), (seed, call, r)
                assert torch.equal(_view(bufs[r] + (call & 1) * m_total * s, m_total, dtype), full)
    finally:
        for p in bufs:
            L.lib().cabl_peer_free(C.c_void_p(p))
        for p in mbs:
            L.lib().cabl_peer_mailbox_destroy(C.c_void_p(p))
