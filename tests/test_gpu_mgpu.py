"""The multi-GPU C ABI (cabl_mgpu_*) through ctypes on the devices of this
box (world = every visible GPU; 1 on the round's boxes, where the clique has
one member and the path still runs ncclCommInitAll, the collectives, the
rank-ordered combines and the fused peer kernels).  Every result is checked
bitwise against the same shards run one by one through the single-GPU C ABI,
plus the failure contract: a timed-out call raises CablExchangeError, aborts
the context, and every later call fails the same way instead of hanging."""
from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu

SEED = 42


def _dev_count():
    return torch.cuda.device_count()


def _fill(n, dtype, stream, dev, offset=0):
    import paper_2108_02025_b200 as cb
    t = torch.empty(n, dtype=dtype, device=dev)
    if n:
        cb.fill_uniform(t, SEED, stream, offset)
    return t


@pytest.fixture(scope="module")
def mg():
    from paper_2108_02025_b200.mgpu import MultiGpu
    ctx = MultiGpu(list(range(_dev_count())))
    yield ctx
    ctx.close()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("exchange", ["nccl", "peer"])
@pytest.mark.parametrize("n", [1000, (1 << 22) + 3])
def test_mgpu_dot_is_the_rank_ordered_sum(mg, dtype, exchange, n):
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200.mgpu import partition
    G = mg.size
    pol = cb.default_policy(1)
    xs, ys, expect = [], [], 0.0
    parts = []
    for r in range(G):
        b, e = partition(n, G, r)
        xs.append(_fill(e - b, dtype, 1, f"cuda:{r}", b))
        ys.append(_fill(e - b, dtype, 2, f"cuda:{r}", b))
        with torch.cuda.device(r):
            parts.append(cb.dot(xs[r], ys[r], 0.0, pol))
    # reference kernels.hpp:160-163: partials in order, alpha0 last (in T)
    acc = torch.zeros((), dtype=dtype)
    for p in parts:
        acc = acc + torch.tensor(p, dtype=dtype)
    expect = float(acc + torch.tensor(0.75, dtype=dtype))
    got = mg.dot(xs, ys, 0.75, pol, exchange=exchange)
    assert got == expect
    assert mg.dot(xs, ys, 0.75, pol, exchange=exchange) == got  # reproducible


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("exchange", ["nccl", "peer"])
@pytest.mark.parametrize("gather", [False, True])
def test_mgpu_gemv_rows_equal_per_shard_calls(mg, dtype, exchange, gather):
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200.mgpu import partition
    G = mg.size
    m, n = 8192, 4096
    pol = cb.default_policy(1)
    As, xs, cs, want = [], [], [], []
    for r in range(G):
        b, e = partition(m, G, r)
        dev = f"cuda:{r}"
        A = cb.DenseMatrix.wrap(_fill((e - b) * n, dtype, 3, dev, b * n), e - b, n, cb.Layout.RowMajor)
        x = _fill(n, dtype, 1, dev)
        c = _fill(e - b, dtype, 4, dev, b)
        w = c.clone()
        with torch.cuda.device(r):
            cb.gemv_row_major(A, x, w, pol)
        As.append(A), xs.append(x), cs.append(c), want.append(w)
    full = [torch.full((m,), float("nan"), dtype=dtype, device=f"cuda:{r}") for r in range(G)] \
        if gather else None
    mg.gemv_rm(As, xs, cs, pol, exchange=exchange, c_full=full)
    for r in range(G):
        assert torch.equal(cs[r], want[r])
    if gather:
        cat = torch.cat([w.cpu() for w in want])
        for r in range(G):
            assert torch.equal(full[r].cpu(), cat)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("exchange", ["nccl", "peer"])
def test_mgpu_gemv_cols_every_replica_gets_the_ordered_sum(mg, dtype, exchange):
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200.mgpu import partition
    G = mg.size
    m, n = 256, 30001
    pol = cb.default_policy(1)
    As, xs, cs = [], [], []
    total = torch.zeros(m, dtype=dtype)
    c0 = _fill(m, dtype, 4, "cuda:0").cpu()
    for r in range(G):
        b, e = partition(n, G, r)
        dev = f"cuda:{r}"
        A = cb.DenseMatrix.wrap(_fill(m * (e - b), dtype, 3, dev, m * b), m, e - b, cb.Layout.ColMajor)
        x = _fill(e - b, dtype, 1, dev, b)
        p = torch.zeros(m, dtype=dtype, device=dev)
        with torch.cuda.device(r):
            cb.gemv_col_major(A, x, p, pol)
        total = total + p.cpu()
        As.append(A), xs.append(x), cs.append(c0.to(dev))
    want = c0 + total
    mg.gemv_cm_cols(As, xs, cs, pol, exchange=exchange)
    for r in range(G):
        assert torch.equal(cs[r].cpu(), want)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_mgpu_ger_rows_equal_per_shard_calls(mg, dtype):
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200.mgpu import partition
    G = mg.size
    m, n = 4099, 2048
    pol = cb.default_policy(1)
    xs, ys, Cs, want = [], [], [], []
    for r in range(G):
        b, e = partition(m, G, r)
        dev = f"cuda:{r}"
        C = cb.DenseMatrix.wrap(_fill((e - b) * n, dtype, 5, dev, b * n), e - b, n, cb.Layout.RowMajor)
        x, y = _fill(e - b, dtype, 1, dev, b), _fill(n, dtype, 2, dev)
        W = cb.DenseMatrix.wrap(C.data.clone(), e - b, n, cb.Layout.RowMajor)
        with torch.cuda.device(r):
            cb.ger(x, y, W, pol)
        xs.append(x), ys.append(y), Cs.append(C), want.append(W)
    mg.ger_rm(xs, ys, Cs, pol)
    for r in range(G):
        assert torch.equal(Cs[r].data, want[r].data)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_mgpu_dot_segmented_is_gpu_count_invariant(mg, dtype):
    """cabl_mgpu_dot_segmented: one partial per fixed global segment, summed in index
    order.  On this box's devices it must give the bits of shard.sharded_dot_invariant
    run on the whole vectors by one rank (which tests/test_gpu_dist.py shows equal to
    the per-rank work of 1, 2, 3, 4 and 8 GPUs combined), and reject shards that are not
    whole segments."""
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200 import shard
    G = mg.size
    pol = cb.default_policy(1)
    seg = 1 << 20
    n = 9 * seg + 4321  # 10 segments, ragged last
    xs, ys = [], []
    for r in range(G):
        b, e = shard.invariant_range(n, seg, G, r)
        xs.append(_fill(e - b, dtype, 1, f"cuda:{r}", b))
        ys.append(_fill(e - b, dtype, 2, f"cuda:{r}", b))
    got = mg.dot_segmented(xs, ys, 0.75, seg, pol)
    x_all = _fill(n, dtype, 1, "cuda:0")
    y_all = _fill(n, dtype, 2, "cuda:0")
    want = torch.zeros(1, dtype=dtype, device="cuda:0")
    with torch.cuda.device(0):
        shard.sharded_dot_invariant(x_all, y_all, 0.75, want, pol, n_total=n, segment=seg)
    assert got == float(want.item())
    assert mg.dot_segmented(xs, ys, 0.75, seg, pol) == got  # and run to run
    # empty input: alpha0
    empty = [_fill(0, dtype, 1, f"cuda:{r}") for r in range(G)]
    assert mg.dot_segmented(empty, empty, 0.75, seg, pol) == 0.75
    with pytest.raises(ValueError, match="segment must be > 0"):
        mg.dot_segmented(xs, ys, 0.0, 0, pol)
    with pytest.raises(ValueError, match="multiple of 64"):
        mg.dot_segmented(xs, ys, 0.0, 1000, pol)
    if G > 1:  # a first shard that is not whole segments
        bad = [_fill(seg + 1, dtype, 1, f"cuda:{r}") for r in range(G)]
        with pytest.raises(ValueError, match="whole number of segments"):
            mg.dot_segmented(bad, bad, 0.0, seg, pol)


def test_mgpu_validates_every_shard_before_launching(mg):
    import paper_2108_02025_b200 as cb
    G = mg.size
    x = [_fill(100, torch.float32, 1, f"cuda:{r}") for r in range(G)]
    y = [_fill(101, torch.float32, 2, f"cuda:{r}") for r in range(G)]
    with pytest.raises(ValueError, match="lengths differ"):
        mg.dot(x, y, 0.0)
    # the C ABI's own check (bypassing the mirror): a null shard pointer
    from paper_2108_02025_b200 import _lib
    import ctypes as C
    nulls = (C.c_void_p * G)(*([None] * G))
    ns = (C.c_uint64 * G)(*([100] * G))
    out = C.c_float()
    rc = _lib.lib().cabl_mgpu_dot_f32(mg._ctx, nulls, nulls, ns, C.c_float(0), 8192, 0, C.byref(out))
    assert rc == _lib.CABL_EINVAL
    # a gathering GEMV whose shard cannot take the sweep kernel: rejected for
    # every rank before any kernel (no peer left waiting), context still usable
    A = [cb.DenseMatrix.wrap(_fill(3 * 5, torch.float32, 3, f"cuda:{r}"), 3, 5, cb.Layout.RowMajor)
         for r in range(G)]
    xs = [_fill(5, torch.float32, 1, f"cuda:{r}") for r in range(G)]
    cs = [_fill(3, torch.float32, 4, f"cuda:{r}") for r in range(G)]
    full = [torch.zeros(3 * G, device=f"cuda:{r}") for r in range(G)]
    with pytest.raises(ValueError, match="sweep kernel"):
        mg.gemv_rm(A, xs, cs, exchange="peer", c_full=full)
    x2 = [_fill(100, torch.float32, 1, f"cuda:{r}") for r in range(G)]
    assert mg.dot(x2, x2, 0.0) > 0


def test_mgpu_timeout_aborts_and_poisons_the_context():
    """A call that does not finish within the timeout raises
    CablExchangeError (after ncclCommAbort); later calls fail the same way."""
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200._lib import CablExchangeError
    from paper_2108_02025_b200.mgpu import MultiGpu
    G = _dev_count()
    n = 1 << 31  # 2 x 8 GiB per device: ~2.3 ms of DOT, well past a 1 ms timeout
    xs = [torch.ones(n // G, device=f"cuda:{r}") for r in range(G)]
    mg = MultiGpu(list(range(G)), timeout_ms=1)
    try:
        with pytest.raises(CablExchangeError, match="not complete after 1 ms"):
            for _ in range(20):  # the first call may win the race; a queue of them cannot
                mg.dot(xs, xs, 0.0, cb.default_policy(1))
        with pytest.raises(CablExchangeError, match="aborted"):
            mg.dot(xs[:G], xs[:G], 0.0)
    finally:
        mg.close()
        torch.cuda.synchronize()
    del xs
    torch.cuda.empty_cache()


def test_mgpu_randomised_shapes_equal_single_gpu_calls(mg):
    """40 seeded cases over every op, dtype, exchange and ragged shape: each
    multi-GPU call equals the same shards run through the single-GPU API, bit
    for bit (world = all visible GPUs; 1 on the round's boxes)."""
    import random

    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200.mgpu import partition
    rng = random.Random(20261020)
    G = mg.size
    pol = cb.default_policy(1)
    for case in range(40):
        dt = rng.choice([torch.float32, torch.float64])
        op = rng.choice(["dot", "gemv_rm", "gemv_cm", "ger"])
        ex = rng.choice(["nccl", "peer"])
        if op == "dot":
            n = rng.randint(1, 3_000_000)
            xs, ys, parts = [], [], []
            for r in range(G):
                b, e = partition(n, G, r)
                xs.append(_fill(e - b, dt, 1, f"cuda:{r}", b))
                ys.append(_fill(e - b, dt, 2, f"cuda:{r}", b))
                with torch.cuda.device(r):
                    parts.append(cb.dot(xs[r], ys[r], 0.0, pol) if e > b else 0.0)
            acc = torch.zeros((), dtype=dt)
            for p in parts:
                acc = acc + torch.tensor(p, dtype=dt)
            want = float(acc + torch.tensor(-0.5, dtype=dt))
            assert mg.dot(xs, ys, -0.5, pol, exchange=ex) == want, (case, n)
        elif op == "gemv_rm":
            m, n = rng.randint(G, 20_000), rng.choice([1, 7, 64, 1000, 4096, 8195])
            As, xs, cs, want = [], [], [], []
            for r in range(G):
                b, e = partition(m, G, r)
                A = cb.DenseMatrix.wrap(_fill((e - b) * n, dt, 3, f"cuda:{r}", b * n), e - b, n,
                                        cb.Layout.RowMajor)
                x, c = _fill(n, dt, 1, f"cuda:{r}"), _fill(e - b, dt, 4, f"cuda:{r}", b)
                w = c.clone()
                with torch.cuda.device(r):
                    cb.gemv_row_major(A, x, w, pol)
                As.append(A), xs.append(x), cs.append(c), want.append(w)
            mg.gemv_rm(As, xs, cs, pol, exchange="nccl")
            for r in range(G):
                assert torch.equal(cs[r], want[r]), (case, m, n)
        elif op == "gemv_cm":
            m, n = rng.choice([1, 8, 256, 1000, 4096]), rng.randint(G, 50_000)
            As, xs, cs = [], [], []
            total = torch.zeros(m, dtype=dt)
            c0 = _fill(m, dt, 4, "cuda:0").cpu()
            for r in range(G):
                b, e = partition(n, G, r)
                A = cb.DenseMatrix.wrap(_fill(m * (e - b), dt, 3, f"cuda:{r}", m * b), m, e - b,
                                        cb.Layout.ColMajor)
                x = _fill(e - b, dt, 1, f"cuda:{r}", b)
                p = torch.zeros(m, dtype=dt, device=f"cuda:{r}")
                with torch.cuda.device(r):
                    cb.gemv_col_major(A, x, p, pol)
                total = total + p.cpu()
                As.append(A), xs.append(x), cs.append(c0.to(f"cuda:{r}"))
            mg.gemv_cm_cols(As, xs, cs, pol, exchange=ex)
            for r in range(G):
                assert torch.equal(cs[r].cpu(), c0 + total), (case, m, n)
        else:
            m, n = rng.randint(G, 5000), rng.choice([1, 5, 64, 777, 4096])
            xs, ys, Cs, want = [], [], [], []
            for r in range(G):
                b, e = partition(m, G, r)
                C = cb.DenseMatrix.wrap(_fill((e - b) * n, dt, 5, f"cuda:{r}", b * n), e - b, n,
                                        cb.Layout.RowMajor)
                x, y = _fill(e - b, dt, 1, f"cuda:{r}", b), _fill(n, dt, 2, f"cuda:{r}")
                W = cb.DenseMatrix.wrap(C.data.clone(), e - b, n, cb.Layout.RowMajor)
                with torch.cuda.device(r):
                    cb.ger(x, y, W, pol)
                xs.append(x), ys.append(y), Cs.append(C), want.append(W)
            mg.ger_rm(xs, ys, Cs, pol)
            for r in range(G):
                assert torch.equal(Cs[r].data, want[r].data), (case, m, n)
