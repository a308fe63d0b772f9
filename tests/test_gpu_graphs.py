"""Every kernel family inside a CUDA graph (stream capture + replay).

The C ABI takes a stream, so a caller may capture its calls into a CUDA graph (the
resident-operator pipeline of bench.py's e2e_resident does).  What must hold for that:
nothing in a call may be host-side state that a replay would not repeat — the work
queues' counters reset themselves in the kernel, DOT's epoch and the tickets live in
device memory, the PDL-chained combine kernels are captured as a dependent pair — and
the scratch must come from the entry the warm-up call created (no allocation while
capturing).  Each case warms up once, captures ONE call, replays it three times and
compares bit for bit with the same number of eager calls.  (The shapes were checked
with an ncu launch list to reach the kernel named beside each one.)

Reference semantics being preserved: c += A x, C += x (x) y accumulate in place
(kernels.hpp:187-313), so k replays equal k eager calls on the same operands.
"""
from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu

SEED = 42


def _fill(n, dtype, stream, dev):
    import paper_2108_02025_b200 as cb
    return cb.fill_uniform(torch.empty(n, dtype=dtype, device=dev), SEED, stream)


def _policy():
    import paper_2108_02025_b200 as cb
    return cb.default_policy(1)


def _replay_equals_eager(call, outputs, replays=3):
    """call() updates `outputs` in place.  Returns after asserting that warm-up +
    `replays` graph replays leave the same bits as warm-up + `replays` eager calls."""
    start = [o.clone() for o in outputs]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        call()  # warm-up: sizes the (device, stream) scratch entry
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        call()
    # capture does not execute: outputs hold exactly one (warm-up) update here
    for _ in range(replays):
        g.replay()
    torch.cuda.synchronize()
    got = [o.clone() for o in outputs]
    for o, st in zip(outputs, start):
        o.copy_(st)
    for _ in range(1 + replays):
        call()
    torch.cuda.synchronize()
    for a, b in zip(got, outputs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("n", [5000, 1 << 20, (1 << 22) + 3])
def test_dot_in_a_graph(cuda, dtype, n):
    """Small path, the one-launch kernel with its epoch-tagged collector, odd length."""
    import paper_2108_02025_b200 as cb
    x, y = _fill(n, dtype, 1, cuda), _fill(n, dtype, 2, cuda)
    out = torch.zeros(1, dtype=dtype, device=cuda)
    pol = _policy()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        cb.dot_into(x, y, 0.25, out, pol)
    s.synchronize()
    want = out.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        cb.dot_into(x, y, 0.25, out, pol)
    for _ in range(4):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, want)


@pytest.mark.parametrize("dtype,m,n", [
    (torch.float32, 8192, 2048),     # sweep (static)
    (torch.float32, 2048, 8200),     # 8 x 1 sweep shape
    (torch.float32, 4, 1 << 20),     # few long rows: chunk queue + per-row tickets
    (torch.float32, 100_000, 40),    # one thread per row
    (torch.float64, 3000, 1024),     # 8 x 1 sweep, fp64
    (torch.float32, 50_000, 256),    # sub-CTA sweep, one warp per row (1 KB rows)
    (torch.float32, 10_000, 1536),   # sub-CTA sweep, one row per pass (6 KB rows)
    (torch.float64, 20_000, 264),    # G lanes per row (66 of 128 lanes: below fp64's fill rule)
    (torch.float32, 1000, 4097),     # few long scalar rows: one CTA per row
    (torch.float32, 20_000, 129),    # many scalar rows: the scalar sub-CTA sweep
    (torch.float32, 5000, 129),      # fewer scalar rows: G lanes per row, scalar loads
    (torch.float64, 7, 5),           # small (single CTA, reference order)
])
def test_gemv_row_major_in_a_graph(cuda, dtype, m, n):
    import paper_2108_02025_b200 as cb
    A = cb.DenseMatrix.wrap(_fill(m * n, dtype, 3, cuda), m, n, cb.Layout.RowMajor)
    x, c = _fill(n, dtype, 1, cuda), _fill(m, dtype, 4, cuda)
    pol = _policy()
    _replay_equals_eager(lambda: cb.gemv_row_major(A, x, c, pol), [c])


@pytest.mark.parametrize("dtype,m,n", [
    (torch.float64, 1 << 18, 32),    # tall
    (torch.float32, 1 << 20, 4),     # narrow tall
    (torch.float64, 256, 1 << 14),   # bulk ring + one-wave combine
    (torch.float32, 4096, 1024),     # full-column sweep + PDL-chained combine
    (torch.float32, 16384, 256),     # two row vectors per thread + 16-byte combine
    (torch.float64, 8192, 512),      # 2-D split, per-tile tickets or external combine
    (torch.float32, 3001, 700),      # full-column bulk ring (odd m)
    (torch.float32, 40001, 64),      # realigning split
    (torch.float32, 1001, 300),      # bulk ring, scalar consumers
    (torch.float32, 300_001, 8),     # tall, one row per lane (odd m)
])
def test_gemv_col_major_in_a_graph(cuda, dtype, m, n):
    import paper_2108_02025_b200 as cb
    A = cb.DenseMatrix.wrap(_fill(m * n, dtype, 3, cuda), m, n, cb.Layout.ColMajor)
    x, c = _fill(n, dtype, 1, cuda), _fill(m, dtype, 4, cuda)
    pol = _policy()
    _replay_equals_eager(lambda: cb.gemv_col_major(A, x, c, pol), [c])


@pytest.mark.parametrize("dtype,layout,m,n", [
    (torch.float32, "row", 2048, 4096),   # tile queue
    (torch.float64, "col", 1024, 2048),
    (torch.float32, "row", 4096, 64),     # flat vector sweep
    (torch.float32, "row", 1000, 1001),   # flat any-width sweep
    (torch.float64, "col", 1, 1 << 20),   # one-element rows (AXPY)
    (torch.float32, "row", 5, 7),         # small
])
def test_ger_in_a_graph(cuda, dtype, layout, m, n):
    import paper_2108_02025_b200 as cb
    lay = cb.Layout.RowMajor if layout == "row" else cb.Layout.ColMajor
    C_ = cb.DenseMatrix.wrap(_fill(m * n, dtype, 5, cuda), m, n, lay)
    # small factors keep three accumulations far from overflow and still exact-order
    x, y = _fill(m, dtype, 1, cuda), _fill(n, dtype, 2, cuda)
    pol = _policy()
    _replay_equals_eager(lambda: cb.ger(x, y, C_, pol), [C_.data])
