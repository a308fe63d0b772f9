"""Randomised shapes, alignments and dtypes across every dispatch path, against
the CPU oracle (oracle/, a restatement of reference kernels.hpp pinned to the
compiled reference): GER bitwise (one FMA per element, reference
kernels.hpp:264-313), DOT and GEMV within the BASELINE contract bound and the
fp64-truth bound, every result bitwise reproducible on a second run.  The
shapes are drawn from a fixed seed so a failure reproduces; each case is small
enough for the oracle to finish in well under a second.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from tests import tolerances as T
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _draw(rng, kind):
    """(m, n) spread over the shape classes the dispatch distinguishes."""
    if kind == "dot":
        return 0, int(rng.choice([rng.integers(1, 64), rng.integers(64, 9000),
                                  rng.integers(9000, 400_000), rng.integers(400_000, 3_000_000)]))
    cls = rng.integers(0, 6)
    if cls == 0:   # tiny (ordered single-CTA paths)
        return int(rng.integers(1, 40)), int(rng.integers(1, 40))
    if cls == 1:   # short rows, many of them
        return int(rng.integers(5000, 60_000)), int(rng.integers(1, 80))
    if cls == 2:   # few long rows
        return int(rng.integers(1, 20)), int(rng.integers(20_000, 400_000))
    if cls == 3:   # mid
        return int(rng.integers(200, 3000)), int(rng.integers(200, 3000))
    if cls == 4:   # tall-ish
        return int(rng.integers(20_000, 160_000)), int(rng.integers(2, 40))
    return int(rng.integers(1000, 9000)), int(rng.integers(1000, 9000)) | 1  # odd widths


def _dev(a, off, cuda):
    """A device copy of numpy array `a` starting `off` elements past a 256-byte boundary."""
    t = torch.empty(a.size + off, dtype=torch.from_numpy(a[:0]).dtype, device=cuda)
    t[off:] = torch.from_numpy(a)
    return t[off:]


KINDS = ("dot", "gemv-row", "gemv-col", "ger-row", "ger-col")
CASES = [(kind, seed) for kind in KINDS for seed in range(30)]


@pytest.mark.parametrize("kind,seed", CASES)
def test_random_shapes_against_oracle(cuda, kind, seed):
    import paper_2108_02025_b200 as cb
    rng = np.random.default_rng(1000 * seed + KINDS.index(kind))
    dt = np.float32 if rng.integers(0, 2) == 0 else np.float64
    off = int(rng.choice([0, 0, 1, 3]))
    m, n = _draw(rng, kind)
    if dt == np.float64 and m * n > 20_000_000:
        n = max(1, 20_000_000 // max(m, 1))
    pol = cb.default_policy(1)
    eps = float(np.finfo(dt).eps)
    if kind == "dot":
        x, y = O.gen_uniform(n, dt, seed, 1), O.gen_uniform(n, dt, seed, 2)
        xd, yd = _dev(x, off, cuda), _dev(y, 2 * off % 5, cuda)
        got = cb.dot(xd, yd, 0.375, pol)
        assert cb.dot(xd, yd, 0.375, pol) == got
        truth, sumabs = O.dot_truth(x, y, 0.375)
        assert abs(got - float(O.dot_ref(x, y, 0.375))) <= 4 * n * eps * (sumabs + 0.375)
        assert abs(got - truth) <= T.truth_tol(n, sumabs, 0.375, dt)
        return
    lay = cb.Layout.RowMajor if kind.endswith("row") else cb.Layout.ColMajor
    if kind.startswith("gemv"):
        A = O.gen_uniform(m * n, dt, seed, 3)
        x, c0 = O.gen_uniform(n, dt, seed, 1), O.gen_uniform(m, dt, seed, 4)
        Ad, xd = _dev(A, off, cuda), _dev(x, 0, cuda)
        c1, c2 = _dev(c0, 0, cuda), _dev(c0, 0, cuda)
        f = cb.gemv_row_major if lay == cb.Layout.RowMajor else cb.gemv_col_major
        Am = cb.DenseMatrix.wrap(Ad, m, n, lay)
        f(Am, xd, c1, pol)
        f(Am, xd, c2, pol)
        assert torch.equal(c1, c2)
        got = c1.cpu().numpy().astype(np.float64)
        want = c0.copy()
        O.gemv_ref(A, int(lay), x, want)
        truth, rowabs = O.gemv_truth(A, int(lay), x, c0)
        assert np.all(np.abs(got - want) <= T.contract_tol(n, rowabs, np.abs(c0), dt))
        chain = T.gemv_rm_chain(n, dt) if lay == cb.Layout.RowMajor else T.gemv_cm_chain(m, n, dt)
        assert np.all(np.abs(got - truth) <= T.truth_tol(chain, rowabs, np.abs(c0), dt))
        return
    x, y = O.gen_uniform(m, dt, seed, 1), O.gen_uniform(n, dt, seed, 2)
    C0 = O.gen_uniform(m * n, dt, seed, 5)
    Cd = _dev(C0, off, cuda)
    cb.ger(_dev(x, off, cuda), _dev(y, off, cuda), cb.DenseMatrix.wrap(Cd, m, n, lay), pol)
    want = C0.copy()
    O.ger_ref(x, y, want, int(lay))
    np.testing.assert_array_equal(Cd.cpu().numpy(), want)
