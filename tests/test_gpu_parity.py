"""GPU parity: libcabl_cuda.so (through the C ABI) vs the CPU oracle.

Inputs are the seeded SplitMix64 fills generated on the device and copied to
the host, so both sides see identical bits.  Bars (tests/tolerances.py):
GER and the ordered paths bitwise; DOT/GEMV within BASELINE's contract bound
against the oracle AND a non-vacuous bound against extended-precision truth;
every kernel bitwise reproducible run to run.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests import tolerances as T

pytestmark = pytest.mark.gpu

SEED = 42


def dev_uniform(n, dtype, stream, cuda, seed=SEED):
    import paper_2108_02025_b200 as cb
    t = torch.empty(n, dtype=dtype, device=cuda)
    if n:
        cb.fill_uniform(t, seed, stream)
    return t


def np_of(t):
    return t.detach().cpu().numpy()


def policy():
    import paper_2108_02025_b200 as cb
    return cb.default_policy(1)


def plan_for(dtype):
    """Plan derived with element_bytes = sizeof(T), as the reference bench does."""
    import paper_2108_02025_b200 as cb
    md = cb.default_machine()
    md.element_bytes = torch.tensor([], dtype=dtype).element_size()
    return cb.ExecPolicy(cb.derive_blocking_plan(md), 1)


DTYPES = [torch.float32, torch.float64]


# ------------------------------------------------------------------ DOT
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 33, 1000, 8192, 8193, 16384, 16385, 100_003,
                               1_000_000, 1 << 24])
def test_dot_matches_oracle(cuda, dtype, n):
    import paper_2108_02025_b200 as cb
    x, y = dev_uniform(n, dtype, 1, cuda), dev_uniform(n, dtype, 2, cuda)
    pol = plan_for(dtype)
    got = cb.dot(x, y, 0.25, pol)
    probe = cb.last_exec()
    xn, yn = np_of(x), np_of(y)
    want = O.dot_ref(xn, yn, 0.25)
    truth, sumabs = O.dot_truth(xn, yn, 0.25)
    npdt = xn.dtype
    assert abs(got - float(want)) <= T.contract_tol(n, sumabs, 0.25, npdt)
    assert abs(got - truth) <= T.truth_tol(T.dot_chain(n, npdt), sumabs, 0.25, npdt)
    if n <= pol.plan.dot_cutoff:
        assert probe.variant == cb.KernelVariant.dot_small and probe.threads_used == 1
    else:
        assert probe.variant == cb.KernelVariant.dot_blocked and probe.threads_used >= 2


@pytest.mark.parametrize("dtype", DTYPES)
def test_dot_unaligned_operands(cuda, dtype):
    """Different misalignments (scalar path) and a shared one (head peeled,
    then the vector path): truth bound, and run-to-run bitwise."""
    import paper_2108_02025_b200 as cb
    n = 300_001
    x, y = dev_uniform(n + 8, dtype, 1, cuda), dev_uniform(n + 8, dtype, 2, cuda)
    for ox, oy in [(1, 3), (1, 1), (3, 3), (7, 7), (2, 2)]:
        xs, ys = x[ox:ox + n], y[oy:oy + n]
        got = cb.dot(xs, ys, -1.5, policy())
        assert cb.dot(xs, ys, -1.5, policy()) == got
        xn, yn = np_of(xs), np_of(ys)
        truth, sumabs = O.dot_truth(xn, yn, -1.5)
        assert abs(got - truth) <= T.truth_tol(n, sumabs, 1.5, xn.dtype), (ox, oy)


def test_dot_hand_values(cuda):
    import paper_2108_02025_b200 as cb
    # reference test_kernels.cpp:54-62, :96-98
    t = lambda v: torch.tensor(v, dtype=torch.float64, device=cuda)
    assert cb.dot(t([1, 2, 3]), t([4, 5, 6]), 0.0, policy()) == 32.0
    assert cb.dot(t([0.5, -1.25, 3.0]), t([0.0, 0.0, 0.0]), 7.5, policy()) == 7.5
    assert cb.dot(t([0.0, 1.0, 0.0]), t([0.0, 1.0, 0.0]), 0.0, policy()) == 1.0
    assert cb.dot(t([]), t([]), 2.5, policy()) == 2.5
    with pytest.raises(ValueError, match="dot: x and y lengths differ"):
        cb.dot(t([1.0, 2.0]), t([1.0]), 0.0, policy())


# ----------------------------------------------------------------- GEMV
def _gemv_case(cuda, dtype, m, n, layout, seed=SEED):
    import paper_2108_02025_b200 as cb
    A = dev_uniform(m * n, dtype, 3, cuda, seed)
    x = dev_uniform(n, dtype, 1, cuda, seed)
    c0 = dev_uniform(m, dtype, 4, cuda, seed)
    Am = cb.DenseMatrix.wrap(A, m, n, layout)
    c = c0.clone()
    pol = plan_for(dtype)
    if layout == cb.Layout.RowMajor:
        cb.gemv_row_major(Am, x, c, pol)
    else:
        cb.gemv_col_major(Am, x, c, pol)
    probe = cb.last_exec()
    An, xn, c0n = np_of(A), np_of(x), np_of(c0)
    want = c0n.copy()
    O.gemv_ref(An, int(layout), xn, want)
    truth, rowabs = O.gemv_truth(An, int(layout), xn, c0n)
    return np_of(c), want, truth, rowabs, c0n, probe, pol


RM_SHAPES = [(1, 777), (3, 3), (8, 8), (40, 200), (257, 259), (1000, 1000), (2000, 500),
             (33, 16392), (4097, 1024), (8192, 8192), (4736, 100), (5000, 1028), (9001, 3000),
             # short rows: one thread per row (bitwise), vector and scalar loads
             (9472, 64), (100_000, 16), (20_001, 5), (9472, 256), (30_000, 255), (1 << 18, 1),
             (9472, 1024), (12_000, 999),
             # rows of 1 / 2 / 4 warps of 32-byte vectors: the sub-CTA sweep (full and
             # partly filled row slots, ragged last group), and the G-lanes kernel
             # where a slot would be < 3/4 full
             (9473, 512), (9600, 200), (9999, 776), (12_345, 1000), (9472, 96), (9500, 384),
             (9473, 264), (10_000, 520),
             # odd rows of 65 .. 2048 elements: the scalar sub-CTA sweep (every slot width)
             (9473, 65), (10_000, 129), (9600, 1001), (9500, 2047), (20_000, 300), (9999, 513),
             # 4 - 8 KiB rows: fp32 one-row slots of the sub-CTA sweep, fp64 the 8 x 1 sweep
             (9473, 2048), (9600, 1280), (10_001, 1032),
             # rows of whole 16-byte (not 32-byte) vectors: the scalar-load kernel
             (20_000, 2052), (3000, 20_002), (1800, 65_540),
             # odd rows, long and short: the G-lanes scalar kernel
             (8192, 8193), (7200, 1001), (8000, 249),
             # few long rows: the chunked kernel (units of row x chunk, queue, row tickets)
             (1, 1 << 20), (3, 300_000), (8, 65_536), (2, 1_000_000),
             # few long odd rows: one CTA per row (scalar loads, block sum)
             (1000, 65_537), (37, 100_001), (4096, 16_385)]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("m,n", RM_SHAPES)
def test_gemv_row_major_matches_oracle(cuda, dtype, m, n):
    import paper_2108_02025_b200 as cb
    got, want, truth, rowabs, c0, probe, pol = _gemv_case(cuda, dtype, m, n, cb.Layout.RowMajor)
    dt = got.dtype
    assert probe.variant == cb.KernelVariant.gemv_row
    if m * n + m + n <= pol.plan.dot_cutoff:
        # ordered single-CTA path: bit for bit the compiled reference gemv_ref
        assert probe.threads_used == 1
        np.testing.assert_array_equal(got, want)
    if T.rm_is_ordered(m, n, dt) or T.rm_is_lane(m, n, dt):
        # reference-order kernels: bit for bit the compiled reference gemv_ref
        np.testing.assert_array_equal(got, want)
    tol_c = T.contract_tol(n, rowabs, np.abs(c0), dt)
    assert np.all(np.abs(got.astype(np.float64) - want) <= tol_c)
    tol_t = T.truth_tol(T.gemv_rm_chain(n, dt), rowabs, np.abs(c0), dt)
    assert np.all(np.abs(got.astype(np.float64) - truth) <= tol_t)


@pytest.mark.parametrize("cfg", ["", "tma"])
def test_gemv_row_major_reference_order_mode_subprocess(cuda, cfg):
    """CABL_GEMV_RM_ORDER=reference (read once per process): rerun the
    row-major parity cases in a child process, where tolerances.rm_is_ordered
    turns the reference-order shapes into bitwise assertions.  cfg "tma" runs
    the tensor-map producer variant (CABL_ORD_CFG=tma)."""
    import os
    import subprocess
    import sys
    if os.environ.get("CABL_GEMV_RM_ORDER") == "reference":
        pytest.skip("already the reference-order process")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CABL_TUNING="1", CABL_GEMV_RM_ORDER="reference")
    if cfg:
        env["CABL_ORD_CFG"] = cfg
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py",
                        "tests/test_gpu_bounds.py", "-m", "gpu", "-q", "-x", "-p", "no:cacheprovider",
                        "-k", "(row_major_matches or 65536_square or gemv_guard) and not subprocess"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


CM_SHAPES = [(3, 3), (8, 8), (257, 259), (1000, 1000), (256, 65536), (2047, 300),
             (2048, 100), (4096, 4096), (5000, 3001), (65536, 256), (70001, 37),
             (151552, 40), (303104, 24), (160001, 9),
             # short-wide with few rows: tiles wider than the ring's x slot
             (1, 1 << 20), (3, 300_000), (8, 400_000), (64, 100_000), (100, 50_000),
             # tall and narrow (n < 16): several row vectors per thread, bitwise
             (303_104, 4), (1 << 20, 5), (1 << 20, 15), (1 << 21, 1), (1 << 20, 8),
             # tall from half the SMs' worth of 256-vector units up (bitwise)
             (151_552, 33), (200_000, 20), (151_544, 7),
             # odd m >= 1024: the realigning split (aligned 256-bit loads + warp shuffles)
             (1025, 3000), (8193, 2000), (3001, 5003), (12_345, 777), (100_003, 64),
             # aligned mid-size m: the row-tiled bulk ring (ragged last tile and
             # column parts, stages wider and narrower than the x slot, n < parts)
             (512, 70_001), (1000, 20_003), (4096, 16_384), (4104, 5_001), (12_000, 5_592),
             (16_384, 4_096), (24_576, 777), (65_536, 1_030), (131_072, 130), (8_192, 3)]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("m,n", CM_SHAPES)
def test_gemv_col_major_matches_oracle(cuda, dtype, m, n):
    import paper_2108_02025_b200 as cb
    got, want, truth, rowabs, c0, probe, pol = _gemv_case(cuda, dtype, m, n, cb.Layout.ColMajor)
    dt = got.dtype
    assert probe.variant == cb.KernelVariant.gemv_col_blocked
    if T.cm_is_tall(m, dt) or m * n + m + n <= pol.plan.dot_cutoff:
        # tall kernel / ordered path keep the reference order and rounding
        np.testing.assert_array_equal(got, want)
    tol_c = T.contract_tol(n, rowabs, np.abs(c0), dt)
    assert np.all(np.abs(got.astype(np.float64) - want) <= tol_c)
    tol_t = T.truth_tol(T.gemv_cm_chain(m, n, dt), rowabs, np.abs(c0), dt)
    assert np.all(np.abs(got.astype(np.float64) - truth) <= tol_t)


# full-column sweep (aligned 512 <= m, m/V <= 1024) with its in-kernel combine:
# grids below the 64 combiners (several row-vector passes per combiner warp),
# row-vector counts that do not divide by the combiners, 1 and 2 column lanes
FULLCOL_SHAPES = [(8192, 40), (2048, 100), (4096, 65), (4104, 5001), (1536, 593), (1032, 70_001),
                  (8192, 8192), (520, 148), (2048, 1)]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("m,n", FULLCOL_SHAPES)
def test_gemv_col_major_fullcol_combine(cuda, dtype, m, n):
    import paper_2108_02025_b200 as cb
    got, want, truth, rowabs, c0, probe, pol = _gemv_case(cuda, dtype, m, n, cb.Layout.ColMajor)
    dt = got.dtype
    tol_c = T.contract_tol(n, rowabs, np.abs(c0), dt)
    assert np.all(np.abs(got.astype(np.float64) - want) <= tol_c)
    tol_t = T.truth_tol(T.gemv_cm_chain(m, n, dt), rowabs, np.abs(c0), dt)
    assert np.all(np.abs(got.astype(np.float64) - truth) <= tol_t)


# fp32 8192 < m <= 16384: the two-row-vector full-column sweep and its 16-byte
# combine (a second row vector live for 1 thread, grids below 16 parts, one
# column); fp64 at the same m: the 2-D split finishing in the same combine
# kernel (row tiles, >= 2 parts) or in-kernel (1 part)
TWO_RV_SHAPES = [(8200, 300), (16384, 7), (9000, 1), (16376, 4097), (12000, 160), (8208, 148)]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("m,n", TWO_RV_SHAPES)
def test_gemv_col_major_two_row_vectors_and_combine16(cuda, dtype, m, n):
    import paper_2108_02025_b200 as cb
    got, want, truth, rowabs, c0, probe, pol = _gemv_case(cuda, dtype, m, n, cb.Layout.ColMajor)
    dt = got.dtype
    tol_c = T.contract_tol(n, rowabs, np.abs(c0), dt)
    assert np.all(np.abs(got.astype(np.float64) - want) <= tol_c)
    tol_t = T.truth_tol(T.gemv_cm_chain(m, n, dt), rowabs, np.abs(c0), dt)
    assert np.all(np.abs(got.astype(np.float64) - truth) <= tol_t)
    # run to run: the same bits
    A = cb.DenseMatrix.wrap(dev_uniform(m * n, dtype, 3, cuda), m, n, cb.Layout.ColMajor)
    x, c1 = dev_uniform(n, dtype, 1, cuda), dev_uniform(m, dtype, 4, cuda)
    c2 = c1.clone()
    cb.gemv_col_major(A, x, c1, pol)
    cb.gemv_col_major(A, x, c2, pol)
    assert torch.equal(c1, c2)
    np.testing.assert_array_equal(np_of(c1), got)


def test_gemv_col_major_fullcol_tickets_interleaved(cuda):
    """The full-column sweep's arrival/departure tickets live in the stream's
    shared counters: back-to-back launches with different grids, interleaved
    with the 2-D split and the DOT on the same stream, must each give the bits
    of a lone call."""
    import paper_2108_02025_b200 as cb
    pol = policy()
    cases = []
    for i, (m, n, dt) in enumerate([(4096, 16_384, torch.float32), (8192, 40, torch.float32),
                                    (16_384, 300, torch.float32), (2048, 5000, torch.float64)]):
        A = cb.DenseMatrix.wrap(dev_uniform(m * n, dt, 3 + i, cuda), m, n, cb.Layout.ColMajor)
        cases.append((A, dev_uniform(n, dt, 1, cuda), dev_uniform(m, dt, 4, cuda)))

    def run(k):
        A, x, c0 = cases[k]
        c = c0.clone()
        cb.gemv_col_major(A, x, c, pol)
        return c

    lone = [run(k).cpu() for k in range(len(cases))]
    xd, yd = dev_uniform(1 << 22, torch.float32, 1, cuda), dev_uniform(1 << 22, torch.float32, 2, cuda)
    d0 = cb.dot(xd, yd, 0.0, pol)
    order = [0, 1, 0, 2, 1, 3, 0, 0, 2, 3, 1]
    outs = []
    for k in order:
        outs.append((k, run(k)))
        if k == 2:
            assert cb.dot(xd, yd, 0.0, pol) == d0
    torch.cuda.synchronize()
    for k, c in outs:
        assert torch.equal(c.cpu(), lone[k]), k


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("off", [1, 3])
@pytest.mark.parametrize("m,n", [(4096, 2048), (2048, 4096), (1024, 1000), (5000, 300),
                                 (257, 20_000), (100, 65_536), (3, 300_000), (1000, 3000)])
def test_gemv_col_major_misaligned_a(cuda, dtype, off, m, n):
    """A starting `off` elements past a 32-byte boundary (every column
    misaligned): the realigning split, within the contract and truth bounds,
    and bitwise run to run."""
    import paper_2108_02025_b200 as cb
    A = dev_uniform(m * n + off, dtype, 3, cuda)[off:]
    x = dev_uniform(n, dtype, 1, cuda)
    c0 = dev_uniform(m, dtype, 4, cuda)
    Am = cb.DenseMatrix.wrap(A, m, n, cb.Layout.ColMajor)
    c, c2 = c0.clone(), c0.clone()
    cb.gemv_col_major(Am, x, c, plan_for(dtype))
    cb.gemv_col_major(Am, x, c2, plan_for(dtype))
    assert torch.equal(c, c2)
    An, xn, c0n = np_of(A), np_of(x), np_of(c0)
    want = c0n.copy()
    O.gemv_ref(An, 1, xn, want)
    truth, rowabs = O.gemv_truth(An, 1, xn, c0n)
    got = np_of(c)
    dt = got.dtype
    assert np.all(np.abs(got.astype(np.float64) - want) <= T.contract_tol(n, rowabs, np.abs(c0n), dt))
    tol_t = T.truth_tol(T.gemv_cm_chain(m, n, dt), rowabs, np.abs(c0n), dt)
    assert np.all(np.abs(got.astype(np.float64) - truth) <= tol_t)


def _bulk_scalar_tc(m, s):
    """Columns per stage of the scalar bulk ring for an A off a 16-byte
    boundary (csrc/gemv_cm.cu split_bulk_geom with the 49152 - 32 budget)."""
    q = 16 // s
    return max(q, (49152 - 32 + 1024) // ((m + 1) * s) // q * q)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("off", [1, 2])
@pytest.mark.parametrize("m", [1, 2])
@pytest.mark.parametrize("rag", [1, 2])
def test_gemv_col_major_misaligned_ragged_tail_tiny_m(cuda, dtype, off, m, rag):
    """A off a 16-byte boundary with 1-2 rows and a last tile of 1-2 columns:
    that tile ends inside its first 16 bytes, so the ring copies nothing for it
    and every element must come from global memory (regression: the in-smem
    count wrapped and the tile read a stale stage)."""
    import paper_2108_02025_b200 as cb
    s = torch.tensor([], dtype=dtype).element_size()
    if off * s % 16 == 0:
        pytest.skip("offset keeps A 16-byte aligned")
    n = _bulk_scalar_tc(m, s) * 40 + rag
    A = dev_uniform(m * n + off, dtype, 3, cuda)[off:]
    x = dev_uniform(n, dtype, 1, cuda)
    c0 = dev_uniform(m, dtype, 4, cuda)
    c = c0.clone()
    cb.gemv_col_major(cb.DenseMatrix.wrap(A, m, n, cb.Layout.ColMajor), x, c, plan_for(dtype))
    An, xn, c0n = np_of(A), np_of(x), np_of(c0)
    want = c0n.copy()
    O.gemv_ref(An, 1, xn, want)
    truth, rowabs = O.gemv_truth(An, 1, xn, c0n)
    got = np_of(c)
    dt = got.dtype
    assert np.all(np.abs(got.astype(np.float64) - want) <= T.contract_tol(n, rowabs, np.abs(c0n), dt))
    tol_t = T.truth_tol(T.gemv_cm_chain(m, n, dt), rowabs, np.abs(c0n), dt)
    assert np.all(np.abs(got.astype(np.float64) - truth) <= tol_t)


@pytest.mark.parametrize("m,n", [(1 << 20, 256), (256, 1 << 20)])
def test_gemv_col_major_baseline_configs_fp64_normal(cuda, m, n):
    """BASELINE config 4 (G2 / G3): fp64 col-major, N(0,1) inputs."""
    import paper_2108_02025_b200 as cb
    A = cb.fill_normal(torch.empty(m * n, dtype=torch.float64, device=cuda), SEED, 3)
    x = cb.fill_normal(torch.empty(n, dtype=torch.float64, device=cuda), SEED, 1)
    c0 = cb.fill_normal(torch.empty(m, dtype=torch.float64, device=cuda), SEED, 4)
    c = c0.clone()
    cb.gemv_col_major(cb.DenseMatrix.wrap(A, m, n, cb.Layout.ColMajor), x, c, policy())
    An, xn, c0n = np_of(A), np_of(x), np_of(c0)
    want = c0n.copy()
    O.gemv_ref(An, 1, xn, want)
    truth, rowabs = O.gemv_truth(An, 1, xn, c0n)
    got = np_of(c)
    if T.cm_is_tall(m, np.float64):
        np.testing.assert_array_equal(got, want)
    assert np.all(np.abs(got - want) <= T.contract_tol(n, rowabs, np.abs(c0n), np.float64))
    assert np.all(np.abs(got - truth) <=
                  T.truth_tol(T.gemv_cm_chain(m, n, np.float64), rowabs, np.abs(c0n), np.float64))


def test_gemv_hand_values_and_contracts(cuda):
    import paper_2108_02025_b200 as cb
    t = lambda v: torch.tensor(v, dtype=torch.float64, device=cuda)
    # reference test_kernels.cpp:114-147, :180-186
    I = cb.DenseMatrix(3, 3, cb.Layout.ColMajor, device=cuda)
    for i in range(3):
        I[i, i] = 1.0
    c = t([0.0, 0.0, 0.0])
    cb.gemv_col_major(I, t([1, 2, 3]), c, policy())
    assert c.tolist() == [1, 2, 3]
    ones = cb.DenseMatrix(2, 3, cb.Layout.RowMajor, 1.0, device=cuda)
    co = t([1.0, 1.0])
    cb.gemv_row_major(ones, t([1.0, 1.0, 1.0]), co, policy())
    assert co.tolist() == [4, 4]
    with pytest.raises(ValueError, match="matrix is not col-major"):
        cb.gemv_col_major(ones, t([1.0, 1.0, 1.0]), co, policy())
    with pytest.raises(ValueError, match="gemv: A.cols != x.len"):
        cb.gemv_row_major(ones, t([1.0] * 4), co, policy())
    x = t([1.0, 2.0, 3.0])
    with pytest.raises(ValueError, match="gemv: c must not alias x"):
        cb.gemv_col_major(cb.DenseMatrix(3, 3, cb.Layout.ColMajor, 1.0, device=cuda), x, x,
                          policy())
    # zero-size operands are no-ops (test_kernels.cpp:282-300)
    c5 = t([3.0] * 5)
    cb.gemv_row_major(cb.DenseMatrix(5, 0, cb.Layout.RowMajor, device=cuda), t([]), c5, policy())
    assert c5.tolist() == [3.0] * 5


def test_gemv_single_row_equals_dot_ref_bitwise(cuda):
    """Reference test_kernels.cpp:199-208: a 1 x 777 row at threads=1 equals
    dot_ref(row, x, c0) exactly — here through the ordered small path."""
    import paper_2108_02025_b200 as cb
    n = 777
    A = dev_uniform(n, torch.float64, 3, cuda)
    x = dev_uniform(n, torch.float64, 1, cuda)
    c = torch.tensor([0.125], dtype=torch.float64, device=cuda)
    cb.gemv_row_major(cb.DenseMatrix.wrap(A, 1, n, cb.Layout.RowMajor), x, c, policy())
    assert c.item() == float(O.dot_ref(np_of(A), np_of(x), 0.125))
    assert cb.last_exec().threads_used == 1


# ------------------------------------------------------------------ GER
GER_SHAPES = [(1, 1), (2, 3), (3, 3), (500, 500), (777, 1001), (1000, 8), (8, 1000),
              (1024, 1024), (3000, 4096), (8192, 8192),
              # short aligned rows (flat vector sweep) and short odd rows (flat scalar)
              (20_000, 64), (64, 20_000), (100_000, 8), (50_000, 5), (5, 50_000), (1, 300_000),
              # rows of whole 16-byte vectors (flat 16-byte sweep)
              (3000, 4100), (12, 100_004), (40_000, 12),
              # odd rows of >= 8 elements (flat 32-byte sweep of C, rows straddling vectors)
              (1001, 777), (400, 1003), (3, 200_001), (200_001, 9), (8192, 8193),
              # one-element rows (row-major n = 1, col-major m = 1): the AXPY kernel
              (400_001, 1), (1, 400_003)]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("layout", ["row", "col"])
@pytest.mark.parametrize("m,n", GER_SHAPES)
def test_ger_bitwise_equals_oracle(cuda, dtype, layout, m, n):
    import paper_2108_02025_b200 as cb
    if dtype == torch.float64 and m * n > (1 << 24):
        pytest.skip("fp64 at 8192^2 covered by the fp32 BASELINE config")
    lay = cb.Layout.RowMajor if layout == "row" else cb.Layout.ColMajor
    x, y = dev_uniform(m, dtype, 1, cuda), dev_uniform(n, dtype, 2, cuda)
    C0 = dev_uniform(m * n, dtype, 5, cuda)
    Cm = cb.DenseMatrix.wrap(C0.clone(), m, n, lay)
    cb.ger(x, y, Cm, plan_for(dtype))
    assert cb.last_exec().variant == cb.KernelVariant.ger
    want = np_of(C0)
    O.ger_ref(np_of(x), np_of(y), want, int(lay))
    np.testing.assert_array_equal(np_of(Cm.data), want)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("off", [1, 2, 3, 5])
@pytest.mark.parametrize("m,n", [(1000, 4096), (777, 1001), (2048, 2048)])
def test_ger_misaligned_c_bitwise(cuda, dtype, off, m, n):
    """C (and x, y) starting off elements past a 32-byte boundary: the flat
    sweep's scalar head/tail plus 32-byte body, still one FMA per element."""
    import paper_2108_02025_b200 as cb
    x = dev_uniform(m + off, dtype, 1, cuda)[off:]
    y = dev_uniform(n + off, dtype, 2, cuda)[off:]
    big = dev_uniform(m * n + off, dtype, 5, cuda)
    C0 = big[off:].clone()
    view = big[off:]
    cb.ger(x, y, cb.DenseMatrix.wrap(view, m, n, cb.Layout.RowMajor), plan_for(dtype))
    want = np_of(C0)
    O.ger_ref(np_of(x), np_of(y), want, 0)
    np.testing.assert_array_equal(np_of(view), want)


def test_ger_hand_values(cuda):
    import paper_2108_02025_b200 as cb
    t = lambda v: torch.tensor(v, dtype=torch.float64, device=cuda)
    C = cb.DenseMatrix(3, 3, cb.Layout.ColMajor, 0.0, device=cuda)
    cb.ger(t([0, 1, 0]), t([0, 0, 1]), C, policy())
    for i in range(3):
        for j in range(3):
            assert C(i, j).item() == (1.0 if (i, j) == (1, 2) else 0.0)
    C2 = cb.DenseMatrix(2, 3, cb.Layout.RowMajor, 0.0, device=cuda)
    cb.ger(t([1, 2]), t([3, 4, 5]), C2, policy())
    assert [[C2(i, j).item() for j in range(3)] for i in range(2)] == [[3, 4, 5], [6, 8, 10]]
    with pytest.raises(ValueError, match="ger: C.cols != y.len"):
        cb.ger(t([1, 2]), t([3]), cb.DenseMatrix(2, 2, cb.Layout.ColMajor, device=cuda), policy())
    cb.ger(t([]), t([]), cb.DenseMatrix(0, 0, cb.Layout.ColMajor, device=cuda), policy())


# --------------------------------------------------------- determinism
def test_bitwise_reproducible_run_to_run(cuda):
    import paper_2108_02025_b200 as cb
    pol = policy()
    n = (1 << 24) + 7
    x, y = dev_uniform(n, torch.float32, 1, cuda), dev_uniform(n, torch.float32, 2, cuda)
    first = cb.dot(x, y, 1.25, pol)
    assert all(cb.dot(x, y, 1.25, pol) == first for _ in range(50))
    for (m, k, lay) in [(8192, 8192, cb.Layout.RowMajor), (4097, 1000, cb.Layout.RowMajor),
                        (256, 1 << 18, cb.Layout.ColMajor)]:
        A = cb.DenseMatrix.wrap(dev_uniform(m * k, torch.float32, 3, cuda), m, k, lay)
        xv = dev_uniform(k, torch.float32, 1, cuda)
        c0 = dev_uniform(m, torch.float32, 4, cuda)
        fn = cb.gemv_row_major if lay == cb.Layout.RowMajor else cb.gemv_col_major
        ref = c0.clone()
        fn(A, xv, ref, pol)
        for _ in range(20):
            c = c0.clone()
            fn(A, xv, c, pol)
            assert torch.equal(c, ref)


# ------------------------------------------------- host-buffer entry points
def test_host_buffer_path_equals_device_path(cuda):
    import paper_2108_02025_b200 as cb
    pol = policy()
    n = 123_457
    x, y = dev_uniform(n, torch.float64, 1, cuda), dev_uniform(n, torch.float64, 2, cuda)
    assert cb.dot(x.cpu(), y.cpu(), 0.5, pol) == cb.dot(x, y, 0.5, pol)
    m, k = 999, 1001
    A = dev_uniform(m * k, torch.float32, 3, cuda)
    xv = dev_uniform(k, torch.float32, 1, cuda)
    c0 = dev_uniform(m, torch.float32, 4, cuda)
    for lay, fn in [(cb.Layout.RowMajor, cb.gemv_row_major), (cb.Layout.ColMajor, cb.gemv_col_major)]:
        cd = c0.clone()
        fn(cb.DenseMatrix.wrap(A, m, k, lay), xv, cd, pol)
        ch = c0.cpu().clone()
        fn(cb.DenseMatrix.wrap(A.cpu(), m, k, lay), xv.cpu(), ch, pol)
        assert torch.equal(cd.cpu(), ch)
    gx, gy = dev_uniform(m, torch.float32, 1, cuda), dev_uniform(k, torch.float32, 2, cuda)
    Cd = cb.DenseMatrix.wrap(A.clone(), m, k, cb.Layout.RowMajor)
    Ch = cb.DenseMatrix.wrap(A.cpu().clone(), m, k, cb.Layout.RowMajor)
    cb.ger(gx, gy, Cd, pol)
    cb.ger(gx.cpu(), gy.cpu(), Ch, pol)
    assert torch.equal(Cd.data.cpu(), Ch.data)


@pytest.mark.parametrize("pinned", [False, True])
def test_host_staged_copies_equal_device_path(cuda, pinned):
    """Host containers above the 4 MiB staging threshold: pageable buffers go
    through the multi-threaded pinned-slot staging (capi.cu staged_copy, H2D
    and D2H, several 8 MiB chunks and a ragged last one), pinned ones straight
    to the DMA engine.  Results equal the device-resident call bit for bit."""
    import paper_2108_02025_b200 as cb
    pol = policy()
    host = (lambda t: t.cpu().pin_memory()) if pinned else (lambda t: t.cpu())
    n = 5_000_003
    x, y = dev_uniform(n, torch.float64, 1, cuda), dev_uniform(n, torch.float64, 2, cuda)
    assert cb.dot(host(x), host(y), 0.25, pol) == cb.dot(x, y, 0.25, pol)
    m, k = 3000, 5001
    A = dev_uniform(m * k, torch.float32, 3, cuda)
    xv, c0 = dev_uniform(k, torch.float32, 1, cuda), dev_uniform(m, torch.float32, 4, cuda)
    cd = c0.clone()
    cb.gemv_row_major(cb.DenseMatrix.wrap(A, m, k, cb.Layout.RowMajor), xv, cd, pol)
    ch = host(c0)
    cb.gemv_row_major(cb.DenseMatrix.wrap(host(A), m, k, cb.Layout.RowMajor), host(xv), ch, pol)
    assert torch.equal(cd.cpu(), ch)
    gx, gy = dev_uniform(m, torch.float32, 5, cuda), dev_uniform(k, torch.float32, 6, cuda)
    Cd = cb.DenseMatrix.wrap(A.clone(), m, k, cb.Layout.ColMajor)
    Ch = cb.DenseMatrix.wrap(host(A), m, k, cb.Layout.ColMajor)
    cb.ger(gx, gy, Cd, pol)
    cb.ger(host(gx), host(gy), Ch, pol)
    assert torch.equal(Cd.data.cpu(), Ch.data)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("layout", ["row", "col"])
@pytest.mark.parametrize("m,n", [(8192, 8192), (3001, 5003), (40_000, 777)])
def test_host_ger_pipeline_equals_device_path(cuda, dtype, layout, m, n):
    """Pinned host C above two slabs: the full-duplex pipeline (H2D of slab
    k+1, GER of slab k and D2H of slab k-1 on three streams, capi.cu
    host_ger_pipelined) — bit for bit the device-resident call, ragged last
    slab included, and x / y slices at the slab offsets."""
    import paper_2108_02025_b200 as cb
    lay = cb.Layout.RowMajor if layout == "row" else cb.Layout.ColMajor
    C0 = dev_uniform(m * n, dtype, 5, cuda)
    gx, gy = dev_uniform(m, dtype, 1, cuda), dev_uniform(n, dtype, 2, cuda)
    Cd = cb.DenseMatrix.wrap(C0.clone(), m, n, lay)
    cb.ger(gx, gy, Cd, policy())
    Ch = cb.DenseMatrix.wrap(C0.cpu().pin_memory(), m, n, lay)
    cb.ger(gx.cpu(), gy.cpu(), Ch, policy())
    assert torch.equal(Cd.data.cpu(), Ch.data)
    want = np_of(C0).copy()
    O.ger_ref(np_of(gx), np_of(gy), want, int(lay))
    np.testing.assert_array_equal(Ch.data.numpy(), want)


# ------------------------------------------------- full BASELINE sizes
def test_generator_matches_host_oracle(cuda):
    for dtype, npdt in [(torch.float32, np.float32), (torch.float64, np.float64)]:
        t = dev_uniform(100_003, dtype, 7, cuda, seed=1234)
        np.testing.assert_array_equal(np_of(t), O.gen_uniform(100_003, npdt, 1234, 7))
    import paper_2108_02025_b200 as cb
    g = cb.fill_normal(torch.empty(4096, dtype=torch.float64, device=cuda), 9, 3)
    h = O.gen_normal_f64(4096, 9, 3)
    np.testing.assert_allclose(np_of(g), h, rtol=1e-13, atol=1e-13)


@pytest.mark.slow
def test_gemv_65536_square_fp32_sampled_rows(cuda):
    """BASELINE config 5 (G4): 16 GiB A.  Every row against the CPU oracle
    gemv_ref (contract tolerance, and the truth bound from extended
    precision), and against an fp64 torch matvec on the device."""
    import paper_2108_02025_b200 as cb
    m = n = 65536
    A = dev_uniform(m * n, torch.float32, 3, cuda)
    x = dev_uniform(n, torch.float32, 1, cuda)
    c0 = dev_uniform(m, torch.float32, 4, cuda)
    c = c0.clone()
    cb.gemv_row_major(cb.DenseMatrix.wrap(A, m, n, cb.Layout.RowMajor), x, c, policy())
    # every row against the CPU oracle (gemv_ref), 4096-row blocks copied to
    # the host in turn (~4 s of oracle time for the 4.3e9 multiply-adds)
    xn = np_of(x)
    got_all = np_of(c)
    c0_all = np_of(c0)
    for r0 in range(0, m, 4096):
        An = np_of(A.view(m, n)[r0:r0 + 4096]).reshape(-1)
        c0n = c0_all[r0:r0 + 4096]
        want = c0n.copy()
        O.gemv_ref(An, 0, xn, want)
        truth, rowabs = O.gemv_truth(An, 0, xn, c0n)
        got = got_all[r0:r0 + 4096]
        if T.rm_is_ordered(m, n, np.float32):
            np.testing.assert_array_equal(got, want)
        assert np.all(np.abs(got - want) <= T.contract_tol(n, rowabs, np.abs(c0n), np.float32))
        assert np.all(np.abs(got - truth) <=
                      T.truth_tol(T.gemv_rm_chain(n, np.float32), rowabs, np.abs(c0n), np.float32))
    # all rows: fp64 torch reference (exact products, fp64 sums)
    ref = c0.double().clone()
    for r0 in range(0, m, 4096):
        ref[r0:r0 + 4096] += A.view(m, n)[r0:r0 + 4096].double() @ x.double()
    absA = torch.zeros(m, dtype=torch.float64, device=cuda)
    for r0 in range(0, m, 4096):
        absA[r0:r0 + 4096] = A.view(m, n)[r0:r0 + 4096].double().abs() @ x.double().abs()
    err = (c.double() - ref).abs()
    bound = (T.gemv_rm_chain(n, np.float32) + 4) * T.EPS[np.dtype(np.float32)] * (absA + c0.double().abs())
    assert bool((err <= bound).all())
    # the row-block shards of 2 / 4 / 8 GPUs (BASELINE config 5's partition), each run
    # as its own call: bit for bit the rows of the single-GPU result, so the sharded
    # G4 gives the same c at every GPU count (a row's order depends on n and on the
    # sweep shape, which these shards share with the whole matrix)
    from paper_2108_02025_b200 import shard
    for G in (2, 4, 8):
        for g in range(G):
            b, e = shard.partition(m, G, g)
            cs = c0[b:e].clone()
            cb.gemv_row_major(cb.DenseMatrix.wrap(A[b * n:e * n], e - b, n, cb.Layout.RowMajor),
                              x, cs, policy())
            assert torch.equal(cs, c[b:e]), (G, g)


def test_concurrent_host_threads_share_a_stream_safely(cuda):
    """Several host threads issue calls on the same (legacy default) stream
    while the per-stream scratch keeps growing (DOT partials, split-GEMV
    partials): results must equal the single-threaded ones bitwise.  Guards
    the scratch lease in csrc/capi.cu."""
    import threading
    import paper_2108_02025_b200 as cb
    pol = policy()
    jobs = []
    for i, n in enumerate([10_000, 1 << 20, 3 << 20, 1 << 22]):
        x, y = dev_uniform(n, torch.float32, 1 + i, cuda), dev_uniform(n, torch.float32, 7 + i, cuda)
        jobs.append(("dot", x, y))
    for i, (m, k) in enumerate([(256, 1 << 16), (128, 1 << 18), (1024, 1 << 15)]):
        A = cb.DenseMatrix.wrap(dev_uniform(m * k, torch.float64, 3 + i, cuda), m, k, cb.Layout.ColMajor)
        jobs.append(("gemv", A, dev_uniform(k, torch.float64, 1, cuda), dev_uniform(m, torch.float64, 4, cuda)))

    def run(job):
        if job[0] == "dot":
            return cb.dot(job[1], job[2], 0.5, pol)
        c = job[3].clone()
        cb.gemv_col_major(job[1], job[2], c, pol)
        torch.cuda.synchronize()
        return c.cpu()

    want = [run(j) for j in jobs]
    errors = []

    def worker(seed):
        order = list(range(len(jobs)))
        rng = np.random.default_rng(seed)
        for _ in range(20):
            rng.shuffle(order)
            for k in order:
                got = run(jobs[k])
                same = got == want[k] if jobs[k][0] == "dot" else torch.equal(got, want[k])
                if not same:
                    errors.append((seed, k))

    threads = [threading.Thread(target=worker, args=(s,)) for s in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[:5]


@pytest.mark.slow
def test_dot_chunked_large_n(cuda):
    """2ns >= 512 MiB takes the chunked, queue-scheduled DOT (csrc/dot.cu):
    n = 2^28 + 3 fp32 (1 GiB per operand, 513 chunks, 3 trailing elements)."""
    import paper_2108_02025_b200 as cb
    n = (1 << 28) + 3
    x, y = dev_uniform(n, torch.float32, 1, cuda), dev_uniform(n, torch.float32, 2, cuda)
    pol = plan_for(torch.float32)
    got = cb.dot(x, y, 0.25, pol)
    assert cb.last_exec().variant == cb.KernelVariant.dot_blocked
    again = [cb.dot(x, y, 0.25, pol) for _ in range(5)]
    assert all(a == got for a in again)
    xn, yn = np_of(x), np_of(y)
    truth, sumabs = O.dot_truth(xn, yn, 0.25)
    assert abs(got - float(O.dot_ref(xn, yn, 0.25))) <= T.contract_tol(n, sumabs, 0.25, np.float32)
    assert abs(got - truth) <= T.truth_tol(T.dot_chain(n, np.float32), sumabs, 0.25, np.float32)


@pytest.mark.slow
def test_dot_2pow32_baseline_config(cuda):
    """BASELINE config 5 (D2): n = 2^32 fp32, 32 GiB of operands.  Size-
    independent properties (exact power-of-two scaling, symmetry, run-to-run
    bits), the non-vacuous truth bound against an fp64 torch reduction
    computed chunk by chunk on the device (fp32 products are exact in fp64),
    and the CPU oracle dot_ref over all 2^32 terms."""
    import paper_2108_02025_b200 as cb
    n = 1 << 32
    x = dev_uniform(n, torch.float32, 1, cuda)
    y = dev_uniform(n, torch.float32, 2, cuda)
    pol = plan_for(torch.float32)
    got = cb.dot(x, y, 0.0, pol)
    assert cb.dot(x, y, 0.0, pol) == got
    assert cb.dot(y, x, 0.0, pol) == got          # fma(a,b,c) == fma(b,a,c)
    x.mul_(2.0)                                    # exact: a power of two
    assert cb.dot(x, y, 0.0, pol) == 2.0 * got
    x.mul_(0.5)
    truth = 0.0
    sumabs = 0.0
    step = 1 << 28
    for b in range(0, n, step):
        p = x[b:b + step].double() * y[b:b + step].double()
        truth += float(p.sum())
        sumabs += float(p.abs().sum())
    eps = float(np.finfo(np.float32).eps)
    # fp64 chunk sums carry ~1e-16 relative error: far below the fp32 bound
    assert abs(got - truth) <= (T.dot_chain(n, np.float32) + 2) * eps * sumabs
    # the CPU oracle dot_ref over all 2^32 terms: its sequential chain
    # continues exactly from chunk to chunk (chunks are multiples of its
    # 16-byte vector prefix), so this is dot_ref of the whole vectors
    ref = np.float32(0.0)
    for b in range(0, n, step):
        ref = O.dot_ref(np_of(x[b:b + step]), np_of(y[b:b + step]), float(ref))
    assert abs(got - float(ref)) <= T.contract_tol(n, sumabs, 0.0, np.float32)
    # both are far inside the fp32 truth bound; the GPU's short chains are the
    # more accurate (reported in the assertion message if this ever fails)
    assert abs(got - truth) <= abs(float(ref) - truth) + 64 * eps * sumabs, (got, float(ref), truth)


def test_resident_gemv_operator_graph_equals_direct_call(cuda):
    """operators.ResidentGemv (A resident, x/c streamed, CUDA-graph step)
    gives the same bits as the plain call, call after call."""
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200.operators import ResidentGemv
    for lay, m, n in [(cb.Layout.RowMajor, 8192, 8192), (cb.Layout.ColMajor, 256, 1 << 16)]:
        A = cb.DenseMatrix.wrap(dev_uniform(m * n, torch.float32, 3, cuda), m, n, lay)
        pol = policy()
        ops = [ResidentGemv(A, pol, use_graph=True), ResidentGemv(A, pol, use_graph=False)]
        for step in range(3):
            x = dev_uniform(n, torch.float32, 10 + step, cuda)
            c = dev_uniform(m, torch.float32, 20 + step, cuda)
            want = c.clone()
            (cb.gemv_row_major if lay == cb.Layout.RowMajor else cb.gemv_col_major)(A, x, want, pol)
            for op in ops:
                got = op(x.cpu(), c.cpu())
                assert torch.equal(got, want.cpu())


@pytest.mark.parametrize("depth", [2, 4])
def test_gemv_pipeline_results_in_order(cuda, depth):
    """operators.GemvPipeline: with `depth` steps in flight (bench.py's e2e
    runs 4) every step's result is the GEMV of that step's inputs (no buffer
    reuse before read-back), returned in submission order."""
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200.operators import GemvPipeline
    m, n = 4096, 4096
    A = cb.DenseMatrix.wrap(dev_uniform(m * n, torch.float32, 3, cuda), m, n, cb.Layout.RowMajor)
    pol = policy()
    pipe = GemvPipeline(A, pol, depth=depth)
    xs = [dev_uniform(n, torch.float32, 30 + k, cuda) for k in range(9)]
    cs = [dev_uniform(m, torch.float32, 40 + k, cuda) for k in range(9)]
    wants = []
    for x, c in zip(xs, cs):
        w = c.clone()
        cb.gemv_row_major(A, x, w, pol)
        wants.append(w.cpu())
    got = []
    for x, c in zip(xs, cs):
        r = pipe.step(x.cpu(), c.cpu())
        if r is not None:
            got.append(r.clone())
    got += [r.clone() for r in pipe.drain()]
    assert len(got) == 9
    for g, w in zip(got, wants):
        assert torch.equal(g, w)


@pytest.mark.parametrize("dtype", DTYPES)
def test_special_values_propagate_like_the_oracle(cuda, dtype):
    """NaN / Inf / signed zero / subnormals flow through every kernel as they
    do through the reference's CPU code (no flush-to-zero, no fast math)."""
    import paper_2108_02025_b200 as cb
    npdt = np.float32 if dtype == torch.float32 else np.float64
    tiny = np.finfo(npdt).smallest_subnormal
    pol = policy()
    # DOT: NaN poisons, +Inf survives, subnormal products are kept
    for n in (100, 100_003):
        x = np.full(n, 0.5, npdt)
        y = np.full(n, 2.0, npdt)
        y[7] = np.nan
        assert np.isnan(cb.dot(torch.from_numpy(x).to(cuda), torch.from_numpy(y).to(cuda), 0.0, pol))
        y[7] = np.inf
        assert cb.dot(torch.from_numpy(x).to(cuda), torch.from_numpy(y).to(cuda), 0.0, pol) == np.inf
        xs = np.full(n, tiny, npdt)
        ys = np.ones(n, npdt)
        got = cb.dot(torch.from_numpy(xs).to(cuda), torch.from_numpy(ys).to(cuda), 0.0, pol)
        assert got == float(O.dot_ref(xs, ys, 0.0)) and got > 0
    # signed zero: alpha0 added last to +0 (reference kernels.hpp:142)
    e = torch.empty(0, dtype=dtype, device=cuda)
    assert str(cb.dot(e, e, -0.0, pol)) == "0.0"
    # GEMV / GER with a NaN and an Inf planted: same non-finite pattern as the oracle
    m, n = 300, 1024
    for lay in (cb.Layout.RowMajor, cb.Layout.ColMajor):
        A = O.gen_uniform(m * n, npdt, 42, 3)
        A[5] = np.nan
        A[777] = np.inf
        x = O.gen_uniform(n, npdt, 42, 1)
        c0 = O.gen_uniform(m, npdt, 42, 4)
        c = torch.from_numpy(c0.copy()).to(cuda)
        f = cb.gemv_row_major if lay == cb.Layout.RowMajor else cb.gemv_col_major
        f(cb.DenseMatrix.wrap(torch.from_numpy(A).to(cuda), m, n, lay), torch.from_numpy(x).to(cuda), c, pol)
        want = c0.copy()
        O.gemv_ref(A, int(lay), x, want)
        got = c.cpu().numpy()
        np.testing.assert_array_equal(np.isnan(got), np.isnan(want))
        np.testing.assert_array_equal(np.isinf(got), np.isinf(want))
        C0 = O.gen_uniform(m * n, npdt, 42, 5)
        C0[3] = np.nan
        gx = O.gen_uniform(m, npdt, 42, 1)
        gx[2] = np.inf
        gy = O.gen_uniform(n, npdt, 42, 2)
        Cm = cb.DenseMatrix.wrap(torch.from_numpy(C0.copy()).to(cuda), m, n, lay)
        cb.ger(torch.from_numpy(gx).to(cuda), torch.from_numpy(gy).to(cuda), Cm, pol)
        want = C0.copy()
        O.ger_ref(gx, gy, want, int(lay))
        np.testing.assert_array_equal(Cm.data.cpu().numpy(), want)  # NaN == NaN positions too


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("layout", ["row", "col"])
@pytest.mark.parametrize("m,n", [(16, 1 << 20), (256, 1 << 16), (4, 300_000), (2048, 4096)])
def test_gemv_misaligned_x(cuda, dtype, layout, m, n):
    """x = v[1:] of an aligned buffer with an aligned A: the row-major path
    stages x into aligned scratch, the col-major bulk ring reads x with plain
    loads (a bulk copy needs 16-byte alignment)."""
    import paper_2108_02025_b200 as cb
    lay = cb.Layout.RowMajor if layout == "row" else cb.Layout.ColMajor
    A = dev_uniform(m * n, dtype, 3, cuda)
    x = dev_uniform(n + 1, dtype, 1, cuda)[1:]
    c0 = dev_uniform(m, dtype, 4, cuda)
    c, c2 = c0.clone(), c0.clone()
    f = cb.gemv_row_major if layout == "row" else cb.gemv_col_major
    Am = cb.DenseMatrix.wrap(A, m, n, lay)
    f(Am, x, c, plan_for(dtype))
    f(Am, x, c2, plan_for(dtype))
    torch.cuda.synchronize()
    assert torch.equal(c, c2)
    An, xn, c0n = np_of(A), np_of(x), np_of(c0)
    want = c0n.copy()
    O.gemv_ref(An, int(lay), xn, want)
    truth, rowabs = O.gemv_truth(An, int(lay), xn, c0n)
    got = np_of(c).astype(np.float64)
    dt = np_of(c).dtype
    assert np.all(np.abs(got - want) <= T.contract_tol(n, rowabs, np.abs(c0n), dt))
    chain = T.gemv_rm_chain(n, dt) if layout == "row" else T.gemv_cm_chain(m, n, dt)
    assert np.all(np.abs(got - truth) <= T.truth_tol(chain, rowabs, np.abs(c0n), dt))
