"""Pinning the CPU oracle (no GPU needed).

1. The restatement (oracle/cabl_oracle.c) reproduces the golden outputs the
   COMPILED, UNMODIFIED reference produced (tests/golden/reference_golden.npz,
   made by tests/golden/make_golden.py) bit for bit: dot_ref, gemv_ref (both
   layouts), ger_ref (both layouts).
2. Where the reference is mounted, the same against a live build of it
   (oracle/_ref) on randomized shapes, including the reference's own
   randomized pools (acceptance.cpp:108-114).
3. The reference's hand-computed known answers (test_kernels.cpp:54-62,
   :114-135, :218-243).
4. The generator is pinned (first SplitMix64 outputs, exact U[-1,1) mapping).
"""
from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = Path(__file__).resolve().parent / "golden" / "reference_golden.npz"


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def _gen(dt, seed, stream, n):
    return O.gen_uniform(int(n), dt, int(seed), int(stream))


def test_generator_is_pinned(golden):
    key = O.lib().oracle_sm64_key(42, 1)
    assert key == int(golden["sm64/key_42_1"][0])
    got = [O.lib().oracle_sm64(key, i) for i in range(8)]
    assert got == [int(v) for v in golden["sm64/first8"]]
    u = O.gen_uniform(100_000, np.float32, 1, 2)
    assert u.min() >= -1.0 and u.max() < 1.0
    # exact: every value is k * 2^-23 - 1
    k = (u.astype(np.float64) + 1.0) * 2.0 ** 23
    assert np.array_equal(k, np.round(k))


def _cases(golden, prefix):
    seen = set()
    for k in golden.files:
        if k.startswith(prefix):
            seen.add(k.rsplit("/", 1)[0])
    return sorted(seen)


def test_dot_ref_matches_compiled_reference(golden):
    seed = int(golden["seed"][0])
    n_cases = 0
    for case in _cases(golden, "dot/"):
        _, tag, n = case.split("/")
        dt = np.dtype(tag).type
        s1, s2 = golden[case + "/streams"]
        x, y = _gen(dt, seed, s1, n), _gen(dt, seed, s2, n)
        assert O.dot_ref(x, y, 0.25) == golden[case + "/ref"][0], case
        n_cases += 1
    assert n_cases == 28


@pytest.mark.parametrize("op,lay", [("gemv-row", 0), ("gemv-col", 1)])
def test_gemv_ref_matches_compiled_reference(golden, op, lay):
    seed = int(golden["seed"][0])
    cases = _cases(golden, op + "/")
    assert len(cases) == 22
    for case in cases:
        _, tag, shape = case.split("/")
        m, n = map(int, shape.split("x"))
        dt = np.dtype(tag).type
        sA, sx, sc = golden[case + "/streams"]
        A, x, c = _gen(dt, seed, sA, m * n), _gen(dt, seed, sx, n), _gen(dt, seed, sc, m)
        O.gemv_ref(A, lay, x, c)
        np.testing.assert_array_equal(c, golden[case + "/ref"], err_msg=case)
        if op == "gemv-row":
            # the reference's threaded row-major path is the same per-row chain
            np.testing.assert_array_equal(golden[case + "/t1"], golden[case + "/ref"])
            np.testing.assert_array_equal(golden[case + "/t4"], golden[case + "/ref"])


@pytest.mark.parametrize("ln,lay", [("row", 0), ("col", 1)])
def test_ger_ref_matches_compiled_reference(golden, ln, lay):
    seed = int(golden["seed"][0])
    cases = _cases(golden, f"ger-{ln}/")
    assert len(cases) == 12
    for case in cases:
        _, tag, shape = case.split("/")
        m, n = map(int, shape.split("x"))
        dt = np.dtype(tag).type
        sC, sx, sy = golden[case + "/streams"]
        C0, x, y = _gen(dt, seed, sC, m * n), _gen(dt, seed, sx, m), _gen(dt, seed, sy, n)
        O.ger_ref(x, y, C0, lay)
        assert hashlib.sha256(C0.tobytes()).hexdigest() == str(golden[case + "/ref_sha256"][0]), case
        # the reference's threaded GER is bitwise its oracle (kernels.hpp:272-276)
        assert str(golden[case + "/t4_sha256"][0]) == str(golden[case + "/ref_sha256"][0])


def test_reference_known_answers():
    f64 = np.float64
    a = np.array([1, 2, 3], f64)
    assert O.dot_ref(a, np.array([4, 5, 6], f64), 0.0) == 32.0
    assert O.dot_ref(np.array([0.5, -1.25, 3.0]), np.zeros(3), 7.5) == 7.5
    e1 = np.array([0.0, 1.0, 0.0])
    assert O.dot_ref(e1, e1, 0.0) == 1.0
    with pytest.raises(ValueError):
        O.dot_ref(a, np.zeros(2), 0.0)
    ident = np.eye(3).reshape(-1)
    c = np.zeros(3)
    O.gemv_ref(ident, 1, np.array([1.0, 2.0, 3.0]), c)
    assert c.tolist() == [1, 2, 3]
    co = np.ones(2)
    O.gemv_ref(np.ones(6), 0, np.ones(3), co)
    assert co.tolist() == [4, 4]
    C = np.zeros(6)
    O.ger_ref(np.array([1.0, 2.0]), np.array([3.0, 4.0, 5.0]), C, 0)
    assert C.reshape(2, 3).tolist() == [[3, 4, 5], [6, 8, 10]]
    B = np.zeros(9)
    O.ger_ref(np.array([0.0, 1.0, 0.0]), np.array([0.0, 0.0, 1.0]), B, 1)
    assert np.flatnonzero(B).tolist() == [1 + 2 * 3]


needs_ref = pytest.mark.skipif(not (O.ref_available() or O.REF_INCLUDE.is_dir()),
                               reason="reference not mounted and oracle/_ref not built")


@needs_ref
def test_restatement_equals_live_reference_on_random_pools():
    if not O.ref_available():
        O.build(ref=True)
    rng = np.random.default_rng(20260810)
    dims = [0, 1, 7, 8, 9, 255, 256, 257, 512, 515] + list(rng.integers(1, 420, 30))
    bad = 0
    for dt in (np.float32, np.float64):
        for i in range(60):
            m, n = int(dims[i % len(dims)]), int(dims[(7 * i + 3) % len(dims)])
            lay = i % 2
            A = rng.uniform(-1, 1, m * n).astype(dt)
            x = rng.uniform(-1, 1, n).astype(dt)
            c = rng.uniform(-1, 1, m).astype(dt)
            s = O.RefSession("gemv-col" if lay else "gemv-row", dt, lay, m, n, A, x, c)
            s.run(True)
            want = c.copy()
            O.gemv_ref(A, lay, x, want)
            bad += not np.array_equal(s.output(), want)
            s.close()
            xd, yd = rng.uniform(-1, 1, n).astype(dt), rng.uniform(-1, 1, n).astype(dt)
            sd = O.RefSession("dot", dt, 0, 0, n, None, xd, yd, 0.5)
            bad += sd.run(True) != O.dot_ref(xd, yd, 0.5)
            sd.close()
            gx, gy = rng.uniform(-1, 1, m).astype(dt), rng.uniform(-1, 1, n).astype(dt)
            C0 = rng.uniform(-1, 1, m * n).astype(dt)
            sg = O.RefSession("ger", dt, lay, m, n, C0, gx, gy)
            sg.run(True)
            O.ger_ref(gx, gy, C0, lay)
            bad += not np.array_equal(sg.output(), C0)
            sg.close()
    assert bad == 0


@needs_ref
def test_reference_dispatch_probe_semantics():
    """The probe values the GPU drop-in mirrors (kernels.hpp:140-163, :240-256)."""
    if not O.ref_available():
        O.build(ref=True)
    md_cutoff = 8192  # default fp64 plan: 2 * 32 KiB / 8 B
    x = np.ones(md_cutoff)
    s = O.RefSession("dot", np.float64, 0, 0, md_cutoff, None, x, x, 0.0, cores=8)
    s.run(False, 4)
    assert (s.variant, s.threads_used) == (1, 1)  # dot_small, 1
    x1 = np.ones(md_cutoff + 1)
    s1 = O.RefSession("dot", np.float64, 0, 0, md_cutoff + 1, None, x1, x1, 0.0, cores=8)
    s1.run(False, 4)
    assert s1.variant == 2 and s1.threads_used >= 2  # dot_blocked


def test_truth_is_more_accurate_than_tolerance():
    x = O.gen_uniform(1 << 16, np.float32, 5, 1)
    y = O.gen_uniform(1 << 16, np.float32, 5, 2)
    truth, sumabs = O.dot_truth(x, y, 0.0)
    exact = float(np.sum(x.astype(np.float64) * y.astype(np.float64), dtype=np.float64))
    assert abs(truth - exact) <= 1e-9 * sumabs
    assert sumabs > 0
