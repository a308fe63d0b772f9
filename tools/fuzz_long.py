"""Long randomised differential run of every kernel path against the CPU oracle
(test infrastructure, like tests/test_gpu_fuzz.py, but time-bounded and much
wider): shapes drawn around every dispatch threshold of csrc/*.cu, A / x / y /
c each at its own misalignment, operands framed by guard bands (NaN around the
inputs, a sentinel around the output), every result run twice (bitwise equal)
and held to

  * GER: bitwise equality with ger_ref (reference kernels.hpp:264-313);
  * DOT / GEMV: the BASELINE contract bound against dot_ref / gemv_ref and the
    non-vacuous fp64/fp80-truth bound of tests/tolerances.py.

    python tools/fuzz_long.py --seconds 600 --seed 1 > gpurun_out/fuzz_long.jsonl

Prints one JSON line per failure and a summary line; exit code 1 on any failure.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as O  # noqa: E402
from tests import tolerances as T  # noqa: E402

PAD = 512
SENT = 1234.5678
MAX_ELEMS = 6_000_000

CM_M = [1, 2, 3, 4, 7, 8, 9, 15, 16, 17, 31, 32, 33, 255, 256, 257, 511, 512, 513, 1000, 1023,
        1024, 1025, 2047, 2048, 2049, 3001, 4095, 4096, 4097, 7001, 8191, 8192, 8193, 9215, 9216,
        9217, 12275, 12276, 12277, 14001, 16383, 16384, 16385, 18423, 18424, 18425, 32768, 40001,
        65535, 65536, 65537, 75775, 75776, 75777, 151551, 151552, 151553, 300000, 1 << 20]
SMALL_N = [1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33, 63, 64, 65, 147, 148, 149, 255, 256,
           257, 295, 296, 297, 591, 592, 593]
RM_N = [1, 2, 3, 5, 7, 8, 9, 16, 24, 25, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257,
        1023, 1024, 1025, 1028, 4095, 4096, 4097, 8191, 8192, 8193, 12001, 16384, 40000, 65536,
        65537, 262144, 1 << 20]
RM_M = [1, 2, 3, 5, 15, 16, 17, 40, 255, 256, 257, 1000, 4095, 4096, 4735, 4736, 4737, 9471, 9472,
        9473, 20000, 60000, 200000]


def pick(rng, values, lo, hi):
    """A listed boundary value (half the time, +-2 jitter now and then) or a uniform draw."""
    if rng.integers(0, 2) == 0:
        v = int(rng.choice(values))
        if rng.integers(0, 4) == 0:
            v = max(1, v + int(rng.integers(-2, 3)))
        return v
    return int(np.exp(rng.uniform(np.log(lo), np.log(hi))))


def shape(rng, kind):
    if kind == "dot":
        n = int(rng.choice([int(rng.integers(0, 70)), int(rng.integers(70, 10_000)),
                            int(rng.integers(10_000, 600_000)), int(rng.integers(600_000, MAX_ELEMS)),
                            int(rng.choice([8192, 8193, 148 * 512 * 8, 296 * 512 * 16 + 1, 1 << 22]))]))
        return 0, n
    if kind == "gemv-col":
        m = pick(rng, CM_M, 1, 400_000)
        cap = max(1, MAX_ELEMS // m)
        n = pick(rng, SMALL_N, 1, cap) if rng.integers(0, 3) else int(rng.integers(1, cap + 1))
        return m, max(1, min(n, cap))
    if kind.endswith("col"):  # GER col-major = row-major of the transpose
        n = pick(rng, RM_M, 1, 200_000)
        cap = max(1, MAX_ELEMS // n)
        m = pick(rng, RM_N, 1, cap)
        return max(1, min(m, cap)), n
    if rng.integers(0, 2):
        n = pick(rng, RM_N, 1, 1 << 20)
        cap = max(1, MAX_ELEMS // n)
        m = pick(rng, RM_M, 1, cap)
        return max(1, min(m, cap)), n
    m = pick(rng, RM_M, 1, 200_000)
    cap = max(1, MAX_ELEMS // m)
    n = pick(rng, RM_N, 1, cap)
    return m, max(1, min(n, cap))


def framed(a, off, fill, dev):
    """Device copy of `a` starting `off` elements past a 256-byte boundary,
    with PAD elements of `fill` on either side; returns (whole buffer, view)."""
    t = torch.full((PAD + off + a.size + PAD,), fill, dtype=torch.from_numpy(a[:0]).dtype, device=dev)
    if a.size:
        t[PAD + off:PAD + off + a.size] = torch.from_numpy(a)
    return t, t[PAD + off:PAD + off + a.size]


def bands_ok(buf, off, size):
    lo, hi = PAD + off, PAD + off + size
    return bool((buf[:lo] == SENT).all()) and bool((buf[hi:] == SENT).all())


def one_case(cb, rng, kind, seed, dev):
    dt = np.float32 if rng.integers(0, 2) == 0 else np.float64
    offs = [int(rng.choice([0, 0, 0, 1, 2, 3, 4, 5, 7, 8])) for _ in range(3)]
    if rng.integers(0, 3) == 0:
        offs = [offs[0]] * 3  # shared misalignment (slices of one aligned buffer)
    m, n = shape(rng, kind)
    info = {"kind": kind, "dtype": np.dtype(dt).name, "m": m, "n": n, "offs": offs, "seed": seed}
    pol = cb.default_policy(1)
    nan = float("nan")
    if kind == "dot":
        x, y = O.gen_uniform(n, dt, seed, 1), O.gen_uniform(n, dt, seed, 2)
        _, xd = framed(x, offs[0], nan, dev)
        _, yd = framed(y, offs[1], nan, dev)
        ob, ov = framed(np.zeros(1, dt), offs[2], SENT, dev)
        cb.dot_into(xd, yd, 0.375, ov, pol)
        got = float(ov.cpu()[0])
        cb.dot_into(xd, yd, 0.375, ov, pol)
        if float(ov.cpu()[0]) != got and not (np.isnan(got)):
            return dict(info, fail="not reproducible")
        if not bands_ok(ob, offs[2], 1):
            return dict(info, fail="write outside out")
        truth, sumabs = O.dot_truth(x, y, 0.375)
        if not abs(got - float(O.dot_ref(x, y, 0.375))) <= T.contract_tol(n, sumabs, 0.375, dt):
            return dict(info, fail="contract", got=got, truth=truth)
        if not abs(got - truth) <= T.truth_tol(T.dot_chain(n, dt) + 8, sumabs, 0.375, dt):
            return dict(info, fail="truth", got=got, truth=truth)
        return None
    lay = cb.Layout.RowMajor if kind.endswith("row") else cb.Layout.ColMajor
    if kind.startswith("gemv"):
        A = O.gen_uniform(m * n, dt, seed, 3)
        x, c0 = O.gen_uniform(n, dt, seed, 1), O.gen_uniform(m, dt, seed, 4)
        _, Ad = framed(A, offs[0], nan, dev)
        _, xd = framed(x, offs[1], nan, dev)
        b1, c1 = framed(c0, offs[2], SENT, dev)
        b2, c2 = framed(c0, offs[2], SENT, dev)
        f = cb.gemv_row_major if lay == cb.Layout.RowMajor else cb.gemv_col_major
        Am = cb.DenseMatrix.wrap(Ad, m, n, lay)
        f(Am, xd, c1, pol)
        f(Am, xd, c2, pol)
        torch.cuda.synchronize()
        if not torch.equal(c1, c2):
            return dict(info, fail="not reproducible")
        if not (bands_ok(b1, offs[2], m) and bands_ok(b2, offs[2], m)):
            return dict(info, fail="write outside c")
        got = c1.cpu().numpy().astype(np.float64)
        if not np.all(np.isfinite(got)):
            return dict(info, fail="read outside an input (non-finite c)")
        want = c0.copy()
        O.gemv_ref(A, int(lay), x, want)
        truth, rowabs = O.gemv_truth(A, int(lay), x, c0)
        bad = ~(np.abs(got - want) <= T.contract_tol(n, rowabs, np.abs(c0), dt))
        if bad.any():
            i = int(np.argmax(bad))
            return dict(info, fail="contract", row=i, rows_bad=int(bad.sum()), got=got[i], want=float(want[i]))
        if lay == cb.Layout.RowMajor:
            chain = T.gemv_rm_chain(n, dt)
        else:
            chain = max(T.gemv_cm_chain(m, n, dt), min(n, 600) + 1)
        bad = ~(np.abs(got - truth) <= T.truth_tol(chain, rowabs, np.abs(c0), dt))
        if bad.any():
            i = int(np.argmax(bad))
            return dict(info, fail="truth", row=i, rows_bad=int(bad.sum()), got=got[i], truth=float(truth[i]))
        return None
    x, y = O.gen_uniform(m, dt, seed, 1), O.gen_uniform(n, dt, seed, 2)
    C0 = O.gen_uniform(m * n, dt, seed, 5)
    Cb, Cd = framed(C0, offs[0], SENT, dev)
    _, xd = framed(x, offs[1], nan, dev)
    _, yd = framed(y, offs[2], nan, dev)
    cb.ger(xd, yd, cb.DenseMatrix.wrap(Cd, m, n, lay), pol)
    torch.cuda.synchronize()
    if not bands_ok(Cb, offs[0], m * n):
        return dict(info, fail="write outside C")
    want = C0.copy()
    O.ger_ref(x, y, want, int(lay))
    got = Cd.cpu().numpy()
    if not np.array_equal(got, want):
        bad = np.flatnonzero(got != want)
        return dict(info, fail="bits", first=int(bad[0]), count=int(bad.size))
    return None


def main():
    global MAX_ELEMS
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--kinds", default="dot,gemv-row,gemv-col,gemv-col,ger-row,ger-col")
    ap.add_argument("--max-elems", type=int, default=MAX_ELEMS,
                    help="largest operand in elements (the CPU oracle's time per case grows with it)")
    args = ap.parse_args()
    MAX_ELEMS = args.max_elems
    import paper_2108_02025_b200 as cb
    dev = torch.device("cuda:0")
    kinds = args.kinds.split(",")
    t0 = time.time()
    done, fails, per = 0, 0, {}
    case = args.seed * 1_000_000
    while time.time() - t0 < args.seconds:
        kind = kinds[done % len(kinds)]
        rng = np.random.default_rng(case)
        try:
            r = one_case(cb, rng, kind, case % 100_000, dev)
        except Exception as e:  # a raised error is a failure of the case, not of the run
            r = {"kind": kind, "case": case, "fail": f"exception: {e!r}"[:300]}
        if r is not None:
            fails += 1
            r["case"] = case
            print(json.dumps(r, default=float), flush=True)
        per[kind] = per.get(kind, 0) + 1
        done += 1
        case += 1
    print(json.dumps({"summary": True, "cases": done, "failures": fails, "per_kind": per,
                      "seconds": round(time.time() - t0, 1), "seed": args.seed,
                      "max_elems": MAX_ELEMS}), flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
