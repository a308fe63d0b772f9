#!/usr/bin/env python
"""Generate tests/golden/reference_golden.npz from the COMPILED, UNMODIFIED
reference (oracle/_ref/libcabl_ref.so: /root/reference/proj/include/cabl/
kernels.hpp built with the reference flags by oracle/Makefile).

Run in the build container (where /root/reference is mounted):

    make -C oracle all ref && python tests/golden/make_golden.py

Inputs are NOT stored: each case records the (seed, stream) of its seeded
SplitMix64 inputs (oracle/cabl_oracle.c; the generator's first outputs are
pinned in the file) and the reference's outputs of the naive oracles dot_ref / gemv_ref / ger_ref
(kernels.hpp:119-127, :171-181, :264-270) and of the threaded paths dot /
gemv_row_major / gemv_col_major / ger (:134-313) at threads = 1 and 4, so the
oracle restatement and the GPU path can be checked against the reference's
own bits on a machine where the reference is absent (the GPU box).
"""
from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402

OUT = Path(__file__).resolve().parent / "reference_golden.npz"
SEED = 20260810  # the reference acceptance suite's seed (acceptance.cpp:106)

DOT_N = [0, 1, 3, 7, 8, 9, 31, 33, 1000, 4097, 8192, 8193, 16385, 20001]
GEMV_SHAPES = [(0, 5), (5, 0), (1, 1), (1, 777), (3, 3), (8, 8), (9, 7), (31, 33), (256, 257),
               (257, 256), (100, 1000)]
GER_SHAPES = [(1, 1), (2, 3), (7, 9), (33, 31), (256, 257), (500, 40)]


def main():
    if not O.ref_available():
        O.build(ref=True)
    rec = {}
    case = 0
    for dt in (np.float32, np.float64):
        tag = np.dtype(dt).name
        for n in DOT_N:
            x = O.gen_uniform(n, dt, SEED, 1 + case)
            y = O.gen_uniform(n, dt, SEED, 1001 + case)
            s = O.RefSession("dot", dt, 0, 0, n, None, x, y, 0.25, cores=4)
            rec[f"dot/{tag}/{n}/streams"] = np.array([1 + case, 1001 + case], np.uint64)
            rec[f"dot/{tag}/{n}/ref"] = np.array([s.run(True)], dt)
            rec[f"dot/{tag}/{n}/t1"] = np.array([s.run(False, 1)], dt)
            rec[f"dot/{tag}/{n}/t4"] = np.array([s.run(False, 4)], dt)
            s.close()
            case += 1
        for lay, op in ((0, "gemv-row"), (1, "gemv-col")):
            for m, n in GEMV_SHAPES:
                A = O.gen_uniform(m * n, dt, SEED, 2001 + case)
                x = O.gen_uniform(n, dt, SEED, 3001 + case)
                c = O.gen_uniform(m, dt, SEED, 4001 + case)
                key = f"{op}/{tag}/{m}x{n}"
                rec[key + "/streams"] = np.array([2001 + case, 3001 + case, 4001 + case], np.uint64)
                s = O.RefSession(op, dt, lay, m, n, A, x, c, cores=4)
                s.run(True)
                rec[key + "/ref"] = s.output()
                for t in (1, 4):
                    s.set_output(c)
                    s.run(False, t)
                    rec[key + f"/t{t}"] = s.output()
                s.close()
                case += 1
        for lay, ln in ((0, "row"), (1, "col")):
            for m, n in GER_SHAPES:
                C0 = O.gen_uniform(m * n, dt, SEED, 5001 + case)
                x = O.gen_uniform(m, dt, SEED, 6001 + case)
                y = O.gen_uniform(n, dt, SEED, 7001 + case)
                key = f"ger-{ln}/{tag}/{m}x{n}"
                rec[key + "/streams"] = np.array([5001 + case, 6001 + case, 7001 + case], np.uint64)
                s = O.RefSession("ger", dt, lay, m, n, C0, x, y, cores=4)
                s.run(True)
                out = s.output()
                rec[key + "/ref_sha256"] = np.array([hashlib.sha256(out.tobytes()).hexdigest()])
                rec[key + "/ref_head"] = out[:16]
                s.set_output(C0)
                s.run(False, 4)
                rec[key + "/t4_sha256"] = np.array(
                    [hashlib.sha256(s.output().tobytes()).hexdigest()])
                s.close()
                case += 1
    # first SplitMix64 outputs, pinned
    key = O.lib().oracle_sm64_key(42, 1)
    rec["sm64/key_42_1"] = np.array([key], np.uint64)
    rec["seed"] = np.array([SEED], np.uint64)
    rec["sm64/first8"] = np.array([O.lib().oracle_sm64(key, i) for i in range(8)], np.uint64)
    np.savez_compressed(OUT, **rec)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(rec)} arrays)")


if __name__ == "__main__":
    main()
