"""Error bounds used by the parity tests (written down once, cited everywhere).

BASELINE.json's contract for fp32 DOT and GEMV (per output element):

    |gpu - oracle| <= 4 * n * eps * sum_i |a_i * b_i|

It matches the reference tests' own bound (reference test_kernels.cpp:36-50,
acceptance.cpp:142,158,177) up to the factor 4, and becomes vacuous for fp32
once 4 n eps >= 1 (n >= 2^21) — SURVEY.md §0 finding 3.  The reference's form
also omits the initial |c_i|, which breaks its own criterion 1 on one
instance; we add |c_i| (|alpha0|) to the sum.

Next to the contract, every DOT/GEMV result is held to a NON-VACUOUS bound
against extended-precision truth (fp32: exact products summed in 80-bit;
fp64: Dot2 compensated) — the standard a priori bound gamma_L * S with
L = the longest chain of roundings any output passes through on the GPU:

    |gpu - truth| <= (L + 2) * eps * (S + |c0|)

L is stated per kernel below from its decomposition (a per-lane sequential
chain, then fixed trees of adds).  GER is held to bitwise equality with the
oracle (one FMA per element, reference kernels.hpp:264-313).
"""
from __future__ import annotations

import math

import os

import numpy as np

EPS = {np.dtype(np.float32): float(np.finfo(np.float32).eps),
       np.dtype(np.float64): float(np.finfo(np.float64).eps)}

SMS = 148  # B200


def contract_tol(n: int, sumabs, c0abs, dtype):
    """BASELINE.json: 4 n eps (sum |a b| + |c0|) — with the |c0| term added."""
    return 4.0 * max(n, 1) * EPS[np.dtype(dtype)] * (np.asarray(sumabs) + np.asarray(c0abs))


def log2c(v: int) -> int:
    return max(1, math.ceil(math.log2(max(v, 2))))


def dot_chain(n: int, dtype, block: int = 512, unroll: int = 2, ctas_per_sm: int = 2) -> int:
    """dot_kernel (csrc/dot.cu): grid G <= 148*ctas_per_sm CTAs x block
    threads, each thread one FMA chain per accumulator over its share (U
    accumulators, V elements per vector), then U-1 adds, a 5-level warp
    butterfly, log2(warps) levels across warps, a sequential pass of
    ceil(G/block) partials per thread in the last CTA, the same two trees
    again, and + alpha0."""
    V = 32 // np.dtype(dtype).itemsize
    nvec = n // V
    if 2 * n * np.dtype(dtype).itemsize >= (512 << 20) and nvec >= SMS * ctas_per_sm:
        # chunked kernel (csrc/dot.cu chunk_vecs): power-of-two chunks of
        # <= nvec / 2048 vectors in [4096, 65536], partials summed in order
        cv = 4096
        while cv * 2 <= 65536 and cv * 2 * 2048 <= nvec:
            cv *= 2
        chunks = math.ceil(nvec / cv)
        per_acc = math.ceil(cv / (block * unroll)) * V
        tree = 5 + log2c(block // 32)
        return per_acc + unroll + tree + math.ceil(chunks / block) + tree + V + 1
    G = max(1, min(math.ceil(nvec / (block * unroll)), SMS * ctas_per_sm))
    per_thread = math.ceil(max(nvec, 1) / (G * block)) * V + V
    tree = 5 + log2c(block // 32)
    return per_thread + unroll + tree + math.ceil(G / block) + tree + 1


def gemv_rm_chain(n: int, dtype) -> int:
    """gemv_rm_vec_kernel: each lane FMA-chains n/32 elements of a row, a
    5-level butterfly, then at most (warps touching the row) adds of partials
    and + c_i.  A row touches at most ceil(row units / per-warp units)+1 warps;
    bounded by 64 here for every shape the tests use."""
    return math.ceil(n / 32) + 5 + 64 + 1


def rm_is_ordered(m: int, n: int, dtype, aligned: bool = True) -> bool:
    """csrc/gemv_rm_ordered.cu gemv_rm_ordered_ok: with CABL_GEMV_RM_ORDER=
    reference the reference-order row-major kernel (bitwise gemv_ref) runs when
    rows are 16-byte multiples, operands 16-byte aligned and m >= 148 * 32 (a
    full warp of rows per CTA)."""
    return os.environ.get("CABL_TUNING") == "1" and os.environ.get("CABL_GEMV_RM_ORDER") == "reference" and aligned and (n * np.dtype(dtype).itemsize) % 16 == 0 and m >= SMS * 32


def rm_is_lane(m: int, n: int, dtype, aligned: bool = True) -> bool:
    """csrc/gemv_rm.cu gemv_rm_is_lane: rows of <= 256 B and >= 148 * 64 of
    them take the one-thread-per-row kernel — the reference's order and
    rounding, so bitwise gemv_ref — when the rows are whole 32-byte vectors,
    or (scalar loads) at most 24 elements long."""
    s = np.dtype(dtype).itemsize
    vec = aligned and n % (32 // s) == 0
    return n * s <= 256 and m >= SMS * 64 and (vec or n <= 24)


def cm_is_tall(m: int, dtype, aligned: bool = True) -> bool:
    """csrc/gemv_cm.cu cm_path: the bit-exact tall kernels run when m/V >= 74
    units of 256 row vectors (half the SMs; V = 32/s, aligned, m % V == 0) or,
    otherwise, m >= 148 * 1024."""
    V = 32 // np.dtype(dtype).itemsize
    if aligned and m % V == 0:
        return m // V >= (SMS // 2) * 256
    return m >= SMS * 1024


def gemv_cm_chain(m: int, n: int, dtype) -> int:
    """Tall kernels: one sequential chain per row over all n columns (the
    reference order).  Split kernels (csrc/gemv_cm.cu): <= 148 column parts,
    each thread a chain over <= ceil(n / G) columns, then its column lanes
    summed in order (< 512 adds in the bulk kernels, where a row can have up
    to 512 column lanes), the G part partials summed in order, + c_i.  The
    full-column sweep: <= ceil(n / 296) columns per thread, <= 8 column lanes,
    <= 296 CTA partials in 32 groups (<= 10 adds, then a 5-level tree), + c_i; with two
    row vectors per thread (fp32 8192 < m <= 16384) <= 148 partials in 16 groups (<= 10
    adds, then a 4-level tree): inside the same bound."""
    if cm_is_tall(m, dtype):
        return n + 1
    G = max(1, min(SMS, n))
    return math.ceil(n / G) + 512 + G + 2


def truth_tol(chain: int, sumabs, c0abs, dtype):
    return (chain + 2) * EPS[np.dtype(dtype)] * (np.asarray(sumabs) + np.asarray(c0abs))
