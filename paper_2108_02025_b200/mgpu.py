"""Python mirror of the multi-GPU C ABI (``cabl_mgpu_*``, include/cabl_cuda.h):
one process driving several devices, the process model of SURVEY.md §8(e)
(``include/cabl/nccl.hpp`` is the C++ mirror).  Shards are lists of CUDA
tensors, shard r on ``devices[r]``; the partition is the caller's (balanced
contiguous ranges, ``partition``, as the reference's parallel_chunks,
thread_pool.hpp:153-164).

Every call is synchronous and validated on all shards before anything runs.
A failed exchange (NCCL error, asynchronous NCCL error, timed-out peer
exchange, context timeout) raises ``CablExchangeError`` after the library
aborted the communicators; the context must then be closed.

    with MultiGpu([0, 1]) as mg:
        total = mg.dot(xs, ys, alpha0, exchange="nccl")
"""
from __future__ import annotations

import ctypes as C

from . import _lib
from . import cabl

EXCHANGE = {"nccl": _lib.CABL_MGPU_NCCL, "peer": _lib.CABL_MGPU_PEER}


def partition(total: int, parts: int, rank: int) -> tuple[int, int]:
    q, r = divmod(total, parts)
    b = rank * q + min(rank, r)
    return b, b + q + (1 if rank < r else 0)


def nccl_version() -> int:
    v = C.c_int()
    _lib.call("cabl_mgpu_nccl_version", C.byref(v))
    return v.value


def _ptrs(ts) -> C.Array:
    return (C.c_void_p * len(ts))(*[t.data_ptr() if t is not None and t.numel() else None
                                   for t in ts])


def _u64s(vals) -> C.Array:
    return (C.c_uint64 * len(vals))(*vals)


class MultiGpu:
    def __init__(self, devices: list[int], timeout_ms: int | None = None):
        self.devices = list(devices)
        arr = (C.c_int * len(self.devices))(*self.devices)
        self._ctx = C.c_void_p()
        _lib.call("cabl_mgpu_init", arr, len(self.devices), C.byref(self._ctx))
        if timeout_ms is not None:
            _lib.call("cabl_mgpu_set_timeout_ms", self._ctx, int(timeout_ms))

    # -- lifecycle
    def close(self) -> None:
        if self._ctx is not None and self._ctx.value:
            _lib.lib().cabl_mgpu_finalize(self._ctx)
        self._ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass

    @property
    def size(self) -> int:
        return _lib.lib().cabl_mgpu_size(self._ctx)

    def stream(self, rank: int) -> int:
        return _lib.lib().cabl_mgpu_stream(self._ctx, rank)

    def set_timeout_ms(self, ms: int) -> None:
        _lib.call("cabl_mgpu_set_timeout_ms", self._ctx, int(ms))

    def last_call_ms(self) -> list[float]:
        """Device time of the last call on every rank (CUDA events around its
        work on the rank's stream); the multi-GPU time is the max."""
        out = []
        for r in range(len(self.devices)):
            v = C.c_float()
            _lib.call("cabl_mgpu_last_call_ms", self._ctx, r, C.byref(v))
            out.append(v.value)
        return out

    # -- checks shared by the ops
    def _shards(self, what: str, *groups) -> str:
        G = len(self.devices)
        sfx = None
        for grp in groups:
            cabl._require(len(grp) == G, f"{what}: one shard per device")
            for r, t in enumerate(grp):
                cabl._require(t.is_cuda and t.device.index == self.devices[r],
                              f"{what}: shard {r} must be on cuda:{self.devices[r]}")
                cabl._require(t.is_contiguous(), f"{what}: shards must be contiguous")
                s = cabl._suffix(t)
                cabl._require(sfx in (None, s), f"{what}: shards must share one dtype")
                sfx = s
        # the context's streams do not wait on the caller's: let the work that
        # produced the shards (torch's current stream per device) finish first
        import torch
        for d in self.devices:
            torch.cuda.current_stream(d).synchronize()
        return sfx

    # -- ops
    def dot(self, xs, ys, alpha0: float, policy=None, exchange: str = "nccl") -> float:
        sfx = self._shards("dot", xs, ys)
        for x, y in zip(xs, ys):
            cabl._require(x.numel() == y.numel(), "dot: x and y lengths differ")
        pol = policy or cabl.default_policy(1)
        out = C.c_float() if sfx == "f32" else C.c_double()
        val = C.c_float(alpha0) if sfx == "f32" else C.c_double(alpha0)
        _lib.call(f"cabl_mgpu_dot_{sfx}", self._ctx, _ptrs(xs), _ptrs(ys),
                  _u64s([x.numel() for x in xs]), val, pol.plan.dot_cutoff, EXCHANGE[exchange],
                  C.byref(out))
        return out.value

    def dot_segmented(self, xs, ys, alpha0: float, segment: int, policy=None) -> float:
        """alpha0 + the partials of the fixed global segments (every `segment` elements of
        the concatenated shards) summed in index order: the same bits for every device
        count.  Every shard before the last non-empty one must be whole segments."""
        sfx = self._shards("dot", xs, ys)
        for x, y in zip(xs, ys):
            cabl._require(x.numel() == y.numel(), "dot: x and y lengths differ")
        pol = policy or cabl.default_policy(1)
        out = C.c_float() if sfx == "f32" else C.c_double()
        val = C.c_float(alpha0) if sfx == "f32" else C.c_double(alpha0)
        _lib.call(f"cabl_mgpu_dot_segmented_{sfx}", self._ctx, _ptrs(xs), _ptrs(ys),
                  _u64s([x.numel() for x in xs]), C.c_uint64(segment), val, pol.plan.dot_cutoff,
                  C.byref(out))
        return out.value

    def gemv_rm(self, As, xs, cs, policy=None, exchange: str = "nccl", c_full=None) -> None:
        """c[r] += A[r] x[r] (row blocks, A[r] a row-major DenseMatrix); with
        c_full every device also receives the whole updated c."""
        Ad = [a.data for a in As]
        groups = [Ad, xs, cs] + ([c_full] if c_full is not None else [])
        sfx = self._shards("gemv_row_major", *groups)
        n = As[0].cols()
        for a, x, c in zip(As, xs, cs):
            cabl._require(a.layout() == cabl.Layout.RowMajor, "gemv_row_major: matrix is not row-major")
            cabl._require(a.cols() == x.numel() == n, "gemv: A.cols != x.len")
            cabl._require(a.rows() == c.numel(), "gemv: A.rows != c.len")
        pol = policy or cabl.default_policy(1)
        _lib.call(f"cabl_mgpu_gemv_rm_{sfx}", self._ctx, _ptrs(Ad), _u64s([a.rows() for a in As]),
                  n, _ptrs(xs), _ptrs(cs), pol.plan.dot_cutoff, EXCHANGE[exchange],
                  _ptrs(c_full) if c_full is not None else None)

    def gemv_cm_cols(self, As, xs, cs, policy=None, exchange: str = "nccl") -> None:
        """Column blocks: every replica c[r] += rank-ordered sum of A[r] x[r]."""
        Ad = [a.data for a in As]
        sfx = self._shards("gemv_col_major", Ad, xs, cs)
        m = cs[0].numel()
        for a, x, c in zip(As, xs, cs):
            cabl._require(a.layout() == cabl.Layout.ColMajor, "gemv_col_major: matrix is not col-major")
            cabl._require(a.cols() == x.numel(), "gemv: A.cols != x.len")
            cabl._require(a.rows() == m and c.numel() == m,
                          "sharded_gemv_cols: col-major blocks of m rows, c replicas of length m")
        pol = policy or cabl.default_policy(1)
        _lib.call(f"cabl_mgpu_gemv_cm_cols_{sfx}", self._ctx, _ptrs(Ad), m,
                  _u64s([a.cols() for a in As]), _ptrs(xs), _ptrs(cs), pol.plan.dot_cutoff,
                  EXCHANGE[exchange])

    def ger_rm(self, xs, ys, Cs, policy=None) -> None:
        """C[r] += x[r] (x) y[r] on row blocks of a row-major C (no exchange)."""
        Cd = [c.data for c in Cs]
        sfx = self._shards("ger", xs, ys, Cd)
        n = Cs[0].cols()
        for x, y, c in zip(xs, ys, Cs):
            cabl._require(c.layout() == cabl.Layout.RowMajor, "ger: multi-GPU row blocks need a row-major C")
            cabl._require(c.rows() == x.numel(), "ger: C.rows != x.len")
            cabl._require(c.cols() == y.numel() == n, "ger: C.cols != y.len")
        pol = policy or cabl.default_policy(1)
        _lib.call(f"cabl_mgpu_ger_rm_{sfx}", self._ctx, _ptrs(xs), _u64s([c.rows() for c in Cs]),
                  _ptrs(ys), n, _ptrs(Cd), pol.plan.dot_cutoff)


__all__ = ["MultiGpu", "partition", "nccl_version", "EXCHANGE"]
