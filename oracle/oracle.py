"""TEST INFRASTRUCTURE ONLY — Python access to the CPU oracle.

Two libraries live under ``oracle/``:

* ``libcabl_oracle.so`` — the plain-C restatement in ``cabl_oracle.c`` (naive
  oracles with pinned FP semantics, the SplitMix64 generator, extended
  precision truth).  Always buildable (gcc only).
* ``_ref/libcabl_ref.so`` — the UNMODIFIED reference templates
  (``/root/reference/proj/include/cabl/kernels.hpp``) behind ``ref_shim.cpp``.
  Built only where the reference is mounted; it travels to the GPU box as a
  prebuilt file and is then used as the timed CPU baseline.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline /
``--impl reference``) may import this module, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "libcabl_oracle.so"
REF_SO = HERE / "_ref" / "libcabl_ref.so"
REF_INCLUDE = Path("/root/reference/proj/include")

u64 = C.c_uint64
vp = C.c_void_p

OP = {"dot": 0, "gemv-row": 1, "gemv-col": 2, "ger": 3}
ROW, COL = 0, 1


def build(ref: bool | None = None) -> None:
    """Compile the restatement, and the reference shim when the reference is mounted."""
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    if ref is None:
        ref = REF_INCLUDE.is_dir()
    if ref:
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


_lib = None
_ref = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not ORACLE_SO.exists():
            build(ref=False)
        L = C.CDLL(str(ORACLE_SO))
        L.oracle_sm64_key.restype = u64
        L.oracle_sm64_key.argtypes = [u64, u64]
        L.oracle_sm64.restype = u64
        L.oracle_sm64.argtypes = [u64, u64]
        for nm in ("oracle_gen_uniform_f32", "oracle_gen_uniform_f64", "oracle_gen_normal_f64"):
            getattr(L, nm).argtypes = [vp, u64, u64, u64, u64]
            getattr(L, nm).restype = None
        L.oracle_dot_ref_f32.restype = C.c_float
        L.oracle_dot_ref_f32.argtypes = [vp, vp, u64, C.c_float, C.c_uint]
        L.oracle_dot_ref_f64.restype = C.c_double
        L.oracle_dot_ref_f64.argtypes = [vp, vp, u64, C.c_double, C.c_uint]
        for s in ("f32", "f64"):
            getattr(L, f"oracle_gemv_ref_{s}").argtypes = [vp, C.c_int, u64, u64, vp, vp, C.c_uint]
            getattr(L, f"oracle_ger_ref_{s}").argtypes = [vp, vp, vp, C.c_int, u64, u64]
            getattr(L, f"oracle_dot_truth_{s}").argtypes = [vp, vp, u64,
                                                            C.c_float if s == "f32" else C.c_double,
                                                            vp, vp]
            getattr(L, f"oracle_gemv_truth_{s}").argtypes = [vp, C.c_int, u64, u64, vp, vp, vp, vp]
        _lib = L
    return _lib


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")
        L = C.CDLL(str(REF_SO))
        L.cabl_ref_new.restype = vp
        L.cabl_ref_new.argtypes = [C.c_int, C.c_int, C.c_int, u64, u64, vp, vp, vp, C.c_double,
                                   C.c_uint]
        L.cabl_ref_run.restype = C.c_int
        L.cabl_ref_run.argtypes = [vp, C.c_int, C.c_uint, C.POINTER(C.c_double)]
        L.cabl_ref_get.argtypes = [vp, vp]
        L.cabl_ref_set_out.argtypes = [vp, vp]
        L.cabl_ref_last_threads.restype = C.c_uint
        L.cabl_ref_last_threads.argtypes = [vp]
        L.cabl_ref_last_variant.restype = C.c_int
        L.cabl_ref_last_variant.argtypes = [vp]
        L.cabl_ref_free.argtypes = [vp]
        L.cabl_ref_last_error.restype = C.c_char_p
        _ref = L
    return _ref


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"] or a.flags["F_CONTIGUOUS"]
    return a.ctypes.data


def _suffix(dtype) -> str:
    return "f32" if np.dtype(dtype) == np.float32 else "f64"


# ----------------------------------------------------------------- generator
def gen_uniform(n: int, dtype, seed: int, stream: int, offset: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=dtype)
    getattr(lib(), f"oracle_gen_uniform_{_suffix(dtype)}")(_p(out), n, seed, stream, offset)
    return out


def gen_normal_f64(n: int, seed: int, stream: int, offset: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib().oracle_gen_normal_f64(_p(out), n, seed, stream, offset)
    return out


# ----------------------------------------------------- restated naive oracles
# ``vec``: how many leading terms (a multiple of vec) accumulate as separately
# rounded mul-then-add before the FMA remainder — see cabl_oracle.c.  The
# default, 16 // itemsize, is the compiled reference's own semantics.
def ref_vec(dtype) -> int:
    return 16 // np.dtype(dtype).itemsize


def dot_ref(x: np.ndarray, y: np.ndarray, alpha0: float, vec: int | None = None):
    if x.shape != y.shape:
        raise ValueError("dot: x and y lengths differ")
    v = ref_vec(x.dtype) if vec is None else vec
    f = getattr(lib(), f"oracle_dot_ref_{_suffix(x.dtype)}")
    return x.dtype.type(f(_p(x), _p(y), x.size, alpha0, v))


def gemv_ref(A: np.ndarray, layout: int, x: np.ndarray, c: np.ndarray,
             vec: int | None = None) -> None:
    """c += A x in place.  ``A`` is the flat storage buffer of an m x n matrix."""
    m, n = c.size, x.size
    assert A.size == m * n
    v = ref_vec(A.dtype) if vec is None else vec
    getattr(lib(), f"oracle_gemv_ref_{_suffix(A.dtype)}")(_p(A), layout, m, n, _p(x), _p(c), v)


def ger_ref(x: np.ndarray, y: np.ndarray, C_: np.ndarray, layout: int) -> None:
    m, n = x.size, y.size
    assert C_.size == m * n
    getattr(lib(), f"oracle_ger_ref_{_suffix(C_.dtype)}")(_p(x), _p(y), _p(C_), layout, m, n)


def dot_truth(x: np.ndarray, y: np.ndarray, alpha0: float) -> tuple[float, float]:
    t, s = C.c_double(), C.c_double()
    getattr(lib(), f"oracle_dot_truth_{_suffix(x.dtype)}")(_p(x), _p(y), x.size, alpha0,
                                                          C.byref(t), C.byref(s))
    return t.value, s.value


def gemv_truth(A, layout, x, c0) -> tuple[np.ndarray, np.ndarray]:
    m, n = c0.size, x.size
    truth = np.empty(m, np.float64)
    rowabs = np.empty(m, np.float64)
    getattr(lib(), f"oracle_gemv_truth_{_suffix(A.dtype)}")(_p(A), layout, m, n, _p(x), _p(c0),
                                                           _p(truth), _p(rowabs))
    return truth, rowabs


# ------------------------------------------------- the compiled reference path
class RefSession:
    """One reference call site with inputs already inside reference containers."""

    def __init__(self, op: str, dtype, layout: int, m: int, n: int, a=None, x=None, y=None,
                 alpha0: float = 0.0, cores: int | None = None):
        self.L = ref()
        self.op, self.m, self.n = op, m, n
        self.dtype = np.dtype(dtype)
        self.cores = cores or os.cpu_count() or 1
        self.h = self.L.cabl_ref_new(OP[op], self.dtype.itemsize, layout, m, n, _p(a), _p(x),
                                     _p(y), float(alpha0), self.cores)
        if not self.h:
            raise ValueError(self.L.cabl_ref_last_error().decode())

    def run(self, use_ref: bool, threads: int = 1):
        out = C.c_double()
        rc = self.L.cabl_ref_run(self.h, int(use_ref), threads, C.byref(out))
        if rc:
            raise ValueError(self.L.cabl_ref_last_error().decode())
        return self.dtype.type(out.value) if self.op == "dot" else None

    def output(self) -> np.ndarray:
        size = self.m if self.op.startswith("gemv") else self.m * self.n
        out = np.empty(size, self.dtype)
        self.L.cabl_ref_get(self.h, _p(out))
        return out

    def set_output(self, src: np.ndarray) -> None:
        self.L.cabl_ref_set_out(self.h, _p(np.ascontiguousarray(src, self.dtype)))

    @property
    def threads_used(self) -> int:
        return self.L.cabl_ref_last_threads(self.h)

    @property
    def variant(self) -> int:
        return self.L.cabl_ref_last_variant(self.h)

    def close(self):
        if self.h:
            self.L.cabl_ref_free(self.h)
            self.h = None

    __del__ = close


def time_ref(session: RefSession, use_ref: bool, threads: int, reps: int,
             reset=None) -> list[float]:
    """Median-of-reps timing of the reference call (reference bench.hpp:191-211 style)."""
    times = []
    session.run(use_ref, threads)  # warm-up
    for _ in range(reps):
        if reset is not None:
            reset()
        t0 = time.perf_counter()
        session.run(use_ref, threads)
        times.append(time.perf_counter() - t0)
    return times
