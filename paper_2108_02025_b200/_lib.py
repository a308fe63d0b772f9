"""ctypes binding of libcabl_cuda.so (the C ABI in include/cabl_cuda.h).

The library is built in-tree (``make -C paper_2108_02025_b200/csrc``, or
``__graft_entry__.build()``).  There is no fallback of any kind: if the
library is missing this module raises at import of the first call, and every
compute entry point returns CABL_ECUDA when no GPU is usable.
"""
from __future__ import annotations

import ctypes as C
import subprocess
import threading
from pathlib import Path

PKG = Path(__file__).resolve().parent
import os as _os

# CABL_LIB points at another build of the library (A/B measurements only)
LIB_PATH = Path(_os.environ["CABL_LIB"]) if _os.environ.get("CABL_LIB") else PKG / "libcabl_cuda.so"
CSRC = PKG / "csrc"

CABL_OK, CABL_EINVAL, CABL_ECUDA, CABL_ENOMEM, CABL_ENCCL = 0, 1, 2, 3, 4
CABL_MGPU_NCCL, CABL_MGPU_PEER = 0, 1
ROW_MAJOR, COL_MAJOR = 0, 1

u64 = C.c_uint64
u32 = C.c_uint32
vp = C.c_void_p
f32 = C.c_float
f64 = C.c_double
i32 = C.c_int


class Probe(C.Structure):
    _fields_ = [("variant", C.c_int), ("threads_used", C.c_uint)]


_P = C.POINTER(Probe)


class GpuMachineC(C.Structure):
    """cabl_gpu_machine (include/cabl_cuda.h)."""
    _fields_ = [("device", C.c_int32), ("cc_major", C.c_int32), ("cc_minor", C.c_int32),
                ("sm_count", C.c_uint32), ("max_threads_per_sm", C.c_uint32),
                ("line_bytes", C.c_uint32), ("smem_per_sm", C.c_uint64),
                ("smem_per_block_optin", C.c_uint64), ("l2_bytes", C.c_uint64),
                ("hbm_bytes", C.c_uint64), ("mem_bus_bits", C.c_uint32), ("reserved", C.c_uint32),
                ("queue_threshold_bytes", C.c_uint64), ("name", C.c_char * 96)]

# symbol -> argtypes (restype is int unless listed in _RESTYPE)
SIGNATURES: dict[str, list] = {
    "cabl_last_error": [],
    "cabl_abi_version": [],
    "cabl_device_count": [],
    "cabl_describe_device": [i32, C.POINTER(GpuMachineC)],
    "cabl_cuda_dot_f32": [vp, vp, u64, f32, vp, u64, _P, vp],
    "cabl_cuda_dot_f64": [vp, vp, u64, f64, vp, u64, _P, vp],
    "cabl_cuda_combine_partials_f32": [vp, u32, f32, vp, vp],
    "cabl_cuda_combine_partials_f64": [vp, u32, f64, vp, vp],
    "cabl_cuda_combine_rows_f32": [vp, u32, u64, vp, vp],
    "cabl_cuda_combine_rows_f64": [vp, u32, u64, vp, vp],
    "cabl_cuda_gemv_rm_f32": [vp, u64, u64, vp, vp, u64, _P, vp],
    "cabl_cuda_gemv_rm_f64": [vp, u64, u64, vp, vp, u64, _P, vp],
    "cabl_cuda_gemv_cm_f32": [vp, u64, u64, vp, vp, u64, _P, vp],
    "cabl_cuda_gemv_cm_f64": [vp, u64, u64, vp, vp, u64, _P, vp],
    "cabl_cuda_ger_rm_f32": [vp, vp, vp, u64, u64, u64, _P, vp],
    "cabl_cuda_ger_rm_f64": [vp, vp, vp, u64, u64, u64, _P, vp],
    "cabl_cuda_ger_cm_f32": [vp, vp, vp, u64, u64, u64, _P, vp],
    "cabl_cuda_ger_cm_f64": [vp, vp, vp, u64, u64, u64, _P, vp],
    "cabl_host_dot_f32": [vp, vp, u64, f32, vp, u64, _P, vp],
    "cabl_host_dot_f64": [vp, vp, u64, f64, vp, u64, _P, vp],
    "cabl_host_gemv_f32": [vp, i32, u64, u64, vp, vp, u64, _P, vp],
    "cabl_host_gemv_f64": [vp, i32, u64, u64, vp, vp, u64, _P, vp],
    "cabl_host_ger_f32": [vp, vp, vp, i32, u64, u64, u64, _P, vp],
    "cabl_host_ger_f64": [vp, vp, vp, i32, u64, u64, u64, _P, vp],
    "cabl_peer_mailbox_create": [C.POINTER(vp)],
    "cabl_peer_mailbox_destroy": [vp],
    "cabl_peer_mailbox_export": [vp, C.c_char_p],
    "cabl_peer_mailbox_import": [C.c_char_p, C.POINTER(vp)],
    "cabl_peer_mailbox_unmap": [vp],
    "cabl_peer_mailbox_state": [vp, C.POINTER(u64), C.POINTER(u64)],
    "cabl_cuda_dot_peer_f32": [vp, vp, u64, f32, vp, vp, i32, i32, u64, _P, vp],
    "cabl_cuda_dot_peer_f64": [vp, vp, u64, f64, vp, vp, i32, i32, u64, _P, vp],
    "cabl_cuda_dot_peer_emulate_f32": [i32, vp, vp, vp, f32, vp, vp, u64, vp],
    "cabl_cuda_dot_peer_emulate_f64": [i32, vp, vp, vp, f64, vp, vp, u64, vp],
    "cabl_peer_alloc": [u64, C.POINTER(vp)],
    "cabl_peer_free": [vp],
    "cabl_cuda_gemv_rm_gather_f32": [vp, u64, u64, vp, vp, u64, u64, vp, vp, i32, i32, _P, vp],
    "cabl_cuda_gemv_rm_gather_f64": [vp, u64, u64, vp, vp, u64, u64, vp, vp, i32, i32, _P, vp],
    "cabl_cuda_gemv_rm_gather_emulate_f32": [i32, vp, vp, u64, vp, vp, vp, u64, vp, vp, vp],
    "cabl_cuda_gemv_rm_gather_emulate_f64": [i32, vp, vp, u64, vp, vp, vp, u64, vp, vp, vp],
    "cabl_cuda_combine_rows_peer_f32": [vp, u64, vp, vp, vp, i32, i32, vp],
    "cabl_cuda_combine_rows_peer_f64": [vp, u64, vp, vp, vp, i32, i32, vp],
    "cabl_cuda_combine_rows_peer_emulate_f32": [i32, vp, u64, vp, vp, vp, vp],
    "cabl_cuda_combine_rows_peer_emulate_f64": [i32, vp, u64, vp, vp, vp, vp],
    "cabl_cuda_gemv_rm_gather_supported_f32": [vp, u64, u64, vp, C.POINTER(i32)],
    "cabl_cuda_gemv_rm_gather_supported_f64": [vp, u64, u64, vp, C.POINTER(i32)],
    "cabl_mgpu_nccl_version": [C.POINTER(i32)],
    "cabl_mgpu_init": [C.POINTER(i32), i32, C.POINTER(vp)],
    "cabl_mgpu_finalize": [vp],
    "cabl_mgpu_size": [vp],
    "cabl_mgpu_device": [vp, i32],
    "cabl_mgpu_stream": [vp, i32],
    "cabl_mgpu_set_timeout_ms": [vp, u64],
    "cabl_mgpu_last_call_ms": [vp, i32, C.POINTER(f32)],
    "cabl_mgpu_dot_f32": [vp, vp, vp, vp, f32, u64, i32, C.POINTER(f32)],
    "cabl_mgpu_dot_f64": [vp, vp, vp, vp, f64, u64, i32, C.POINTER(f64)],
    "cabl_mgpu_dot_segmented_f32": [vp, vp, vp, vp, u64, f32, u64, C.POINTER(f32)],
    "cabl_mgpu_dot_segmented_f64": [vp, vp, vp, vp, u64, f64, u64, C.POINTER(f64)],
    "cabl_mgpu_gemv_rm_f32": [vp, vp, vp, u64, vp, vp, u64, i32, vp],
    "cabl_mgpu_gemv_rm_f64": [vp, vp, vp, u64, vp, vp, u64, i32, vp],
    "cabl_mgpu_gemv_cm_cols_f32": [vp, vp, u64, vp, vp, vp, u64, i32],
    "cabl_mgpu_gemv_cm_cols_f64": [vp, vp, u64, vp, vp, vp, u64, i32],
    "cabl_mgpu_ger_rm_f32": [vp, vp, vp, vp, u64, vp, u64],
    "cabl_mgpu_ger_rm_f64": [vp, vp, vp, vp, u64, vp, u64],
    "cabl_cuda_fill_uniform_f32": [vp, u64, u64, u64, u64, vp],
    "cabl_cuda_fill_uniform_f64": [vp, u64, u64, u64, u64, vp],
    "cabl_cuda_fill_normal_f64": [vp, u64, u64, u64, u64, vp],
}
_RESTYPE = {"cabl_last_error": C.c_char_p, "cabl_mgpu_stream": C.c_void_p}

_lock = threading.Lock()
_lib: C.CDLL | None = None


def build(verbose: bool = False) -> Path:
    """Compile libcabl_cuda.so for sm_100a (nvcc cross-compiles without a GPU)."""
    cmd = ["make", "-C", str(CSRC), "-j8"]
    if not verbose:
        cmd.insert(1, "-s")
    subprocess.run(cmd, check=True)
    return LIB_PATH


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with "
                        "`make -C paper_2108_02025_b200/csrc` (no CPU fallback exists)")
                L = C.CDLL(str(LIB_PATH))
                for name, args in SIGNATURES.items():
                    fn = getattr(L, name)
                    fn.argtypes = args
                    fn.restype = _RESTYPE.get(name, C.c_int)
                _lib = L
    return _lib


class CablError(RuntimeError):
    """CUDA-side failure (CABL_ECUDA / CABL_ENOMEM)."""


class CablExchangeError(CablError):
    """Multi-GPU exchange failure (CABL_ENCCL): NCCL error, asynchronous NCCL
    error, timed-out peer exchange or context timeout; the context is aborted."""


def check(rc: int) -> None:
    if rc == CABL_OK:
        return
    msg = lib().cabl_last_error().decode()
    if rc == CABL_EINVAL:
        # the reference throws std::invalid_argument (kernels.hpp:59-61)
        raise ValueError(msg)
    if rc == CABL_ENCCL:
        raise CablExchangeError(msg)
    raise CablError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
