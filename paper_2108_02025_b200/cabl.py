"""Python mirror of the reference ``cabl`` hot-path API, backed by libcabl_cuda.so.

Same names, argument meaning and error behaviour as the reference C++
templates (``/root/reference/proj/include/cabl/kernels.hpp``):

=====================  ==================================================
reference (C++)         here
=====================  ==================================================
``dot`` :134           ``dot(x, y, alpha0, policy) -> scalar``
``gemv_col_major`` :187 ``gemv_col_major(A, x, c, policy)`` (c updated in place)
``gemv_row_major`` :230 ``gemv_row_major(A, x, c, policy)``
``ger`` :277           ``ger(x, y, C, policy)`` (C updated in place)
``ExecPolicy`` :28     ``ExecPolicy(plan, threads)``
``last_exec()`` :54    ``last_exec()`` (thread-local probe)
``DenseMatrix`` dense.hpp:42  ``DenseMatrix`` (flat tensor + rows/cols/layout)
``Vector`` dense.hpp:16       a 1-D ``torch.Tensor``
=====================  ==================================================

Operands may live on the GPU (``torch.cuda`` tensors: the call only enqueues
on the current stream, except ``dot`` which returns a host scalar) or on the
host (CPU tensors / numpy arrays: staged through the device by the C ABI's
``cabl_host_*`` entry points).  Precondition violations raise ``ValueError``
with the reference's message text (the reference throws
``std::invalid_argument``, kernels.hpp:59-61).  There is no CPU compute path.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import enum
import math
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import Probe

# --------------------------------------------------------------------------
# Layout and dense containers (reference dense.hpp)
# --------------------------------------------------------------------------


class Layout(enum.IntEnum):
    RowMajor = _lib.ROW_MAJOR
    ColMajor = _lib.COL_MAJOR


def layout_name(layout: Layout) -> str:
    return "row-major" if layout == Layout.RowMajor else "col-major"


class DenseMatrix:
    """Dense m x n matrix over one flat buffer; element (i, j) at j + i*cols
    (row-major) or i + j*rows (col-major), reference dense.hpp:54-56."""

    def __init__(self, rows: int, cols: int, layout: Layout, value: float = 0.0, *,
                 dtype=torch.float64, device="cpu", data: torch.Tensor | None = None):
        self._rows, self._cols, self._layout = int(rows), int(cols), Layout(layout)
        if data is None:
            data = torch.full((self._rows * self._cols,), value, dtype=dtype, device=device)
        else:
            if data.numel() != self._rows * self._cols:
                raise ValueError("DenseMatrix: data size != rows*cols")
            data = data.reshape(-1)
        self.data = data

    @classmethod
    def wrap(cls, data: torch.Tensor, rows: int, cols: int, layout: Layout) -> "DenseMatrix":
        return cls(rows, cols, layout, data=data)

    def rows(self) -> int:
        return self._rows

    def cols(self) -> int:
        return self._cols

    def layout(self) -> Layout:
        return self._layout

    def size(self) -> int:
        return self._rows * self._cols

    def index(self, i: int, j: int) -> int:
        return i + j * self._rows if self._layout == Layout.ColMajor else j + i * self._cols

    def __call__(self, i: int, j: int):
        return self.data[self.index(i, j)]

    def __setitem__(self, ij, v):
        self.data[self.index(*ij)] = v

    def to(self, device) -> "DenseMatrix":
        return DenseMatrix(self._rows, self._cols, self._layout, data=self.data.to(device))

    def clone(self) -> "DenseMatrix":
        return DenseMatrix(self._rows, self._cols, self._layout, data=self.data.clone())

    def __eq__(self, other) -> bool:
        return (isinstance(other, DenseMatrix) and self._rows == other._rows
                and self._cols == other._cols and self._layout == other._layout
                and torch.equal(self.data.cpu(), other.data.cpu()))


# --------------------------------------------------------------------------
# Machine model and plan (reference machine.hpp) — policy carrier only: the
# GPU kernels ignore the CPU cache parameters; dot_cutoff drives the
# small-problem dispatch exactly as in the reference.
# --------------------------------------------------------------------------


class DescriptorError(RuntimeError):
    pass


@dataclass
class CacheLevel:
    line_bytes: int = 0
    associativity: int = 0
    num_sets: int = 0
    shared: bool = False

    def size_bytes(self) -> int:
        return self.line_bytes * self.associativity * self.num_sets


@dataclass
class MachineDescriptor:
    levels: list = field(default_factory=list)
    cores: int = 1
    element_bytes: int = 8

    def capacity_elements(self, i: int) -> int:
        if self.element_bytes < 1:
            raise DescriptorError("element_bytes must be >= 1")
        return self.levels[i].size_bytes() // self.element_bytes


def validate_machine(md: MachineDescriptor) -> None:
    """Rules of reference machine.hpp:55-74."""
    if md.element_bytes < 1:
        raise DescriptorError("element_bytes must be >= 1")
    if md.cores < 1:
        raise DescriptorError("cores must be >= 1")
    if len(md.levels) < 2:
        raise DescriptorError("at least two cache levels are required")
    for lv in md.levels:
        if lv.line_bytes < 1 or lv.associativity < 1 or lv.num_sets < 1:
            raise DescriptorError("line_bytes, associativity and num_sets must all be >= 1")
        if lv.line_bytes & (lv.line_bytes - 1):
            raise DescriptorError("line size must be a power of two")
    for prev, cur in zip(md.levels, md.levels[1:]):
        if cur.line_bytes != md.levels[0].line_bytes:
            raise DescriptorError("line size differs across levels")
        if cur.size_bytes() <= prev.size_bytes():
            raise DescriptorError("level sizes must increase")
    if md.levels[0].shared:
        raise DescriptorError("level 1 must be private (shared = false)")


def default_machine(cores: int = 8) -> MachineDescriptor:
    """32 KiB private L1 + 512 KiB shared L2, 64 B lines (reference machine.hpp:78-88)."""
    md = MachineDescriptor(levels=[CacheLevel(64, 8, 64, False), CacheLevel(64, 8, 1024, True)],
                           cores=cores, element_bytes=8)
    validate_machine(md)
    return md


@dataclass(frozen=True)
class BlockingPlan:
    m_c: int = 0
    n_c: int = 0
    m_r: int = 0
    dot_block: int = 0
    dot_cutoff: int = 0
    max_threads: int = 1


def derive_blocking_plan(md: MachineDescriptor, m_r_hint: int | None = None) -> BlockingPlan:
    """Reference machine.hpp:116-136: m_c = n_c = floor(sqrt(M_L2)) rounded down
    to m_r, dot_block = M_L1 / 2, dot_cutoff = 2 M_L1."""
    validate_machine(md)
    m_r = 8 if m_r_hint is None else m_r_hint
    if m_r < 1:
        raise DescriptorError("m_r must be >= 1")
    side = math.isqrt(md.capacity_elements(1))
    if side < m_r:
        raise DescriptorError("L2 capacity too small: floor(sqrt(M_L2)) < m_r")
    cap_l1 = md.capacity_elements(0)
    return BlockingPlan(m_c=side - side % m_r, n_c=side - side % m_r, m_r=m_r,
                        dot_block=cap_l1 // 2, dot_cutoff=2 * cap_l1, max_threads=md.cores)


class ExecPolicy:
    """Reference kernels.hpp:28-36."""

    def __init__(self, plan: BlockingPlan, threads: int):
        if threads < 1 or threads > plan.max_threads:
            raise ValueError("ExecPolicy: threads must be in [1, plan.max_threads]")
        self.plan = plan
        self.threads = threads


def default_policy(threads: int = 1) -> ExecPolicy:
    return ExecPolicy(derive_blocking_plan(default_machine()), threads)


# --------------------------------------------------------------------------
# Execution-path probe (reference kernels.hpp:38-55), thread-local
# --------------------------------------------------------------------------


class KernelVariant(enum.IntEnum):
    none = 0
    dot_small = 1
    dot_blocked = 2
    gemv_col_blocked = 3
    gemv_row = 4
    ger = 5


@dataclass
class ExecProbe:
    variant: KernelVariant = KernelVariant.none
    threads_used: int = 0


_tls = threading.local()


def last_exec() -> ExecProbe:
    return getattr(_tls, "probe", ExecProbe())


def _record(p: Probe) -> None:
    _tls.probe = ExecProbe(KernelVariant(p.variant), int(p.threads_used))


def _require(ok: bool, msg: str) -> None:
    if not ok:
        raise ValueError(msg)


# --------------------------------------------------------------------------
# operand plumbing
# --------------------------------------------------------------------------


def _as_tensor(a) -> torch.Tensor:
    if isinstance(a, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(a))
    return a


def _suffix(t: torch.Tensor) -> str:
    if t.dtype == torch.float32:
        return "f32"
    if t.dtype == torch.float64:
        return "f64"
    raise ValueError(f"cabl: unsupported dtype {t.dtype} (float32 / float64)")


def _ptr(t: torch.Tensor):
    return t.data_ptr() if t.numel() else None


def _on_device(dev: torch.device):
    """The C ABI launches on the current CUDA device: make it the operands'."""
    if dev.index is None or dev.index == torch.cuda.current_device():
        return contextlib.nullcontext()
    return torch.cuda.device(dev)


def _stream_of(t: torch.Tensor):
    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _check_same(ts, what: str) -> tuple[str, bool]:
    dev = {t.device.type for t in ts}
    if len(dev) != 1:
        raise ValueError(f"{what}: operands must all be on the host or all on the GPU")
    if len({t.device for t in ts}) != 1:
        raise ValueError(f"{what}: CUDA operands must be on one device")
    dts = {t.dtype for t in ts}
    if len(dts) != 1:
        raise ValueError(f"{what}: operands must share one dtype")
    for t in ts:
        if not t.is_contiguous():
            raise ValueError(f"{what}: operands must be contiguous")
    return _suffix(ts[0]), ts[0].is_cuda


# --------------------------------------------------------------------------
# DOT (reference kernels.hpp:134-164)
# --------------------------------------------------------------------------


def dot_into(x: torch.Tensor, y: torch.Tensor, alpha0: float, out: torch.Tensor,
             policy: ExecPolicy) -> None:
    """Device-resident DOT: out[0] = alpha0 + x.y, enqueued on the current stream."""
    _require(x.numel() == y.numel(), "dot: x and y lengths differ")
    sfx, cuda = _check_same([x, y, out], "dot")
    _require(cuda, "dot_into: operands must be CUDA tensors")
    p = Probe()
    with _on_device(x.device):
        _lib.call(f"cabl_cuda_dot_{sfx}", _ptr(x), _ptr(y), x.numel(), float(alpha0),
                  out.data_ptr(), policy.plan.dot_cutoff, C.byref(p), _stream_of(x))
    _record(p)


def dot(x, y, alpha0: float, policy: ExecPolicy):
    x, y = _as_tensor(x), _as_tensor(y)
    _require(x.numel() == y.numel(), "dot: x and y lengths differ")
    sfx, cuda = _check_same([x, y], "dot")
    if cuda:
        out = torch.empty(1, dtype=x.dtype, device=x.device)
        dot_into(x, y, alpha0, out, policy)
        return out.item()
    res = (C.c_float if sfx == "f32" else C.c_double)()
    p = Probe()
    _lib.call(f"cabl_host_dot_{sfx}", _ptr(x), _ptr(y), x.numel(), float(alpha0), C.byref(res),
              policy.plan.dot_cutoff, C.byref(p), None)
    _record(p)
    return res.value


# --------------------------------------------------------------------------
# GEMV (reference kernels.hpp:187-257)
# --------------------------------------------------------------------------


def _gemv(A: DenseMatrix, x, c, policy: ExecPolicy, layout: Layout, who: str) -> None:
    _require(A.layout() == layout, f"{who}: matrix is not {'col' if layout else 'row'}-major")
    x, c = _as_tensor(x), _as_tensor(c)
    _require(A.cols() == x.numel(), "gemv: A.cols != x.len")
    _require(A.rows() == c.numel(), "gemv: A.rows != c.len")
    _require(not (c.numel() and x.numel() and c.data_ptr() == x.data_ptr()),
             "gemv: c must not alias x")
    sfx, cuda = _check_same([A.data, x, c], "gemv")
    p = Probe()
    m, n = A.rows(), A.cols()
    if cuda:
        tag = "rm" if layout == Layout.RowMajor else "cm"
        with _on_device(c.device):
            _lib.call(f"cabl_cuda_gemv_{tag}_{sfx}", _ptr(A.data), m, n, _ptr(x), _ptr(c),
                      policy.plan.dot_cutoff, C.byref(p), _stream_of(c))
    else:
        _lib.call(f"cabl_host_gemv_{sfx}", _ptr(A.data), int(layout), m, n, _ptr(x), _ptr(c),
                  policy.plan.dot_cutoff, C.byref(p), None)
    _record(p)


def gemv_col_major(A: DenseMatrix, x, c, policy: ExecPolicy) -> None:
    _gemv(A, x, c, policy, Layout.ColMajor, "gemv_col_major")


def gemv_row_major(A: DenseMatrix, x, c, policy: ExecPolicy) -> None:
    _gemv(A, x, c, policy, Layout.RowMajor, "gemv_row_major")


# --------------------------------------------------------------------------
# GER (reference kernels.hpp:277-313)
# --------------------------------------------------------------------------


def ger(x, y, C_: DenseMatrix, policy: ExecPolicy) -> None:
    x, y = _as_tensor(x), _as_tensor(y)
    _require(C_.rows() == x.numel(), "ger: C.rows != x.len")
    _require(C_.cols() == y.numel(), "ger: C.cols != y.len")
    if C_.size():
        _require(not ((x.numel() and C_.data.data_ptr() == x.data_ptr())
                      or (y.numel() and C_.data.data_ptr() == y.data_ptr())),
                 "ger: C must not alias x or y")
    sfx, cuda = _check_same([x, y, C_.data], "ger")
    p = Probe()
    m, n = C_.rows(), C_.cols()
    if cuda:
        tag = "rm" if C_.layout() == Layout.RowMajor else "cm"
        with _on_device(C_.data.device):
            _lib.call(f"cabl_cuda_ger_{tag}_{sfx}", _ptr(x), _ptr(y), _ptr(C_.data), m, n,
                      policy.plan.dot_cutoff, C.byref(p), _stream_of(C_.data))
    else:
        _lib.call(f"cabl_host_ger_{sfx}", _ptr(x), _ptr(y), _ptr(C_.data), int(C_.layout()),
                  m, n, policy.plan.dot_cutoff, C.byref(p), None)
    _record(p)


# --------------------------------------------------------------------------
# seeded inputs on the device (bit-identical to oracle/cabl_oracle.c)
# --------------------------------------------------------------------------


def fill_uniform(t: torch.Tensor, seed: int, stream_id: int, offset: int = 0) -> torch.Tensor:
    sfx = _suffix(t)
    _require(t.is_cuda and t.is_contiguous(), "fill_uniform: needs a contiguous CUDA tensor")
    with _on_device(t.device):
        _lib.call(f"cabl_cuda_fill_uniform_{sfx}", _ptr(t), t.numel(), seed, stream_id, offset,
                  _stream_of(t))
    return t


def fill_normal(t: torch.Tensor, seed: int, stream_id: int, offset: int = 0) -> torch.Tensor:
    _require(t.dtype == torch.float64, "fill_normal: float64 only")
    _require(t.is_cuda and t.is_contiguous(), "fill_normal: needs a contiguous CUDA tensor")
    with _on_device(t.device):
        _lib.call("cabl_cuda_fill_normal_f64", _ptr(t), t.numel(), seed, stream_id, offset,
                  _stream_of(t))
    return t


def device_count() -> int:
    return _lib.lib().cabl_device_count()
