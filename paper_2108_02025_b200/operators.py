"""Resident operators: the matrix stays in HBM, each call streams the vectors.

For iterative use of GEMV (power iterations, Krylov solvers, decode-style
serving) the matrix is loaded once and every call moves only x in and c out.
``ResidentGemv`` packages that pattern behind one call and captures the whole
step — H2D of x and c, the GEMV kernel (``cabl_cuda_gemv_*`` through the C
ABI), D2H of c — into a CUDA graph, so a step is one graph launch plus one
stream synchronize instead of four API calls.

The reference has no such object (its containers live in host memory); this
is the B200 way to call the same ``gemv_row_major`` / ``gemv_col_major``
repeatedly without paying PCIe for A every time.
"""
from __future__ import annotations

import torch

from . import cabl


class ResidentGemv:
    """c_out = c_in + A x for host vectors, A resident on the device.

    ``A`` is a :class:`cabl.DenseMatrix` on a CUDA device.  ``x`` / ``c`` are
    host tensors (pinned for asynchronous copies); results land in the pinned
    buffer returned by :meth:`__call__`.
    """

    def __init__(self, A: cabl.DenseMatrix, policy: cabl.ExecPolicy, use_graph: bool = True):
        if not A.data.is_cuda:
            raise ValueError("ResidentGemv: A must be resident on a CUDA device")
        self.A, self.policy = A, policy
        dev, dt = A.data.device, A.data.dtype
        self.x_dev = torch.empty(A.cols(), dtype=dt, device=dev)
        self.c_dev = torch.empty(A.rows(), dtype=dt, device=dev)
        self.x_host = torch.empty(A.cols(), dtype=dt).pin_memory()
        self.c_host = torch.empty(A.rows(), dtype=dt).pin_memory()
        self.out_host = torch.empty(A.rows(), dtype=dt).pin_memory()
        self._fn = (cabl.gemv_row_major if A.layout() == cabl.Layout.RowMajor
                    else cabl.gemv_col_major)
        self.stream = torch.cuda.Stream(device=dev)
        self.graph = None
        if use_graph:
            self._capture()

    def _step(self):
        self.x_dev.copy_(self.x_host, non_blocking=True)
        self.c_dev.copy_(self.c_host, non_blocking=True)
        self._fn(self.A, self.x_dev, self.c_dev, self.policy)
        self.out_host.copy_(self.c_dev, non_blocking=True)

    def _capture(self):
        # warm up outside capture: the library sizes its per-stream scratch on
        # first use, and allocation must not happen inside the graph
        with torch.cuda.stream(self.stream):
            self._step()
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self._step()
        self.stream.synchronize()

    def submit(self, x: torch.Tensor | None = None, c: torch.Tensor | None = None) -> None:
        """Enqueue one step (H2D x, c -> GEMV -> D2H c) without waiting.  The
        result is valid in ``out_host`` after :meth:`wait`.  The staging
        buffers must not be rewritten until then."""
        if x is not None:
            self.x_host.copy_(x)
        if c is not None:
            self.c_host.copy_(c)
        # a graph replays on the current stream: make it ours
        with torch.cuda.stream(self.stream):
            if self.graph is not None:
                self.graph.replay()
            else:
                self._step()

    def wait(self) -> torch.Tensor:
        self.stream.synchronize()
        return self.out_host

    def __call__(self, x: torch.Tensor | None = None, c: torch.Tensor | None = None):
        """One synchronous step; ``x`` / ``c`` (host tensors) are copied into
        the pinned staging buffers when given (``None`` reuses what the caller
        already wrote into ``x_host`` / ``c_host``)."""
        self.submit(x, c)
        return self.wait()


class GemvPipeline:
    """``depth`` ResidentGemv instances over the same resident A, used round
    robin: step k's copies and kernel are enqueued while step k-1 is still in
    flight, and step k's result is read back (waited for) before its staging
    buffers are reused ``depth`` steps later — the serving pattern with
    ``depth`` requests in flight."""

    def __init__(self, A: cabl.DenseMatrix, policy: cabl.ExecPolicy, depth: int = 2):
        self.ops = [ResidentGemv(A, policy) for _ in range(depth)]
        self.k = 0
        self.pending = [False] * depth

    def step(self, x: torch.Tensor | None = None, c: torch.Tensor | None = None):
        """Submit one step; returns the finished result of the step submitted
        ``depth`` calls ago (None while the pipeline fills)."""
        i = self.k % len(self.ops)
        done = None
        if self.pending[i]:
            done = self.ops[i].wait()
        self.ops[i].submit(x, c)
        self.pending[i] = True
        self.k += 1
        return done

    def drain(self) -> list:
        out = []
        for j in range(len(self.ops)):
            i = (self.k + j) % len(self.ops)
            if self.pending[i]:
                out.append(self.ops[i].wait())
                self.pending[i] = False
        return out
