"""Multi-GPU partitioning of the hot path — one process per GPU, torch.distributed.

The reference parallelises over CPU threads with contiguous chunks
(reference thread_pool.hpp:153-164) and combines DOT partials in chunk order
(kernels.hpp:160-163).  Lifted to GPUs:

* DOT — rank g owns the contiguous chunk [g n/G, (g+1) n/G) of x and y and
  computes a partial with the single-GPU kernel (alpha0 = 0).  The only
  exchange is one all-gather of the G partials (4 or 8 bytes each) over
  NCCL; every rank then sums them IN RANK ORDER on the device and adds
  alpha0 last (``cabl_cuda_combine_partials_*``), so the result does not
  depend on NCCL's reduction algorithm: bitwise reproducible, and identical
  on every rank.  ``sharded_dot_fused`` gives the same bits from ONE kernel
  per rank: the partials are exchanged over peer memory (NVLink P2P stores
  into every rank's mailbox, csrc/peer.cu) inside the DOT kernel, with no
  NCCL call and no combine launch.
* GEMV (row-major or col-major tall) — rank g owns a block of rows of A and
  of c, x is replicated; no exchange is needed.  ``gather=True`` assembles
  the full c on every rank with one all-gather (slices padded to equal size).
* GER — rank g owns a block of rows of C and of x, y is replicated; no
  communication at all.
* GEMV col-major by columns (short-wide, e.g. G3) — rank g owns a block of
  columns; partial c vectors are all-gathered and added in rank order.
* ``sharded_gemv_cols_fused`` — the column-sharded GEMV with its combine as one
  peer-memory kernel (partials pushed into every rank's slots, rank-ordered
  sum), no collective call.
* ``GatherGemv`` — row-block GEMV whose c all-gather runs inside the GEMV
  kernel: every finished row is stored into every rank's (double-buffered)
  gathered c over peer memory (csrc/peer_gemv.cu), no NCCL call.

The collective and the local compute are injectable so the partition and
combine logic can be exercised by CPU ``gloo`` tests (tests/test_shard_gloo.py)
without a GPU; the defaults are the CUDA kernels and nothing else.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable

import torch
import torch.distributed as dist

from . import cabl


def partition(total: int, parts: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split: the first total % parts ranks get one extra."""
    q, r = divmod(total, parts)
    b = rank * q + min(rank, r)
    return b, b + q + (1 if rank < r else 0)


def _device_partial(x, y, out, policy):
    cabl.dot_into(x, y, 0.0, out, policy)


def _device_combine(partials: torch.Tensor, alpha0: float, out: torch.Tensor) -> None:
    from . import _lib
    sfx = cabl._suffix(partials)
    with cabl._on_device(partials.device):
        _lib.call(f"cabl_cuda_combine_partials_{sfx}", partials.data_ptr(), partials.numel(),
                  float(alpha0), out.data_ptr(), cabl._stream_of(partials))


def sharded_dot(x_local: torch.Tensor, y_local: torch.Tensor, alpha0: float, out: torch.Tensor,
                policy: "cabl.ExecPolicy", group=None, *,
                partial_fn: Callable = _device_partial,
                combine_fn: Callable = _device_combine,
                gathered: torch.Tensor | None = None) -> torch.Tensor:
    """out[0] = alpha0 + sum over ranks (in rank order) of this rank's partial."""
    world = dist.get_world_size(group)
    part = torch.empty(1, dtype=x_local.dtype, device=x_local.device)
    partial_fn(x_local, y_local, part, policy)
    if gathered is None:
        gathered = torch.empty(world, dtype=x_local.dtype, device=x_local.device)
    dist.all_gather_into_tensor(gathered, part, group=group)
    combine_fn(gathered, alpha0, out)
    return out


# --------------------------------------------------------------------------
# DOT whose bits do not depend on the GPU count ("optional
# G-invariant result: fixed-size global segments with per-segment partials
# gathered and summed in index order" — the reference's own block decomposition,
# kernels.hpp:145-163, with the block a fixed number of elements instead of a
# share of n / threads)

INVARIANT_SEGMENT = 1 << 26  # elements per global segment (256 MiB of fp32 per vector)


def invariant_segments(n_total: int, segment: int, world: int, rank: int) -> tuple[int, int]:
    """The global segments [kb, ke) rank owns: whole segments, balanced, in rank order."""
    return partition(-(-n_total // segment), world, rank)


def invariant_range(n_total: int, segment: int, world: int, rank: int) -> tuple[int, int]:
    """The element range of x and y rank must hold for sharded_dot_invariant."""
    kb, ke = invariant_segments(n_total, segment, world, rank)
    return min(kb * segment, n_total), min(ke * segment, n_total)


def invariant_partials(x_local: torch.Tensor, y_local: torch.Tensor, segment: int,
                       policy: "cabl.ExecPolicy", *, width: int | None = None,
                       partial_fn: Callable = _device_partial) -> torch.Tensor:
    """One partial per global segment of this rank's range, each from its own launch of
    the single-GPU kernel (alpha0 = 0): a segment's partial is a function of its data
    and length only, whoever computes it.  Returns `width` values (>= the segment
    count; the rest zero)."""
    n = x_local.numel()
    count = -(-n // segment)
    out = torch.zeros(max(count, width or 0, 1), dtype=x_local.dtype, device=x_local.device)
    for k in range(count):
        lo, hi = k * segment, min((k + 1) * segment, n)
        partial_fn(x_local[lo:hi], y_local[lo:hi], out[k:k + 1], policy)
    return out


def sharded_dot_invariant(x_local: torch.Tensor, y_local: torch.Tensor, alpha0: float,
                          out: torch.Tensor, policy: "cabl.ExecPolicy", *, n_total: int,
                          segment: int = INVARIANT_SEGMENT, group=None,
                          partial_fn: Callable = _device_partial,
                          combine_fn: Callable = _device_combine) -> torch.Tensor:
    """out[0] = alpha0 + the global segments' partials summed in index order: the same
    bits on every rank AND for every GPU count (1 GPU included), as long as the
    vectors' base addresses share their 32-byte alignment class.  Rank r holds
    elements invariant_range(n_total, segment, world, r) of x and y.  One all-gather
    of ceil(K / world) values per rank; with the default 2^26-element segments D2 is
    64 launches in all (8 per GPU at N = 8)."""
    grouped = dist.is_available() and dist.is_initialized()
    world = dist.get_world_size(group) if grouped else 1
    rank = dist.get_rank(group) if grouped else 0
    # cut points must not move a segment's alignment class relative to its shard's
    # base (the kernel's vector path depends on it): whole 64-element units
    cabl._require(segment > 0 and segment % 64 == 0,
                  "sharded_dot_invariant: segment must be a positive multiple of 64 elements")
    b, e = invariant_range(n_total, segment, world, rank)
    cabl._require(x_local.numel() == e - b and y_local.numel() == e - b,
                  f"sharded_dot_invariant: rank {rank} must hold elements [{b}, {e}) of x and y")
    counts = [(lambda kk: kk[1] - kk[0])(invariant_segments(n_total, segment, world, r))
              for r in range(world)]
    width = max(1, max(counts))
    mine = invariant_partials(x_local, y_local, segment, policy, width=width,
                              partial_fn=partial_fn)
    if world == 1:
        ordered = mine[:counts[0]]
    else:
        slab = torch.empty(world * width, dtype=mine.dtype, device=mine.device)
        dist.all_gather_into_tensor(slab, mine[:width].contiguous(), group=group)
        ordered = slab if all(c == width for c in counts) else torch.cat(
            [slab[r * width: r * width + counts[r]] for r in range(world)])
    combine_fn(ordered, alpha0, out)
    return out


def sharded_gemv_rows(A_local: "cabl.DenseMatrix", x: torch.Tensor, c_local: torch.Tensor,
                      policy: "cabl.ExecPolicy", *, gather: bool = False, m_total: int = 0,
                      group=None, local_fn: Callable | None = None,
                      out: torch.Tensor | None = None) -> torch.Tensor | None:
    """c_local += A_local x on this rank's row block; optionally all-gather c
    (into ``out``, m_total values, when given: no allocation per call).  Equal
    slices (m_total % world == 0, e.g. G4 over 2/4/8 GPUs) are gathered straight
    from c_local into the result, one collective and nothing else; ragged ones are
    padded to the widest slice and cut again."""
    if local_fn is None:
        local_fn = (cabl.gemv_row_major if A_local.layout() == cabl.Layout.RowMajor
                    else cabl.gemv_col_major)
    local_fn(A_local, x, c_local, policy)
    if not gather:
        return None
    world = dist.get_world_size(group)
    if out is not None:
        cabl._require(out.numel() == m_total and out.dtype == c_local.dtype
                      and out.device == c_local.device and out.is_contiguous(),
                      "sharded_gemv_rows: out must hold m_total values of c's dtype on c's device")
    if m_total % world == 0 and c_local.numel() * world == m_total and c_local.is_contiguous():
        full = out if out is not None else torch.empty(m_total, dtype=c_local.dtype,
                                                       device=c_local.device)
        dist.all_gather_into_tensor(full, c_local, group=group)
        return full
    widest = partition(m_total, world, 0)
    width = widest[1] - widest[0]
    padded = torch.zeros(width, dtype=c_local.dtype, device=c_local.device)
    padded[:c_local.numel()] = c_local
    slab = torch.empty(world * width, dtype=c_local.dtype, device=c_local.device)
    dist.all_gather_into_tensor(slab, padded, group=group)
    pieces = []
    for r in range(world):
        b, e = partition(m_total, world, r)
        pieces.append(slab[r * width: r * width + (e - b)])
    return torch.cat(pieces, out=out) if out is not None else torch.cat(pieces)


def _device_combine_rows(parts: torch.Tensor, world: int, c: torch.Tensor) -> None:
    from . import _lib
    sfx = cabl._suffix(parts)
    with cabl._on_device(parts.device):
        _lib.call(f"cabl_cuda_combine_rows_{sfx}", parts.data_ptr(), world, c.numel(),
                  c.data_ptr(), cabl._stream_of(parts))


def sharded_gemv_cols(A_local: "cabl.DenseMatrix", x_local: torch.Tensor, c: torch.Tensor,
                      policy: "cabl.ExecPolicy", group=None, *,
                      local_fn: Callable | None = None,
                      combine_fn: Callable = _device_combine_rows) -> torch.Tensor:
    """Column-sharded col-major GEMV ("G3 by columns"): rank g
    owns the contiguous column block A[:, cols_g] (col-major, so one dense
    m x |cols_g| block) and x[cols_g]; c is replicated.  Each rank computes its
    partial A[:, cols_g] x[cols_g] from zero, the G partials are all-gathered,
    and every rank adds them to c in rank order (cabl_cuda_combine_rows_*):
    c is bitwise identical on every rank, independent of the collective's
    reduction order."""
    cabl._require(A_local.layout() == cabl.Layout.ColMajor,
                  "sharded_gemv_cols: A must be col-major (its column blocks are contiguous)")
    world = dist.get_world_size(group)
    m = c.numel()
    part = torch.zeros(m, dtype=c.dtype, device=c.device)
    (local_fn or cabl.gemv_col_major)(A_local, x_local, part, policy)
    gathered = torch.empty(world * m, dtype=c.dtype, device=c.device)
    dist.all_gather_into_tensor(gathered, part, group=group)
    combine_fn(gathered, world, c)
    return c


def sharded_ger_rows(x_local: torch.Tensor, y: torch.Tensor, C_local: "cabl.DenseMatrix",
                     policy: "cabl.ExecPolicy", *, local_fn: Callable | None = None) -> None:
    """C_local += x_local (x) y on this rank's row block — no communication."""
    (local_fn or cabl.ger)(x_local, y, C_local, policy)


# --------------------------------------------------------------------------
# DOT with the exchange fused into the kernel (csrc/peer.cu)

class PeerMailboxes:
    """This rank's peer-DOT mailbox and every other rank's, mapped here.

    Each rank creates a 512-byte mailbox on its device and exports a CUDA IPC
    handle; the handles are all-gathered over the process group (any backend:
    this is setup, not data path) and every peer's is imported.  ``table`` is
    the mailbox pointer table of ``cabl_cuda_dot_peer_*`` in rank order.  At
    world size 1 nothing is exchanged.  ``create``/``export``/``import_``
    are injectable so the exchange can be tested on CPU over gloo.
    """

    def __init__(self, device: torch.device, group=None, *, create=None, export=None,
                 import_=None):
        from . import _lib
        grouped = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if grouped else 1
        self.rank = dist.get_rank(group) if grouped else 0
        self.device = device
        if self.world > 8:
            raise ValueError("peer DOT: at most 8 ranks (one NVLink domain)")
        real = create is None and import_ is None  # library-owned mappings to release on failure
        create = create or self._create
        export = export or self._export
        import_ = import_ or self._import
        with cabl._on_device(device):
            self.own = create()
            self.mapped = {}
            if self.world > 1:
                handles: list = [None] * self.world
                dist.all_gather_object(handles, export(self.own), group=group)
                err = None
                try:
                    for g, h in enumerate(handles):
                        if g != self.rank:
                            self.mapped[g] = import_(h)
                except Exception as e:  # noqa: BLE001 - reported collectively below
                    err = e
                # every rank must agree before any kernel spins on a peer
                flag = torch.tensor([0 if err else 1], dtype=torch.int32,
                                    device=device if device.type == "cuda" else "cpu")
                dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
                if int(flag.item()) == 0:
                    if real:
                        for p in self.mapped.values():  # return codes ignored: failing anyway
                            _lib.lib().cabl_peer_mailbox_unmap(C.c_void_p(p))
                        _lib.lib().cabl_peer_mailbox_destroy(C.c_void_p(self.own))
                    raise RuntimeError(f"peer mailbox exchange failed on at least one rank"
                                       f"{': ' + str(err) if err else ''}")
        ptrs = [self.own if g == self.rank else self.mapped[g] for g in range(self.world)]
        self.table = (C.c_void_p * self.world)(*ptrs)
        self._lib = _lib

    @staticmethod
    def _create() -> int:
        from . import _lib
        p = C.c_void_p()
        _lib.call("cabl_peer_mailbox_create", C.byref(p))
        return p.value

    @staticmethod
    def _export(ptr: int) -> bytes:
        from . import _lib
        buf = C.create_string_buffer(64)
        _lib.call("cabl_peer_mailbox_export", C.c_void_p(ptr), buf)
        return buf.raw

    @staticmethod
    def _import(handle: bytes) -> int:
        from . import _lib
        p = C.c_void_p()
        _lib.call("cabl_peer_mailbox_import", C.c_char_p(handle), C.byref(p))
        return p.value

    def state(self) -> tuple[int, int]:
        """(completed calls, epoch of a timed-out call or 0) of this rank's mailbox."""
        e, f = C.c_uint64(), C.c_uint64()
        with cabl._on_device(self.device):
            self._lib.call("cabl_peer_mailbox_state", C.c_void_p(self.own), C.byref(e), C.byref(f))
        return e.value, f.value

    def close(self) -> None:
        if self.own is None:
            return
        with cabl._on_device(self.device):
            for p in self.mapped.values():
                self._lib.call("cabl_peer_mailbox_unmap", C.c_void_p(p))
            self._lib.call("cabl_peer_mailbox_destroy", C.c_void_p(self.own))
        self.own, self.mapped = None, {}


def sharded_dot_fused(x_local: torch.Tensor, y_local: torch.Tensor, alpha0: float,
                      out: torch.Tensor, policy: "cabl.ExecPolicy",
                      mailboxes: PeerMailboxes) -> torch.Tensor:
    """out[0] = alpha0 + sum over ranks (rank order) of each rank's shard partial,
    in one kernel per rank (``cabl_cuda_dot_peer_*``): bitwise ``sharded_dot``'s
    result.  Collective: every rank of the mailboxes' group must call it."""
    from . import _lib
    cabl._require(x_local.numel() == y_local.numel(), "dot: x and y lengths differ")
    sfx, cuda = cabl._check_same([x_local, y_local, out], "dot")
    cabl._require(cuda, "sharded_dot_fused: operands must be CUDA tensors")
    p = cabl.Probe()
    with cabl._on_device(x_local.device):
        _lib.call(f"cabl_cuda_dot_peer_{sfx}", cabl._ptr(x_local), cabl._ptr(y_local),
                  x_local.numel(), float(alpha0), out.data_ptr(), mailboxes.table,
                  mailboxes.world, mailboxes.rank, policy.plan.dot_cutoff, C.byref(p),
                  cabl._stream_of(x_local))
    cabl._record(p)
    return out


# --------------------------------------------------------------------------
# Row-major GEMV with the c all-gather fused into the kernel (csrc/peer_gemv.cu)

class _CudaArray:
    """Zero-copy view of library-owned device memory for torch.as_tensor."""

    def __init__(self, ptr: int, n: int, dtype: torch.dtype):
        self.__cuda_array_interface__ = {
            "shape": (n,), "typestr": "<f4" if dtype == torch.float32 else "<f8",
            "data": (ptr, False), "version": 3, "strides": None}


class GatherGemv:
    """c_slice += A_slice x on every rank, with the full c assembled on every
    rank by the same kernel (``cabl_cuda_gemv_rm_gather_*``): each finished row
    is stored into every rank's gathered buffer over NVLink P2P, no NCCL call.

    Rank g owns rows ``row_off[g] .. row_off[g] + m_g`` of A and c (x
    replicated), like ``sharded_gemv_rows``.  The gathered buffer is library
    memory, double-buffered: call k returns the view of half k & 1.  With the
    ranks in separate processes that view must be consumed (or cloned), in
    stream order, before this rank issues call k + 1: a faster peer starts
    pushing call k + 2 into the same half as soon as it sees this rank's call
    k + 1 (``cabl_cuda_gemv_rm_gather_*`` in include/cabl_cuda.h).
    Collective: every rank of the group calls, in the same order.  The slice
    shape must take the sweep kernel (long aligned rows, enough of them); other
    shapes raise ValueError — use ``sharded_gemv_rows(gather=True)`` there.
    ``alloc``/``create``/``export``/``import_`` are injectable for CPU tests.
    """

    def __init__(self, device: torch.device, m_total: int, dtype: torch.dtype, group=None, *,
                 alloc=None, create=None, export=None, import_=None):
        from . import _lib
        self._lib = _lib
        self.device, self.m_total, self.dtype = device, m_total, dtype
        real = alloc is None and import_ is None
        s = torch.tensor([], dtype=dtype).element_size()
        alloc = alloc or (lambda nbytes: GatherGemv._alloc(nbytes))
        create = create or PeerMailboxes._create
        export = export or PeerMailboxes._export
        import_ = import_ or PeerMailboxes._import
        grouped = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if grouped else 1
        self.rank = dist.get_rank(group) if grouped else 0
        if self.world > 8:
            raise ValueError("gather GEMV: at most 8 ranks (one NVLink domain)")
        with cabl._on_device(device):
            self.buf = alloc(2 * m_total * s)
            self.mbox = create()
            self.mapped: dict[int, tuple[int, int]] = {}
            if self.world > 1:
                handles: list = [None] * self.world
                dist.all_gather_object(handles, (export(self.buf), export(self.mbox)), group=group)
                err = None
                try:
                    for g, (hb, hm) in enumerate(handles):
                        if g != self.rank:
                            self.mapped[g] = (import_(hb), import_(hm))
                except Exception as e:  # noqa: BLE001 - reported collectively below
                    err = e
                flag = torch.tensor([0 if err else 1], dtype=torch.int32,
                                    device=device if device.type == "cuda" else "cpu")
                dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
                if int(flag.item()) == 0:
                    if real:
                        self.close()
                    raise RuntimeError(f"gather buffer exchange failed on at least one rank"
                                       f"{': ' + str(err) if err else ''}")
        bufs = [self.buf if g == self.rank else self.mapped[g][0] for g in range(self.world)]
        mbs = [self.mbox if g == self.rank else self.mapped[g][1] for g in range(self.world)]
        self.cfull_table = (C.c_void_p * self.world)(*bufs)
        self.mbox_table = (C.c_void_p * self.world)(*mbs)
        self.calls = 0
        self._views = None
        if device.type == "cuda":
            self._views = [torch.as_tensor(_CudaArray(self.buf + h * m_total * s, m_total, dtype),
                                           device=device) for h in (0, 1)]

    @staticmethod
    def _alloc(nbytes: int) -> int:
        from . import _lib
        p = C.c_void_p()
        _lib.call("cabl_peer_alloc", nbytes, C.byref(p))
        return p.value

    def __call__(self, A_local: "cabl.DenseMatrix", x: torch.Tensor, c_local: torch.Tensor,
                 row_off: int) -> torch.Tensor:
        cabl._require(A_local.layout() == cabl.Layout.RowMajor, "gemv_row_major: A must be row-major")
        sfx, on_gpu = cabl._check_same([A_local.data, x, c_local], "gemv_row_major")
        # the peer buffers hold m_total values of self.dtype on self.device: an
        # operand of another dtype or device would write past them on every rank
        cabl._require(on_gpu and c_local.dtype == self.dtype and c_local.device == self.device,
                      f"gather GEMV: operands must be {self.dtype} on {self.device} "
                      "(the dtype and device the gathered buffers were built for)")
        m, n = A_local.rows(), A_local.cols()
        cabl._require(x.numel() == n and c_local.numel() == m, "gemv_row_major: shape mismatch")
        p = cabl.Probe()
        with cabl._on_device(self.device):
            self._lib.call(f"cabl_cuda_gemv_rm_gather_{sfx}", A_local.data.data_ptr(), m, n,
                           x.data_ptr(), c_local.data_ptr(), row_off, self.m_total,
                           self.cfull_table, self.mbox_table, self.world, self.rank, C.byref(p),
                           cabl._stream_of(c_local))
        cabl._record(p)
        self.calls += 1
        return self._views[self.calls & 1]

    def state(self) -> tuple[int, int]:
        """(completed calls, epoch of a timed-out call or 0) of this rank's mailbox."""
        e, f = C.c_uint64(), C.c_uint64()
        with cabl._on_device(self.device):
            self._lib.call("cabl_peer_mailbox_state", C.c_void_p(self.mbox), C.byref(e), C.byref(f))
        return e.value, f.value

    def close(self) -> None:
        if getattr(self, "buf", None) is None:
            return
        L = self._lib.lib()
        with cabl._on_device(self.device):
            for pb, pm in self.mapped.values():  # return codes ignored on teardown
                L.cabl_peer_mailbox_unmap(C.c_void_p(pb))
                L.cabl_peer_mailbox_unmap(C.c_void_p(pm))
            L.cabl_peer_free(C.c_void_p(self.buf))
            L.cabl_peer_mailbox_destroy(C.c_void_p(self.mbox))
        self.buf, self.mapped, self._views = None, {}, None


# --------------------------------------------------------------------------
# Column-sharded col-major GEMV with the combine over peer memory (csrc/peer.cu)

class PeerRows:
    """Slot buffer (2 x 8 x m values) and mailbox of this rank, and every
    peer's, mapped here: the tables ``cabl_cuda_combine_rows_peer_*`` takes.
    Exchange and failure agreement as in ``GatherGemv``."""

    def __init__(self, device: torch.device, m: int, dtype: torch.dtype, group=None, *,
                 alloc=None, create=None, export=None, import_=None):
        from . import _lib
        self._lib = _lib
        self.device, self.m, self.dtype = device, m, dtype
        real = alloc is None and import_ is None
        s = torch.tensor([], dtype=dtype).element_size()
        alloc = alloc or GatherGemv._alloc
        create = create or PeerMailboxes._create
        export = export or PeerMailboxes._export
        import_ = import_ or PeerMailboxes._import
        grouped = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if grouped else 1
        self.rank = dist.get_rank(group) if grouped else 0
        if self.world > 8:
            raise ValueError("peer combine: at most 8 ranks (one NVLink domain)")
        with cabl._on_device(device):
            self.buf = alloc(2 * 8 * max(m, 1) * s)
            self.mbox = create()
            self.mapped: dict[int, tuple[int, int]] = {}
            if self.world > 1:
                handles: list = [None] * self.world
                dist.all_gather_object(handles, (export(self.buf), export(self.mbox)), group=group)
                err = None
                try:
                    for g, (hb, hm) in enumerate(handles):
                        if g != self.rank:
                            self.mapped[g] = (import_(hb), import_(hm))
                except Exception as e:  # noqa: BLE001 - reported collectively below
                    err = e
                flag = torch.tensor([0 if err else 1], dtype=torch.int32,
                                    device=device if device.type == "cuda" else "cpu")
                dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
                if int(flag.item()) == 0:
                    if real:
                        self.close()
                    raise RuntimeError(f"peer slot exchange failed on at least one rank"
                                       f"{': ' + str(err) if err else ''}")
        self.slot_table = (C.c_void_p * self.world)(
            *[self.buf if g == self.rank else self.mapped[g][0] for g in range(self.world)])
        self.mbox_table = (C.c_void_p * self.world)(
            *[self.mbox if g == self.rank else self.mapped[g][1] for g in range(self.world)])

    def state(self) -> tuple[int, int]:
        e, f = C.c_uint64(), C.c_uint64()
        with cabl._on_device(self.device):
            self._lib.call("cabl_peer_mailbox_state", C.c_void_p(self.mbox), C.byref(e), C.byref(f))
        return e.value, f.value

    def close(self) -> None:
        if getattr(self, "buf", None) is None:
            return
        L = self._lib.lib()
        with cabl._on_device(self.device):
            for pb, pm in self.mapped.values():  # return codes ignored on teardown
                L.cabl_peer_mailbox_unmap(C.c_void_p(pb))
                L.cabl_peer_mailbox_unmap(C.c_void_p(pm))
            L.cabl_peer_free(C.c_void_p(self.buf))
            L.cabl_peer_mailbox_destroy(C.c_void_p(self.mbox))
        self.buf, self.mapped = None, {}


def sharded_gemv_cols_fused(A_local: "cabl.DenseMatrix", x_local: torch.Tensor, c: torch.Tensor,
                            policy: "cabl.ExecPolicy", peers: PeerRows) -> torch.Tensor:
    """``sharded_gemv_cols`` with the all-gather + rank-ordered combine replaced by
    one peer-memory kernel (``cabl_cuda_combine_rows_peer_*``): bitwise the same
    c on every rank, no collective call.  Collective over ``peers``' group."""
    from . import _lib
    cabl._require(A_local.layout() == cabl.Layout.ColMajor,
                  "sharded_gemv_cols: A must be col-major (its column blocks are contiguous)")
    m = c.numel()
    _, on_gpu = cabl._check_same([A_local.data, x_local, c], "sharded_gemv_cols")
    cabl._require(on_gpu and c.dtype == peers.dtype and c.device == peers.device,
                  f"sharded_gemv_cols_fused: operands must be {peers.dtype} on {peers.device} "
                  "(the dtype and device the peer slots were built for)")
    cabl._require(m == peers.m, "sharded_gemv_cols_fused: c length differs from the slot size")
    part = torch.zeros(m, dtype=c.dtype, device=c.device)
    cabl.gemv_col_major(A_local, x_local, part, policy)
    sfx = cabl._suffix(c)
    with cabl._on_device(c.device):
        _lib.call(f"cabl_cuda_combine_rows_peer_{sfx}", part.data_ptr(), m, c.data_ptr(),
                  peers.slot_table, peers.mbox_table, peers.world, peers.rank,
                  cabl._stream_of(c))
    return c
