"""GPU machine descriptor — SURVEY §8(f)4.

The reference derives every tuning parameter from a declared memory hierarchy
(proj/include/cabl/machine.hpp:43-136) stored as a flat JSON document
(descriptor_json.hpp:3-15: element_bytes, cores, levels L1 outward).  This
module describes a GPU in that same format, read live from the driver through
the C ABI (``cabl_describe_device``):

  cores  = streaming multiprocessors (the units a grid is sized by)
  L1     = the per-SM shared-memory capacity, private (128-byte lines, 4 ways)
  L2     = the device L2, shared (128-byte lines, 16 ways)

plus a ``gpu`` object the reference loader ignores (name, compute capability,
HBM bytes, opt-in shared memory per CTA).  The document passes the
reference's validation rules unchanged, so ``derive_blocking_plan`` works on
it, and ``derive_gpu_plan`` turns it into the launch parameters this library
uses (grid sizes, the work-queue threshold, the bench's L2 policy) instead of
hard-coded B200 numbers.  ``machines/b200.json`` is the document captured on
a B200 of this pool.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from pathlib import Path

from . import _lib
from .cabl import CacheLevel, DescriptorError, MachineDescriptor, validate_machine

LINE_BYTES = 128
L1_WAYS = 4
L2_WAYS = 16
B200_JSON = Path(__file__).resolve().parents[1] / "machines" / "b200.json"


@dataclass(frozen=True)
class GpuInfo:
    """cabl_gpu_machine as read from the driver."""
    device: int
    name: str
    cc: tuple
    sm_count: int
    max_threads_per_sm: int
    line_bytes: int
    smem_per_sm: int
    smem_per_block_optin: int
    l2_bytes: int
    hbm_bytes: int
    mem_bus_bits: int
    queue_threshold_bytes: int


def describe_device(device: int = 0) -> GpuInfo:
    """Live device facts through the C ABI (raises CablError without a GPU)."""
    g = _lib.GpuMachineC()
    _lib.check(_lib.lib().cabl_describe_device(device, C.byref(g)))
    return GpuInfo(device=g.device, name=g.name.decode(), cc=(g.cc_major, g.cc_minor),
                   sm_count=g.sm_count, max_threads_per_sm=g.max_threads_per_sm,
                   line_bytes=g.line_bytes, smem_per_sm=g.smem_per_sm,
                   smem_per_block_optin=g.smem_per_block_optin, l2_bytes=g.l2_bytes,
                   hbm_bytes=g.hbm_bytes, mem_bus_bits=g.mem_bus_bits,
                   queue_threshold_bytes=g.queue_threshold_bytes)


def _level(size: int, ways: int, shared: bool) -> CacheLevel:
    sets = size // (LINE_BYTES * ways)
    if sets < 1:
        raise DescriptorError("line_bytes, associativity and num_sets must all be >= 1")
    return CacheLevel(LINE_BYTES, ways, sets, shared)


def descriptor_of(info: GpuInfo, element_bytes: int = 4) -> dict:
    """The reference's flat descriptor document for a GPU (+ a 'gpu' object)."""
    md = MachineDescriptor(levels=[_level(info.smem_per_sm, L1_WAYS, False),
                                   _level(info.l2_bytes, L2_WAYS, True)],
                           cores=info.sm_count, element_bytes=element_bytes)
    validate_machine(md)
    return {
        "element_bytes": element_bytes,
        "cores": info.sm_count,
        "levels": [{"line_bytes": lv.line_bytes, "associativity": lv.associativity,
                    "num_sets": lv.num_sets, "shared": lv.shared} for lv in md.levels],
        "gpu": {"name": info.name, "cc": f"{info.cc[0]}.{info.cc[1]}",
                "hbm_bytes": info.hbm_bytes, "smem_per_block_optin": info.smem_per_block_optin,
                "max_threads_per_sm": info.max_threads_per_sm,
                "mem_bus_bits": info.mem_bus_bits},
    }


def load_descriptor(text: str) -> MachineDescriptor:
    """Reference descriptor_json.hpp:25-52: parse, read the three keys, validate
    (extra keys such as 'gpu' are ignored, as nlohmann's at() lookups do)."""
    try:
        d = json.loads(text)
    except json.JSONDecodeError as e:
        raise DescriptorError(f"descriptor parse failure: {e}") from None
    try:
        levels = [CacheLevel(int(lv["line_bytes"]), int(lv["associativity"]),
                             int(lv["num_sets"]), bool(lv["shared"])) for lv in d["levels"]]
        md = MachineDescriptor(levels=levels, cores=int(d["cores"]),
                               element_bytes=int(d["element_bytes"]))
    except (KeyError, TypeError, ValueError) as e:
        raise DescriptorError(f"descriptor parse failure: {e!r}") from None
    validate_machine(md)
    return md


def load_descriptor_file(path) -> MachineDescriptor:
    p = Path(path)
    if not p.exists():
        raise DescriptorError(f"cannot open descriptor file: {path}")
    return load_descriptor(p.read_text())


def gpu_machine(device: int = 0, element_bytes: int = 4) -> MachineDescriptor:
    """Live GPU descriptor as a reference MachineDescriptor."""
    return load_descriptor(json.dumps(descriptor_of(describe_device(device), element_bytes)))


def _pow2_ceil(v: int) -> int:
    t = 1
    while t < v:
        t <<= 1
    return t


@dataclass(frozen=True)
class GpuPlan:
    """Launch parameters derived from a GPU descriptor."""
    sm_count: int
    l2_bytes: int
    smem_per_sm: int
    queue_threshold_bytes: int  # operands >= this use the atomic work queues
    l2_flush_bytes: int         # bench: flush buffer (write then read) between steps
    dot_ctas: int               # DOT grid: 2 CTAs of 512 threads per SM


def derive_gpu_plan(md: MachineDescriptor) -> GpuPlan:
    """Rules (csrc/capi.cu queue_threshold_bytes, dot.cu, gemv_rm_ordered.cu,
    bench.py L2Flush):
      * queue threshold = 4 x L2 rounded up to a power of two (512 MiB on B200);
      * L2 flush = the same (> 4 x L2, so no step input survives);
      * DOT grid = 2 x SMs.
    The library applies the same rules to the live device (capi.cu reads
    the SM count and L2 size from the driver); this function makes them
    available for a descriptor document, e.g. machines/b200.json."""
    validate_machine(md)
    sms = md.cores
    l1 = md.levels[0].size_bytes()
    l2 = md.levels[-1].size_bytes()
    q = _pow2_ceil(4 * l2)
    return GpuPlan(sm_count=sms, l2_bytes=l2, smem_per_sm=l1, queue_threshold_bytes=q,
                   l2_flush_bytes=q, dot_ctas=2 * sms)
