"""B200-native DOT / GEMV / GER — the hot path of arXiv 2108.02025 (`cabl`).

The product is ``libcabl_cuda.so`` (hand-written sm_100a kernels behind the C
ABI in ``include/cabl_cuda.h``) with two host faces that mirror the reference
API: the C++ drop-in header ``include/cabl/kernels.hpp`` and this Python
module.  ``shard`` adds the multi-GPU partitioning (one process per GPU,
``torch.distributed``).
"""
from . import _lib
from .cabl import (BlockingPlan, CacheLevel, DenseMatrix, DescriptorError, ExecPolicy,
                   ExecProbe, KernelVariant, Layout, MachineDescriptor, default_machine,
                   default_policy, derive_blocking_plan, device_count, dot, dot_into,
                   fill_normal, fill_uniform, gemv_col_major, gemv_row_major, ger, last_exec,
                   layout_name, validate_machine)

__all__ = [
    "BlockingPlan", "CacheLevel", "DenseMatrix", "DescriptorError", "ExecPolicy", "ExecProbe",
    "KernelVariant", "Layout", "MachineDescriptor", "default_machine", "default_policy",
    "derive_blocking_plan", "device_count", "dot", "dot_into", "fill_normal", "fill_uniform",
    "gemv_col_major", "gemv_row_major", "ger", "last_exec", "layout_name", "validate_machine",
    "_lib",
]
