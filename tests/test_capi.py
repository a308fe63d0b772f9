"""The C-ABI library without a GPU: it loads, exports exactly what
include/cabl_cuda.h declares, and fails loudly (CABL_ECUDA + message) instead
of computing anything on the CPU.  Plus the Python mirror's host-side
validation, which must match the reference's messages (kernels.hpp)."""
from __future__ import annotations

import ctypes as C
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "cabl_cuda.h"


def declared_symbols() -> set[str]:
    text = HEADER.read_text()
    return set(re.findall(r"CABL_API\s+[\w\s\*]+?\b(cabl_\w+)\s*\(", text))


def test_library_builds_for_sm100a():
    from paper_2108_02025_b200 import _lib
    _lib.build()
    assert _lib.LIB_PATH.exists()
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_every_declared_symbol_is_exported():
    from paper_2108_02025_b200 import _lib
    declared = declared_symbols()
    assert len(declared) >= 24
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                        text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in nm.splitlines() if " T " in ln}
    assert declared <= exported, declared - exported
    # and nothing else leaks (hidden visibility for internals)
    assert {s for s in exported if s.startswith("cabl_")} == declared
    assert declared == set(_lib.SIGNATURES)
    L = _lib.lib()
    for name in declared:
        assert getattr(L, name) is not None


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_gpu_means_loud_failure_not_fallback():
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200 import _lib
    L = _lib.lib()
    assert L.cabl_device_count() == 0
    x = np.ones(4, np.float32)
    out = np.zeros(1, np.float32)
    rc = L.cabl_cuda_dot_f32(x.ctypes.data, x.ctypes.data, 4, C.c_float(0.0), out.ctypes.data,
                             8192, None, None)
    assert rc == _lib.CABL_ECUDA
    assert "no CUDA device" in L.cabl_last_error().decode()
    assert out[0] == 0.0  # nothing was computed
    with pytest.raises(_lib.CablError, match="no CPU fallback"):
        cb.dot(torch.ones(3, dtype=torch.float64), torch.ones(3, dtype=torch.float64), 0.0,
               cb.default_policy(1))
    A = cb.DenseMatrix(4, 4, cb.Layout.RowMajor, 1.0)
    with pytest.raises(_lib.CablError):
        cb.gemv_row_major(A, torch.ones(4, dtype=torch.float64),
                          torch.zeros(4, dtype=torch.float64), cb.default_policy(1))


def test_abi_version():
    from paper_2108_02025_b200 import _lib
    assert _lib.lib().cabl_abi_version() >= 100


# ---------------------------------------------------- host-side validation
def test_plan_derivation_matches_reference_defaults():
    import paper_2108_02025_b200 as cb
    plan = cb.derive_blocking_plan(cb.default_machine())
    # reference README: m_c = n_c = 256, m_r = 8, dot_block = 2048, dot_cutoff = 8192
    assert (plan.m_c, plan.n_c, plan.m_r, plan.dot_block, plan.dot_cutoff) == (256, 256, 8, 2048, 8192)
    md = cb.default_machine()
    md.element_bytes = 4
    p32 = cb.derive_blocking_plan(md)
    assert (p32.dot_block, p32.dot_cutoff) == (4096, 16384)
    with pytest.raises(ValueError, match=r"ExecPolicy: threads must be in \[1, plan.max_threads\]"):
        cb.ExecPolicy(plan, 0)
    with pytest.raises(ValueError):
        cb.ExecPolicy(plan, plan.max_threads + 1)
    bad = cb.MachineDescriptor(levels=[cb.CacheLevel(64, 8, 64, True), cb.CacheLevel(64, 8, 1024)])
    with pytest.raises(cb.DescriptorError, match="level 1 must be private"):
        cb.validate_machine(bad)


def test_reference_precondition_messages():
    import paper_2108_02025_b200 as cb
    pol = cb.default_policy(1)
    f = lambda *v: torch.tensor(v, dtype=torch.float64)  # noqa: E731
    with pytest.raises(ValueError, match="dot: x and y lengths differ"):
        cb.dot(f(1, 2), f(1), 0.0, pol)
    A = cb.DenseMatrix(2, 3, cb.Layout.RowMajor, 1.0)
    with pytest.raises(ValueError, match="gemv_col_major: matrix is not col-major"):
        cb.gemv_col_major(A, f(1, 1, 1), f(0, 0), pol)
    with pytest.raises(ValueError, match="gemv: A.cols != x.len"):
        cb.gemv_row_major(A, f(1, 1), f(0, 0), pol)
    with pytest.raises(ValueError, match="gemv: A.rows != c.len"):
        cb.gemv_row_major(A, f(1, 1, 1), f(0, 0, 0), pol)
    sq = cb.DenseMatrix(3, 3, cb.Layout.ColMajor, 1.0)
    x = f(1, 2, 3)
    with pytest.raises(ValueError, match="gemv: c must not alias x"):
        cb.gemv_col_major(sq, x, x, pol)
    C2 = cb.DenseMatrix(2, 2, cb.Layout.ColMajor)
    with pytest.raises(ValueError, match="ger: C.cols != y.len"):
        cb.ger(f(1, 2), f(3), C2, pol)
    with pytest.raises(ValueError, match="ger: C.rows != x.len"):
        cb.ger(f(1, 2, 3), f(3, 4), C2, pol)


def test_dense_matrix_indexing_matches_reference_layout():
    import paper_2108_02025_b200 as cb
    rm = cb.DenseMatrix(2, 3, cb.Layout.RowMajor)
    cm = cb.DenseMatrix(2, 3, cb.Layout.ColMajor)
    assert rm.index(1, 2) == 2 + 1 * 3   # j + i*cols
    assert cm.index(1, 2) == 1 + 2 * 2   # i + j*rows


def test_product_never_touches_the_oracle():
    """The oracle is test infrastructure: the package sources never import it
    and the shipped library links none of its objects."""
    import re
    import subprocess
    pkg = ROOT / "paper_2108_02025_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        text = f.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle\b", text, re.M), f
        assert not re.search(r"#\s*include\s*[<\"][^>\"]*oracle", text), f
        assert "libcabl_oracle" not in text and "libcabl_ref" not in text, f
    needed = subprocess.run(["readelf", "-d", str(pkg / "libcabl_cuda.so")],
                            capture_output=True, text=True).stdout
    assert "oracle" not in needed and "cabl_ref" not in needed
    syms = subprocess.run(["nm", "-D", "--defined-only", str(pkg / "libcabl_cuda.so")],
                          capture_output=True, text=True).stdout
    assert "dot_ref" not in syms and "gemv_ref" not in syms and "ger_ref" not in syms


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_peer_entry_points_without_a_gpu():
    """The peer-memory entry points validate their arguments the reference way
    (EINVAL + message) and otherwise fail loudly without a device (ECUDA)."""
    from paper_2108_02025_b200 import _lib
    L = _lib.lib()
    p = C.c_void_p()
    assert L.cabl_peer_mailbox_create(C.byref(p)) == _lib.CABL_ECUDA
    assert L.cabl_peer_alloc(1024, C.byref(p)) == _lib.CABL_ECUDA
    x = np.ones(16, np.float32)
    fake = (C.c_void_p * 2)(x.ctypes.data, x.ctypes.data)
    rc = L.cabl_cuda_dot_peer_f32(x.ctypes.data, x.ctypes.data, 16, C.c_float(0), x.ctypes.data,
                                  fake, 9, 0, 8192, None, None)
    assert rc == _lib.CABL_EINVAL and "world" in L.cabl_last_error().decode()
    rc = L.cabl_cuda_dot_peer_f32(x.ctypes.data, x.ctypes.data, 16, C.c_float(0), x.ctypes.data,
                                  fake, 2, 0, 8192, None, None)
    assert rc == _lib.CABL_ECUDA
    rc = L.cabl_cuda_gemv_rm_gather_f32(x.ctypes.data, 4, 4, x.ctypes.data, x.ctypes.data, 0, 4,
                                        fake, fake, 2, 0, None, None)
    assert rc == _lib.CABL_ECUDA
    rc = L.cabl_cuda_combine_rows_peer_f32(x.ctypes.data, 4, x.ctypes.data, fake, fake, 2, 5, None)
    assert rc == _lib.CABL_EINVAL and "rank" in L.cabl_last_error().decode()
    rc = L.cabl_cuda_combine_rows_peer_f32(x.ctypes.data, 4, x.ctypes.data, fake, fake, 2, 1, None)
    assert rc == _lib.CABL_ECUDA
    assert x[0] == 1.0  # nothing was written


def test_mgpu_entry_points_without_a_gpu():
    """The multi-GPU C ABI: NCCL is found and loaded at run time; arguments
    are validated the reference way (EINVAL + message); without a device the
    context cannot be created (ECUDA), and no call proceeds without one."""
    from paper_2108_02025_b200 import _lib
    L = _lib.lib()
    v = C.c_int()
    assert L.cabl_mgpu_nccl_version(C.byref(v)) == _lib.CABL_OK
    assert v.value >= 21800  # 2.18+; this image ships 2.27 (system) / 2.28 (torch)
    ctx = C.c_void_p()
    assert L.cabl_mgpu_init(None, 0, C.byref(ctx)) == _lib.CABL_EINVAL
    devs = (C.c_int * 2)(0, 0)
    assert L.cabl_mgpu_init(devs, 2, C.byref(ctx)) == _lib.CABL_EINVAL
    assert "twice" in L.cabl_last_error().decode()
    if not torch.cuda.is_available():
        devs = (C.c_int * 1)(0)
        assert L.cabl_mgpu_init(devs, 1, C.byref(ctx)) == _lib.CABL_ECUDA
        assert ctx.value is None
    out = C.c_float()
    n = (C.c_uint64 * 1)(4)
    assert L.cabl_mgpu_dot_f32(None, None, None, n, C.c_float(0), 8192, 0,
                               C.byref(out)) == _lib.CABL_EINVAL
    assert "null context" in L.cabl_last_error().decode()
    assert L.cabl_mgpu_ger_rm_f32(None, None, n, None, 4, None, 8192) == _lib.CABL_EINVAL
    assert L.cabl_mgpu_finalize(None) == _lib.CABL_OK
    assert L.cabl_mgpu_size(None) == 0 and L.cabl_mgpu_stream(None, 0) is None


def test_mgpu_reports_a_missing_nccl():
    """CABL_NCCL_LIB pointing nowhere: CABL_ENCCL with the loader's message,
    never a crash (the single-GPU entry points do not need NCCL at all)."""
    code = ("import ctypes as C; from paper_2108_02025_b200 import _lib; L = _lib.lib(); "
            "v = C.c_int(); rc = L.cabl_mgpu_nccl_version(C.byref(v)); "
            "print(rc, L.cabl_last_error().decode())")
    import os
    env = dict(os.environ, CABL_NCCL_LIB="/nonexistent/libnccl.so.2")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr
    rc, msg = r.stdout.split(" ", 1)
    assert int(rc) == 4 and "cannot load NCCL" in msg
