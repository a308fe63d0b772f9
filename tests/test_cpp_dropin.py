"""The C++ drop-in (include/cabl/*.hpp over libcabl_cuda.so).

CPU: the header compiles against the reference-shaped test program and the
device-container example, and the binaries link.  GPU: the re-hosted
reference test obligations (tests/cpp/dropin_tests.cpp: test_kernels.cpp's
hot-path cases + acceptance criteria 1, 7, 9) and the device example pass.
"""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

CPP = Path(__file__).resolve().parent / "cpp"
LIB = Path(__file__).resolve().parents[1] / "paper_2108_02025_b200" / "libcabl_cuda.so"


def _build():
    if not LIB.exists():
        pytest.fail("libcabl_cuda.so is not built (make -C paper_2108_02025_b200/csrc)")
    r = subprocess.run(["make", "-s", "-C", str(CPP)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_dropin_header_compiles_and_links():
    _build()
    assert (CPP / "dropin_tests").exists() and (CPP / "device_example").exists()
    assert (CPP / "mgpu_example").exists()


def test_dropin_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    _build()
    r = subprocess.run([str(CPP / "dropin_tests")], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0
    assert "no CUDA device available" in r.stdout


@pytest.mark.gpu
def test_rehosted_reference_tests_pass_on_gpu(cuda):
    _build()
    r = subprocess.run([str(CPP / "dropin_tests")], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all groups passed" in r.stdout


@pytest.mark.gpu
def test_device_container_example(cuda):
    _build()
    r = subprocess.run([str(CPP / "device_example")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_multi_gpu_nccl_example(cuda):
    """include/cabl/nccl.hpp: one process, an NCCL clique over every visible
    device; sharded DOT / GEMV / GER bitwise equal to the shard-by-shard runs."""
    _build()
    r = subprocess.run([str(CPP / "mgpu_example")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "MISMATCH" not in r.stdout


def _cmake_consumer(tmp_path):
    """a reference-shaped consumer switched to the drop-in
    by CMake target alone (tests/cpp/cmake_consumer)."""
    import shutil
    if shutil.which("cmake") is None:
        pytest.skip("cmake not available")
    if not LIB.exists():
        pytest.fail("libcabl_cuda.so is not built")
    build = tmp_path / "build"
    gen = ["-G", "Ninja"] if shutil.which("ninja") else []
    r = subprocess.run(["cmake", "-S", str(CPP / "cmake_consumer"), "-B", str(build), *gen],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    r = subprocess.run(["cmake", "--build", str(build)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    return build / "consumer"


def test_cmake_consumer_builds(tmp_path):
    import torch
    exe = _cmake_consumer(tmp_path)
    assert exe.exists()
    if not torch.cuda.is_available():
        r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
        assert r.returncode == 3 and "no CUDA device available" in r.stdout


@pytest.mark.gpu
def test_cmake_consumer_runs(cuda, tmp_path):
    exe = _cmake_consumer(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
