"""GPU mode of the reference bench harness / CLI (paper_2108_02025_b200.benchcli),
checked against the reference's own CLI contract (acceptance criterion 10,
reference acceptance.cpp:533-580): exit status, one CSV record per
(kernel, size, threads), CSV round trip, an SVG with one polyline per
(kernel, threads)."""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import pytest
import torch

from paper_2108_02025_b200 import benchcli as B

ROOT = Path(__file__).resolve().parents[1]


def test_parse_sizes_and_rects():
    assert B.parse_sizes("256,1024,4096") == [256, 1024, 4096]
    assert B.parse_sizes("256:1048576:4") == [256, 1024, 4096, 16384, 65536, 262144, 1048576]
    with pytest.raises(ValueError):
        B.parse_sizes("1:10")
    with pytest.raises(ValueError):
        B.parse_sizes("0:10:2")
    assert B.parse_rects("256x1048576,8x9") == [(256, 1048576), (8, 9)]


def test_csv_round_trip_and_svg():
    recs = []
    for k in B.KERNELS:
        for size in (64, 256):
            for t in (1, 2):
                recs.append(B.BenchRecord(k, 0 if k == "dot" else size, size, t, 3,
                                          1.0e-5 * size, 1.1e-5 * size, 3.14159265 * size,
                                          -0.123456789e3, "f32", 1234.5678, 0.1885))
    text = B.emit_csv(recs)
    assert text.splitlines()[0] == B.CSV_HEADER + B.CSV_GPU_SUFFIX
    back = B.parse_csv(text)
    assert len(back) == 16
    assert B.emit_csv(back) == text
    # the reference's own 9-column CSV still parses
    plain = B.CSV_HEADER + "\n" + "dot,0,64,1,3,1e-05,2e-05,3,4\n"
    assert B.parse_csv(plain)[0].kernel == "dot"
    svg = B.emit_svg(recs)
    assert svg.startswith("<?xml") and svg.rstrip().endswith("</svg>")
    assert svg.count("<polyline") == 8


def test_descriptor_loading(tmp_path):
    p = tmp_path / "m.json"
    p.write_text('{"element_bytes": 8, "cores": 16, "levels": ['
                 '{"line_bytes": 64, "associativity": 8, "num_sets": 64, "shared": false},'
                 '{"line_bytes": 64, "associativity": 8, "num_sets": 1024, "shared": true}]}')
    md = B.load_descriptor(str(p))
    assert md.cores == 16 and md.levels[1].size_bytes() == 512 * 1024


def test_bounds_columns_round_trip():
    r = B.BenchRecord("gemv-row", 8192, 8192, 1, 3, 4.1e-5, 4.2e-5, 3.2e3, 1.0, "f32", 6.4e3,
                      0.98, alg_bytes=268533760, hbm_bound_s=268533760 / 6547.8e9)
    text = B.emit_csv([r])
    assert text.splitlines()[0].endswith(B.CSV_BOUNDS_SUFFIX)
    back = B.parse_csv(text)
    assert back[0].alg_bytes == 268533760 and B.emit_csv(back) == text


def test_cli_errors_exit_2():
    r = subprocess.run([sys.executable, "-m", "paper_2108_02025_b200.benchcli", "--sizes", "0"],
                       capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 2
    if not torch.cuda.is_available():
        r = subprocess.run([sys.executable, "-m", "paper_2108_02025_b200.benchcli", "--sizes", "64",
                            "--reps", "3"], capture_output=True, text=True, cwd=ROOT, timeout=300)
        assert r.returncode == 2 and "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_cli_contract_criterion_10(cuda, tmp_path):
    csv, svg = tmp_path / "sweep.csv", tmp_path / "sweep.svg"
    r = subprocess.run([sys.executable, "-m", "paper_2108_02025_b200.benchcli", "--kernel", "all",
                        "--sizes", "64,256", "--threads", "1,2", "--reps", "3", "--seed", "7",
                        "--csv", str(csv), "--svg", str(svg)],
                       capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr
    text = csv.read_text()
    recs = B.parse_csv(text)
    assert len(recs) == 4 * 2 * 2
    assert B.emit_csv(recs) == text
    s = svg.read_text()
    assert s.startswith("<?xml") and "</svg>" in s and s.count("<polyline") == 8
    assert all(rec.gbs > 0 and rec.median_s > 0 for rec in recs)


@pytest.mark.gpu
def test_cli_fp32_rectangular_baseline_shapes(cuda, tmp_path):
    csv = tmp_path / "rect.csv"
    r = subprocess.run([sys.executable, "-m", "paper_2108_02025_b200.benchcli", "--kernel",
                        "gemv-col", "--sizes", "4096", "--rect", "256x262144,262144x256",
                        "--dtype", "f64", "--reps", "3", "--csv", str(csv)],
                       capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr
    recs = B.parse_csv(csv.read_text())
    assert [(x.m, x.n) for x in recs] == [(4096, 4096), (256, 262144), (262144, 256)]
    assert all(x.dtype == "f64" and x.roofline_frac > 0.2 for x in recs)


def test_gpus_layout_and_dram_columns_round_trip():
    r = B.BenchRecord("gemv-col", 256, 1 << 20, 1, 3, 3.0e-4, 3.1e-4, 1.7e3, 2.0, "f64", 7.0e3,
                      0.53, gpus=2, layout="col-major", alg_bytes=2155876352,
                      hbm_bound_s=2155876352 / (2 * 6552.6e9), dram_bytes=2.156e9,
                      dram_per_alg=1.0001)
    text = B.emit_csv([r])
    head = text.splitlines()[0]
    assert head == B.CSV_HEADER + B.CSV_GPU_SUFFIX + B.CSV_BOUNDS_SUFFIX
    assert head.split(",")[12:14] == ["gpus", "layout"]
    back = B.parse_csv(text)[0]
    assert (back.gpus, back.layout, back.dram_per_alg) == (2, "col-major", 1.0001)
    assert B.emit_csv([back]) == text


def test_round1_documents_still_parse():
    old = B.CSV_HEADER + B.CSV_GPU_SUFFIX_R1 + "\n" + "ger,64,64,1,3,1e-05,2e-05,3,4,f32,5,0.5\n"
    r = B.parse_csv(old)[0]
    assert r.gpus == 1 and r.layout == "row-major" and r.gbs == 5
    oldb = (B.CSV_HEADER + B.CSV_GPU_SUFFIX_R1 + B.CSV_BOUNDS_SUFFIX_R1 + "\n"
            + "dot,0,64,1,3,1e-05,2e-05,3,4,f32,5,0.5,512,7e-11\n")
    r = B.parse_csv(oldb)[0]
    assert r.alg_bytes == 512 and r.dram_bytes != r.dram_bytes  # nan: not measured


def test_alg_bytes_count_replicated_operands_per_gpu():
    # x once per GPU for row blocks, y once per GPU for GER
    assert B._alg_bytes("gemv-row", 65536, 65536, 4, 8) == 17182490624
    assert B._alg_bytes("ger", 8192, 8192, 4, 4) == 537034752
    assert B._alg_bytes("dot", 0, 1 << 32, 4, 8) == 1 << 35
    assert B._split("gemv-col", 256, 1000, 3) == [(0, 334), (334, 667), (667, 1000)]
    assert B._split("ger", 10, 7, 4) == [(0, 3), (3, 6), (6, 8), (8, 10)]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_ger_exact_sample_is_ger_ref_bitwise(dtype):
    """The GER spot check's exact-rational rule agrees with the compiled
    oracle's ger_ref (one fma per element) and catches a one-ulp error."""
    import numpy as np

    from oracle import oracle as O
    rng = np.random.default_rng(3)
    npdt = np.float32 if dtype == torch.float32 else np.float64
    m, n = 37, 53
    x = rng.uniform(-1, 1, m).astype(npdt)
    y = rng.uniform(-1, 1, n).astype(npdt)
    C0 = rng.uniform(-1, 1, m * n).astype(npdt)
    C1 = C0.copy()
    O.ger_ref(x, y, C1, 0)
    t = lambda a: torch.from_numpy(a)  # noqa: E731
    assert B._ger_exact_sample(t(x), t(y), t(C0), t(C1), m, n, dtype, k=m * n) is None
    C1[5 * n + 7] = np.nextafter(C1[5 * n + 7], npdt(2))
    assert "C(5,7)" in B._ger_exact_sample(t(x), t(y), t(C0), t(C1), m, n, dtype, k=m * n)


@pytest.mark.gpu
def test_bounds_measured_dram_matches_algorithmic_bytes(cuda, tmp_path):
    """--bounds --measure-dram: ncu's DRAM bytes for a G1-shaped row-major
    GEMV are the algorithmic bytes (no re-reads)."""
    import shutil
    if not (shutil.which("ncu") or Path("/usr/local/cuda/bin/ncu").exists()):
        pytest.skip("ncu not installed")
    csv = tmp_path / "b.csv"
    r = subprocess.run([sys.executable, "-m", "paper_2108_02025_b200.benchcli", "--kernel",
                        "gemv-row", "--sizes", "8192", "--dtype", "f32", "--reps", "3",
                        "--bounds", "--measure-dram", "--csv", str(csv)],
                       capture_output=True, text=True, cwd=ROOT, timeout=900)
    if r.returncode != 0 and "ncu failed" in r.stderr and "closed" in r.stderr.lower():
        pytest.skip("ncu is closed on this pool")
    assert r.returncode == 0, r.stderr
    rec = B.parse_csv(csv.read_text())[0]
    assert rec.alg_bytes == 268533760
    assert 0.95 <= rec.dram_per_alg <= 1.10, rec.dram_per_alg


@pytest.mark.gpu
def test_cli_through_the_multi_gpu_c_abi(cuda, tmp_path):
    """--mgpu: every kernel through the cabl_mgpu C ABI (all visible GPUs with
    --gpus; here world = 1), spot-checked, device-timed, gpus column set."""
    csv = tmp_path / "m.csv"
    g = torch.cuda.device_count()
    r = subprocess.run([sys.executable, "-m", "paper_2108_02025_b200.benchcli", "--kernel", "all",
                        "--sizes", "256,4096", "--rect", "256x262144", "--dtype", "f32",
                        "--reps", "3", "--gpus", str(g), "--mgpu", "--csv", str(csv)],
                       capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr
    recs = B.parse_csv(csv.read_text())
    assert len(recs) == 2 + 3 * 3
    assert all(x.gpus == g and x.gbs > 0 for x in recs)
    assert {x.layout for x in recs} == {"vector", "row-major", "col-major"}


def test_cabl_bench_executable_exit_codes():
    """bin/cabl-bench: the reference CLI's name and exit codes (2 on an error)."""
    exe = ROOT / "bin" / "cabl-bench"
    r = subprocess.run([str(exe), "--sizes", "0"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "sizes must be >= 1" in r.stderr
    r = subprocess.run([str(exe), "--machine", "/nonexistent.json", "--sizes", "64"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "cannot open descriptor file" in r.stderr
