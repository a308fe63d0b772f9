"""bench.py contract pieces that run without a GPU: the reference arm (the
compiled reference's CPU path timed on the host cores) prints one JSON line
with the agreed keys; the GPU arm refuses to run without a device."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps",
                        "2", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["unit"] == "GB/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["config"]["workload"].startswith("G1")


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_gpu_arm_refuses_without_gpu():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 2
    assert "no CUDA device" in r.stdout


@pytest.mark.parametrize("wid", ["D1", "G1", "R1", "G3"])
def test_cpu_reference_sample_paths(wid):
    """The --cpu-table leg on a small sample of each op: the threaded path and
    the naive oracle both run and report algorithmic GB/s."""
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2108_02025_b200 import workloads as WL
    w = WL.WORKLOADS[wid]
    for naive in (False, True):
        r = bench.cpu_reference_sample(w, max_bytes=4 << 20, reps=1, threads=2, naive=naive)
        assert r["value"] > 0 and r["unit"] == "GB/s"
        assert r["cores"] == (1 if naive or r["kind"] == "port" else 2)
        assert ("naive oracle" in r["sample"]) == (naive and r["kind"] == "reference")
