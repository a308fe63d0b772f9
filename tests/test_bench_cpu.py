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


def test_launcher_spawns_gpus_ranks_over_gloo():
    """`bench.py --gpus 2` without torchrun re-executes itself under
    torch.distributed.run with 2 ranks (checked on CPU over gloo)."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--launch-check"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2
    assert sorted(x["rank"] for x in d["ranks"]) == [0, 1]
    assert len({x["pid"] for x in d["ranks"]}) == 2  # one process per rank


@pytest.mark.skipif(torch.cuda.device_count() >= 2, reason="checks the too-few-GPUs refusal")
def test_launcher_refuses_more_gpus_than_visible():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode != 0
    assert "needs 2 visible GPUs" in r.stderr


def test_launcher_refuses_world_size_mismatch():
    import os
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--steps", "3"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode != 0
    assert "WORLD_SIZE=2 but --gpus 4" in r.stderr


def test_both_arms_share_the_workload_config():
    """The driver matches our line with the reference arm's by `config`: both
    are built by one function and carry only workload-defining fields."""
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2108_02025_b200 import workloads as WL
    for w in WL.WORKLOADS.values():
        cfg = bench.workload_config(w)
        assert set(cfg) == {"workload", "m_per_gpu", "n", "layout", "dtype", "l2"}
        assert cfg == bench.workload_config(w)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps",
                        "1", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["config"] == bench.workload_config(WL.WORKLOADS["G1"])


def test_l2_policy_follows_the_footprint_not_the_algorithmic_bytes():
    """A GER shard whose in-place C fits in L2 must be flushed between steps even
    though its read + write bytes exceed the L2 (R1 over 4 GPUs: 64 MiB of C, 134 MB
    algorithmic; back to back it runs out of L2 at 9.8 TB/s,
    profiles/r02_shard_share.jsonl)."""
    import dataclasses
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2108_02025_b200 import workloads as WL
    r1 = WL.WORKLOADS["R1"]
    assert r1.footprint_bytes() == 8192 * 8192 * 4 + 2 * 8192 * 4
    assert r1.alg_bytes(1) == 2 * 8192 * 8192 * 4 + 2 * 8192 * 4
    assert bench.l2_mode(r1.footprint_bytes()) == "stream"
    quarter = dataclasses.replace(r1, m=r1.m // 4)
    assert quarter.alg_bytes(1) > bench.L2_BYTES > quarter.footprint_bytes()
    assert bench.l2_mode(quarter.footprint_bytes()) == "flush"
    for wid in ("D1", "G1", "G2", "G3", "G4", "D2"):  # read-only inputs: footprint ~ alg bytes
        w = WL.WORKLOADS[wid]
        assert bench.l2_mode(w.footprint_bytes()) == "stream"
        assert 0 <= w.alg_bytes(1) - w.footprint_bytes() <= w.m * w.s
