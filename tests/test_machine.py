"""GPU machine descriptor (paper_2108_02025_b200/machine.py).

CPU: the document format and rules against the reference's loader/validator
semantics (descriptor_json.hpp:25-61, machine.hpp:55-136) and the committed
B200 capture machines/b200.json.  GPU: the live device equals the capture
and the C ABI's derived work-queue threshold equals derive_gpu_plan's."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

from paper_2108_02025_b200 import cabl, machine as MC

ROOT = Path(__file__).resolve().parents[1]

B200 = MC.GpuInfo(device=0, name="NVIDIA B200", cc=(10, 0), sm_count=148,
                  max_threads_per_sm=2048, line_bytes=128, smem_per_sm=233472,
                  smem_per_block_optin=232448, l2_bytes=132644864, hbm_bytes=191502876672,
                  mem_bus_bits=7680, queue_threshold_bytes=512 << 20)


def test_descriptor_document_follows_the_reference_format_and_rules():
    doc = MC.descriptor_of(B200, 4)
    assert set(doc) >= {"element_bytes", "cores", "levels"}
    assert doc["cores"] == 148 and doc["element_bytes"] == 4
    l1, l2 = doc["levels"]
    assert (l1["line_bytes"], l1["shared"], l2["line_bytes"], l2["shared"]) == (128, False, 128, True)
    assert l1["line_bytes"] * l1["associativity"] * l1["num_sets"] == 233472
    assert l2["line_bytes"] * l2["associativity"] * l2["num_sets"] == 132644864
    md = MC.load_descriptor(json.dumps(doc))  # extra 'gpu' key ignored
    plan = cabl.derive_blocking_plan(md)      # the reference derivation accepts it
    assert plan.max_threads == 148
    assert plan.dot_cutoff == 2 * 233472 // 4


def test_gpu_plan_rules():
    p = MC.derive_gpu_plan(MC.load_descriptor(json.dumps(MC.descriptor_of(B200, 8))))
    assert p.sm_count == 148 and p.dot_ctas == 296
    assert p.queue_threshold_bytes == 512 << 20 == p.l2_flush_bytes
    assert p.l2_bytes == 132644864
    # the rule is 4 x L2 rounded up to a power of two
    small = MC.GpuInfo(**{**B200.__dict__, "l2_bytes": 50 << 20})
    assert MC.derive_gpu_plan(MC.load_descriptor(json.dumps(MC.descriptor_of(small)))) \
        .queue_threshold_bytes == 256 << 20


def test_loader_errors_carry_reference_messages(tmp_path):
    with pytest.raises(cabl.DescriptorError, match="descriptor parse failure"):
        MC.load_descriptor("{not json")
    with pytest.raises(cabl.DescriptorError, match="descriptor parse failure"):
        MC.load_descriptor(json.dumps({"cores": 1, "levels": []}))
    with pytest.raises(cabl.DescriptorError, match="cannot open descriptor file"):
        MC.load_descriptor_file(tmp_path / "missing.json")
    bad = MC.descriptor_of(B200)
    bad["levels"][0]["shared"] = True
    with pytest.raises(cabl.DescriptorError, match="level 1 must be private"):
        MC.load_descriptor(json.dumps(bad))


def test_committed_b200_capture_is_valid():
    md = MC.load_descriptor_file(MC.B200_JSON)
    assert md.cores == 148
    p = MC.derive_gpu_plan(md)
    assert p.queue_threshold_bytes == 512 << 20
    assert 120e6 < p.l2_bytes < 140e6
    doc = json.loads(MC.B200_JSON.read_text())
    assert doc["gpu"]["cc"] == "10.0"


def test_describe_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception):
        MC.describe_device(0)


@pytest.mark.gpu
def test_live_device_matches_capture_and_library_rule(cuda):
    info = MC.describe_device(0)
    assert info.sm_count == 148 and info.cc == (10, 0)
    live = MC.descriptor_of(info, 4)
    cap = json.loads(MC.B200_JSON.read_text())
    assert live["levels"] == cap["levels"] and live["cores"] == cap["cores"]
    plan = MC.derive_gpu_plan(MC.gpu_machine(0))
    assert info.queue_threshold_bytes == plan.queue_threshold_bytes  # C ABI == Python rule


@pytest.mark.gpu
def test_benchcli_describe_prints_the_live_descriptor(cuda):
    r = subprocess.run([sys.executable, "-m", "paper_2108_02025_b200.benchcli", "--describe",
                        "--dtype", "f32"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    doc = json.loads(r.stdout)
    assert doc["cores"] == 148
    MC.load_descriptor(r.stdout)
