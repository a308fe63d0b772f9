"""The C++ descriptor loader (include/cabl/descriptor_json.hpp, the reference
descriptor_json.hpp:25-61 without its JSON dependency) agrees with the Python
loader on valid documents — the B200 descriptor and the reference's generic
one — and rejects malformed ones with a DescriptorError.  CPU only."""
from __future__ import annotations

import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def loader(tmp_path_factory):
    exe = tmp_path_factory.mktemp("desc") / "descriptor_test"
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror",
                    f"-I{ROOT / 'include'}", str(ROOT / "tests/cpp/descriptor_test.cpp"),
                    "-o", str(exe)], check=True)
    return exe


def run(loader, docs, tmp_path):
    paths = []
    for i, d in enumerate(docs):
        p = tmp_path / f"d{i}.json"
        p.write_text(d)
        paths.append(str(p))
    out = subprocess.run([str(loader), *paths], capture_output=True, text=True, check=True)
    return out.stdout.splitlines()


GENERIC = ('{"element_bytes": 8, "cores": 8, "levels": ['
           '{"line_bytes": 64, "associativity": 8, "num_sets": 64, "shared": false},'
           '{"line_bytes": 64, "associativity": 8, "num_sets": 1024, "shared": true}]}')


def test_valid_documents_match_the_python_loader(loader, tmp_path):
    from paper_2108_02025_b200 import machine as M
    b200 = (ROOT / "machines" / "b200.json").read_text()
    esc = GENERIC.replace('"cores"', '"c\\u006fres"')  # escapes in keys decode
    lines = run(loader, [GENERIC, b200, esc], tmp_path)
    for text, line in zip([GENERIC, b200, GENERIC], lines):
        md = M.load_descriptor(text)
        assert line.startswith("ok "), line
        f = dict(kv.split("=") for kv in line.split()[1:])
        assert int(f["cores"]) == md.cores and int(f["element_bytes"]) == md.element_bytes
        assert int(f["l1"]) == md.levels[0].size_bytes() and int(f["l2"]) == md.levels[1].size_bytes()
    # the reference defaults (README: m_c = n_c = 256, dot_block 2048, dot_cutoff 8192)
    f = dict(kv.split("=") for kv in lines[0].split()[1:])
    assert (f["m_c"], f["dot_block"], f["dot_cutoff"]) == ("256", "2048", "8192")


@pytest.mark.parametrize("doc,needle", [
    ("{", "descriptor parse failure"),
    ("[]", "descriptor parse failure"),
    ('{"element_bytes": 8, "cores": 8}', "missing key 'levels'"),
    ('{"element_bytes": -8, "cores": 8, "levels": []}', "non-negative integer"),
    ('{"element_bytes": 8.5, "cores": 8, "levels": []}', "non-negative integer"),
    ('{"element_bytes": 8, "cores": 8, "levels": [{"line_bytes": 64, "associativity": 8, '
     '"num_sets": 64, "shared": 0}]}', "must be a boolean"),
    (GENERIC + " x", "trailing characters"),
    (GENERIC.replace('"num_sets": 1024', '"num_sets": 32'), "level sizes must increase"),
    (GENERIC.replace('"line_bytes": 64, "associativity": 8, "num_sets": 64',
                     '"line_bytes": 48, "associativity": 8, "num_sets": 64'),
     "line size must be a power of two"),
    (GENERIC.replace('"cores": 8', '"cores": 0'), "cores must be >= 1"),
])
def test_malformed_documents_raise(loader, tmp_path, doc, needle):
    (line,) = run(loader, [doc], tmp_path)
    assert line.startswith("error ") and needle in line, line


def test_missing_file(loader):
    out = subprocess.run([str(loader), "/nonexistent/m.json"], capture_output=True, text=True,
                         check=True).stdout
    assert out.strip() == "error cannot open descriptor file: /nonexistent/m.json"


def test_b200_document_is_valid_json():
    d = json.loads((ROOT / "machines" / "b200.json").read_text())
    assert d["cores"] == 148 and len(d["levels"]) == 2
