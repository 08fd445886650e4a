"""The host library's free-id bitmap (csrc/aqua_idset.h: lowest-first block
and slot allocation, reading R4) against a std::set model on random single
and bulk operations -- ids present or absent, duplicates, sorted runs --
with the size, membership, ascending iteration and scan checked after every
operation.  g++ only, no CUDA."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_idset_matches_set_model(tmp_path):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not available")
    exe = tmp_path / "idset_test"
    r = subprocess.run([gxx, "-O2", "-std=c++17", "-Wall", "-I", os.path.join(ROOT, "paper_2407_21255_b200", "csrc"),
                        os.path.join(ROOT, "tests", "c", "idset_test.cpp"), "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("ok ")
