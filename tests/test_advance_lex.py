"""CPU test of device code: the staged cuPC-E kernel's set stepper advance_lex<L> (pcs_device.cuh),
compiled for the host by nvcc and checked against a full lexicographic enumeration
(comb.hpp:50-67's order) for L = 2, 3."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_advance_lex_matches_enumeration(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = str(tmp_path / "test_advance_lex")
    src = os.path.join(ROOT, "tests", "cpp", "test_advance_lex.cu")
    inc = os.path.join(ROOT, "paper_1812_08491_b200", "csrc")
    subprocess.run([nvcc, "-std=c++17", "-O1", "-I", inc, src, "-o", exe], check=True, capture_output=True, timeout=300)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("ok"), out.stdout
