"""The C++ drop-in header (include/pcstable_b200.hpp): builds against the C ABI
without a GPU; on a GPU the reference-style C++ test program runs against the
device library and the CPU oracle."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_1812_08491_b200", "build")
EXE = os.path.join(BUILD, "test_dropin")


def build_dropin_test() -> str:
    import paper_1812_08491_b200 as pcs
    from oracle import pyoracle
    pyoracle.lib()
    os.makedirs(BUILD, exist_ok=True)
    pkg = os.path.dirname(pcs.LIB_PATH)
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"),
           pcs.LIB_PATH, os.path.join(ROOT, "oracle", "libpcs_oracle.so"),
           f"-Wl,-rpath,{pkg}", f"-Wl,-rpath,{os.path.join(ROOT, 'oracle')}", "-o", EXE]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return EXE


def test_dropin_header_compiles_and_links():
    exe = build_dropin_test()
    assert os.path.exists(exe)


def test_dropin_header_is_c_compatible():
    """include/pcstable_b200.h is plain C (the ABI a cgo/ctypes/JNI binding consumes)."""
    src = "#include \"pcstable_b200.h\"\nint main(void){pcs_config c; pcs_config_default(&c); return c.max_level + 1;}\n"
    exe = os.path.join(BUILD, "c_abi_probe")
    os.makedirs(BUILD, exist_ok=True)
    import paper_1812_08491_b200 as pcs
    res = subprocess.run(["gcc", "-std=c99", "-Wall", "-x", "c", "-", "-x", "none", "-I", os.path.join(ROOT, "include"),
                          pcs.LIB_PATH, f"-Wl,-rpath,{os.path.dirname(pcs.LIB_PATH)}", "-o", exe],
                         input=src, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    assert subprocess.run([exe]).returncode == 0  # pcs_config_default needs no GPU


@pytest.mark.gpu
def test_dropin_program_on_device(pcs):
    exe = build_dropin_test()
    res = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
