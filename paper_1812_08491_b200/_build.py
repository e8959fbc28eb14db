"""In-tree build of libpcstable_b200.so for sm_100a (nvcc, no JIT cache).

level.cu is compiled with -fmad=false so every CI decision keeps the
reference's two-rounding a*b+c (bit parity with the oracle); corr.cu keeps
FMA/DMMA (the Gram's summation order is not pinned by the reference).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libpcstable_b200.so")
BUILD = os.path.join(PKG, "build")
CLI = os.path.join(PKG, "pcstable_b200")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
          "--expt-relaxed-constexpr", "-I", CSRC, "-I", os.path.join(ROOT, "include")]
UNITS = {
    "level.cu": ["-fmad=false"],
    "level1t.cu": ["-fmad=false"],
    "datagen_dev.cu": ["-fmad=false"],
    "corr.cu": [],
    "host.cu": ["-Xcompiler", "-ffp-contract=off"],
    "probe.cu": [],
    "orient.cu": ["-Xcompiler", "-ffp-contract=off"],
}


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "pcstable_b200.h"))
    objs = []
    for unit, extra in UNITS.items():
        src = os.path.join(CSRC, unit)
        obj = os.path.join(BUILD, unit.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [src, *headers, __file__]):
            cmd = [nvcc(), *ARCH, *COMMON, *extra, "-c", src, "-o", obj]
            res = subprocess.run(cmd, capture_output=True, text=True)
            log = os.path.join(BUILD, unit + ".ptxas.log")
            with open(log, "w") as f:
                f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
            if res.returncode != 0:
                sys.stderr.write(res.stderr)
                raise RuntimeError(f"nvcc failed for {unit}")
            if verbose:
                sys.stderr.write(res.stderr)
    # host-only datagen: plain g++, no FMA contraction (reference Release build has none)
    dsrc = os.path.join(CSRC, "datagen.cpp")
    dobj = os.path.join(BUILD, "datagen.o")
    objs.append(dobj)
    if force or _stale(dobj, [dsrc, *headers, __file__]):
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-c", dsrc, "-o", dobj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stderr)
            raise RuntimeError("g++ failed for datagen.cpp")
    if force or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stderr)
            raise RuntimeError("link failed")
    # the reference CLI (pcstable_main.cpp) on the device path: host C++20 over the drop-in header
    cli_src = os.path.join(PKG, "cli", "pcstable_b200.cpp")
    if force or _stale(CLI, [cli_src, LIB, os.path.join(ROOT, "include", "pcstable_b200.hpp")]):
        cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), cli_src, LIB,
               "-Wl,-rpath,$ORIGIN", "-o", CLI]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stderr)
            raise RuntimeError("g++ failed for cli/pcstable_b200.cpp")
    return LIB


def build_variant(name: str, defines: list[str], source: str | None = None) -> str:
    """Tuning experiments (tools/variants.py): the library with level.cu rebuilt under extra -D knobs
    (or from another level.cu `source`, e.g. an older revision for A/B timing) into
    variants/libpcstable_b200_<name>.so (knobs never change results)."""
    build()
    vdir = os.path.join(BUILD, "var_" + name)
    os.makedirs(vdir, exist_ok=True)
    out_dir = os.path.join(PKG, "variants")
    os.makedirs(out_dir, exist_ok=True)
    lib = os.path.join(out_dir, f"libpcstable_b200_{name}.so")
    obj = os.path.join(vdir, "level.o")
    cmd = [nvcc(), *ARCH, *COMMON, *UNITS["level.cu"], *[f"-D{d}" for d in defines], "-c",
           source or os.path.join(CSRC, "level.cu"), "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    with open(os.path.join(vdir, "level.cu.ptxas.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr)
        raise RuntimeError(f"nvcc failed for variant {name}")
    objs = [obj] + [os.path.join(BUILD, u.replace(".cu", ".o")) for u in UNITS if u != "level.cu"]
    objs.append(os.path.join(BUILD, "datagen.o"))
    cmd = [nvcc(), *ARCH, "-shared", "-o", lib, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stderr)
        raise RuntimeError("variant link failed")
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
