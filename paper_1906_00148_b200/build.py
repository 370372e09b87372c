"""In-tree build of libshe.so (sm_100a) and the test-only host emulation.

    python -m paper_1906_00148_b200.build

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo; the .so lands next to
this file so gpurun ships it with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libshe.so")
EMU = os.path.join(HERE, "libshe_hostemu.so")

CUDA_SOURCES = ["engine.cu"]
CXX_SOURCES = ["client.cpp", "scheduler.cpp"]

NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
HOST_FLAGS = "-fPIC,-fopenmp,-ffp-contract=off,-march=x86-64-v3"
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xptxas", "-v", "--expt-relaxed-constexpr", "-DGL_ADDSUB_PTX",
              "-Xcompiler", HOST_FLAGS]


def _inputs():
    # every source and header under csrc/ (a new header is covered automatically)
    files = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
             if f.endswith((".cu", ".cuh", ".h", ".cpp", ".hpp"))]
    files.append(os.path.join(os.path.dirname(HERE), "include", "she.h"))
    files.append(os.path.join(os.path.dirname(HERE), "she_inputs", "she_rng.h"))
    files.append(os.path.abspath(__file__))
    return [f for f in files if os.path.exists(f)]


def _stale(target: str) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(f) > t for f in _inputs())


def build_lib(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale(LIB):
        return LIB
    objs = []
    for src in CUDA_SOURCES + CXX_SOURCES:
        path = os.path.join(CSRC, src)
        if not os.path.exists(path):
            continue
        obj = os.path.join(CSRC, src + ".o")
        cmd = [NVCC, *ARCH, *NVCC_FLAGS, "-c", path, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC,-fopenmp", *objs, "-o", tmp,
           "-lcudart", "-lgomp"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


def build_emu(force: bool = False) -> str:
    if not force and not _stale(EMU):
        return EMU
    cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", os.path.join(CSRC, "host_emu.cpp"),
           "-o", EMU]
    subprocess.run(cmd, check=True)
    return EMU


def build(force: bool = False, verbose: bool = False) -> None:
    build_lib(force, verbose)
    build_emu(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
