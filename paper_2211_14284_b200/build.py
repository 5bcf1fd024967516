"""Builds the in-tree shared library paper_2211_14284_b200/librm.so (C ABI of include/rm.h).

Host setup code: g++ -O3 -fopenmp; kernels: nvcc for sm_100a only
(-gencode arch=compute_100a,code=sm_100a -lineinfo).  Incremental: objects are rebuilt when
their source or any header in csrc/ or include/ is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "librm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CXX_SRC = ["basis.cpp", "model.cpp", "patches.cpp", "coarse.cpp", "abi.cpp"]
CU_SRC = ["kernels.cu", "apply.cu", "apply_kform.cu", "apply_tri.cu", "patch_solve.cu", "coarse.cu", "dsetup.cu", "sc_ph.cu"]


def _headers():
    hs = []
    for d in (CSRC, os.path.join(ROOT, "include")):
        hs += [os.path.join(d, f) for f in os.listdir(d) if f.endswith((".h", ".hpp", ".cuh"))]
    return hs


def _stale(obj, src, headers):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(x) > t for x in [src] + headers)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[0]} {os.path.basename(cmd[-1])}")
    return r


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = _headers()
    objs = []
    inc = ["-I", CSRC, "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include"]
    if os.environ.get("RM_BUILD_EXPERIMENTS"):   # instrumentation build (exp_env.hpp); rebuild from clean
        inc += ["-DRM_EXPERIMENTS"]
    if os.environ.get("RM_BUILD_DEFS"):   # tuning sweeps: extra -D definitions (rebuild from clean)
        inc += os.environ["RM_BUILD_DEFS"].split()
    for s in CXX_SRC:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if _stale(obj, src, headers):
            # host code via nvcc's host compiler settings for consistency (g++, -O3, OpenMP)
            _run(["g++", "-std=c++17", "-O3", "-march=x86-64-v3", "-fopenmp", "-fPIC", "-Wall",
                  "-Wno-unused-function", *inc, "-c", "-o", obj, src])
    for s in CU_SRC:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if _stale(obj, src, headers):
            _run([NVCC, "-std=c++17", "-O3", *ARCH, "-lineinfo", "-Xptxas", "-v", "-Xcompiler", "-fPIC",
                  "--expt-relaxed-constexpr", *inc, "-c", "-o", obj, src])
    if not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        _run([NVCC, "-shared", *ARCH, "-o", LIB, *objs, "-Xcompiler", "-fopenmp", "-lgomp", "-cudart", "static"])
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
