"""Builds tests/native/libemu.so (test-only host re-enactment of the product's setup code)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
CSRC = os.path.join(ROOT, "paper_2211_14284_b200", "csrc")
LIB = os.path.join(HERE, "libemu.so")


def build():
    srcs = [os.path.join(HERE, "emu.cpp")] + [os.path.join(CSRC, f) for f in ("basis.cpp", "model.cpp", "patches.cpp", "coarse.cpp")]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".h"))]
    if os.path.exists(LIB) and all(os.path.getmtime(LIB) > os.path.getmtime(s) for s in deps):
        return LIB
    cmd = ["g++", "-std=c++17", "-O2", "-fopenmp", "-fPIC", "-shared", "-I", CSRC, "-o", LIB] + srcs
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    return LIB


if __name__ == "__main__":
    print(build())
