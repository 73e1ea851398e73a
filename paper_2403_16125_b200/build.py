"""Build libcrius.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcrius.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-fmad=false"]


def sources():
    srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))]
    srcs.append(os.path.join(ROOT, "include", "crius.h"))
    return srcs


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources())


def build_debug(out=None):
    """libcrius with the device-side invariant checks (-DCRIUS_DEBUG)."""
    out = out or os.path.join(ROOT, "variants", "libcrius_debug.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [os.environ.get("NVCC", "nvcc")] + NVCC_FLAGS + ["-DCRIUS_DEBUG", "-o", out,
                                                           os.path.join(CSRC, "crius_lib.cu")]
    subprocess.check_call(cmd)
    return out


def build_variant(name, defines):
    """libcrius compiled with extra -D flags into variants/<name> (experiments only)."""
    out = os.path.join(ROOT, "variants", name)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [os.environ.get("NVCC", "nvcc")] + NVCC_FLAGS + ["-D" + d for d in defines] + [
        "-o", out, os.path.join(CSRC, "crius_lib.cu")]
    subprocess.check_call(cmd)
    return out


def build(force=False, verbose=False):
    if not force and up_to_date():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc] + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose else []) + [
        "-o", LIB, os.path.join(CSRC, "crius_lib.cu")]
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
