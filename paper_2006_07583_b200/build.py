"""In-tree build of libadi.so for sm_100a (nvcc; no JIT cache, no site-packages)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "libadi.so")
SOURCES = [os.path.join(HERE, "csrc", "adi_runtime.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", "adi_line.cuh"),
        os.path.join(HERE, "csrc", "adi_thread.cuh"),
        os.path.join(HERE, "csrc", "adi_warp.cuh"), os.path.join(ROOT, "include", "adi.h")]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "177"]


def build(force: bool = False, verbose: bool = False) -> str:
    nvcc = os.environ.get("NVCC", "nvcc")
    stale = (not os.path.exists(LIB_PATH)) or any(
        os.path.getmtime(d) > os.path.getmtime(LIB_PATH) for d in DEPS)
    if force or stale:
        cmd = [nvcc] + NVCC_FLAGS + ["-I", os.path.join(ROOT, "include"), "-o", LIB_PATH] + SOURCES
        if verbose:
            cmd += ["-Xptxas", "-v"]
        subprocess.run(cmd, check=True)
    return LIB_PATH
