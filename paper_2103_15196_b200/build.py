"""Build the in-tree CUDA library ``libcsph.so`` for sm_100a (nvcc, no torch JIT).

Flags: ``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false``.
``-fmad=false`` forbids implicit FMA contraction so every kernel expression
rounds exactly as written in DESIGN.md section 3 (bitwise parity with the CPU
oracle).  NCCL is opened lazily with dlopen (only the headers are needed here).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libcsph.so")
SOURCES = ["csph_api.cu", "csph_staged.cu", "csph_fused.cu"]
HEADERS = ["csph_internal.cuh", "csph_real.cuh", "csph_launch.h", "../../include/csph.h"]


def _nccl_include() -> str:
    try:
        import nvidia.nccl  # type: ignore
        for p in nvidia.nccl.__path__:
            inc = os.path.join(p, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except ImportError:
        pass
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include"
    raise RuntimeError("nccl.h not found")


def nvcc_cmd(out: str = SO) -> list[str]:
    return [
        "nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
        "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
        "-I" + _nccl_include(), "-shared", "-o", out,
    ] + [os.path.join(CSRC, s) for s in SOURCES] + ["-ldl"]


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        r = subprocess.run(nvcc_cmd(), capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libcsph.so")
        if verbose:
            sys.stderr.write(r.stderr)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(SO)
