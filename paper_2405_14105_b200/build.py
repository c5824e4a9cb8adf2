"""Build libdsi_sim.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libdsi_sim.so")
SOURCES = [os.path.join(CSRC, "dsi_host.cpp"), os.path.join(CSRC, "dsi_heatmap.cpp"),
           os.path.join(CSRC, "dsi_kernel.cu"), os.path.join(CSRC, "dsi_crn.cu"),
           os.path.join(CSRC, "dsi_reduce_dev.cu"), os.path.join(CSRC, "dsi_crn2.cu"),
           os.path.join(CSRC, "dsi_multi.cu"), os.path.join(CSRC, "dsi_seg.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "dsi_device.h"), os.path.join(CSRC, "dsi_common.cuh"),
                  os.path.join(CSRC, "dsi_crn_common.cuh"),
                  os.path.join(ROOT, "include", "dsi_sim.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def command(out: str = LIB, extra=()) -> list:
    return [nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O2", "-shared",
            "-I" + os.path.join(ROOT, "include"), "-o", out, *SOURCES, "-ldl", *extra]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build_library(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        cmd = command(extra=["-Xptxas", "-v"] if verbose else [])
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libdsi_sim.so")
        if verbose:
            sys.stderr.write(r.stderr)
    return LIB


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose="-v" in sys.argv))
