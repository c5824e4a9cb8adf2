"""Build the simulator library in-tree for sm_100a (nvcc cross-compiles without a GPU).

Four builds of the same sources:
  libdsi_sim.so         the product (no test hooks, no developer knobs)
  libdsi_sim_test.so    -DDSI_TEST_HOOKS: adds include/dsi_sim_testing.h (host all-reduce hook,
                        A/B knobs) for the multi-rank-on-one-GPU tests and A/B runs
  libdsi_sim_mutant.so  -DDSI_TEST_HOOKS -DDSI_MUTANT_CG -DDSI_MUTANT_TIES: every DSI segment cost
                        C(g), g >= 2, one tick too large, and the halves layout's tie-break dropped
                        (ties left as rejections) -- the mutation test (tests/test_mutation.py)
                        checks that GPU parity against the oracle FAILS with it
  libdsi_sim_checked.so -DDSI_TEST_HOOKS -DDSI_BOUNDS_CHECK: the kernels' computed indices checked
                        (DSI_CHECK traps) -- tests/test_bounds_checked.py runs every kernel variant
                        under it (compute-sanitizer is closed on the GPU pool)
Each library embeds the SHA-256 of its sources and flags (dsi_build_id()); a build is redone
whenever the embedded id differs from that of the current sources, so a snapshot shipped to a
GPU box always runs a build of exactly the tree it carries.  Objects compile in parallel.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = ["dsi_validate.cpp", "dsi_plan.cpp", "dsi_collective.cpp", "dsi_runtime.cpp",
        "dsi_multi_host.cpp", "dsi_heatmap.cpp"]
DEVICE = ["dsi_kernel.cu", "dsi_crn.cu", "dsi_reduce_dev.cu", "dsi_crn2.cu", "dsi_multi.cu", "dsi_seg.cu",
          "dsi_stage.cu"]
SOURCES = [os.path.join(CSRC, f) for f in HOST + DEVICE]
HEADERS = [os.path.join(CSRC, f) for f in ("dsi_host.h", "dsi_device.h", "dsi_convert.h", "dsi_common.cuh",
                                                  "dsi_crn_common.cuh")] + \
          [os.path.join(ROOT, "include", f) for f in ("dsi_sim.h", "dsi_sim_testing.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
VARIANTS = {"product": ("libdsi_sim.so", []),
            "test": ("libdsi_sim_test.so", ["-DDSI_TEST_HOOKS"]),
            "mutant": ("libdsi_sim_mutant.so", ["-DDSI_TEST_HOOKS", "-DDSI_MUTANT_CG", "-DDSI_MUTANT_TIES"]),
            "checked": ("libdsi_sim_checked.so", ["-DDSI_TEST_HOOKS", "-DDSI_BOUNDS_CHECK"])}
LIB = os.path.join(PKG, VARIANTS["product"][0])
TEST_LIB = os.path.join(PKG, VARIANTS["test"][0])
MUTANT_LIB = os.path.join(PKG, VARIANTS["mutant"][0])
COMMON = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden"]
# per-source ptxas settings: the trial kernels' register allocation at -regUsageLevel=2 (default 5):
# the 32-bit layout's kernel takes 80 registers instead of 91 and runs 1.7% faster on the cfg3
# sample (cfg4 1.6%, cfg5 and the halves / fresh-verifier variants unchanged;
# profiles/r02o_ab_*_ru2*.jsonl, r02o_ab_*_reglevel.jsonl); the two-pass shared-stream kernels at
# -regUsageLevel=8: cfg3 12.77 -> 12.5 ms (profiles/r02s_ab_shared_reglevel.jsonl)
PER_SOURCE = {"dsi_kernel.cu": ["-Xptxas", "-regUsageLevel=2"], "dsi_crn2.cu": ["-Xptxas", "-regUsageLevel=8"]}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build_id(variant: str = "product") -> str:
    """SHA-256 over the source and header contents and the variant's flags."""
    h = hashlib.sha256()
    for p in SOURCES + HEADERS:
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(COMMON + VARIANTS[variant][1]).encode())
    h.update(repr(sorted(PER_SOURCE.items())).encode())
    return h.hexdigest()


def embedded_id(lib: str):
    """The id a built library carries (read from its bytes, without loading it)."""
    try:
        data = open(lib, "rb").read()
    except OSError:
        return None
    i = data.find(b"DSI_BUILD_ID=")
    return data[i + 13:i + 77].decode(errors="replace") if i >= 0 else None


def stale(variant: str = "product") -> bool:
    lib = os.path.join(PKG, VARIANTS[variant][0])
    return embedded_id(lib) != build_id(variant)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError("nvcc failed: " + os.path.basename(cmd[-1]))
    return r.stderr


def build_variant(variant: str = "product", force: bool = False, verbose: bool = False, jobs: int = 0) -> str:
    name, flags = VARIANTS[variant]
    lib = os.path.join(PKG, name)
    if not force and not stale(variant):
        return lib
    bid = build_id(variant)
    odir = os.path.join(PKG, "build", variant)
    os.makedirs(odir, exist_ok=True)
    extra = ["-Xptxas", "-v"] if verbose else []

    def compile_one(src):
        obj = os.path.join(odir, os.path.basename(src) + ".o")
        defs = ["-DDSI_BUILD_ID=\"" + bid + "\""] if src.endswith("dsi_validate.cpp") else []
        per = PER_SOURCE.get(os.path.basename(src), [])
        return _run([nvcc(), *COMMON, *flags, *per, *defs, *extra, "-I" + os.path.join(ROOT, "include"), "-c",
                     "-o", obj, src]), obj

    with ThreadPoolExecutor(max_workers=jobs or min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    if verbose:
        for log, _ in results:
            sys.stderr.write(log)
    tmp = lib + ".tmp"
    _run([nvcc(), *ARCH, "-shared", "-o", tmp, *[o for _, o in results], "-ldl"])
    os.replace(tmp, lib)
    return lib


def build_library(force: bool = False, verbose: bool = False,
                  variants=("product", "test", "mutant", "checked")) -> str:
    """Build every variant whose embedded id is not the current one; returns the product path."""
    with ThreadPoolExecutor(max_workers=len(variants)) as ex:
        list(ex.map(lambda v: build_variant(v, force=force, verbose=verbose and v == "product",
                                            jobs=max(2, (os.cpu_count() or 4) // len(variants))), variants))
    return LIB


def command(out: str = LIB, extra=()) -> list:
    """One-shot nvcc command of a library from the product sources (profiles/ A/B scripts).  One nvcc
    call cannot give one source its own flags: PER_SOURCE is not applied (pass it in `extra` to
    apply it to every source)."""
    return [nvcc(), *COMMON, "-shared", "-I" + os.path.join(ROOT, "include"), "-o", out, *SOURCES, "-ldl", *extra]


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose="-v" in sys.argv))
