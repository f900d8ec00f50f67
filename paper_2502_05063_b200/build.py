"""Build libvr.so in-tree for sm_100a (nvcc; no JIT cache, so the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvr.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["vr_api.cu", "tables.cu", "sort.cu", "hotpath.cu", "sparse.cu", "hypha.cu", "hypha_host.cpp", "netsimplex.cpp", "w1.cu", "host.cpp", "probe.cu", "comm.cu", "residual_prep.cu"]
HEADERS = ["vr_common.cuh", "vr_internal.h", "vr_types.h"]

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3,-pthread",
    "-shared",
    "--expt-relaxed-constexpr",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "vr.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


LIB_CHECKS = os.path.join(HERE, "libvr_checks.so")


def build(force: bool = False, verbose: bool = False, checks: bool = False) -> str:
    """checks: the bounds-checked variant (device asserts, -DVR_CHECKS) -> libvr_checks.so"""
    lib = LIB_CHECKS if checks else LIB
    if not force and not checks and not _stale():
        return LIB
    srcs = [os.path.join(CSRC, f) for f in SOURCES]
    tmp = lib + ".tmp"
    cmd = [NVCC, *FLAGS, *(["-DVR_CHECKS"] if checks else []), "-I", os.path.join(HERE, "..", "include"), "-o", tmp,
           *srcs, "-ldl"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checks="--checks" in sys.argv))
