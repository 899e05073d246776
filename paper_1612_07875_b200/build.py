"""Build libsdmd.so (the C-ABI library, include/sdmd.h) in-tree for sm_100a with nvcc.

Usage: python -m paper_1612_07875_b200.build [--force] [--verbose]
The .so is written next to this file (git-ignored, travels to the GPU box with the repo).
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsdmd.so")
SOURCES = ["sdmd_api.cu", "k1_gram.cu", "k1b_batch.cu", "k2_dmma.cu", "k3_sparse.cu", "k4_eigen.cu", "k6_background.cu"]
HEADERS = ["sdmd_internal.cuh", os.path.join("..", "..", "include", "sdmd.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include() -> str:
    cands = []
    try:
        import nvidia.nccl as nn  # type: ignore
        for p in list(getattr(nn, "__path__", [])):
            cands.append(os.path.join(p, "include"))
    except Exception:
        pass
    cands.append(os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl", "include"))
    cands.append("/usr/include")
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found (needed for types; libnccl is dlopen'ed at run time)")


def _digest() -> str:
    h = hashlib.sha256()
    for f in SOURCES + HEADERS:
        with open(os.path.join(CSRC, f), "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(ARCH).encode())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = False) -> str:
    stamp = LIB + ".stamp"
    dig = _digest()
    if not force and os.path.exists(LIB) and os.path.exists(stamp):
        if open(stamp).read().strip() == dig:
            return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    objs = []
    inc = ["-I", CSRC, "-I", os.path.join(ROOT, "include"), "-I", _nccl_include()]
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-v" if verbose else "-O3"] + ARCH + inc
    bdir = os.path.join(HERE, "build")
    os.makedirs(bdir, exist_ok=True)
    for s in SOURCES:
        o = os.path.join(bdir, s.replace(".cu", ".o"))
        cmd = [nvcc, "-c", os.path.join(CSRC, s), "-o", o] + common
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {s}")
        objs.append(o)
    tmp = LIB + ".tmp"
    cmd = [nvcc, "-shared", "-o", tmp] + objs + ARCH + ["-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, LIB)
    with open(stamp, "w") as fh:
        fh.write(dig)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
