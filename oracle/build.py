"""Build the ORACLE's C library (test infrastructure, not the product): oracle/liboracle.so from
oracle/csrc/sdmd_oracle.c with gcc (plain C99, OpenMP for the optional row-chunk threads, no
BLAS).  Called lazily by oracle/sdmd_oracle.py and by __graft_entry__.build()."""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "sdmd_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
# -ffp-contract=off: no silent fma contraction (the compensated sums rely on exact IEEE steps);
# no -march=native: the .so built here also runs on the GPU box's host
FLAGS = ["-O2", "-std=c99", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math"]


def _digest() -> str:
    h = hashlib.sha256(open(SRC, "rb").read())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()[:16]


def build(force: bool = False) -> str:
    stamp = LIB + ".stamp"
    dig = _digest()
    if not force and os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read().strip() == dig:
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cc = shutil.which("gcc") or "gcc"
    r = subprocess.run([cc] + FLAGS + [SRC, "-o", tmp, "-lm"], capture_output=True, text=True)
    if r.returncode != 0:      # no libgomp: the same code, single-threaded (pragmas ignored)
        flags = [f for f in FLAGS if f != "-fopenmp"]
        r = subprocess.run([cc] + flags + [SRC, "-o", tmp, "-lm"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + r.stdout + r.stderr)
    os.replace(tmp, LIB)
    with open(stamp, "w") as fh:
        fh.write(dig)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
