"""Build a variant of libsdmd.so with extra -D flags on one source (kernel-tuning experiments).
Usage: python scripts/build_variant.py NAME SOURCE.cu -DFOO=1 ...  -> variants/libsdmd_NAME.so
Load it with SDMD_LIB=<path>.  The default library must be built first (shares its objects)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1612_07875_b200 import build as B  # noqa: E402

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
bdir = os.path.join(B.HERE, "build")
out = os.path.join(ROOT, "variants")
os.makedirs(out, exist_ok=True)
inc = ["-I", B.CSRC, "-I", os.path.join(ROOT, "include"), "-I", B._nccl_include()]
common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"] + B.ARCH + inc
vo = os.path.join(out, f"{name}_{src.replace('.cu', '.o')}")
subprocess.run([os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc"), "-c", os.path.join(B.CSRC, src), "-o", vo]
               + common + defs, check=True)
objs = [vo if s == src else os.path.join(bdir, s.replace(".cu", ".o")) for s in B.SOURCES]
lib = os.path.join(out, f"libsdmd_{name}.so")
subprocess.run(["/usr/local/cuda/bin/nvcc", "-shared", "-o", lib] + objs + B.ARCH + ["-ldl"], check=True)
print(lib)
