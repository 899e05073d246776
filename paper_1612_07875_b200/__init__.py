"""B200-native streaming method-of-snapshots SVD / DMD (arXiv 1612.07875 hot path).

The product is the C-ABI library ``libsdmd.so`` (include/sdmd.h) built from ``csrc/`` for sm_100a;
``sdmd`` is its thin ctypes binding.  Importing this package does not load the library; the first
call does, and fails loudly if it was not built (there is no CPU fallback).
"""
from .sdmd import (StreamingDMD, SDMDError, lib, nccl_unique_id, row_partition,  # noqa: F401
                   LIB_PATH, EXPORTS)
