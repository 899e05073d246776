"""B200-native streaming method-of-snapshots SVD / DMD (arXiv 1612.07875 hot path).

The product is the C-ABI library ``libsdmd.so`` (include/sdmd.h) built from ``csrc/`` for sm_100a;
``sdmd`` is its thin ctypes binding.  Importing this package does not load the library; the first
call does, and fails loudly if it was not built (there is no CPU fallback).
"""
import os as _os


def recommended_env() -> None:
    """Opt-in helper: set CUDA_DEVICE_MAX_CONNECTIONS=32 unless the user set it.  The engine runs
    the Gram pass, the copy stream and up to 2·workers eigen streams concurrently; CUDA's default of
    8 hardware work queues makes some of them share a queue, so an eigen stage waits behind an
    unrelated stream-wait (measured +5.5 ms per frame of K4 latency).  Only effective if called
    before CUDA initialises in this process; importing the package does NOT change the environment
    (other libraries in the process may rely on their own setting)."""
    _os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


from .sdmd import (StreamingDMD, SDMDError, lib, nccl_unique_id, row_partition,  # noqa: F401
                   LIB_PATH, EXPORTS)
