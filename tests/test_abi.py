"""CPU checks of the C-ABI boundary: libsdmd.so loads and exports every symbol include/sdmd.h
declares; host-side argument validation fails before any device work; the binding's config
struct matches the header layout.  No compute calls (no GPU here)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sdmd.h")


@pytest.fixture(scope="module")
def libpath():
    from paper_1612_07875_b200.build import build
    return build()


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sdmd_\w+)\s*\(", txt, re.M)))


def test_header_declares_expected_symbols():
    from paper_1612_07875_b200 import EXPORTS
    assert header_symbols() == sorted(EXPORTS)


def test_library_exports_every_header_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True)
    syms = set(re.findall(r"\sT\s(sdmd_\w+)", out.stdout))
    missing = [s for s in header_symbols() if s not in syms]
    assert not missing, missing
    L = ctypes.CDLL(libpath)
    for s in header_symbols():
        assert getattr(L, s) is not None


def test_sm100a_code_present(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath],
                         capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_status_strings_and_version(libpath):
    from paper_1612_07875_b200 import sdmd
    L = sdmd.lib()
    assert L.sdmd_abi_version() == 4
    assert L.sdmd_status_string(2).decode() == "non-finite frame rejected"
    assert L.sdmd_status_string(999).decode() == "unknown status"


def test_config_layout_and_validation(libpath):
    from paper_1612_07875_b200 import sdmd
    L = sdmd.lib()
    cfg = sdmd.Config()
    assert L.sdmd_config_init(ctypes.byref(cfg)) == 0
    assert abs(cfg.rank_tol - 1e-7) < 1e-20 and abs(cfg.threshold - 0.2) < 1e-7
    assert cfg.dmd == 1 and cfg.workers == 4 and cfg.nranks == 1
    # the binding's structs have the C layout of include/sdmd.h (sizes from a gcc-compiled probe)
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "sz.c")
        with open(src, "w") as fh:
            fh.write('#include <stdio.h>\n#include "sdmd.h"\nint main(){printf("%zu %zu %zu %zu", '
                     'sizeof(sdmd_config), sizeof(sdmd_info), sizeof(sdmd_stats), sizeof(sdmd_scores));return 0;}\n')
        exe = os.path.join(d, "sz")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        c_sizes = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    assert c_sizes == [ctypes.sizeof(sdmd.Config), ctypes.sizeof(sdmd.Info), ctypes.sizeof(sdmd.Stats),
                       ctypes.sizeof(sdmd.Scores)]
    assert cfg.eigen_shard == 1 and cfg.batch_max == 0
    h = ctypes.c_void_p()
    # invalid shapes are rejected before any CUDA call (works without a GPU)
    cfg.n_local = cfg.n_global = 100
    cfg.m = 1
    assert L.sdmd_create(ctypes.byref(cfg), ctypes.byref(h)) == sdmd.E_INVALID
    cfg.m = 300
    assert L.sdmd_create(ctypes.byref(cfg), ctypes.byref(h)) == sdmd.E_INVALID
    cfg.m = 10
    cfg.nranks = 2
    cfg.nccl_uid = None
    assert L.sdmd_create(ctypes.byref(cfg), ctypes.byref(h)) == sdmd.E_INVALID
    assert L.sdmd_push_dense(None, None, 0) == sdmd.E_INVALID
    assert L.sdmd_sync(None, None) == sdmd.E_INVALID


def test_row_partition_covers_rows():
    from paper_1612_07875_b200 import row_partition
    for n in (24883200, 1000, 89351):
        for P in (1, 2, 4, 8):
            spans = [row_partition(n, P, r) for r in range(P)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a < b
            if P > 1 and n >= 32 * P:
                assert all(a % 32 == 0 for a, _ in spans)


def test_binding_input_checks():
    """the binding checks dtype, length and contiguity of every input buffer
    before passing a raw pointer, converts numpy inputs it can, and returns the converted object so
    the caller keeps it alive."""
    import torch
    from paper_1612_07875_b200.sdmd import _checked
    with pytest.raises(TypeError):
        _checked(torch.zeros(10, dtype=torch.float64), np.float32, 10, "push")
    with pytest.raises(ValueError):
        _checked(torch.zeros(10, dtype=torch.float32), np.float32, 11, "push")
    with pytest.raises(ValueError):
        _checked(torch.zeros((10, 4), dtype=torch.float32)[:, 1], np.float32, 10, "push")
    a, p, where = _checked([1.0, 2.0, 3.0], np.float32, 3, "push")
    assert a.dtype == np.float32 and p.value == a.ctypes.data and where == 0
    x64 = np.arange(6.0)
    a, p, _ = _checked(x64, np.float32, 6, "push")
    assert a.dtype == np.float32 and np.array_equal(a, x64.astype(np.float32))
    # (n, k) C-ordered numpy -> Fortran copy (columns contiguous); (k, n) C-ordered kept as is
    Z = np.arange(12.0).reshape(4, 3)
    a, p, _ = _checked(Z, np.float64, 12, "init_window", n=4)
    assert a.flags.f_contiguous and np.array_equal(a, Z)
    Zt = np.ascontiguousarray(Z.T)
    a, p, _ = _checked(Zt, np.float64, 12, "init_window", n=4)
    assert a is Zt
    with pytest.raises(ValueError):
        _checked(np.zeros(5), np.float64, 6, "push")


def test_import_does_not_change_environment(monkeypatch):
    """importing the package leaves CUDA_DEVICE_MAX_CONNECTIONS alone."""
    import importlib
    import sys
    monkeypatch.delenv("CUDA_DEVICE_MAX_CONNECTIONS", raising=False)
    for k in [k for k in sys.modules if k.startswith("paper_1612_07875_b200")]:
        monkeypatch.delitem(sys.modules, k)
    importlib.import_module("paper_1612_07875_b200")
    import os
    assert "CUDA_DEVICE_MAX_CONNECTIONS" not in os.environ


def test_sparse_basis_and_grid_validation(libpath):
    """NEXT-3 config rules are enforced before any device work: the RFFT basis needs its grid
    (n_global = rows·(cols/2+1)); a sparse background needs the DCT basis, one rank and a
    power-of-two grid covering n; Fourier bases need sparse storage."""
    from paper_1612_07875_b200 import sdmd
    L = sdmd.lib()
    h = ctypes.c_void_p()

    def cfg(**kw):
        c = sdmd.Config()
        L.sdmd_config_init(ctypes.byref(c))
        c.m, c.storage, c.nnz_cap = 8, sdmd.SPARSE, 100
        c.n_local = c.n_global = 64 * 64
        for k, v in kw.items():
            setattr(c, k, v)
        return c
    bad = [
        cfg(basis=sdmd.BASIS_RFFT),                                  # no grid
        cfg(basis=sdmd.BASIS_RFFT, grid_rows=64, grid_cols=64),      # 64*33 != n
        cfg(basis=3),
        cfg(storage=sdmd.DENSE, basis=sdmd.BASIS_FFT),
        cfg(background=1),                                           # no grid
        cfg(background=1, grid_rows=64, grid_cols=64, basis=sdmd.BASIS_FFT),
        cfg(background=1, grid_rows=32, grid_cols=128, n_local=4096, n_global=4096, nranks=2),
        cfg(background=1, grid_rows=48, grid_cols=48, n_local=48 * 48, n_global=48 * 48),  # not 2^k
        cfg(grid_rows=64, grid_cols=0),
    ]
    for c in bad:
        assert L.sdmd_create(ctypes.byref(c), ctypes.byref(h)) == sdmd.E_INVALID


def _build_c_consumer(libpath, d):
    src = os.path.join(ROOT, "tests", "c_consumer", "sdmd_consumer.c")
    exe = os.path.join(d, "sdmd_consumer")
    libdir = os.path.dirname(libpath)
    subprocess.run(["gcc", "-std=c99", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", exe,
                    "-L", libdir, "-lsdmd", f"-Wl,-rpath,{libdir}", "-lm"], check=True)
    return exe


def test_c_consumer_compiles_and_validates(libpath):
    """A gcc-compiled C program (no Python) links libsdmd.so through include/sdmd.h; on a host
    without a GPU every call it makes fails cleanly with the documented status."""
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        exe = _build_c_consumer(libpath, d)
        out = subprocess.run([exe, "cpu"], capture_output=True, text=True, timeout=60)
        assert out.returncode == 0, out.stdout + out.stderr
        assert "cpu ok" in out.stdout


@pytest.mark.gpu
def test_c_consumer_streams_dmd_on_gpu(libpath):
    """The same C program streams a planted rank-2 signal through the library on the GPU and
    recovers its eigenvalue pair ρe^{±iθ} to 1e-9."""
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        exe = _build_c_consumer(libpath, d)
        out = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
        assert out.returncode == 0, out.stdout + out.stderr
