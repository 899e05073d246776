"""Thin Python binding of libsdmd (include/sdmd.h) — argument marshalling only.

Every step of the streaming SVD/DMD path runs in the CUDA library; this module only converts
torch tensors / numpy arrays to pointers and status codes to exceptions.  There is no CPU
fallback: if ``libsdmd.so`` is missing or no CUDA device is present, the calls fail loudly.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SDMD_LIB: load a variant build of the same library (kernel-tuning experiments only)
LIB_PATH = os.environ.get("SDMD_LIB") or os.path.join(_HERE, "libsdmd.so")

OK, E_INVALID, E_NONFINITE, E_WINDOW_NOT_FULL, E_ZERO_MATRIX = 0, 1, 2, 3, 4
E_NO_CONVERGENCE, W_SINGULAR, E_NO_VIABLE_MODE, E_CUDA, E_NCCL, E_OOM, E_STATE = (
    5, 6, 7, 8, 9, 10, 11)
F32, F64 = 0, 1
DENSE, SPARSE = 0, 1
BASIS_DCT, BASIS_FFT, BASIS_RFFT = 0, 1, 2
HOST, DEVICE, HOST_ASYNC, DEVICE_READY = 0, 1, 2, 3
MAX_M, MAX_R = 256, 224

# every symbol include/sdmd.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "sdmd_config_init", "sdmd_create", "sdmd_destroy", "sdmd_init_window", "sdmd_push_dense",
    "sdmd_push_sparse", "sdmd_push_batch", "sdmd_acquire_slot", "sdmd_commit_slot", "sdmd_join",
    "sdmd_sync",
    "sdmd_get_info",
    "sdmd_get_gram", "sdmd_get_partial_gram_column", "sdmd_get_svd", "sdmd_get_spectrum",
    "sdmd_get_eigvecs", "sdmd_get_modes", "sdmd_get_background", "sdmd_get_frame_diag",
    "sdmd_score_background", "sdmd_get_scores", "sdmd_get_background_window",
    "sdmd_set_timing",
    "sdmd_get_stats", "sdmd_get_timeline", "sdmd_nccl_unique_id", "sdmd_status_string", "sdmd_last_error",
    "sdmd_abi_version",
]


class Config(ctypes.Structure):
    _fields_ = [
        ("n_global", ctypes.c_int64), ("row_begin", ctypes.c_int64), ("n_local", ctypes.c_int64),
        ("m", ctypes.c_int32), ("dtype", ctypes.c_int32), ("storage", ctypes.c_int32),
        ("nnz_cap", ctypes.c_int32), ("r_max", ctypes.c_int32), ("rank_tol", ctypes.c_double),
        ("threshold", ctypes.c_float), ("background", ctypes.c_int32), ("dmd", ctypes.c_int32),
        ("workers", ctypes.c_int32), ("device", ctypes.c_int32), ("stream", ctypes.c_void_p),
        ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("nccl_uid", ctypes.c_void_p),
        ("lag", ctypes.c_int32), ("eigen_shard", ctypes.c_int32),
        ("batch_max", ctypes.c_int32), ("bg_modes", ctypes.c_int32), ("buildup", ctypes.c_int32),
        ("modes_every_frame", ctypes.c_int32), ("basis", ctypes.c_int32),
        ("grid_rows", ctypes.c_int32), ("grid_cols", ctypes.c_int32),
    ]


class Info(ctypes.Structure):
    _fields_ = [("frames", ctypes.c_int64), ("window", ctypes.c_int32), ("lag", ctypes.c_int32),
                ("ring_slots", ctypes.c_int32), ("workers", ctypes.c_int32),
                ("ring_bytes", ctypes.c_int64), ("ld", ctypes.c_int64),
                ("cluster_workers", ctypes.c_int32), ("k1_grid", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("k1_launches", ctypes.c_int64), ("k1_ms", ctypes.c_double),
                ("k4_launches", ctypes.c_int64), ("k4_ms", ctypes.c_double),
                ("gpu_launches", ctypes.c_int64), ("k1_gap_ms", ctypes.c_double),
                ("k1_wait_ms", ctypes.c_double), ("collectives", ctypes.c_int64)]


class Scores(ctypes.Structure):
    _fields_ = [("frames", ctypes.c_int64), ("tp", ctypes.c_int64), ("fp", ctypes.c_int64),
                ("fn", ctypes.c_int64), ("tn", ctypes.c_int64), ("recall", ctypes.c_double),
                ("precision", ctypes.c_double), ("f_measure", ctypes.c_double),
                ("psnr", ctypes.c_double), ("empty_gt", ctypes.c_int32),
                ("empty_mask", ctypes.c_int32)]


class SDMDError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"sdmd status {status} ({status_string(status)}): {msg}")
        self.status = status


_lib = None


def lib():
    """Load libsdmd.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not built — run `python -m paper_1612_07875_b200.build`; "
                           "the streaming DMD path has no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, dp = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
    sig = {
        "sdmd_config_init": [ctypes.POINTER(Config)],
        "sdmd_create": [ctypes.POINTER(Config), ctypes.POINTER(vp)],
        "sdmd_destroy": [vp],
        "sdmd_init_window": [vp, vp, i64, ctypes.c_int],
        "sdmd_push_dense": [vp, vp, ctypes.c_int],
        "sdmd_push_sparse": [vp, i32, vp, vp, ctypes.c_int],
        "sdmd_push_batch": [vp, i32, vp, i64, ctypes.c_int, i32],
        "sdmd_acquire_slot": [vp, ctypes.POINTER(vp)],
        "sdmd_commit_slot": [vp],
        "sdmd_join": [vp],
        "sdmd_sync": [vp, ctypes.POINTER(i64)],
        "sdmd_get_info": [vp, ctypes.POINTER(Info)],
        "sdmd_get_gram": [vp, dp, ctypes.POINTER(i32)],
        "sdmd_get_partial_gram_column": [vp, dp, ctypes.POINTER(i32)],
        "sdmd_get_svd": [vp, ctypes.POINTER(i32), dp, dp, ctypes.POINTER(i64)],
        "sdmd_get_spectrum": [vp, ctypes.POINTER(i32), dp, dp, ctypes.POINTER(i32),
                              ctypes.POINTER(i64)],
        "sdmd_get_eigvecs": [vp, dp, ctypes.POINTER(i32)],
        "sdmd_get_modes": [vp, vp, i32, vp, i64],
        "sdmd_get_background": [vp, vp, vp, vp, ctypes.POINTER(i64), ctypes.c_int],
        "sdmd_get_frame_diag": [vp, dp],
        "sdmd_score_background": [vp, i64, vp, ctypes.c_int],
        "sdmd_get_scores": [vp, ctypes.POINTER(Scores), ctypes.c_int],
        "sdmd_get_background_window": [vp, vp, vp, vp, i64, ctypes.POINTER(i64)],
        "sdmd_set_timing": [vp, ctypes.c_int],
        "sdmd_get_stats": [vp, ctypes.POINTER(Stats), ctypes.c_int],
        "sdmd_get_timeline": [vp, ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                              ctypes.POINTER(ctypes.c_int)],
        "sdmd_nccl_unique_id": [vp],
        "sdmd_status_string": [ctypes.c_int],
        "sdmd_last_error": [vp],
        "sdmd_abi_version": [],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_char_p if name in ("sdmd_status_string", "sdmd_last_error") \
            else ctypes.c_int
    _lib = L
    return L


def status_string(st: int) -> str:
    try:
        return lib().sdmd_status_string(st).decode()
    except Exception:
        return str(st)


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    st = lib().sdmd_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p))
    if st:
        raise SDMDError(st, "nccl unique id")
    return bytes(buf)


def _ptr(a):
    """(pointer, where) of a torch tensor or numpy array (no copies are made here)."""
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr()), (DEVICE if a.is_cuda else HOST)
    a = np.asarray(a)
    return ctypes.c_void_p(a.ctypes.data), HOST


_TORCH_NP = {"torch.float32": np.float32, "torch.float64": np.float64, "torch.int32": np.int32}


def _checked(a, np_dtype, count: int, what: str, n: int | None = None):
    """(obj, pointer, where) of an input buffer after checking that it holds at least ``count``
    elements of ``np_dtype`` contiguously (the library reads raw memory).  Torch tensors must be
    contiguous with the exact dtype; numpy arrays (or lists) of another dtype or layout are
    converted here, and the converted object is returned so that the caller keeps it alive until
    the (possibly asynchronous) copy has run."""
    if hasattr(a, "data_ptr"):
        dt = _TORCH_NP.get(str(a.dtype))
        if dt is not np_dtype:
            raise TypeError(f"{what}: tensor dtype {a.dtype} does not match the engine dtype "
                            f"{np.dtype(np_dtype).name}")
        if not a.is_contiguous():
            raise ValueError(f"{what}: tensor must be contiguous (pass .contiguous())")
        if a.numel() < count:
            raise ValueError(f"{what}: {a.numel()} elements, need {count}")
        return a, ctypes.c_void_p(a.data_ptr()), (DEVICE if a.is_cuda else HOST)
    arr = np.asarray(a)
    if arr.ndim <= 1:
        if arr.dtype != np_dtype or not arr.flags.c_contiguous:
            arr = np.ascontiguousarray(arr, dtype=np_dtype)
    elif n is not None and arr.ndim == 2 and arr.shape[0] == n and arr.shape[1] != n:
        if arr.dtype != np_dtype or not arr.flags.f_contiguous:
            arr = np.asfortranarray(arr, dtype=np_dtype)        # (n, k): columns contiguous
    elif arr.dtype != np_dtype or not arr.flags.c_contiguous:
        arr = np.ascontiguousarray(arr, dtype=np_dtype)         # (k, n): rows contiguous
    if arr.size < count:
        raise ValueError(f"{what}: {arr.size} elements, need {count}")
    return arr, ctypes.c_void_p(arr.ctypes.data), HOST


def _dp(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


class StreamingDMD:
    """Streaming method-of-snapshots SVD / DMD / background subtraction on one GPU (or one row
    shard).  Mirrors the C ABI one-to-one; see include/sdmd.h for semantics."""

    def __init__(self, n: int, m: int, dtype: str = "f32", storage: str = "dense",
                 nnz_cap: int = 0, r_max: int = 0, rank_tol: float = 1e-7,
                 threshold: float = 0.2, background: bool = False, dmd: bool = True,
                 workers: int = 4, device: int = 0, stream="torch", rank: int = 0,
                 nranks: int = 1, row_begin: int = 0, n_global: int | None = None,
                 nccl_uid: bytes | None = None, lag: int = 0, eigen_shard: int = 1,
                 batch_max: int = 0, bg_modes: int = 0, buildup: bool = False,
                 modes_every_frame: bool = False, basis: str = "dct", grid=None):
        L = lib()
        cfg = Config()
        L.sdmd_config_init(ctypes.byref(cfg))
        cfg.n_local = int(n)
        cfg.row_begin = int(row_begin)
        cfg.n_global = int(n_global if n_global is not None else row_begin + n)
        cfg.m = int(m)
        cfg.dtype = F32 if dtype in ("f32", "float32") else F64
        cfg.storage = SPARSE if storage == "sparse" else DENSE
        cfg.nnz_cap = int(nnz_cap)
        cfg.r_max = int(r_max)
        cfg.rank_tol = float(rank_tol)
        cfg.threshold = float(threshold)
        cfg.background = 1 if background else 0
        cfg.dmd = 1 if dmd else 0
        cfg.workers = int(workers)
        cfg.device = int(device)
        if isinstance(stream, str) and stream == "torch":
            # order library work after the caller's torch stream (device inputs are read in
            # stream order); torch's legacy default stream (handle 0) maps to cudaStreamLegacy
            import torch
            s = int(torch.cuda.current_stream(int(device)).cuda_stream)
            stream = s if s != 0 else 1
        elif stream is not None and hasattr(stream, "cuda_stream"):
            stream = int(stream.cuda_stream) or 1
        cfg.stream = ctypes.c_void_p(int(stream)) if stream is not None else None
        cfg.rank = int(rank)
        cfg.nranks = int(nranks)
        cfg.lag = int(lag)
        cfg.eigen_shard = int(eigen_shard)
        cfg.batch_max = int(batch_max)
        cfg.bg_modes = int(bg_modes)
        cfg.buildup = 1 if buildup else 0
        cfg.modes_every_frame = 1 if modes_every_frame else 0
        cfg.basis = {"dct": BASIS_DCT, "fft": BASIS_FFT, "rfft": BASIS_RFFT}[basis]
        if grid is not None:
            cfg.grid_rows, cfg.grid_cols = int(grid[0]), int(grid[1])
        self._uid = None
        if nccl_uid is not None:
            self._uid = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_uid)
            cfg.nccl_uid = ctypes.cast(self._uid, ctypes.c_void_p)
        self.cfg = cfg
        self.n, self.m = int(n), int(m)
        self.np_dtype = np.float32 if cfg.dtype == F32 else np.float64
        # background outputs: the dense storage dtype; fp64 pixels for a sparse (DCT) context
        self.out_dtype = np.float64 if cfg.storage == SPARSE else self.np_dtype
        # inputs of recent pushes stay referenced until the library no longer reads them (pinned
        # host buffers are copied asynchronously; the ring guard bounds how far the host runs
        # ahead, so 64 pushes is ample); sync() drops them
        import collections
        self._pending = collections.deque(maxlen=64)
        h = ctypes.c_void_p()
        st = L.sdmd_create(ctypes.byref(cfg), ctypes.byref(h))
        if st:
            raise SDMDError(st, "sdmd_create")
        self.h = h

    # ----------------------------------------------------------------------------------
    def _check(self, st, what, ok=(OK,)):
        if st not in ok:
            msg = lib().sdmd_last_error(self.h).decode() if self.h else ""
            raise SDMDError(st, f"{what}: {msg}")
        return st

    def close(self):
        if getattr(self, "h", None):
            lib().sdmd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---------------------------------------------------------------- ingest ----------
    def init_window(self, Z, ldz: int | None = None):
        """Z: (m+1) columns of n values, column-major (a torch (m+1, n) row-major tensor or an
        (n, m+1) Fortran array both work; pass ldz for padded layouts)."""
        if ldz is None:
            ldz = self.n
        Z, p, where = _checked(Z, self.np_dtype, int(ldz) * self.m + self.n, "init_window", self.n)
        self._pending.append(Z)
        return self._check(lib().sdmd_init_window(self.h, p, int(ldz), where), "init_window")

    def push_batch(self, X, dmd_every: bool = True, ldx: int | None = None):
        """k snapshots at once (K1b): a torch (k, n) row-major tensor / (n, k) Fortran array, oldest
        first.  dmd_every=False runs the DMD only for the newest window (catch-up mode)."""
        k = int(X.shape[0]) if hasattr(X, "data_ptr") else int(np.asarray(X).shape[1])
        ld = int(ldx or self.n)
        X, p, where = _checked(X, self.np_dtype, ld * (k - 1) + self.n, "push_batch", self.n)
        self._pending.append(X)
        return self._check(lib().sdmd_push_batch(self.h, k, p, ld, where,
                                                 1 if dmd_every else 0), "push_batch")

    def push(self, x, ready: bool = False):
        """One dense snapshot.  ready=True (CUDA tensors): the tensor's contents are complete now
        (SDMD_DEVICE_READY: copied on the copy stream, overlapping the previous Gram pass)."""
        x, p, where = _checked(x, self.np_dtype, self.n, "push")
        if ready and where == DEVICE:
            where = DEVICE_READY
        self._pending.append(x)
        return self._check(lib().sdmd_push_dense(self.h, p, where), "push_dense")

    def push_sparse(self, idx, val):
        """nnz (index, value) pairs; values fp64 (DCT basis) or complex128 (Fourier bases: numpy
        complex128 arrays, or torch float64 tensors holding 2·nnz interleaved doubles)."""
        nnz = int(idx.shape[0]) if hasattr(idx, "shape") else len(idx)
        idx, pi, wi = _checked(idx, np.int32, nnz, "push_sparse idx")
        vs = 2 if self.cfg.basis != BASIS_DCT else 1
        if vs == 2 and not hasattr(val, "data_ptr"):
            val = np.ascontiguousarray(np.asarray(val, dtype=np.complex128)).view(np.float64)
        val, pv, wv = _checked(val, np.float64, vs * nnz, "push_sparse val")
        if wi != wv:
            raise ValueError("push_sparse: idx and val must both be host or both be device buffers")
        self._pending.append((idx, val))
        return self._check(lib().sdmd_push_sparse(self.h, nnz, pi, pv, wi), "push_sparse")

    def acquire_slot(self) -> int:
        p = ctypes.c_void_p()
        self._check(lib().sdmd_acquire_slot(self.h, ctypes.byref(p)), "acquire_slot")
        return int(p.value)

    def commit_slot(self):
        return self._check(lib().sdmd_commit_slot(self.h), "commit_slot")

    def join(self):
        """Device-side join of the eigen workers into the ctx stream (no host wait)."""
        return self._check(lib().sdmd_join(self.h), "join")

    def background_async(self, mask=None, lowrank=None, sparse=None):
        """Asynchronous D2H of the newest enqueued background outputs into pinned host tensors
        (valid after sync(), or after join() on the ctx stream); returns their frame index."""
        p = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        fr = ctypes.c_int64(-1)
        self._check(lib().sdmd_get_background(self.h, p(lowrank), p(sparse), p(mask),
                                               ctypes.byref(fr), HOST_ASYNC), "get_background")
        return int(fr.value)

    def sync(self) -> int:
        """Wait for all work; returns -1, or raises SDMDError(E_NONFINITE) with .failed_frame."""
        f = ctypes.c_int64(-1)
        st = lib().sdmd_sync(self.h, ctypes.byref(f))
        self._pending.clear()
        if st:
            e = SDMDError(st, lib().sdmd_last_error(self.h).decode())
            e.failed_frame = int(f.value)
            raise e
        return -1

    # ---------------------------------------------------------------- getters ---------
    def info(self) -> dict:
        i = Info()
        self._check(lib().sdmd_get_info(self.h, ctypes.byref(i)), "get_info")
        return {k: getattr(i, k) for k, _ in Info._fields_}

    def gram(self) -> np.ndarray:
        k = self.m + 1
        G = np.zeros((k, k), dtype=np.float64, order="F")
        kk = ctypes.c_int32()
        self._check(lib().sdmd_get_gram(self.h, _dp(G), ctypes.byref(kk)), "get_gram")
        kk = kk.value
        return np.asfortranarray(G.ravel(order="F")[: kk * kk].reshape((kk, kk), order="F"))

    def partial_gram_column(self) -> np.ndarray:
        g = np.zeros(self.m + 1, dtype=np.float64)
        kk = ctypes.c_int32()
        self._check(lib().sdmd_get_partial_gram_column(self.h, _dp(g), ctypes.byref(kk)),
                    "get_partial_gram_column")
        return g[: kk.value]

    def svd(self, with_V: bool = True):
        m = self.m
        sigma = np.zeros(m, dtype=np.float64)
        V = np.zeros((m, MAX_R), dtype=np.float64, order="F") if with_V else None
        r = ctypes.c_int32()
        fr = ctypes.c_int64()
        st = lib().sdmd_get_svd(self.h, ctypes.byref(r), _dp(sigma),
                                _dp(V) if with_V else None, ctypes.byref(fr))
        self._check(st, "get_svd", ok=(OK, E_NO_CONVERGENCE))
        rr = r.value
        if with_V:
            V = V.ravel(order="F")[: m * rr].reshape((m, rr), order="F")
        return dict(sigma=sigma, V=V, r=rr, frame=fr.value, status=st)

    def spectrum(self, with_b: bool = False) -> dict:
        lam = np.zeros(2 * MAX_R, dtype=np.float64)
        b = np.zeros(2 * MAX_R, dtype=np.float64) if with_b else None
        r = ctypes.c_int32()
        idx = ctypes.c_int32()
        fr = ctypes.c_int64()
        st = lib().sdmd_get_spectrum(self.h, ctypes.byref(r), _dp(lam),
                                     _dp(b) if with_b else None, ctypes.byref(idx),
                                     ctypes.byref(fr))
        self._check(st, "get_spectrum", ok=(OK, E_NO_CONVERGENCE, W_SINGULAR, E_NO_VIABLE_MODE))
        rr = r.value
        out = dict(r=rr, idx=idx.value, frame=fr.value, status=st,
                   lam=lam[: 2 * rr].view(np.complex128).copy())
        if with_b:
            out["b"] = b[: 2 * rr].view(np.complex128).copy()
        return out

    def eigvecs(self) -> np.ndarray:
        W = np.zeros(2 * MAX_R * MAX_R, dtype=np.float64)
        r = ctypes.c_int32()
        self._check(lib().sdmd_get_eigvecs(self.h, _dp(W), ctypes.byref(r)), "get_eigvecs")
        rr = r.value
        return W[: 2 * rr * rr].view(np.complex128).reshape((rr, rr), order="F").copy()

    def modes(self, cols, out=None):
        """Φ[:, cols] for this rank's rows as a torch complex128 CUDA tensor (n, len(cols))."""
        import torch
        cols = np.ascontiguousarray(np.asarray(cols, dtype=np.int32))
        nc = int(cols.size)
        if out is None:
            out = torch.empty((nc, self.n), dtype=torch.complex128,
                              device=f"cuda:{self.cfg.device}")
        self._check(lib().sdmd_get_modes(self.h, _dp(cols), nc, ctypes.c_void_p(out.data_ptr()),
                                         self.n), "get_modes")
        return out.T

    def background(self):
        """(lowrank, sparse, mask, frame) as numpy arrays (host copy)."""
        low = np.zeros(self.n, dtype=self.out_dtype)
        sp = np.zeros(self.n, dtype=self.out_dtype)
        mask = np.zeros(self.n, dtype=np.uint8)
        fr = ctypes.c_int64(-1)
        self._check(lib().sdmd_get_background(self.h, _dp(low), _dp(sp), _dp(mask),
                                               ctypes.byref(fr), HOST), "get_background")
        return low, sp, mask.astype(bool), fr.value

    def background_device(self, lowrank=None, sparse=None, mask=None) -> int:
        fr = ctypes.c_int64(-1)
        p = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        self._check(lib().sdmd_get_background(self.h, p(lowrank), p(sparse), p(mask),
                                               ctypes.byref(fr), DEVICE), "get_background")
        return fr.value

    def background_window(self):
        """Alg 3 first-window branch on the newest DMD window: (lowrank, sparse, mask, frame) as
        torch CUDA tensors of shape (m+1, n) — row e is window column e (exponent e)."""
        import torch
        dt = torch.float32 if self.cfg.dtype == F32 else torch.float64
        dev = f"cuda:{self.cfg.device}"
        low = torch.empty((self.m + 1, self.n), dtype=dt, device=dev)
        sp = torch.empty_like(low)
        mask = torch.empty((self.m + 1, self.n), dtype=torch.uint8, device=dev)
        fr = ctypes.c_int64(-1)
        self._check(lib().sdmd_get_background_window(self.h, ctypes.c_void_p(low.data_ptr()),
                                                     ctypes.c_void_p(sp.data_ptr()),
                                                     ctypes.c_void_p(mask.data_ptr()), self.n,
                                                     ctypes.byref(fr)),
                    "get_background_window", ok=(OK, W_SINGULAR))
        return low, sp, mask.bool(), int(fr.value)

    def score(self, frame: int, gt):
        """Accumulate TP/FP/FN of the newest background mask (frame ``frame``) against the ground
        truth ``gt`` (n bytes, nonzero = foreground; numpy host array or torch CUDA uint8)."""
        if hasattr(gt, "data_ptr"):
            if gt.numel() < self.n or str(gt.dtype) not in ("torch.uint8", "torch.bool") \
                    or not gt.is_contiguous():
                raise ValueError("score: gt must be a contiguous tensor of n uint8/bool values")
            g, p, where = gt, ctypes.c_void_p(gt.data_ptr()), (DEVICE if gt.is_cuda else HOST)
        else:
            g = np.ascontiguousarray(np.asarray(gt).astype(np.uint8).ravel())
            if g.size < self.n:
                raise ValueError("score: gt must hold n values")
            p, where = ctypes.c_void_p(g.ctypes.data), HOST
        self._pending.append(g)
        return self._check(lib().sdmd_score_background(self.h, int(frame), p, where), "score_background")

    def scores(self, reset: bool = False) -> dict:
        o = Scores()
        self._check(lib().sdmd_get_scores(self.h, ctypes.byref(o), 1 if reset else 0), "get_scores")
        d = {k: getattr(o, k) for k, _ in Scores._fields_}
        d["empty_gt"], d["empty_mask"] = bool(d["empty_gt"]), bool(d["empty_mask"])
        return d

    def frame_diag(self) -> dict:
        o = np.zeros(24, dtype=np.int64)
        self._check(lib().sdmd_get_frame_diag(self.h, _dp(o)), "get_frame_diag")
        names = ["build_S", "jacobi", "sort_V", "atilde", "hessenberg", "qr", "eigvec_c"]
        return dict(frame=int(o[0]), status=int(o[1]), r=int(o[2]), idx=int(o[3]),
                    sweeps=int(o[4]), qr_its=int(o[5]),
                    cycles={k: int(v) for k, v in zip(names, o[6:13])},
                    qr_steps=int(o[13]), ms_steps=int(o[14]), ms_sweeps=int(o[15]),
                    ms_shift_cycles=int(o[16]), qr_block_its=int(o[17]),
                    ms_chase_ab_cycles=int(o[18]), ms_chase_c_cycles=int(o[19]),
                    aberth_its=int(o[20]), aberth_evals=int(o[21]), commit_wait=int(o[22]))

    def set_timing(self, on: bool = True):
        return self._check(lib().sdmd_set_timing(self.h, 1 if on else 0), "set_timing")

    def stats(self, reset: bool = False) -> dict:
        s = Stats()
        self._check(lib().sdmd_get_stats(self.h, ctypes.byref(s), 1 if reset else 0), "get_stats")
        return {k: getattr(s, k) for k, _ in Stats._fields_}

    def timeline(self) -> np.ndarray:
        """Device timeline since the last stats reset: rows {frame, kind, start_ms, end_ms}, kind
        0 = Gram pass, 1 = K4a, 2 = K4b, 3 = wait for background coefficients."""
        n = ctypes.c_int(0)
        self._check(lib().sdmd_get_timeline(self.h, None, 0, ctypes.byref(n)), "get_timeline")
        out = np.zeros((max(n.value, 1), 4), dtype=np.float64)
        self._check(lib().sdmd_get_timeline(self.h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                            n.value, ctypes.byref(n)), "get_timeline")
        return out[:n.value]


def row_partition(n: int, nranks: int, rank: int, align: int = 32) -> tuple[int, int]:
    """Contiguous row slice [begin, end) of rank ``rank``: equal shares rounded to
    ``align``-element boundaries, the remainder on the last rank."""
    if nranks < 1 or not (0 <= rank < nranks):
        raise ValueError("bad rank/nranks")
    base = n // nranks
    base = (base // align) * align if base >= align else base
    b = rank * base
    e = n if rank == nranks - 1 else (rank + 1) * base
    return b, e
