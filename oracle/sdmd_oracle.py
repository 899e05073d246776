"""ORACLE — test infrastructure, NOT part of the product.

Plain, slow, fp64 CPU implementation of the streaming method-of-snapshots SVD / DMD /
background-subtraction path of arXiv 1612.07875 (reference: /root/reference/PAPER.md, cited as
P:<line>; SPEC.md as S:<line>).  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this module.  It shares no
code with the CUDA path (``paper_1612_07875_b200/``) and never imports it.

The arithmetic lives in ``oracle/csrc/sdmd_oracle.c`` (C99, explicit loops, no BLAS/LAPACK),
called here through ctypes; this module holds the step order of the paper's Algorithms 1-3 and the
conventions (sorting, normalisation, index rules).  Steps follow SURVEY.md §8(c) O1-O13:
  O1  Gram: Neumaier-compensated fp64 row-order sums of exact products      (C: orc_gram/orc_dots)
  O3  symmetric eig of S: cyclic-by-row Jacobi, stable rotation            (C: orc_jacobi)
  O6  eig(Ã): Householder-Hessenberg + Francis double-shift QR + back-substitution
                                                                           (C: orc_eig_real)
  O7  modes Φ = X'(Y W): compensated complex accumulation                  (C: orc_modes)
  O9  b = (WΛ)⁻¹α₁: complex Gaussian elimination with partial pivoting;
      singular fallback: complex column-pivoted Householder least squares  (C: orc_csolve/clstsq)
Small dense products (Ã = Yᵀ G_xy Y, T = Y W, the O(r) sums) use numpy matmul as a library
primitive, as the paper's own pseudo-code does ("*" products, Alg 2).  Readings where
the paper is ambiguous or garbled are DESIGN.md §3; each is cited
as Qk/Rk where used.

Pins (tests/test_oracle.py, ``-m "not gpu"``): closed-form planted spectra, worked examples from
SPEC.md (cited), exact-rational brute force on tiny inputs, streamed == batch, Gram slice
identities, invariance under orthonormal transforms, Eckart-Young, eigenvalue equivalence with
the full operator X' pinv(X), LAPACK (numpy.linalg, test side only — independent of this
module now) on tiny inputs, the singular-amplitude branch on a planted zero eigenvalue, the
first-window background on a constant video, and the Q12 order on hand-built spectra.

Parity unpinned: eigenvalues of Ã for noisy video windows with r ≈ m have no closed form;
they are checked only GPU-vs-oracle within κ(λ)·‖ΔÃ‖ (DESIGN.md §"Parity").
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

# ----------------------------------------------------------------------------------------
# status codes (values of include/sdmd.h redefined here: no shared code)
# ----------------------------------------------------------------------------------------
OK, E_INVALID, E_NONFINITE, E_WINDOW_NOT_FULL, E_ZERO_MATRIX = 0, 1, 2, 3, 4
E_NO_CONVERGENCE, W_SINGULAR, E_NO_VIABLE_MODE = 5, 6, 7

THREADS = int(os.environ.get("ORACLE_THREADS", "0"))   # 0: all host cores (row-chunk sums)


class OracleError(Exception):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"status {code}: {msg}")
        self.code = code


_clib = None


def clib():
    """The oracle's C library (built on first use with gcc; see oracle/build.py)."""
    global _clib
    if _clib is None:
        from oracle.build import build
        L = ctypes.CDLL(build())
        vp, i32, i64, dp = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
        L.orc_dots.argtypes = [vp, i64, i32, vp, i64, i32, i32, dp]
        L.orc_dots.restype = None
        L.orc_gram.argtypes = [vp, i64, i32, i64, i32, i32, dp]
        L.orc_gram.restype = None
        L.orc_jacobi.argtypes = [i32, dp, dp, dp, i32, ctypes.POINTER(ctypes.c_int)]
        L.orc_jacobi.restype = ctypes.c_int
        L.orc_eig_real.argtypes = [i32, dp, dp, dp, dp, dp, ctypes.POINTER(ctypes.c_int)]
        L.orc_eig_real.restype = ctypes.c_int
        L.orc_csolve.argtypes = [i32, dp, dp, dp]
        L.orc_csolve.restype = ctypes.c_int
        L.orc_clstsq.argtypes = [i32, i32, dp, dp, dp]
        L.orc_clstsq.restype = ctypes.c_int
        L.orc_modes.argtypes = [vp, i64, i32, i64, i32, dp, i32, dp, i64, i32]
        L.orc_modes.restype = None
        _clib = L
    return _clib


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _real_cols(cols) -> tuple[np.ndarray, int]:
    """Columns as one Fortran-ordered (n, k) array of float32 (dtype 0) or float64 (dtype 1); fp32
    inputs stay fp32 (promoted exactly inside the C sums, Q9)."""
    arrs = [np.asarray(c) for c in cols]
    if all(a.dtype == np.float32 for a in arrs):
        return np.asfortranarray(np.stack(arrs, axis=1)), 0
    return np.asfortranarray(np.stack([a.astype(np.float64) for a in arrs], axis=1)), 1


# ----------------------------------------------------------------------------------------
# O1  Gram matrix  (Alg 1 first branch "xtx = X.T * X"; §3.1)
# ----------------------------------------------------------------------------------------

def gram(Z) -> np.ndarray:
    """G = Zᵀ Z of the full window Z = [z_0 .. z_m] (n x (m+1)), fp64.

    Alg 1 P:291 ("xtx = X.T * X") applied to the full window (reading Q2: the full-window Gram
    holds both XᵀX = G[0:m,0:m] and XᵀX' = G[0:m,1:m+1]).  Every entry is the Neumaier-
    compensated sum over the rows in increasing order of the exact products (fp32 inputs are
    promoted exactly, Q9; fp64 products carry their fma rounding error)."""
    Z = np.asarray(Z)
    if Z.ndim == 1:
        Z = Z[:, None]
    Zf, dt = _real_cols([Z[:, j] for j in range(Z.shape[1])]) if Z.shape[1] else (Z, 1)
    n, k = Zf.shape
    G = np.zeros((k, k), dtype=np.float64)
    if k:
        clib().orc_gram(_p(Zf), n, k, n, dt, THREADS, _p(G))
    return G


def gram_column(cols, x_new) -> np.ndarray:
    """g_k = <z_k, x_new> for each window column z_k (pass x_new itself last for the self-dot).

    Alg 1 else-branch P:294 ("xtx[:, -1] = X.T * X[:, -1]"); §3.1 P:236 ("only the last row or
    column will need to be recalculated").  Compensated row-order dots (O1)."""
    A, dt = _real_cols(list(cols) + [x_new])
    n, k = A.shape[0], A.shape[1] - 1
    x = np.ascontiguousarray(A[:, -1])
    out = np.zeros(max(k, 1), dtype=np.float64)
    if k:
        clib().orc_dots(_p(A), n, k, _p(x), n, dt, THREADS, _p(out))
    return out[:k]


def sparse_gram_column(slots, x_new, n: int) -> np.ndarray:
    """Sparse variant (§3.5): each snapshot is (idx, val) in an orthonormal coefficient
    basis; g_k is the dot of the *scattered* dense vectors (definition)."""
    def dense(sv):
        idx, val = sv
        d = np.zeros(n, dtype=np.float64)
        d[np.asarray(idx, dtype=np.int64)] = np.asarray(val, dtype=np.float64)
        return d
    return gram_column([dense(s) for s in slots], dense(x_new))


def sparse_window_on_support(slots) -> np.ndarray:
    """The sparse snapshots ``slots`` [(idx, val), ...] scattered onto the union of their supports
    (ascending coefficient index): an (n_support, k) fp64 array whose Gram equals the Gram of the
    scattered dense n-vectors exactly — the omitted rows are zero in every column, and an exact
    zero product leaves the compensated row-order sum (O1) unchanged bit for bit.  Lets the
    oracle evaluate the definition at C5 size (n = 1024², ~1% nonzeros)."""
    sup = np.unique(np.concatenate([np.asarray(i, dtype=np.int64) for i, _ in slots]))
    Z = np.zeros((sup.size, len(slots)), dtype=np.float64, order="F")
    for k, (i, v) in enumerate(slots):
        Z[np.searchsorted(sup, np.asarray(i, dtype=np.int64)), k] = np.asarray(v, dtype=np.float64)
    return Z


class StreamingGram:
    """Sliding-window Gram state (Alg 1 else-branch P:293-295, on the full window, Q2).

    Warm-up: while fewer than m+1 columns are held, push appends a column and extends G (Q14,
    P:496-498).  Full: push drops the oldest column, keeps G[1:,1:] (copied, not
    recomputed) and computes the new last row/column.  A frame whose Gram column is
    not finite is rejected and the state is left unchanged."""

    def __init__(self, m: int):
        self.m = m
        self.cols: list[np.ndarray] = []
        self.G = np.zeros((0, 0))
        self.fresh_dots = 0          # instrumentation: fresh length-n inner products

    @property
    def full(self) -> bool:
        return len(self.cols) == self.m + 1

    def push(self, x) -> None:
        x = np.asarray(x)
        x = (x.astype(np.float32) if x.dtype == np.float32 else x.astype(np.float64)).copy()
        if self.full:
            keep = self.cols[1:]
            Gk = self.G[1:, 1:]                       # "xtx[:-1, :-1] = xtx[1:, 1:]"
        else:
            keep = self.cols
            Gk = self.G
        g = gram_column(keep + [x], x)                 # "xtx[:, -1] = X.T * X[:, -1]"
        if not np.all(np.isfinite(g)):
            raise OracleError(E_NONFINITE, "non-finite frame rejected; state unchanged")
        self.fresh_dots += len(g)
        k = len(keep)
        G = np.zeros((k + 1, k + 1))
        G[:k, :k] = Gk
        G[:, k] = g
        G[k, :] = g                                    # "xtx[-1, :] = xtx[:, -1].T"
        self.cols = keep + [x]
        self.G = G


# ----------------------------------------------------------------------------------------
# O3–O4  Method-of-snapshots SVD from the Gram  (§2.1; Alg 1)
# ----------------------------------------------------------------------------------------

def jacobi_eigh(S, max_sweeps: int = 60):
    """(μ, V, sweeps) of the symmetric S by cyclic-by-row Jacobi (O3; C orc_jacobi): "s, v =
    eig(xtx)" (Alg 1).  μ unsorted, V[:, j] the eigenvector of μ_j.  Raises
    E_NO_CONVERGENCE after max_sweeps sweeps."""
    S = np.ascontiguousarray(np.asarray(S, dtype=np.float64))
    m = S.shape[0]
    mu = np.zeros(m)
    V = np.zeros((m, m), order="F")
    sw = ctypes.c_int(0)
    st = clib().orc_jacobi(m, _p(S), _p(mu), _p(V), int(max_sweeps), ctypes.byref(sw))
    if st:
        raise OracleError(E_NO_CONVERGENCE, f"Jacobi: no convergence in {max_sweeps} sweeps")
    return mu, V, sw.value


def _sign_normalize_real(V: np.ndarray) -> np.ndarray:
    """Q6: make each column's largest-|.| entry positive (first such entry on ties)."""
    V = V.copy()
    for j in range(V.shape[1]):
        i = int(np.argmax(np.abs(V[:, j])))
        if V[i, j] < 0:
            V[:, j] = -V[:, j]
    return V


def svd_from_gram(S, rank_tol: float = 1e-7, r_max: int | None = None):
    """σ, V, r of X from S = XᵀX.

    "s, v = eig(xtx)" (Alg 1; cyclic Jacobi, O3), "sigma = sort(sqrt(abs(s)), 'desc')"
     with V permuted alike (Q6), r = min(r_max, #{σ_i > rank_tol·σ_1}) (Q7).  Raises
    E_ZERO_MATRIX if σ_1 == 0."""
    mu, V, _ = jacobi_eigh(S)
    sigma = np.sqrt(np.abs(mu))
    order = sorted(range(len(sigma)), key=lambda i: (-sigma[i], i))   # stable descending
    sigma = sigma[order]
    V = _sign_normalize_real(V[:, order])
    if sigma.size == 0 or sigma[0] == 0.0:
        raise OracleError(E_ZERO_MATRIX, "sigma_1 == 0")
    r = int(np.count_nonzero(sigma > rank_tol * sigma[0]))
    if r_max is not None:
        r = min(r, int(r_max))
    return sigma, V, r


def left_singular(X, sigma, V, r: int) -> np.ndarray:
    """U = X V Σ⁻¹ (§2.1 Eq. P:95).  Tests only: the paper never forms U."""
    return np.asarray(X, dtype=np.float64) @ (V[:, :r] / sigma[:r])


# ----------------------------------------------------------------------------------------
# O5–O6  Projected operator and its eigendecomposition  (Eq. Atilde; Alg 2)
# ----------------------------------------------------------------------------------------

def eig_real(A):
    """(λ, W) of the real square A (O6; C orc_eig_real): Householder-Hessenberg, Francis double-
    shift QR to real Schur form, eigenvectors by back-substitution ("lambda, w = eig(atilde)",
    Alg 2).  Unordered, unnormalised.  Raises E_NO_CONVERGENCE past 100 r iterations."""
    A = np.ascontiguousarray(np.asarray(A, dtype=np.float64))
    r = A.shape[0]
    wr, wi = np.zeros(r), np.zeros(r)
    Wr, Wi = np.zeros((r, r), order="F"), np.zeros((r, r), order="F")
    its = ctypes.c_int(0)
    st = clib().orc_eig_real(r, _p(A), _p(wr), _p(wi), _p(Wr), _p(Wi), ctypes.byref(its))
    if st:
        raise OracleError(E_NO_CONVERGENCE, "Francis QR: no convergence")
    return wr + 1j * wi, Wr + 1j * Wi


def order_eigs(lam: np.ndarray) -> np.ndarray:
    """Q12: |λ| descending, then Re descending, then Im descending (stable)."""
    keys = [(-abs(l), -l.real, -l.imag, i) for i, l in enumerate(lam)]
    return np.array([k[3] for k in sorted(keys)], dtype=np.int64)


def normalize_eigvecs(W: np.ndarray) -> np.ndarray:
    """Q12: unit 2-norm columns, largest-|.| entry made real positive."""
    W = np.asarray(W, dtype=np.complex128).copy()
    for j in range(W.shape[1]):
        w = W[:, j]
        w = w / np.sqrt(np.sum(np.abs(w) ** 2))
        i = int(np.argmax(np.abs(w)))
        w = w * (np.conj(w[i]) / abs(w[i]))
        W[:, j] = w
    return W


def dmd_from_gram(G, rank_tol: float = 1e-7, r_max: int | None = None) -> dict:
    """Streaming DMD from the full-window Gram (Alg 2 P:308-316 with reading Q2).

    sigma, v from SSVD of X = window[:, :-1] ("SSVD(X[:, :-1])") → S = G[0:m,0:m];
    xty = XᵀX' = G[0:m,1:m+1] ("xty[:, :-1] = xtx[:, 1:]; xty[:, -1] = X[:, :-1].T*X[:, -1]",
    P:310-311); vsi = v Σ⁻¹; atilde = vsiᵀ xty vsi; lambda, w = eig(atilde)
    (P:314)."""
    G = np.asarray(G, dtype=np.float64)
    m = G.shape[0] - 1
    S = G[:m, :m]
    xty = G[:m, 1:m + 1]
    sigma, V, r = svd_from_gram(S, rank_tol, r_max)
    vsi = V[:, :r] / sigma[:r]
    atilde = vsi.T @ xty @ vsi
    lam, W = eig_real(atilde)
    o = order_eigs(lam)
    lam = lam[o]
    W = normalize_eigvecs(W[:, o])
    return dict(m=m, r=r, sigma=sigma, V=V, vsi=vsi, atilde=atilde, lam=lam, W=W, S=S,
                xty=xty)


# ----------------------------------------------------------------------------------------
# O8–O10  Amplitudes and background mode  (§3.3; Alg 3)
# ----------------------------------------------------------------------------------------

def csolve(A, b):
    """x = A⁻¹b (complex, Gaussian elimination with partial pivoting, C orc_csolve); None if a
    pivot is numerically zero."""
    A = np.asfortranarray(np.asarray(A, dtype=np.complex128))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.complex128))
    x = np.zeros(A.shape[0], dtype=np.complex128)
    st = clib().orc_csolve(A.shape[0], _p(A), _p(b), _p(x))
    return None if st else x


def clstsq(A, b):
    """(x, rank): least squares min‖Ax − b‖ by complex Householder QR with column pivoting (C
    orc_clstsq); columns beyond the numerical rank get x = 0."""
    A = np.asfortranarray(np.asarray(A, dtype=np.complex128))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.complex128))
    x = np.zeros(A.shape[1], dtype=np.complex128)
    rk = clib().orc_clstsq(A.shape[0], A.shape[1], _p(A), _p(b), _p(x))
    return x, rk


def amplitudes(d: dict, rank_tol: float = 1e-7) -> tuple[np.ndarray, int]:
    """b = (WΛ)⁻¹ α₁ with α₁ = POD coefficients of x₁ = σ ⊙ V[0, :r] (Q3).

    "alpha1 = sigma * v[:, 0].T; wl = w * lambda; b = lstsq(wl, alpha1)" (Alg 3), §3.3
    P:268.  Reading Q15 (SPEC S:272, S:296 design decision): WΛ is singular when some
    |λ_j| < rank_tol·max|λ| (or elimination meets a zero pivot); those modes are excluded and get
    b = 0, the others are the least-squares solution of the kept columns (min-norm for full column
    rank), and the status is W_SINGULAR.  Otherwise b is the square solve, status OK."""
    r = d["r"]
    alpha1 = (d["sigma"][:r] * d["V"][0, :r]).astype(np.complex128)
    lam, W = d["lam"], d["W"]
    wl = W * lam[None, :]
    amax = float(np.max(np.abs(lam))) if len(lam) else 0.0
    keep = np.abs(lam) >= rank_tol * amax if amax > 0 else np.zeros(len(lam), dtype=bool)
    if keep.all():
        b = csolve(wl, alpha1)
        if b is not None:
            return b, OK
    b = np.zeros(len(lam), dtype=np.complex128)
    if keep.any():
        b[keep] = clstsq(wl[:, keep], alpha1)[0]
    return b, W_SINGULAR


def background_index(lam) -> int:
    """idx = argmin_i |log λ_i| (Alg 3), principal branch, λ = 0 excluded (Q5).

    Ties (conjugate pairs tie exactly): smaller |Im log λ|, then Im(λ) >= 0, then the lowest
    index.  Raises E_NO_VIABLE_MODE when every λ is zero."""
    best, bkey = -1, None
    for i, l in enumerate(np.asarray(lam, dtype=np.complex128)):
        if l == 0:
            continue
        lg = np.log(l)
        key = (abs(lg), abs(lg.imag), 0 if l.imag >= 0 else 1, i)
        if bkey is None or key < bkey:
            best, bkey = i, key
    if best < 0:
        raise OracleError(E_NO_VIABLE_MODE, "all eigenvalues zero")
    return best


# ----------------------------------------------------------------------------------------
# O7, O11–O12  Modes and background/foreground  (Eq. Phi; Alg 3)
# ----------------------------------------------------------------------------------------

def modes(Xp_cols, d: dict, which=None) -> np.ndarray:
    """Φ = X' V Σ⁻¹ W = X' (vsi w)  ("vsiw = vsi * w; phi = X[:, 1:] * vsiw").

    ``Xp_cols``: the m columns of X' (list of n-vectors, or an (n, m) array); ``which``: mode
    indices (default all).  Each entry is a compensated sum over the m columns (O7, C
    orc_modes)."""
    vsiw = d["vsi"] @ d["W"]
    cols = list(range(vsiw.shape[1])) if which is None else list(which)
    if isinstance(Xp_cols, np.ndarray) and Xp_cols.ndim == 2:
        Xp_cols = [Xp_cols[:, k] for k in range(Xp_cols.shape[1])]
    X, dt = _real_cols(Xp_cols)
    n, m = X.shape
    T = np.asfortranarray(vsiw[:, cols].astype(np.complex128))
    Phi = np.zeros((n, len(cols)), dtype=np.complex128, order="F")
    clib().orc_modes(_p(X), n, m, n, dt, _p(T), len(cols), _p(Phi), n, THREADS)
    return Phi


def background_newest(Xp_cols, x_newest, d: dict, b, idx: int, threshold: float = 0.2):
    """Streaming branch of Alg 3 for the newest column:
    l = b[idx] φ_idx λ_idx^e with e = m (Q4; b is fitted to the oldest column, λ⁰),
    s = x − |l| (Q8: complex modulus), mask = s > threshold (strict)."""
    m = d["m"]
    phi = modes(Xp_cols, d, [idx])[:, 0]
    l = b[idx] * phi * d["lam"][idx] ** m
    low = np.abs(l)
    s = np.asarray(x_newest, dtype=np.float64) - low
    return low, s, s > threshold


def background_set(lam, nb: int) -> list:
    """Reading Q25 ("use some small subset of background DMD modes
    rather than just the single slowest changing mode"): the nb modes with the smallest |log λ|,
    ranked by Q5's key (|log λ|, |Im log λ|, Im λ >= 0 first, index), λ = 0 excluded, closed
    under conjugation — if the nb-th mode's conjugate partner is the next in rank it is added
    (at most nb + 1 modes).  nb = 1 gives [background_index(lam)]."""
    ranked = []
    for i, l in enumerate(np.asarray(lam, dtype=np.complex128)):
        if l == 0:
            continue
        lg = np.log(l)
        ranked.append(((abs(lg), abs(lg.imag), 0 if l.imag >= 0 else 1, i), i))
    if not ranked:
        raise OracleError(E_NO_VIABLE_MODE, "all eigenvalues zero")
    order = [i for _, i in sorted(ranked)]
    B = order[:nb]
    lam = np.asarray(lam, dtype=np.complex128)
    if nb < len(order) and lam[B[-1]].imag != 0 and lam[order[nb]] == np.conj(lam[B[-1]]):
        B.append(order[nb])
    return B


def background_newest_multi(Xp_cols, x_newest, d: dict, b, B, threshold: float = 0.2):
    """Streaming branch of Alg 3 with the mode set B (Q25) instead of the single
    idx: l = Σ_{p∈B} b_p φ_p λ_p^m (e = m, Q4), s = x − |l|, mask = s > threshold (Q8)."""
    m = d["m"]
    phi = modes(Xp_cols, d, list(B))
    l = np.zeros(phi.shape[0], dtype=np.complex128)
    for q, p in enumerate(B):
        l += b[p] * phi[:, q] * d["lam"][p] ** m
    low = np.abs(l)
    s = np.asarray(x_newest, dtype=np.float64) - low
    return low, s, s > threshold


def background_first_window(Z_cols, d: dict, b, idx: int, threshold: float = 0.2):
    """First-window branch of Alg 3: exponents 0..m over all m+1 window columns
    (Q24).  Returns (|L|, S, mask) as (n, m+1) arrays."""
    m = d["m"]
    phi = modes(Z_cols[1:], d, [idx])[:, 0]
    pw = d["lam"][idx] ** np.arange(m + 1)
    L = np.abs(b[idx] * np.outer(phi, pw))
    Z = np.stack([np.asarray(c, dtype=np.float64) for c in Z_cols], axis=1)
    S = Z - L
    return L, S, S > threshold


# ----------------------------------------------------------------------------------------
# NEXT-3  Compressed ingestion beyond the real DCT  (§3.5; reading Q10/Q11, Q27)
# ----------------------------------------------------------------------------------------

def rfft_weights(rows: int, cols: int) -> np.ndarray:
    """Weights of the stored half spectrum of a real rows x cols field (numpy.fft.rfft2 layout:
    bin (ky, kx), ky in [0, rows), kx in [0, cols//2], flat index ky*(cols//2+1) + kx).

    Reading Q10's trap: the omitted bins are the complex conjugates of the stored
    bins (kx, ky) -> (-kx, -ky), so Parseval over the full spectrum counts every stored bin twice,
    except the columns kx = 0 and, for even cols, kx = cols/2, whose partners are stored themselves.
    Weight 2 off those columns, 1 on them."""
    h = cols // 2 + 1
    w = np.full((rows, h), 2.0)
    w[:, 0] = 1.0
    if cols % 2 == 0:
        w[:, cols // 2] = 1.0
    return w.ravel()


def fourier_gram_column(slots, x_new, n: int, weights=None) -> np.ndarray:
    """Gram column over complex Fourier-coefficient snapshots (reading Q27): each snapshot is
    (idx, val) with complex val; g_k = Σ_i w_i Re(conj(ẑ_k[i]) x̂[i]) over the scattered dense
    vectors (definition; w = 1 for full-spectrum storage, rfft_weights for the half spectrum).
    With the unitary ("ortho") transform this is the pixel-space inner product (Parseval, P:359
    "unitary transforms"); the real part is exact for Hermitian data, where the imaginary parts
    cancel.  Evaluated as compensated row-order dots (O1) of the real vectors [w·Re ẑ, w·Im ẑ] and
    [Re x̂, Im x̂]: w ∈ {1, 2} scales exactly."""
    wt = np.ones(n) if weights is None else np.asarray(weights, dtype=np.float64)

    def dense(sv, weighted):
        idx, val = sv
        idx = np.asarray(idx, dtype=np.int64)
        d = np.zeros(n, dtype=np.complex128)
        d[idx] = np.asarray(val, dtype=np.complex128)
        if weighted:
            d = d * wt
        return np.concatenate([d.real, d.imag])
    return gram_column([dense(s, True) for s in slots], dense(x_new, False))


def modes_complex(Xp_cols, d: dict, which=None) -> np.ndarray:
    """Φ̂ = X̂'(vsi W) for complex coefficient-space columns (Eq. Phi P:158-160 in the Fourier
    basis, NEXT-3): (A + iB) T = A T + i B T with A = Re X̂', B = Im X̂', each a compensated O7
    sum (C orc_modes)."""
    if isinstance(Xp_cols, np.ndarray) and Xp_cols.ndim == 2:
        Xp_cols = [Xp_cols[:, k] for k in range(Xp_cols.shape[1])]
    cols = [np.asarray(c, dtype=np.complex128) for c in Xp_cols]
    return modes([c.real for c in cols], d, which) + 1j * modes([c.imag for c in cols], d, which)


def dct_matrix(N: int) -> np.ndarray:
    """Orthonormal DCT-II matrix (reading Q11): C[k, p] = w_k cos(π k (2p+1) / (2N)), w_0 = √(1/N),
    w_k = √(2/N).  X̂ = C x;  x = Cᵀ X̂ (DCT-III, the inverse, since C is orthogonal)."""
    k = np.arange(N)[:, None]
    p = np.arange(N)[None, :]
    C = np.cos(np.pi * k * (2 * p + 1) / (2.0 * N))
    C[0, :] *= np.sqrt(1.0 / N)
    C[1:, :] *= np.sqrt(2.0 / N)
    return C


def idct2(coef, rows: int, cols: int) -> np.ndarray:
    """Pixel field (row-major rows x cols, flattened) of orthonormal 2-D DCT-II coefficients
    (flat index ky*cols + kx): x = C_rowsᵀ X̂ C_cols, two matrix products (library primitive)."""
    Xh = np.asarray(coef).reshape(rows, cols)
    if np.iscomplexobj(Xh):
        return idct2(Xh.real, rows, cols) + 1j * idct2(Xh.imag, rows, cols)
    return (dct_matrix(rows).T @ Xh @ dct_matrix(cols)).ravel()


def background_newest_pixel(Xp_slots, x_slot, n: int, rows: int, cols: int, d: dict, b, idx: int,
                            threshold: float = 0.2):
    """Streaming branch of Alg 3 for a sparse-DCT context, returned in pixel space
    (NEXT-3 "an inverse-DCT kernel for pixel-space background", "transfer the compressed
    DMD from the GPU back"): φ̂_idx = X̂'(vsi w_idx) over the scattered coefficient columns (O7),
    l̂ = b_idx φ̂_idx λ_idx^m (e = m, Q4), l = IDCT2(l̂) (the transform is linear and real, so it
    maps the complex coefficient vector part by part), x = IDCT2(x̂_newest), s = x − |l|,
    mask = s > threshold (Q8)."""
    def dense(sv):
        i, v = sv
        z = np.zeros(n)
        z[np.asarray(i, dtype=np.int64)] = np.asarray(v, dtype=np.float64)
        return z
    m = d["m"]
    phi = modes([dense(s) for s in Xp_slots], d, [idx])[:, 0]
    lhat = b[idx] * phi * d["lam"][idx] ** m
    low = np.abs(idct2(lhat, rows, cols))
    x = idct2(dense(x_slot), rows, cols)
    s = x - low
    return low, s, s > threshold


# ----------------------------------------------------------------------------------------
# NEXT-4  BMC-style scoring  (Table 2; reading Q26)
# ----------------------------------------------------------------------------------------

def evaluate(masks, gts) -> dict:
    """Recall, precision, F-measure and PSNR of foreground masks against ground-truth masks
    (Table 2, "BMC Evaluation Wizard"; recall = TP/(TP+FN), precision =
    TP/(TP+FP), F = 2PR/(P+R)).  Reading Q26: counts are pooled over all frames scored (one number
    per sequence, as Table 2 reports); PSNR is that of the binary mask sequence against the
    ground truth at the pixel range's peak (0/1 masks, i.e. 0/255 images): 10·log10(N / (FP+FN))
    over the N pixels scored, +inf when no pixel differs.  Undefined ratios are reported as 0
    with a flag."""
    tp = fp = fn = tn = 0
    for mk, gt in zip(masks, gts):
        mk = np.asarray(mk).astype(bool).ravel()
        gt = np.asarray(gt).astype(bool).ravel()
        if mk.shape != gt.shape:
            raise OracleError(E_INVALID, "mask and ground truth shapes differ")
        tp += int(np.count_nonzero(mk & gt))
        fp += int(np.count_nonzero(mk & ~gt))
        fn += int(np.count_nonzero(~mk & gt))
        tn += int(np.count_nonzero(~mk & ~gt))
    npx = tp + fp + fn + tn
    empty_gt = (tp + fn) == 0
    empty_mask = (tp + fp) == 0
    recall = 0.0 if empty_gt else tp / (tp + fn)
    precision = 0.0 if empty_mask else tp / (tp + fp)
    f = 0.0 if recall + precision == 0 else 2.0 * precision * recall / (precision + recall)
    psnr = math.inf if fp + fn == 0 else 10.0 * math.log10(npx / (fp + fn))
    return dict(tp=tp, fp=fp, fn=fn, tn=tn, recall=recall, precision=precision, f_measure=f,
                psnr=psnr, empty_gt=empty_gt, empty_mask=empty_mask)


# ----------------------------------------------------------------------------------------
# Streaming engine (Fig. 3, §3.2): one push = a2..a11 of SURVEY §8(a)
# ----------------------------------------------------------------------------------------

class StreamingDMD:
    """Oracle counterpart of the C-ABI ``sdmd_push_*`` + getters (one writer).

    Each push slides the Gram (Alg 1), and once the window is full runs SDMD (Alg 2) and the
    streaming branch of SBackSub (Alg 3) for the newest column."""

    def __init__(self, m: int, rank_tol: float = 1e-7, r_max: int | None = None,
                 threshold: float = 0.2, background: bool = True, bg_modes: int = 1,
                 buildup: bool = False):
        self.m, self.rank_tol, self.r_max = m, rank_tol, r_max
        self.threshold, self.background = threshold, background
        self.bg_modes = bg_modes
        # NEXT-4 ("start the algorithm with only 2 columns. Until the matrix is filled,
        # the new columns would be appended without erasing the oldest"): with buildup the DMD
        # also runs on the growing window of 2..m columns (no background before it is full)
        self.buildup = buildup
        self.gram = StreamingGram(m)
        self.frames = 0
        self.last = None

    def init_window(self, Z) -> dict | None:
        """First step (Alg 1 first branch "xtx = X.T * X"): the whole window at once.
        Z: n x (m+1) array (or a list of m+1 columns), oldest first."""
        cols = [np.asarray(c) for c in (Z if isinstance(Z, (list, tuple)) else np.asarray(Z).T)]
        cols = [c.astype(np.float32) if c.dtype == np.float32 else c.astype(np.float64) for c in cols]
        if len(cols) != self.m + 1:
            raise OracleError(E_INVALID, "init_window needs m+1 columns")
        G = gram(np.stack(cols, axis=1))
        if not np.all(np.isfinite(G)):
            raise OracleError(E_NONFINITE, "non-finite window")
        self.gram.cols = cols
        self.gram.G = G
        self.frames = self.m + 1
        return self._dmd()

    def push(self, x) -> dict | None:
        self.gram.push(x)
        self.frames += 1
        if not self.gram.full:
            if self.buildup and len(self.gram.cols) >= 2:
                return self._dmd(background=False)
            self.last = None
            return None
        return self._dmd()

    def _dmd(self, background: bool = True) -> dict:
        G = self.gram.G
        d = dmd_from_gram(G, self.rank_tol, self.r_max)
        b, st = amplitudes(d, self.rank_tol)
        idx = background_index(d["lam"])
        out = dict(d, b=b, amp_status=st, idx=idx, G=G.copy(), frame=self.frames - 1)
        if self.background and background:
            cols = self.gram.cols
            if self.bg_modes <= 1:
                low, s, mask = background_newest(cols[1:], cols[-1], d, b, idx, self.threshold)
            else:
                B = background_set(d["lam"], self.bg_modes)
                low, s, mask = background_newest_multi(cols[1:], cols[-1], d, b, B, self.threshold)
                out.update(bg_set=B)
            out.update(lowrank=low, sparse=s, mask=mask)
        self.last = out
        return out


def dmd_window(Z, rank_tol: float = 1e-7, r_max: int | None = None) -> dict:
    """Batch counterpart: everything from one window Z (n x (m+1)) recomputed from scratch
    (the paper's non-streaming CPU/GPU variants)."""
    G = gram(Z)
    d = dmd_from_gram(G, rank_tol, r_max)
    b, st = amplitudes(d, rank_tol)
    idx = background_index(d["lam"])
    return dict(d, b=b, amp_status=st, idx=idx, G=G)
