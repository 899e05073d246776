"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This module only *generates data*.  It holds none of the method's arithmetic (no Gram
products, no eigensolves, no DMD): it is the one module both the oracle (``oracle/``) and
the CUDA path's harness may import (task rule ③).  Every generator is deterministic given
its seed; the video generator is counter-based (frame ``t`` can be produced on its own, on
any torch device, with bit-identical results on CPU and GPU: integer hashing plus a fixed
sequence of IEEE fp32 element-wise operations, no transcendentals on the per-frame path).

Workload recipes follow SURVEY.md §8(d) (configs C1-C5 of BASELINE.json) and are restated
in DESIGN.md §"Input recipe".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "PlantedModes", "planted_c1", "planted_spec", "cylinder_wake", "VideoStream",
    "SparseDCTStream", "video_config", "CONFIGS",
]

# --------------------------------------------------------------------------------------
# Planted linear dynamics  x_t = sum_j b_j phi_j lambda_j^t   (§2.2.1)
# --------------------------------------------------------------------------------------


@dataclass
class PlantedModes:
    """Real data built from complex-conjugate mode pairs plus optional real modes.

    ``pairs``: list of (lambda, b) for the member with Im(lambda) >= 0; its conjugate
    partner (conj lambda, conj b, conj phi) is implied.  ``reals``: list of (lambda, b)
    with real lambda and a real mode shape.  Snapshot t is
        x_t = sum_pairs 2 Re(b phi lambda^t) + sum_reals b phi lambda^t.
    """

    n: int
    pairs: list
    reals: list = field(default_factory=list)
    seed: int = 0
    normalize: bool = True

    def __post_init__(self):
        rng = np.random.default_rng(self.seed)
        n = self.n
        self.phi_pairs = []
        for _ in self.pairs:
            ph = (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / math.sqrt(2 * n)
            self.phi_pairs.append(ph)
        self.phi_reals = []
        for _ in self.reals:
            ph = rng.standard_normal(n) / math.sqrt(n)
            self.phi_reals.append(ph)

    @property
    def lambdas(self) -> np.ndarray:
        """All planted eigenvalues (each pair contributes lambda and conj(lambda))."""
        out = []
        for lam, _ in self.pairs:
            out += [complex(lam), complex(lam).conjugate()]
        for lam, _ in self.reals:
            out.append(complex(lam))
        return np.array(out, dtype=np.complex128)

    @property
    def rank(self) -> int:
        return 2 * len(self.pairs) + len(self.reals)

    def frames(self, t0: int, t1: int) -> np.ndarray:
        """Columns x_t for t in [t0, t1), shape (n, t1-t0), float64."""
        t = np.arange(t0, t1, dtype=np.float64)
        X = np.zeros((self.n, t1 - t0), dtype=np.float64)
        for (lam, b), ph in zip(self.pairs, self.phi_pairs):
            lam = complex(lam)
            coef = complex(b) * np.power(lam, t)          # (T,)
            X += 2.0 * np.real(np.outer(ph, coef))
        for (lam, b), ph in zip(self.reals, self.phi_reals):
            coef = float(np.real(b)) * np.power(float(np.real(lam)), t)
            X += np.outer(ph, coef)
        return X

    def mode_products(self, t0: int) -> dict:
        """Planted b_j lambda_j^{t0} phi_j for every eigenvalue (the scale-free DMD product
        at a window whose first column is x_{t0}); keyed by eigenvalue."""
        out = {}
        for (lam, b), ph in zip(self.pairs, self.phi_pairs):
            lam = complex(lam)
            v = complex(b) * lam ** t0 * ph
            out[lam] = v
            out[lam.conjugate()] = np.conj(v)
        for (lam, b), ph in zip(self.reals, self.phi_reals):
            lam = complex(lam)
            out[lam] = complex(b) * lam ** t0 * ph.astype(np.complex128)
        return out


def planted_c1(with_unit_mode: bool = False, seed: int = 1612) -> PlantedModes:
    """BASELINE config 1 / SURVEY C1: n=4096, rank 4, lambda = {e^{+-i pi/8}, 0.99 e^{+-i pi/5}},
    b = {e^{+-0.3i}, 0.5 e^{+-1.1i}}.  Variant C1b adds lambda_0 = 1 with a real mode."""
    pairs = [(np.exp(1j * np.pi / 8), np.exp(0.3j)),
             (0.99 * np.exp(1j * np.pi / 5), 0.5 * np.exp(1.1j))]
    reals = [(1.0, 1.0)] if with_unit_mode else []
    return PlantedModes(n=4096, pairs=pairs, reals=reals, seed=seed)


def planted_spec(which: int, n: int = 64, seed: int = 7) -> PlantedModes:
    """SPEC.md acceptance 3 planted spectra: {0.9, 0.5}, {e^{+-i pi/8}},
    {1.0, 0.7 e^{+-0.3i}} at n=64."""
    if which == 0:
        return PlantedModes(n=n, pairs=[], reals=[(0.9, 1.0), (0.5, 0.8)], seed=seed)
    if which == 1:
        return PlantedModes(n=n, pairs=[(np.exp(1j * np.pi / 8), 1.0 + 0.5j)], seed=seed)
    if which == 2:
        return PlantedModes(n=n, pairs=[(0.7 * np.exp(0.3j), 0.6 - 0.2j)],
                            reals=[(1.0, 1.3)], seed=seed)
    raise ValueError(which)


# --------------------------------------------------------------------------------------
# C2: cylinder-wake-shaped periodic field (449 x 199 grid), mean + 10 harmonic pairs
# --------------------------------------------------------------------------------------


def cylinder_wake(nx: int = 449, ny: int = 199, n_harm: int = 10, seed: int = 1613,
                  noise: float = 0.0) -> PlantedModes:
    """Synthetic wake-like field: rank 1 + 2*n_harm, period 30 frames.
    psi_k = exp(-(y(1+0.1k))^2) e^{i(1.3 k x + theta_k)} sigmoid(4x) (cos .7ky + .3i sin ky)
    on x in [-1, 8], y in [-2, 2]; lambda_k = e^{i k 2pi/30}, amplitude 0.7^k."""
    rng = np.random.default_rng(seed)
    x = np.linspace(-1.0, 8.0, nx)
    y = np.linspace(-2.0, 2.0, ny)
    X, Y = np.meshgrid(x, y, indexing="xy")          # (ny, nx), row-major flatten
    sig = 1.0 / (1.0 + np.exp(-4.0 * X))
    omega = 2.0 * np.pi / 30.0
    pm = PlantedModes(n=nx * ny, pairs=[], reals=[], seed=seed)
    pm.phi_pairs, pm.phi_reals = [], []
    pm.reals = [(1.0, 1.0)]
    pm.phi_reals = [(np.exp(-Y ** 2) * sig).ravel()]
    for k in range(1, n_harm + 1):
        th = rng.uniform(0.0, 2.0 * np.pi)
        psi = (np.exp(-(Y * (1.0 + 0.1 * k)) ** 2) * np.exp(1j * (1.3 * k * X + th)) * sig
               * (np.cos(0.7 * k * Y) + 0.3j * np.sin(k * Y)))
        pm.pairs.append((np.exp(1j * k * omega), 0.7 ** k))
        pm.phi_pairs.append(psi.ravel())
    return pm


# --------------------------------------------------------------------------------------
# Counter-based hashing (integer only; identical on numpy / torch CPU / torch CUDA)
# --------------------------------------------------------------------------------------

_M32 = 0xFFFFFFFF


def _mul32_py(x: int, c: int) -> int:
    return (x * c) & _M32


def _hash32_py(x: int) -> int:
    """lowbias32 integer hash on Python ints (for per-frame keys)."""
    x &= _M32
    x ^= x >> 16
    x = _mul32_py(x, 0x7FEB352D)
    x ^= x >> 15
    x = _mul32_py(x, 0x846CA68B)
    x ^= x >> 16
    return x


def _mul32_t(x, c: int):
    """(x * c) mod 2^32 for an int64 tensor x in [0, 2^32) without int64 overflow."""
    lo = c & 0xFFFF
    hi = c >> 16
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & _M32


def _hash32_t(x):
    x = x & _M32
    x = x ^ (x >> 16)
    x = _mul32_t(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32_t(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


# --------------------------------------------------------------------------------------
# C3 / C4: synthetic video (static textured background + moving bright squares + noise)
# --------------------------------------------------------------------------------------


class VideoStream:
    """Counter-based synthetic video, fp32 pixels in [0, 1], planar channel-major flattening
    (index = c*H*W + y*W + x).  Mirrors the paper's workloads (PEViD/BMC: mostly static
    background, sparse moving foreground).

    Frame t = clip(bg_c + noise_t) outside the squares, clip(1.0 + noise_t) inside.
    The background texture is computed once on the host in fp64 and rounded to fp32.
    """

    def __init__(self, H: int, W: int, C: int = 1, seed: int = 1614, n_squares: int = 3,
                 side: int = 96, noise_sigma: float = 0.01,
                 gains=(0.9, 1.0, 1.1)):
        self.H, self.W, self.C = H, W, C
        self.n = H * W * C
        self.seed = seed
        self.side = side
        self.noise_sigma = noise_sigma
        rng = np.random.default_rng(seed)
        yy, xx = np.meshgrid(np.arange(H, dtype=np.float64), np.arange(W, dtype=np.float64),
                             indexing="ij")
        tex = np.zeros((H, W))
        for _ in range(8):
            kx, ky = rng.integers(-4, 5, size=2)
            ph = rng.uniform(0, 2 * np.pi)
            tex += np.cos(2 * np.pi * (kx * xx / W + ky * yy / H) + ph)
        span = tex.max() - tex.min()
        tex = (tex - tex.min()) / (span if span > 0 else 1.0) * 2.0 - 1.0
        bg = np.clip(0.5 + 0.25 * tex, 0.05, 0.95)
        gains = list(gains) if C == 3 else [1.0] * C
        self.bg = np.stack([np.clip(bg * g, 0.0, 1.0) for g in gains[:C]]).astype(np.float32)
        self.sq_x0 = rng.integers(0, W, size=n_squares)
        self.sq_y0 = rng.integers(0, H, size=n_squares)
        self.sq_vx = rng.integers(3, 8, size=n_squares) * rng.choice([-1, 1], size=n_squares)
        self.sq_vy = rng.integers(3, 8, size=n_squares) * rng.choice([-1, 1], size=n_squares)
        self._key = _hash32_py(seed * 0x9E3779B1 + 12345)
        self._bg_cache = {}

    # ---- ground truth ----------------------------------------------------------------
    def square_mask_hw(self, t: int) -> np.ndarray:
        """(H, W) bool mask of the moving squares at frame t (wrap-around motion)."""
        m = np.zeros((self.H, self.W), dtype=bool)
        for q in range(len(self.sq_x0)):
            x0 = int((self.sq_x0[q] + self.sq_vx[q] * t) % self.W)
            y0 = int((self.sq_y0[q] + self.sq_vy[q] * t) % self.H)
            xs = (x0 + np.arange(self.side)) % self.W
            ys = (y0 + np.arange(self.side)) % self.H
            m[np.ix_(ys, xs)] = True
        return m

    def truth_mask(self, t: int) -> np.ndarray:
        return np.tile(self.square_mask_hw(t).ravel(), self.C)

    # ---- frames ----------------------------------------------------------------------
    def frame(self, t: int, device="cpu", row_slice=None):
        """Frame t as a flat fp32 torch tensor (optionally only rows [a, b))."""
        import torch
        a, b = (0, self.n) if row_slice is None else row_slice
        dev = torch.device(device)
        key = (str(dev), a, b)
        if key not in self._bg_cache:
            self._bg_cache[key] = torch.from_numpy(self.bg.ravel()[a:b].copy()).to(dev)
        bg = self._bg_cache[key]
        idx = torch.arange(a, b, dtype=torch.int64, device=dev)
        # noise: Irwin-Hall(4) from four counter-hashed 24-bit uniforms
        kf = _hash32_py(self._key ^ _hash32_py(t + 0x632BE5AB))
        h = _hash32_t(idx ^ kf)
        s = torch.zeros(b - a, dtype=torch.float32, device=dev)
        for j in range(4):
            hj = _hash32_t(h ^ ((0x9E3779B9 * (j + 1)) & _M32))
            s = s + (hj >> 8).to(torch.float32) * np.float32(1.0 / 16777216.0)
        noise = (s - np.float32(2.0)) * np.float32(self.noise_sigma * math.sqrt(3.0))
        # squares (integer geometry)
        hw = self.H * self.W
        p = idx % hw
        yy = p // self.W
        xx = p % self.W
        inside = torch.zeros(b - a, dtype=torch.bool, device=dev)
        for q in range(len(self.sq_x0)):
            x0 = int((self.sq_x0[q] + self.sq_vx[q] * t) % self.W)
            y0 = int((self.sq_y0[q] + self.sq_vy[q] * t) % self.H)
            inside |= (((xx - x0) % self.W) < self.side) & (((yy - y0) % self.H) < self.side)
        base = torch.where(inside, torch.ones_like(bg), bg)
        return torch.clamp(base + noise, 0.0, 1.0)

    def frames(self, t0: int, t1: int, device="cpu", row_slice=None):
        import torch
        cols = [self.frame(t, device, row_slice) for t in range(t0, t1)]
        return torch.stack(cols, dim=1)


def video_config(name: str) -> VideoStream:
    """C3 = 1920x1080 grey, squares of side 96; C4 = 3840x2160x3 planar, side 192.
    Small parity variants: C3s = 192x108 grey (side 24); C4s = 384x216x3 (side 48)."""
    if name == "C3":
        return VideoStream(1080, 1920, 1, seed=1614, side=96)
    if name == "C4":
        return VideoStream(2160, 3840, 3, seed=1615, side=192)
    if name == "C3s":
        return VideoStream(108, 192, 1, seed=1614, side=24)
    if name == "C4s":
        return VideoStream(216, 384, 3, seed=1615, side=48)
    raise ValueError(name)


# --------------------------------------------------------------------------------------
# C5: spectrally sparse turbulence, orthonormal 2D DCT-II coefficient space (1024^2)
# --------------------------------------------------------------------------------------


class SparseDCTStream:
    """Sparse snapshots in an orthonormal DCT-II coefficient space of an N x N field
    (SURVEY Q10/Q11).  Coefficient index = ky*N + kx.  A fixed low-wavenumber
    quarter-disc (|k| <= k_low) carries A(k) cos(omega(k) t + theta_k) with A=(1+k)^-2,
    omega = 0.05 k^(2/3); each frame adds n_shell fresh coefficients drawn from the shell
    k_low < |k| <= N/2 with values A(k) N(0,1).  Values fp64, indices int32 ascending."""

    def __init__(self, N: int = 1024, k_low: float = 110.0, n_shell: int = 1000,
                 seed: int = 1616):
        self.N, self.n = N, N * N
        self.seed = seed
        self.n_shell = n_shell
        ky, kx = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
        kk = np.sqrt(kx.astype(np.float64) ** 2 + ky.astype(np.float64) ** 2).ravel()
        lin = np.arange(N * N)
        self.low_idx = lin[kk <= k_low].astype(np.int64)
        self.shell_idx = lin[(kk > k_low) & (kk <= N / 2)].astype(np.int64)
        self.kmag = kk
        rng = np.random.default_rng(seed)
        self.theta = rng.uniform(0, 2 * np.pi, size=self.low_idx.size)
        k = kk[self.low_idx]
        self.A_low = (1.0 + k) ** -2.0
        self.w_low = 0.05 * k ** (2.0 / 3.0)

    @property
    def nnz_cap(self) -> int:
        return int(self.low_idx.size + self.n_shell)

    def frame(self, t: int):
        """(idx int32 ascending, val float64) of frame t."""
        rng = np.random.default_rng((self.seed, t))
        sh = rng.choice(self.shell_idx, size=self.n_shell, replace=False)
        sv = (1.0 + self.kmag[sh]) ** -2.0 * rng.standard_normal(self.n_shell)
        lv = self.A_low * np.cos(self.w_low * t + self.theta)
        idx = np.concatenate([self.low_idx, sh])
        val = np.concatenate([lv, sv])
        order = np.argsort(idx, kind="stable")
        return idx[order].astype(np.int32), val[order].astype(np.float64)

    def dense(self, t: int) -> np.ndarray:
        idx, val = self.frame(t)
        x = np.zeros(self.n, dtype=np.float64)
        x[idx] = val
        return x


class SparseFourierStream:
    """Sparse snapshots of a real rows x cols field in the unitary 2-D Fourier basis (SURVEY Q10's
    "complex FFT" variant of C5).  Values complex128, indices int32 ascending.

    half=True: the stored half spectrum of numpy.fft.rfft2 (bin (ky, kx), kx <= cols//2, flat
    index ky*(cols//2+1) + kx); half=False: the full spectrum (flat index ky*cols + kx), every
    bin's conjugate partner stored as well.  A fixed low band |k| <= k_low (signed wavenumbers)
    carries A(k) e^{i(ω(k) t + θ_k)}, A = (1+|k|)^-2, ω = 0.05|k|^(2/3); each frame adds n_shell
    fresh bins from the shell k_low < |k| <= min(rows, cols)/2, off the self-conjugate columns
    (kx = 0, cols/2), with values A (N(0,1) + i N(0,1))/√2.  Hermitian consistency (a real field)
    is built in: on the self-conjugate columns X[-ky] = conj(X[ky]) and the self-paired bins are
    real; in the full spectrum every bin's partner (-ky, -kx) holds the conjugate."""

    def __init__(self, rows: int = 1024, cols: int = 1024, k_low: float = 110.0,
                 n_shell: int = 1000, seed: int = 1617, half: bool = True):
        self.rows, self.cols, self.half = rows, cols, half
        self.h = cols // 2 + 1
        self.n = rows * self.h if half else rows * cols
        self.seed, self.n_shell = seed, n_shell
        ky = np.arange(rows)
        kys = np.where(ky <= rows // 2, ky, ky - rows).astype(np.float64)
        kx = np.arange(self.h).astype(np.float64)
        KY, KX = np.meshgrid(kys, kx, indexing="ij")
        kk = np.sqrt(KY ** 2 + KX ** 2)                   # (rows, h)
        self.kmag = kk.ravel()
        self_conj_col = np.zeros(self.h, dtype=bool)
        self_conj_col[0] = True
        if cols % 2 == 0:
            self_conj_col[cols // 2] = True
        flat = np.arange(rows * self.h).reshape(rows, self.h)
        low = kk <= k_low
        # on a self-conjugate column keep only one bin of each conjugate pair (ky <= partner) as
        # the generated one; the partner is filled by conjugation
        partner = (-ky) % rows
        gen = low.copy()
        for c in np.nonzero(self_conj_col)[0]:
            gen[:, c] &= ky <= partner
        self.gen_idx = flat[gen].astype(np.int64)          # half-spectrum bins carrying values
        self.low_idx = flat[low].astype(np.int64)          # all stored low-band bins
        rng = np.random.default_rng(seed)
        self.theta = rng.uniform(0, 2 * np.pi, size=self.gen_idx.size)
        kg = self.kmag[self.gen_idx]
        self.A = (1.0 + kg) ** -2.0
        self.w = 0.05 * kg ** (2.0 / 3.0)
        # bins that must be real (their own partner) and the partner map on self-conjugate columns
        gy, gx = np.divmod(self.gen_idx, self.h)
        self.gen_real = self_conj_col[gx] & (gy == partner[gy])
        shell = (kk > k_low) & (kk <= min(rows, cols) / 2) & ~self_conj_col[None, :]
        self.shell_idx = flat[shell].astype(np.int64)
        self._partner_col = self_conj_col

    @property
    def nnz_cap(self) -> int:
        n_half = int(self.low_idx.size + self.n_shell)
        return n_half if self.half else 2 * n_half

    def _half_frame(self, t: int):
        """dict {half-spectrum flat index: complex value} of frame t."""
        ph = self.w * t + self.theta
        v = self.A * np.exp(1j * ph)
        v = np.where(self.gen_real, v.real + 0j, v)
        vals = dict(zip(self.gen_idx.tolist(), v.tolist()))
        gy, gx = np.divmod(self.gen_idx, self.h)
        for i, y, x, val in zip(self.gen_idx.tolist(), gy.tolist(), gx.tolist(), v.tolist()):
            if self._partner_col[x]:
                p = ((-y) % self.rows) * self.h + x
                if p != i:
                    vals[p] = complex(val).conjugate()
        rng = np.random.default_rng((self.seed, t))
        sh = rng.choice(self.shell_idx, size=self.n_shell, replace=False)
        a = (1.0 + self.kmag[sh]) ** -2.0
        sv = a * (rng.standard_normal(self.n_shell) + 1j * rng.standard_normal(self.n_shell)) / np.sqrt(2.0)
        for i, val in zip(sh.tolist(), sv.tolist()):
            vals[i] = val
        return vals

    def frame(self, t: int):
        """(idx int32 ascending, val complex128) of frame t in this stream's storage."""
        hv = self._half_frame(t)
        if self.half:
            idx = np.array(sorted(hv), dtype=np.int64)
            return idx.astype(np.int32), np.array([hv[i] for i in idx.tolist()], dtype=np.complex128)
        full = {}
        for i, val in hv.items():
            y, x = divmod(i, self.h)
            full[y * self.cols + x] = val
            px = (-x) % self.cols
            if px != x:                                    # the omitted conjugate half
                full[((-y) % self.rows) * self.cols + px] = complex(val).conjugate()
        idx = np.array(sorted(full), dtype=np.int64)
        return idx.astype(np.int32), np.array([full[i] for i in idx.tolist()], dtype=np.complex128)

    def dense(self, t: int) -> np.ndarray:
        idx, val = self.frame(t)
        x = np.zeros(self.n, dtype=np.complex128)
        x[idx] = val
        return x


CONFIGS = {
    # name: (description, n, m, dtype)
    "C1": ("synthetic n=4096, m=16, rank 4 closed-form modes, fp64", 4096, 16, "f64"),
    "C2": ("cylinder-wake-shaped 449x199, m=150, fp64, r=21", 449 * 199, 150, "f64"),
    "C3": ("1920x1080 grey video, m=100, fp32, background/foreground", 1920 * 1080, 100, "f32"),
    "C4": ("3840x2160x3 video, m=200, fp32, row-sharded", 3840 * 2160 * 3, 200, "f32"),
    "C5": ("1024x1024 sparse DCT turbulence (~1% nnz), m=128, fp64", 1024 * 1024, 128, "f64"),
}
