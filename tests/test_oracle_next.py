"""Pins of the oracle's NEXT-row functions against things other
than the oracle: SPEC worked examples (tests/golden/evaluate_examples.json, cited), brute-force
per-pixel counting, closed-form PSNR, Parseval through numpy.fft / scipy.fft (independent library
transforms, test side only) and the dense pixel-space oracle path.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import oracle.sdmd_oracle as O
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "evaluate_examples.json")))


def normwise(Ga, Gb):
    d = np.sqrt(np.abs(np.diag(Gb)))
    den = np.outer(d, d)
    den[den == 0] = 1.0
    return float(np.max(np.abs(Ga - Gb) / den))


# ------------------------------------------------------------- NEXT-4: evaluate ----------

@pytest.mark.parametrize("ex", GOLD["examples"], ids=lambda e: e["name"])
def test_evaluate_spec_worked_examples(ex):
    """SPEC S:371-373 (Table 2 P:437-443 methodology)."""
    r = O.evaluate([np.array(ex["mask"], dtype=bool)], [np.array(ex["gt"], dtype=bool)])
    for k in ("recall", "precision", "f_measure"):
        assert r[k] == pytest.approx(ex[k], abs=1e-15), k
    for k in ("empty_gt", "empty_mask"):
        assert r[k] == ex.get(k, False), k


def test_evaluate_bruteforce_counts_and_psnr():
    """Pooled counts (reading Q26) equal a per-pixel Python loop; PSNR = 10 log10(N/(FP+FN))."""
    rng = np.random.default_rng(11)
    masks = [rng.random(300) < 0.3 for _ in range(4)]
    gts = [rng.random(300) < 0.2 for _ in range(4)]
    tp = fp = fn = tn = 0
    for mk, gt in zip(masks, gts):
        for a, b in zip(mk.tolist(), gt.tolist()):
            tp += a and b
            fp += a and not b
            fn += (not a) and b
            tn += (not a) and (not b)
    r = O.evaluate(masks, gts)
    assert (r["tp"], r["fp"], r["fn"], r["tn"]) == (tp, fp, fn, tn)
    P, R = tp / (tp + fp), tp / (tp + fn)
    assert r["f_measure"] == pytest.approx(2 * P * R / (P + R), rel=1e-15)
    assert r["psnr"] == pytest.approx(10 * math.log10(1200 / (fp + fn)), rel=1e-15)


def test_evaluate_psnr_closed_forms():
    """One wrong pixel of N: PSNR = 10 log10 N (0/255 images: MSE = 255²/N); none: +inf."""
    gt = np.zeros(1000, dtype=bool)
    gt[:10] = True
    mk = gt.copy()
    assert O.evaluate([mk], [gt])["psnr"] == math.inf
    mk[500] = True
    assert O.evaluate([mk], [gt])["psnr"] == pytest.approx(30.0, abs=1e-12)
    mse255 = np.mean((mk.astype(np.float64) * 255 - gt.astype(np.float64) * 255) ** 2)
    assert O.evaluate([mk], [gt])["psnr"] == pytest.approx(10 * math.log10(255.0 ** 2 / mse255), rel=1e-14)


# ----------------------------------------------- NEXT-3: complex Fourier snapshots --------

@pytest.mark.parametrize("rows,cols", [(12, 10), (9, 7), (16, 16)])
def test_fourier_gram_parseval_half_and_full(rows, cols):
    """Reading Q27: the weighted half-spectrum Gram (rfft2, weights 2 off the self-conjugate
    columns) and the full-spectrum Gram (fft2) equal the pixel-space Gram of the real fields
    (Parseval of the unitary transform; numpy.fft, test side)."""
    rng = np.random.default_rng(rows * 100 + cols)
    F = [rng.standard_normal((rows, cols)) for _ in range(5)]
    half = [np.fft.rfft2(f, norm="ortho").ravel() for f in F]
    full = [np.fft.fft2(f, norm="ortho").ravel() for f in F]
    nh = rows * (cols // 2 + 1)
    w = O.rfft_weights(rows, cols)
    sv = lambda v: (np.arange(v.size), v)                  # noqa: E731  (all bins stored)
    g_half = O.fourier_gram_column([sv(v) for v in half[:4]], sv(half[4]), nh, w)
    g_full = O.fourier_gram_column([sv(v) for v in full[:4]], sv(full[4]), rows * cols)
    g_pix = np.array([float(np.sum(F[k] * F[4])) for k in range(4)])
    scale = np.sqrt(np.array([np.sum(F[k] ** 2) for k in range(4)]) * np.sum(F[4] ** 2))
    assert np.max(np.abs(g_half - g_pix) / scale) < 1e-13
    assert np.max(np.abs(g_full - g_pix) / scale) < 1e-13
    # the trap: the unweighted half spectrum is NOT the pixel Gram
    g_bad = O.fourier_gram_column([sv(v) for v in half[:4]], sv(half[4]), nh)
    assert np.max(np.abs(g_bad - g_pix) / scale) > 1e-2


def test_fourier_stream_is_a_real_field_and_storages_agree():
    """synth.SparseFourierStream: its half spectrum round-trips through irfft2/rfft2 (Hermitian
    consistent, i.e. a real field), the full-spectrum storage holds the same field, and the two
    storages give the same Gram (weights vs conjugate partners)."""
    sh = synth.SparseFourierStream(32, 24, k_low=6, n_shell=30, seed=5, half=True)
    sf = synth.SparseFourierStream(32, 24, k_low=6, n_shell=30, seed=5, half=False)
    X = sh.dense(3).reshape(32, 13)
    f = np.fft.irfft2(X, s=(32, 24), norm="ortho")
    assert np.max(np.abs(np.fft.rfft2(f, norm="ortho") - X)) < 1e-15
    f2 = np.fft.ifft2(sf.dense(3).reshape(32, 24), norm="ortho")
    assert np.max(np.abs(f2.imag)) < 1e-15 and np.max(np.abs(f2.real - f)) < 1e-15
    w = O.rfft_weights(32, 24)
    gh = O.fourier_gram_column([sh.frame(t) for t in range(3)], sh.frame(3), sh.n, w)
    gf = O.fourier_gram_column([sf.frame(t) for t in range(3)], sf.frame(3), sf.n)
    assert np.max(np.abs(gh - gf)) < 1e-15 * np.max(np.abs(gh)) * 10


def test_modes_complex_vs_library_product():
    """Φ̂ = X̂'(vsi W) for complex columns (two O7 sums) vs the numpy complex matmul."""
    rng = np.random.default_rng(4)
    n, m = 200, 6
    Z = rng.standard_normal((n, m + 1)) + 1j * rng.standard_normal((n, m + 1))
    d = O.dmd_from_gram(O.gram(np.vstack([Z.real, Z.imag])))
    Phi = O.modes_complex(Z[:, 1:], d)
    ref = Z[:, 1:] @ (d["vsi"] @ d["W"])
    assert np.max(np.abs(Phi - ref)) < 1e-13 * np.max(np.abs(ref))


# ----------------------------------------------- NEXT-3: pixel-space background -------------

@pytest.mark.parametrize("N", [8, 32])
def test_dct_matrix_vs_scipy(N):
    """The oracle's orthonormal DCT-II matrix and 2-D inverse vs scipy.fft (independent)."""
    import scipy.fft as sf
    C = O.dct_matrix(N)
    assert np.max(np.abs(C @ C.T - np.eye(N))) < 1e-14
    x = np.random.default_rng(N).standard_normal(N)
    assert np.max(np.abs(C @ x - sf.dct(x, norm="ortho"))) < 1e-14
    X = np.random.default_rng(N + 1).standard_normal((N, 2 * N))
    assert np.max(np.abs(O.idct2(X.ravel(), N, 2 * N) - sf.idctn(X, norm="ortho").ravel())) < 1e-13


def test_pixel_background_equals_dense_pixel_path():
    """Unitary invariance: the sparse-DCT context's pixel-space background (DMD of the
    coefficient Gram, l = IDCT2(X̂'c)) equals the dense oracle run on the pixel frames (scipy
    idctn of each coefficient plane), for the newest column of several windows."""
    import scipy.fft as sf
    N, m = 32, 8
    st = synth.SparseDCTStream(N=N, k_low=6.0, n_shell=20, seed=9)
    frames = [st.frame(t) for t in range(m + 4)]
    pix = [sf.idctn(st.dense(t).reshape(N, N), norm="ortho").ravel() for t in range(m + 4)]
    dense_eng = O.StreamingDMD(m, background=True, threshold=0.05)
    coef_eng = O.StreamingDMD(m, background=False)
    for t in range(m + 4):
        dense_eng.push(pix[t])
        coef_eng.push(st.dense(t))
        if t < m:
            continue
        out = coef_eng.last
        low, s, mask = O.background_newest_pixel(frames[t - m + 1:t + 1], frames[t], st.n, N, N,
                                                 out, out["b"], out["idx"], threshold=0.05)
        ref = dense_eng.last
        sc = float(np.max(ref["lowrank"]))
        assert np.max(np.abs(low - ref["lowrank"])) < 1e-9 * sc
        assert np.max(np.abs(s - ref["sparse"])) < 1e-9 * max(sc, 1.0)
        amb = np.abs(ref["sparse"] - 0.05) < 1e-9
        assert np.array_equal(mask[~amb], ref["mask"][~amb])
