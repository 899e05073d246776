"""Pins of the oracle (oracle/sdmd_oracle.py + oracle/csrc/sdmd_oracle.c) against things other
than itself: closed forms, SPEC worked examples (tests/golden), exact rational arithmetic,
correctly rounded sums (math.fsum), invariants and independent library routines (LAPACK via
numpy.linalg / scipy, which the oracle itself no longer uses) on small inputs.  CPU only."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle.sdmd_oracle as O
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "spec_worked_examples.json")))


def normwise(Ga, Gb):
    """Q17: max_ij |ΔG_ij| / sqrt(G_ii G_jj) (computed against Gb's diagonal)."""
    d = np.sqrt(np.abs(np.diag(Gb)))
    den = np.outer(d, d)
    den[den == 0] = 1.0
    return float(np.max(np.abs(Ga - Gb) / den))


def match_eigs(a, b):
    """Max |a_i - b_π(i)| under the optimal assignment (Hungarian; scipy)."""
    from scipy.optimize import linear_sum_assignment
    C = np.abs(np.asarray(a)[:, None] - np.asarray(b)[None, :])
    r, c = linear_sum_assignment(C)
    return float(C[r, c].max())


# ---------------------------------------------------------------- Gram (O1) ----------

@pytest.mark.parametrize("ex", GOLD["gram"], ids=lambda e: e["cite"][:20])
def test_gram_worked_examples(ex):
    Z = np.array(ex["Z_cols"], dtype=np.float64).T
    assert np.array_equal(O.gram(Z), np.array(ex["G"], dtype=np.float64))


@pytest.mark.parametrize("ex", GOLD["slide"], ids=lambda e: e["cite"][:20])
def test_slide_worked_examples(ex):
    sg = O.StreamingGram(ex["m"])
    for x in ex["push"]:
        sg.push(np.array(x, dtype=np.float64))
    assert np.array_equal(sg.G, np.array(ex["G_final"], dtype=np.float64))


def test_gram_exact_rational():
    """fp64 Gram vs exact rational arithmetic on a small random window (brute force)."""
    rng = np.random.default_rng(3)
    Z = rng.standard_normal((40, 6))
    G = O.gram(Z)
    F = [[sum(Fraction(Z[k, i]) * Fraction(Z[k, j]) for k in range(Z.shape[0]))
          for j in range(6)] for i in range(6)]
    E = np.array([[float(v) for v in row] for row in F])
    assert normwise(G, E) < 1e-15


def test_gram_fp32_promotion_exact():
    """fp32 inputs: products are exact in fp64 (Q9) — compare with exact rationals."""
    rng = np.random.default_rng(4)
    Z = rng.random((30, 4)).astype(np.float32)
    G = O.gram(Z)
    E = np.array([[float(sum(Fraction(float(Z[k, i])) * Fraction(float(Z[k, j]))
                             for k in range(30))) for j in range(4)] for i in range(4)])
    assert normwise(G, E) < 1e-15


def test_streamed_equals_batch_c1():
    """§3.1 reuse claim: streamed G == batch G of the final window, every slide;
    and exactly m+1 fresh dots per slide."""
    pm = synth.planted_c1()
    m = 16
    X = pm.frames(0, 81)
    sg = O.StreamingGram(m)
    for t in range(81):
        before = sg.fresh_dots
        sg.push(X[:, t])
        if t >= m:
            assert sg.fresh_dots - before == m + 1
            Gb = O.gram(X[:, t - m:t + 1])
            assert normwise(sg.G, Gb) < 1e-13


def test_gram_slices_psd_symmetry():
    rng = np.random.default_rng(5)
    Z = rng.standard_normal((300, 9))
    G = O.gram(Z)
    m = 8
    X, Xp = Z[:, :m], Z[:, 1:]
    # slice identities (BJ north_star): G[0:m,0:m] = XᵀX, G[0:m,1:m+1] = XᵀX'
    Sxx = np.array([[math.fsum(X[:, i] * X[:, j]) for j in range(m)] for i in range(m)])
    Sxy = np.array([[math.fsum(X[:, i] * Xp[:, j]) for j in range(m)] for i in range(m)])
    assert normwise(G[:m, :m], Sxx) < 1e-14
    assert np.max(np.abs(G[:m, 1:] - Sxy)) < 1e-12 * np.max(np.abs(Sxy))
    assert np.array_equal(G, G.T)
    assert np.linalg.eigvalsh(G).min() > -1e-13 * np.trace(G)


def test_nonfinite_rejected_state_unchanged():
    sg = O.StreamingGram(3)
    rng = np.random.default_rng(6)
    for _ in range(5):
        sg.push(rng.standard_normal(20))
    G0, cols0 = sg.G.copy(), [c.copy() for c in sg.cols]
    bad = rng.standard_normal(20)
    bad[7] = np.nan
    with pytest.raises(O.OracleError) as e:
        sg.push(bad)
    assert e.value.code == O.E_NONFINITE
    assert np.array_equal(sg.G, G0) and all(np.array_equal(a, b) for a, b in zip(sg.cols, cols0))


def test_sparse_gram_matches_dense():
    st = synth.SparseDCTStream(N=64, k_low=8.0, n_shell=30, seed=11)
    frames = [st.frame(t) for t in range(5)]
    g = O.sparse_gram_column(frames, frames[-1], st.n)
    D = np.stack([st.dense(t) for t in range(5)], axis=1)
    ref = np.array([math.fsum(D[:, k] * D[:, 4]) for k in range(5)])
    assert np.max(np.abs(g - ref)) <= 1e-15 * np.max(np.abs(ref))


def test_gram_invariant_under_orthonormal_dct():
    """Unitary invariance: Gram of orthonormal DCT-II coefficients == Gram of
    the fields."""
    from scipy.fft import dctn
    rng = np.random.default_rng(8)
    fields = rng.standard_normal((6, 16, 16))
    Z = np.stack([f.ravel() for f in fields], axis=1)
    C = np.stack([dctn(f, norm="ortho").ravel() for f in fields], axis=1)
    assert normwise(O.gram(C), O.gram(Z)) < 1e-13


# ------------------------------------------------------------- SVD (O3-O4) -----------

@pytest.mark.parametrize("ex", GOLD["sym_eig"], ids=lambda e: e["cite"][:20])
def test_svd_from_gram_worked(ex):
    S = np.array(ex["S"], dtype=np.float64)
    sigma, V, r = O.svd_from_gram(S)
    assert np.allclose(sigma ** 2, ex["evals"], atol=1e-13)
    if "r" in ex:
        assert r == ex["r"]
    if "evecs_abs" in ex:
        assert np.allclose(np.abs(V), ex["evecs_abs"], atol=1e-14)


def test_mos_sigma_vs_lapack_svd():
    """MoS σ (eig of XᵀX) vs LAPACK SVD of X itself (acceptance 1): 20 random
    1000x50 matrices."""
    rng = np.random.default_rng(9)
    for _ in range(20):
        X = rng.standard_normal((1000, 50))
        sigma, V, r = O.svd_from_gram(O.gram(X))
        ref = np.linalg.svd(X, compute_uv=False)
        assert r == 50
        assert np.max(np.abs(sigma - ref) / ref) < 1e-12


def test_constant_stream_sigma():
    """the same column repeated m times -> sigma_1 = sqrt(m)·‖x‖, r = 1."""
    rng = np.random.default_rng(10)
    x = rng.random(500)
    m = 12
    sigma, V, r = O.svd_from_gram(O.gram(np.tile(x[:, None], (1, m))))
    assert r == 1
    assert abs(sigma[0] - math.sqrt(m) * np.linalg.norm(x)) < 1e-12 * sigma[0]


def test_left_singular_and_eckart_young():
    rng = np.random.default_rng(12)
    X = rng.standard_normal((400, 10)) @ np.diag(np.logspace(0, -3, 10))
    sigma, V, r = O.svd_from_gram(O.gram(X))
    U = O.left_singular(X, sigma, V, r)
    assert np.max(np.abs(U.T @ U - np.eye(r))) < 1e-8
    assert np.linalg.norm(X - U * sigma[:r] @ V[:, :r].T) < 1e-10 * np.linalg.norm(X)
    for k in (1, 4, 7):
        err = np.linalg.norm(X - (U[:, :k] * sigma[:k]) @ V[:, :k].T)
        assert abs(err - math.sqrt(np.sum(sigma[k:] ** 2))) < 1e-8 * np.linalg.norm(X)


def test_zero_window():
    with pytest.raises(O.OracleError) as e:
        O.svd_from_gram(np.zeros((4, 4)))
    assert e.value.code == O.E_ZERO_MATRIX


# ---------------------------------------------------------- DMD (O5-O9) --------------

@pytest.mark.parametrize("ex", GOLD["eig"], ids=lambda e: e["cite"][:20])
def test_eig_worked(ex):
    """SPEC worked 2x2 examples through the oracle's own O6 (Hessenberg + Francis QR +
    back-substitution), not LAPACK."""
    A = np.array(ex["A"], dtype=np.float64)
    lam, W = O.eig_real(A)
    assert match_eigs(lam, np.array(ex["lam_re"]) + 1j * np.array(ex["lam_im"])) < 1e-14
    for j in range(len(lam)):                    # eigen-pairs where the matrix is diagonalisable
        if np.linalg.norm(W[:, j]) > 0 and not np.allclose(A, np.triu(A, 1)):
            assert np.linalg.norm(A @ W[:, j] - lam[j] * W[:, j]) <= 1e-14 * np.linalg.norm(W[:, j]) * max(1.0, np.abs(A).max())


def test_c1_closed_form_lambda_every_window():
    """BJ north_star: planted x_t = Σ b_j φ_j λ_j^t must recover λ_j to 1e-10 — all 64
    streamed windows of C1 (plus the b_j φ_j products and Φb = x_1)."""
    pm = synth.planted_c1()
    m = 16
    X = pm.frames(0, 81)
    eng = O.StreamingDMD(m, background=False)
    nwin = 0
    for t in range(81):
        out = eng.push(X[:, t])
        if out is None:
            continue
        nwin += 1
        assert out["r"] == 4
        assert match_eigs(out["lam"], pm.lambdas) < 1e-10
        # amplitudes: Φ b reproduces the oldest column x_{t-m}
        cols = eng.gram.cols
        Phi = O.modes(cols[1:], out)
        x1 = cols[0]
        assert np.linalg.norm(Phi @ out["b"] - x1) < 1e-10 * np.linalg.norm(x1)
        # scale-free products b_j φ_j == planted b_j λ_j^{t0} φ_j
        planted = pm.mode_products(t - m)
        for j, lam in enumerate(out["lam"]):
            key = min(planted, key=lambda k: abs(k - lam))
            ref = planted[key]
            assert np.linalg.norm(out["b"][j] * Phi[:, j] - ref) < 1e-9 * np.linalg.norm(ref)
    assert nwin == 65          # initial window + 64 streamed frames


@pytest.mark.parametrize("which", [0, 1, 2])
def test_spec_planted_spectra(which):
    """SPEC acceptance 3: {0.9,0.5}, {e^{±iπ/8}}, {1, 0.7e^{±0.3i}} at n=64, w=12."""
    pm = synth.planted_spec(which)
    Z = pm.frames(0, 12)
    out = O.dmd_window(Z)
    assert out["r"] == pm.rank
    assert match_eigs(out["lam"], pm.lambdas) < 1e-8


def test_eigs_equal_full_operator():
    """§2.2: Ã has the same (nonzero) eigenvalues as A = X' pinv(X)."""
    rng = np.random.default_rng(13)
    for _ in range(10):
        n, w, k = 25, 9, 5
        Z = rng.standard_normal((n, k)) @ rng.standard_normal((k, w))
        out = O.dmd_window(Z)
        X, Xp = Z[:, :-1], Z[:, 1:]
        A = Xp @ np.linalg.pinv(X)
        ev = np.linalg.eigvals(A)
        ev = ev[np.argsort(-np.abs(ev))][:out["r"]]
        assert match_eigs(out["lam"], ev) < 1e-8


def test_amplitudes_equal_least_squares():
    """§3.3: b = (WΛ)⁻¹α₁ equals the high-dimensional b = Φ†x₁ when x₁ is in the
    POD span (exact low-rank data)."""
    pm = synth.planted_spec(2, n=200)
    Z = pm.frames(0, 12)
    out = O.dmd_window(Z)
    Phi = O.modes([Z[:, k] for k in range(1, 12)], out)
    b_ls = np.linalg.pinv(Phi) @ Z[:, 0]
    assert np.linalg.norm(out["b"] - b_ls) < 1e-8 * np.linalg.norm(b_ls)


def test_modes_are_eigvecs_of_A():
    """A Φ_i = λ_i Φ_i with A v = X'(pinv(X) v) on exactly low-rank data."""
    pm = synth.planted_spec(1, n=100)
    Z = pm.frames(0, 12)
    out = O.dmd_window(Z)
    X, Xp = Z[:, :-1], Z[:, 1:]
    Phi = O.modes([Z[:, k] for k in range(1, 12)], out)
    AP = Xp @ (np.linalg.pinv(X) @ Phi)
    assert np.linalg.norm(AP - Phi * out["lam"][None, :]) < 1e-8 * np.linalg.norm(Phi)


def test_alpha1_first_row_reading_Q3():
    """Q3: α₁ = σ ⊙ V[0,:] reproduces x₁ (residual ~1e-15); the column reading does not."""
    pm = synth.planted_c1()
    Z = pm.frames(0, 17)
    out = O.dmd_window(Z)
    Phi = O.modes([Z[:, k] for k in range(1, 17)], out)
    assert np.linalg.norm(Phi @ out["b"] - Z[:, 0]) < 1e-12 * np.linalg.norm(Z[:, 0])
    r = out["r"]
    alt = out["sigma"][:r] * out["V"][:r, 0]
    wl = out["W"] * out["lam"][None, :]
    b_alt = np.linalg.solve(wl, alt.astype(complex))
    assert np.linalg.norm(Phi @ b_alt - Z[:, 0]) > 1e-3 * np.linalg.norm(Z[:, 0])


# --------------------------------------------------- background (O10-O12) ------------

@pytest.mark.parametrize("ex", GOLD["background_index"], ids=lambda e: e["cite"][:20])
def test_background_index_worked(ex):
    lam = np.array(ex["lam_re"]) + 1j * np.array(ex["lam_im"])
    assert O.background_index(lam) == ex["idx"]


def test_background_index_conjugate_tie_and_none():
    lam = np.array([0.5, 0.99 * np.exp(-0.01j), 0.99 * np.exp(0.01j)])
    assert O.background_index(lam) == 2          # tie -> Im >= 0
    with pytest.raises(O.OracleError):
        O.background_index(np.zeros(3, dtype=complex))


def test_exponent_reading_Q4_newest_column():
    """Q4: with b fitted to the oldest column, λ^m reproduces the newest column x_t
    (planted C1b with a λ=1 mode); λ^{m+1} does not."""
    pm = synth.planted_c1(with_unit_mode=True)
    m = 16
    Z = pm.frames(0, m + 1)
    out = O.dmd_window(Z)
    Phi = O.modes([Z[:, k] for k in range(1, m + 1)], out)
    rec_m = Phi @ (out["b"] * out["lam"] ** m)
    rec_m1 = Phi @ (out["b"] * out["lam"] ** (m + 1))
    nz = np.linalg.norm(Z[:, m])
    assert np.linalg.norm(rec_m - Z[:, m]) < 1e-10 * nz
    assert np.linalg.norm(rec_m1 - Z[:, m]) > 1e-2 * nz
    assert abs(out["lam"][out["idx"]] - 1.0) < 1e-10


def test_constant_video_fixed_point():
    """constant stream → λ_idx = 1, |L| = c, s ≈ 0."""
    vs = synth.VideoStream(24, 32, 1, seed=3, n_squares=0, noise_sigma=0.0)
    c = vs.frame(0).numpy().astype(np.float64)
    m = 10
    eng = O.StreamingDMD(m)
    for _ in range(m + 3):
        out = eng.push(c)
    assert abs(out["lam"][out["idx"]] - 1.0) < 1e-9
    assert np.max(np.abs(out["sparse"])) < 1e-6
    assert np.max(np.abs(out["lowrank"] - c)) < 1e-8 * np.max(c)


def test_background_additivity_and_monotone_threshold():
    vs = synth.VideoStream(36, 48, 1, seed=5, side=8)
    m = 12
    eng = O.StreamingDMD(m)
    for t in range(m + 4):
        out = eng.push(vs.frame(t).numpy())
    x = eng.gram.cols[-1]
    assert np.max(np.abs(out["lowrank"] + out["sparse"] - x)) <= 4e-16 * 4
    d = {k: out[k] for k in ("m", "lam", "vsi", "W")}
    masks = [O.background_newest(eng.gram.cols[1:], x, d, out["b"], out["idx"], th)[2]
             for th in (0.1, 0.2, 0.3)]
    assert np.all(masks[1] <= masks[0]) and np.all(masks[2] <= masks[1])


def test_moving_blob_foreground_sanity():
    """S:363 / SURVEY §8(c): synthetic moving squares → per-frame F-measure sanity bar
    (not parity).  Small C3-like stream, m=20."""
    vs = synth.VideoStream(48, 64, 1, seed=21, side=8, n_squares=2)
    m = 20
    eng = O.StreamingDMD(m)
    fs = []
    for t in range(m + 15):
        out = eng.push(vs.frame(t).numpy())
        if out is None:
            continue
        gt = vs.truth_mask(t)
        pred = out["mask"]
        tp = np.sum(pred & gt)
        p = tp / max(1, pred.sum())
        rc = tp / max(1, gt.sum())
        fs.append(0 if tp == 0 else 2 * p * rc / (p + rc))
    assert np.mean(fs) > 0.85


def test_c2_wake_rank_and_lambda():
    """C2 (BJ config 2): r = 21 and λ = {1, e^{±ikω}} (ω = 2π/30, k=1..10) to 1e-10."""
    pm = synth.cylinder_wake()
    m = 150
    Z = pm.frames(0, m + 1)
    out = O.dmd_window(Z)
    assert out["r"] == 21
    ref = [1.0] + [np.exp(s * 1j * k * 2 * np.pi / 30) for k in range(1, 11) for s in (1, -1)]
    assert match_eigs(out["lam"], np.array(ref)) < 1e-10
    assert abs(out["lam"][out["idx"]] - 1.0) < 1e-10


def test_oracle_init_window_equals_streamed():
    """Alg 1 first branch (batch Gram of the first window) == warm-up appends."""
    pm = synth.planted_c1()
    m = 16
    Z = pm.frames(0, m + 1)
    a = O.StreamingDMD(m, background=False)
    out_a = a.init_window(Z)
    b = O.StreamingDMD(m, background=False)
    for t in range(m + 1):
        out_b = b.push(Z[:, t])
    assert normwise(a.gram.G, b.gram.G) < 1e-14
    assert match_eigs(out_a["lam"], out_b["lam"]) < 1e-12
    x = pm.frames(m + 1, m + 2)[:, 0]
    assert match_eigs(a.push(x)["lam"], b.push(x)["lam"]) < 1e-12


# ------------------------------------------- NEXT-2: multi-mode background (reading Q25) -----

def test_background_set_rule_Q25():
    """B = the nb smallest |log λ| in Q5's order, closed under conjugation; nb = 1 is idx."""
    lam = np.array([0.5, np.exp(0.3j), np.exp(-0.3j), 1.0, 0.0, 0.9 * np.exp(1j), 0.9 * np.exp(-1j)])
    assert O.background_set(lam, 1) == [O.background_index(lam)] == [3]
    assert O.background_set(lam, 2) == [3, 1, 2]          # the cut pair is completed
    assert O.background_set(lam, 3) == [3, 1, 2]
    assert O.background_set(lam, 4) == [3, 1, 2, 0]        # |log 0.5| = 0.693 < |log 0.9e^{±i}| = 1.0055
    assert O.background_set(lam, 5) == [3, 1, 2, 0, 5, 6]
    assert O.background_set(lam, 7) == [3, 1, 2, 0, 5, 6]  # λ = 0 is never used
    with pytest.raises(O.OracleError):
        O.background_set(np.zeros(3), 2)


def test_multi_mode_background_closed_form():
    """Planted C1b (λ = 1 plus two conjugate pairs): with B = {1, e^{±iπ/8}} the streamed
    background l = Σ_{p∈B} b_p φ_p λ_p^m equals the planted contributions of exactly those modes
    to the newest frame (closed form), and nb = 1 reproduces the single-mode branch."""
    pm = synth.planted_c1(with_unit_mode=True)
    m, t0 = 16, 5
    Z = pm.frames(t0, t0 + m + 1)
    out = O.dmd_window(Z)
    cols = [Z[:, k] for k in range(m + 1)]
    B = O.background_set(out["lam"], 2)
    lamB = sorted(out["lam"][B], key=lambda z: (z.imag, z.real))
    want = sorted([1.0, np.exp(1j * np.pi / 8), np.exp(-1j * np.pi / 8)], key=lambda z: (z.imag, z.real))
    assert np.max(np.abs(np.array(lamB) - np.array(want))) < 1e-10
    low, s, mask = O.background_newest_multi(cols[1:], cols[-1], out, out["b"], B)
    prods = pm.mode_products(t0 + m)
    l_cf = sum(v for lam, v in prods.items() if abs(lam - 1.0) < 1e-12 or abs(abs(np.angle(lam)) - np.pi / 8) < 1e-12)
    assert np.max(np.abs(low - np.abs(l_cf))) < 1e-10 * np.max(np.abs(l_cf))
    # nb = 1: the single-mode branch (Alg 3 as written)
    l1, s1, m1 = O.background_newest(cols[1:], cols[-1], out, out["b"], out["idx"])
    l1m, s1m, m1m = O.background_newest_multi(cols[1:], cols[-1], out, out["b"], O.background_set(out["lam"], 1))
    assert np.array_equal(l1, l1m) and np.array_equal(m1, m1m)
    # all modes: the newest column itself (Q4 with every mode)
    lall, _, _ = O.background_newest_multi(cols[1:], cols[-1], out, out["b"], list(range(out["r"])))
    assert np.max(np.abs(lall - np.abs(Z[:, m]))) < 1e-10 * np.max(np.abs(Z[:, m]))


# ------------------------------------------------ NEXT-4: DMD during build-up -----

def test_buildup_dmd_closed_form_and_operator():
    """With buildup the oracle decomposes the growing window from 2 columns on.  Planted C1
    (rank 4): from 4 X-columns (frame 4) the spectrum is the planted one (closed form); before
    that eig(Ã) equals the nonzero eigenvalues of the full operator X' pinv(X)."""
    pm = synth.planted_c1()
    m = 16
    X = pm.frames(0, m + 1)
    ref = O.StreamingDMD(m, background=False, buildup=True)
    assert ref.push(X[:, 0]) is None
    for t in range(1, m + 1):
        out = ref.push(X[:, t])
        assert out is not None and out["frame"] == t and out["m"] == t
        if t >= 4:
            assert out["r"] == 4 and match_eigs(out["lam"], pm.lambdas) < 1e-10
        else:
            Xa, Xb = X[:, :t], X[:, 1:t + 1]
            # nonzero eig(X' pinv(X)) = eig(pinv(X) X') (AB and BA share nonzero eigenvalues)
            ev = np.linalg.eigvals(np.linalg.pinv(Xa) @ Xb)
            ev = ev[np.argsort(-np.abs(ev))][:out["r"]]
            assert match_eigs(out["lam"], ev) < 1e-8


# ------------------------------------------- pins of the C arithmetic (round 2) ------------

def test_gram_compensated_vs_correctly_rounded_cancellation():
    """O1 against math.fsum (the correctly rounded sum of the exact products) on fp32 columns with
    heavy cancellation (naive fp64 summation loses ~8 digits here): every entry within 2 ulp."""
    rng = np.random.default_rng(21)
    n = 20000
    base = rng.standard_normal(n).astype(np.float32) * np.float32(1e4)
    Z = np.stack([base, -base + rng.standard_normal(n).astype(np.float32),
                  rng.standard_normal(n).astype(np.float32), base * np.float32(0.5)], axis=1)
    Z = Z.astype(np.float32)
    G = O.gram(Z)
    Zd = Z.astype(np.float64)
    for i in range(4):
        for j in range(4):
            ref = math.fsum(Zd[:, i] * Zd[:, j])          # products exact (fp32 x fp32 in fp64)
            assert abs(G[i, j] - ref) <= 2 * np.spacing(abs(ref)), (i, j)
    naive = float(np.sum(Zd[:, 0] * Zd[:, 1]))
    assert abs(G[0, 1] - math.fsum(Zd[:, 0] * Zd[:, 1])) <= abs(naive - math.fsum(Zd[:, 0] * Zd[:, 1]))


def test_gram_fp64_products_compensated_vs_exact_rational():
    """fp64 inputs whose products round: O1 carries the product error (fma), so each entry matches
    the exact rational dot to ~1 ulp even with cancellation."""
    rng = np.random.default_rng(22)
    a = rng.standard_normal(300)
    b = -a + 1e-9 * rng.standard_normal(300)
    Z = np.stack([a, b, rng.standard_normal(300)], axis=1)
    G = O.gram(Z)
    for i in range(3):
        for j in range(3):
            ex = float(sum(Fraction(Z[k, i]) * Fraction(Z[k, j]) for k in range(300)))
            assert abs(G[i, j] - ex) <= 2 * np.spacing(abs(ex)), (i, j)


def test_gram_threads_agree():
    """Row-chunk threads (timing mode) and the single row-order sum agree to rounding."""
    rng = np.random.default_rng(23)
    Z = rng.random((100000, 5)).astype(np.float32)
    old = O.THREADS
    try:
        O.THREADS = 1
        G1 = O.gram(Z)
        O.THREADS = 7
        G7 = O.gram(Z)
    finally:
        O.THREADS = old
    assert normwise(G1, G7) < 1e-15


def test_gram_column_equals_gram_last_column():
    rng = np.random.default_rng(24)
    Z = rng.standard_normal((777, 6))
    g = O.gram_column([Z[:, k] for k in range(6)], Z[:, 5])
    assert np.array_equal(g, O.gram(Z)[:, 5])


@pytest.mark.parametrize("m", [1, 2, 7, 50, 200])
def test_jacobi_vs_lapack_eigh(m):
    """O3 (cyclic Jacobi) vs LAPACK dsyevd on random symmetric matrices: eigenvalues within
    1e-13·‖S‖, V orthogonal, S V = V diag(μ)."""
    rng = np.random.default_rng(30 + m)
    B = rng.standard_normal((m, m))
    S = B + B.T
    mu, V, sweeps = O.jacobi_eigh(S)
    ref = np.linalg.eigvalsh(S)
    nrm = np.linalg.norm(S, 2)
    assert np.max(np.abs(np.sort(mu) - ref)) < 1e-13 * nrm
    assert np.max(np.abs(V.T @ V - np.eye(m))) < 1e-13
    assert np.linalg.norm(S @ V - V * mu[None, :]) < 1e-13 * nrm * m
    assert sweeps <= 15


def test_jacobi_graded_psd_relative_accuracy():
    """S = XᵀX with σ spread over 1e0..1e-6 (MoS squares it to 1e-12): every eigenvalue meets the
    method-of-snapshots floor of reading Q7, |Δμ_i|/μ_i <= 4u (σ_1/σ_i)^2, against the squared
    LAPACK SVD of X itself (forming XᵀX costs u‖X‖² absolute; Jacobi adds no more)."""
    rng = np.random.default_rng(31)
    Q1, _ = np.linalg.qr(rng.standard_normal((400, 12)))
    Q2, _ = np.linalg.qr(rng.standard_normal((12, 12)))
    sv = np.logspace(0, -6, 12)
    X = (Q1 * sv) @ Q2.T
    mu, V, _ = O.jacobi_eigh(X.T @ X)
    ref = np.linalg.svd(X, compute_uv=False) ** 2
    u = 2.0 ** -53
    rel = np.abs(np.sort(mu)[::-1] - ref) / ref
    assert np.all(rel <= 4 * u * ref[0] / ref + 1e-15)


def test_jacobi_no_convergence_reported():
    rng = np.random.default_rng(32)
    B = rng.standard_normal((20, 20))
    with pytest.raises(O.OracleError) as e:
        O.jacobi_eigh(B + B.T, max_sweeps=1)
    assert e.value.code == O.E_NO_CONVERGENCE


@pytest.mark.parametrize("r", [1, 2, 3, 5, 16, 64, 150, 224])
def test_eig_real_vs_lapack_and_residual(r):
    """O6 on random nonsymmetric matrices: eigenvalues vs LAPACK dgeev (test side) after optimal
    matching, and the eigen-pair residual ‖A w − λ w‖ / (‖A‖‖w‖) ≤ 1e-12."""
    rng = np.random.default_rng(40 + r)
    A = rng.standard_normal((r, r)) / math.sqrt(r)
    lam, W = O.eig_real(A)
    assert match_eigs(lam, np.linalg.eigvals(A)) < 1e-11
    nA = np.linalg.norm(A, 2)
    for j in range(r):
        w = W[:, j]
        assert np.linalg.norm(A @ w - lam[j] * w) <= 1e-12 * nA * np.linalg.norm(w)
    # conjugate pairs come with conjugate vectors
    for j in range(r):
        if lam[j].imag > 0:
            k = int(np.argmin(np.abs(lam - np.conj(lam[j]))))
            assert abs(lam[k] - np.conj(lam[j])) < 1e-12


def test_eig_real_closed_forms():
    """Closed forms: a triangular matrix (λ = its diagonal), a companion matrix with known roots,
    a block-diagonal rotation/scaling (λ = ρ e^{±iθ}), a permutation cycle (roots of unity)."""
    T = np.triu(np.arange(1.0, 26.0).reshape(5, 5))
    assert match_eigs(O.eig_real(T)[0], np.diag(T)) < 1e-12
    roots = np.array([0.9, -0.5, 0.3 + 0.4j, 0.3 - 0.4j, 1.1])
    c = np.poly(roots).real                      # monic coefficients
    C = np.zeros((5, 5))
    C[0, :] = -c[1:]
    C[1:, :-1] = np.eye(4)
    assert match_eigs(O.eig_real(C)[0], roots) < 1e-12
    blocks = [(0.95, 0.3), (0.5, 1.2), (0.99, 0.01)]
    A = np.zeros((6, 6))
    for q, (rho, th) in enumerate(blocks):
        A[2 * q:2 * q + 2, 2 * q:2 * q + 2] = rho * np.array([[math.cos(th), -math.sin(th)],
                                                             [math.sin(th), math.cos(th)]])
    rng = np.random.default_rng(45)
    Qo, _ = np.linalg.qr(rng.standard_normal((6, 6)))
    ref = [rho * np.exp(s * 1j * th) for rho, th in blocks for s in (1, -1)]
    assert match_eigs(O.eig_real(Qo @ A @ Qo.T)[0], ref) < 1e-13
    P = np.roll(np.eye(7), 1, axis=0)
    assert match_eigs(O.eig_real(P)[0], np.exp(2j * np.pi * np.arange(7) / 7)) < 1e-13


def test_eig_real_degenerate():
    """Zero matrix, nilpotent Jordan block, identity: eigenvalues exact, no failure."""
    assert np.all(O.eig_real(np.zeros((4, 4)))[0] == 0)
    J = np.diag(np.ones(4), 1)
    lam, _ = O.eig_real(J)
    assert np.all(lam == 0)
    lam, W = O.eig_real(np.eye(3))
    assert np.all(lam == 1) and np.linalg.matrix_rank(W) == 3


def test_csolve_and_singular_detection():
    rng = np.random.default_rng(50)
    A = rng.standard_normal((30, 30)) + 1j * rng.standard_normal((30, 30))
    b = rng.standard_normal(30) + 1j * rng.standard_normal(30)
    x = O.csolve(A, b)
    assert np.linalg.norm(x - np.linalg.solve(A, b)) < 1e-12 * np.linalg.norm(x)
    A[:, 7] = 0.0
    assert O.csolve(A, b) is None


def test_clstsq_vs_lapack_and_rank():
    rng = np.random.default_rng(51)
    A = rng.standard_normal((40, 12)) + 1j * rng.standard_normal((40, 12))
    b = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    x, rk = O.clstsq(A, b)
    ref = np.linalg.lstsq(A, b, rcond=None)[0]
    assert rk == 12 and np.linalg.norm(x - ref) < 1e-12 * np.linalg.norm(ref)
    A[:, 3] = A[:, 5] * (2 - 1j)                    # rank 11: a basic solution with one zero
    x, rk = O.clstsq(A, b)
    ref = np.linalg.lstsq(A, b, rcond=None)[0]
    assert rk == 11
    assert abs(np.linalg.norm(A @ x - b) - np.linalg.norm(A @ ref - b)) < 1e-10 * np.linalg.norm(b)


def _planted_zero_mode(n=300, m=6, orth=True, seed=60):
    """Real modes, λ = {0, 0.9, -0.7, 0.5}: x_t = Σ b_j φ_j λ_j^t (so φ_0 appears in x_0 only)."""
    rng = np.random.default_rng(seed)
    lam = np.array([0.0, 0.9, -0.7, 0.5])
    b = np.array([1.3, 0.8, -0.6, 1.1])
    Phi = rng.standard_normal((n, 4))
    if orth:
        Phi, _ = np.linalg.qr(Phi)
    X = np.stack([Phi @ (b * lam ** t) for t in range(m + 1)], axis=1)   # 0^0 = 1
    return X, lam, b, Phi


def test_amplitudes_singular_branch_planted_zero_eigenvalue():
    """O9 singular branch (Q15): the window starting at t = 0 of planted
    dynamics with λ_0 = 0 gives Ã an exact zero eigenvalue; the oracle flags W_SINGULAR, gives the
    zero mode b = 0 and, with orthonormal modes (so that α₁'s zero-mode part is orthogonal to the
    kept eigenvectors), recovers the planted b_j of the others as b_j φ_j."""
    X, lam_p, b_p, Phi_p = _planted_zero_mode()
    d = O.dmd_window(X)
    assert d["r"] == 4 and d["amp_status"] == O.W_SINGULAR
    lam = d["lam"]
    assert match_eigs(lam, lam_p) < 1e-10
    j0 = int(np.argmin(np.abs(lam)))
    assert d["b"][j0] == 0
    Phi = O.modes(X[:, 1:], d)
    for j in range(4):
        if j == j0:
            continue
        k = int(np.argmin(np.abs(lam_p - lam[j])))
        assert np.linalg.norm(d["b"][j] * Phi[:, j] - b_p[k] * Phi_p[:, k]) < 1e-9 * abs(b_p[k])


def test_amplitudes_singular_branch_is_least_squares_on_kept_modes():
    """Non-orthogonal modes: the kept b are the least-squares solution of the kept columns of WΛ
    (LAPACK lstsq on the test side), not the oblique (left-eigenvector) solution."""
    X, lam_p, _, _ = _planted_zero_mode(orth=False, seed=61)
    d = O.dmd_window(X)
    assert d["amp_status"] == O.W_SINGULAR
    keep = np.abs(d["lam"]) >= 1e-7 * np.abs(d["lam"]).max()
    alpha1 = d["sigma"][:d["r"]] * d["V"][0, :d["r"]]
    wl = d["W"] * d["lam"][None, :]
    ref = np.linalg.lstsq(wl[:, keep], alpha1.astype(complex), rcond=None)[0]
    assert np.linalg.norm(d["b"][keep] - ref) < 1e-10 * np.linalg.norm(ref)
    assert np.all(d["b"][~keep] == 0)


def test_amplitudes_all_zero_spectrum():
    """Nilpotent window (x_t = 0 for t >= 1): every λ is 0 -> b = 0, W_SINGULAR, and the
    background index reports E_NO_VIABLE_MODE."""
    rng = np.random.default_rng(62)
    X = np.zeros((50, 5))
    X[:, 0] = rng.standard_normal(50)
    with pytest.raises(O.OracleError):
        O.dmd_window(X)                                # σ_1 > 0 but Ã = 0: no viable mode
    G = O.gram(X)
    d = O.dmd_from_gram(G)
    b, st = O.amplitudes(d)
    assert st == O.W_SINGULAR and np.all(b == 0) and np.all(d["lam"] == 0)


def test_order_eigs_rule_Q12():
    lam = np.array([0.5, -0.9, 0.9j, -0.9j, 0.9, 0.3 + 0.4j, 0.3 - 0.4j, 0.5])
    o = O.order_eigs(lam)
    # |λ| = 0.9 group: Re desc (0.9, then 0±0.9i, then -0.9), Im desc within equal Re
    assert list(lam[o]) == [0.9, 0.9j, -0.9j, -0.9, 0.5, 0.5, 0.3 + 0.4j, 0.3 - 0.4j]
    assert list(o[4:6]) == [0, 7]                      # equal keys keep input order


def test_background_first_window_constant_video():
    """Alg 3 first branch (Q24) on a constant video: λ_idx = 1, |L| = x in every column
    e = 0..m, S ≈ 0, empty mask."""
    rng = np.random.default_rng(63)
    x = 0.1 + 0.8 * rng.random(400)
    m = 8
    Z = np.tile(x[:, None], (1, m + 1))
    d = O.dmd_window(Z)
    assert d["r"] == 1 and abs(d["lam"][d["idx"]] - 1) < 1e-13
    L, S, mask = O.background_first_window([Z[:, k] for k in range(m + 1)], d, d["b"], d["idx"])
    assert L.shape == (400, m + 1)
    assert np.max(np.abs(S)) < 1e-12 and not mask.any()


def test_background_first_window_planted_exponents():
    """First branch uses exponents 0..m (Q24): on a planted rank-2 real decaying+constant video the
    background mode's reconstruction reproduces that mode's part of every column."""
    rng = np.random.default_rng(64)
    n, m = 300, 6
    bg = 0.5 + 0.1 * rng.random(n)
    dec = rng.random(n) * 0.2
    Z = np.stack([bg + dec * 0.6 ** t for t in range(m + 1)], axis=1)
    d = O.dmd_window(Z)
    L, S, _ = O.background_first_window([Z[:, k] for k in range(m + 1)], d, d["b"], d["idx"])
    assert abs(d["lam"][d["idx"]] - 1) < 1e-10
    assert np.max(np.abs(L - bg[:, None])) < 1e-9
    assert np.max(np.abs(S - np.stack([dec * 0.6 ** t for t in range(m + 1)], axis=1))) < 1e-9


def test_sparse_window_on_support_equals_dense_definition_bitwise():
    """The support-compressed sparse window has exactly the Gram of the scattered dense vectors."""
    st = synth.SparseDCTStream(N=64, k_low=8.0, n_shell=30, seed=12)
    slots = [st.frame(t) for t in range(6)]
    D = np.stack([st.dense(t) for t in range(6)], axis=1)
    assert np.array_equal(O.gram(O.sparse_window_on_support(slots)), O.gram(D))
