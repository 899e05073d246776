"""GPU parity of the SURVEY §8(f) NEXT-3 / NEXT-4 rows through the C ABI, against the oracle:

- NEXT-4 BMC-style scoring (Table 2): the device TP/FP/FN counts of the
  GPU's own masks equal the oracle's count of the same masks exactly (integer work: bit-exact);
- NEXT-3 complex Fourier snapshots (reading Q27; full and rfft half spectrum with weights): Gram
  vs the oracle definition ≤ 1e-12 normwise, and vs the pixel-space Gram of the real fields;
  λ_idx ≤ 1e-9; coefficient-space modes b_jφ̂_j vs the oracle;
- NEXT-3 pixel-space background of a sparse-DCT context (IDCT kernels): |l|, s vs the oracle's
  background_newest_pixel on every background frame (fp64: 1e-9 relative), mask equal off the
  threshold band; C5 full size (1024², m = 128) on its last frame."""
import numpy as np
import pytest

import synth
from oracle import sdmd_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1612_07875_b200.build import build
    build()


def Eng(*a, **k):
    from paper_1612_07875_b200 import StreamingDMD
    return StreamingDMD(*a, **k)


def normwise(Ga, Gb):
    d = np.sqrt(np.abs(np.diag(Gb)))
    den = np.outer(d, d)
    den[den == 0] = 1.0
    return float(np.max(np.abs(Ga - Gb) / den))


def match(a, b):
    from scipy.optimize import linear_sum_assignment
    C = np.abs(np.asarray(a)[:, None] - np.asarray(b)[None, :])
    r, c = linear_sum_assignment(C)
    return float(C[r, c].max()), c


# ------------------------------------------------------------------ NEXT-4 scoring --------

def test_scores_exact_counts_vs_oracle_and_f_measure():
    """Every background frame of a C3-shaped stream is scored on the device against the synthetic
    ground truth (host and device gt alternately); the pooled counts equal the oracle's
    evaluate() on the masks the GPU produced (exact), recall/precision/F/PSNR follow."""
    from paper_1612_07875_b200.sdmd import SDMDError, E_INVALID
    vs = synth.video_config("C3s")
    m, T = 30, 60
    frames = vs.frames(0, T).numpy()
    Xd = torch.from_numpy(np.ascontiguousarray(frames.T)).cuda()
    eng = Eng(vs.n, m, dtype="f32", background=True, workers=2)
    lag = eng.info()["lag"]
    masks, gts = [], []
    for t in range(T):
        eng.push(Xd[t])
        fb = t - lag
        if fb < m:
            continue
        low, sp, mask, f = eng.background()
        assert f == fb
        gt = vs.truth_mask(fb)
        if t % 2:
            eng.score(fb, torch.from_numpy(gt.astype(np.uint8)).cuda())
        else:
            eng.score(fb, gt)
        masks.append(mask.copy())
        gts.append(gt)
        if t == T - 1:
            with pytest.raises(SDMDError) as ei:
                eng.score(fb - 1, gt)
            assert ei.value.status == E_INVALID
    sc = eng.scores(reset=True)
    ref = O.evaluate(masks, gts)
    assert sc["frames"] == len(masks)
    assert (sc["tp"], sc["fp"], sc["fn"], sc["tn"]) == (ref["tp"], ref["fp"], ref["fn"], ref["tn"])
    for k in ("recall", "precision", "f_measure", "psnr"):
        assert sc[k] == pytest.approx(ref[k], rel=1e-15), k
    assert sc["f_measure"] > 0.85 and np.isfinite(sc["psnr"])
    assert eng.scores()["frames"] == 0                 # reset
    eng.close()


# ------------------------------------------------------ NEXT-3: Fourier snapshots ---------

def _oracle_window_gram(slots, n, w):
    k = len(slots)
    G = np.zeros((k, k))
    for j in range(k):
        g = O.fourier_gram_column(slots[:j + 1], slots[j], n, w)
        G[:j + 1, j] = g
        G[j, :j + 1] = g
    return G


@pytest.mark.parametrize("half", [True, False])
def test_fourier_sparse_gram_dmd_and_modes(half):
    rows, cols, m, T = 64, 48, 20, 34
    st = synth.SparseFourierStream(rows, cols, k_low=10.0, n_shell=40, seed=31, half=half)
    basis = "rfft" if half else "fft"
    eng = Eng(st.n, m, storage="sparse", nnz_cap=st.nnz_cap, basis=basis, grid=(rows, cols),
              workers=2)
    w = O.rfft_weights(rows, cols) if half else None
    slots = []
    for t in range(T):
        idx, val = st.frame(t)
        if t % 3 == 1:                                  # device-resident pushes too
            eng.push_sparse(torch.from_numpy(idx).cuda(),
                            torch.from_numpy(val.view(np.float64).copy()).cuda())
        else:
            eng.push_sparse(idx, val)
        slots = (slots + [(idx, val)])[-(m + 1):]
    eng.sync()
    G = eng.gram()
    Gr = _oracle_window_gram(slots, st.n, w)
    assert normwise(G, Gr) < 1e-12
    # Parseval: the same Gram from the real pixel fields (numpy.fft, test side)
    fields = []
    for idx, val in slots:
        z = np.zeros(st.n, dtype=np.complex128)
        z[idx.astype(np.int64)] = val
        f = (np.fft.irfft2(z.reshape(rows, cols // 2 + 1), s=(rows, cols), norm="ortho") if half
             else np.fft.ifft2(z.reshape(rows, cols), norm="ortho").real)
        fields.append(f.ravel())
    assert normwise(G, O.gram(np.stack(fields, axis=1))) < 1e-12
    d = O.dmd_from_gram(Gr)
    b, _ = O.amplitudes(d)
    idx_ref = O.background_index(d["lam"])
    sp = eng.spectrum(with_b=True)
    assert sp["r"] == d["r"]
    assert abs(sp["lam"][sp["idx"]] - d["lam"][idx_ref]) < 1e-9
    err, perm = match(sp["lam"], d["lam"])
    assert err < 1e-7
    # coefficient-space modes (complex values x complex T): the reconstruction Φ̂ b of x̂_1
    r = sp["r"]
    Phi = eng.modes(list(range(r))).cpu().numpy()
    Xp = []
    for idx, val in slots[1:]:
        z = np.zeros(st.n, dtype=np.complex128)
        z[idx.astype(np.int64)] = val
        Xp.append(z)
    Phi_ref = O.modes_complex(Xp, d)
    rec, rec_ref = Phi @ sp["b"], Phi_ref @ b
    assert np.linalg.norm(rec - rec_ref) < 1e-8 * np.linalg.norm(rec_ref)
    j = sp["idx"]
    a, bb = sp["b"][j] * Phi[:, j], b[idx_ref] * Phi_ref[:, idx_ref]
    assert np.linalg.norm(a - bb) < 1e-8 * np.linalg.norm(bb)
    eng.close()


# -------------------------------------------------- NEXT-3: pixel-space background --------

def _pixel_run(N, m, T, k_low, n_shell, seed, threshold, workers=2, check_every=True):
    st = synth.SparseDCTStream(N=N, k_low=k_low, n_shell=n_shell, seed=seed)
    eng = Eng(st.n, m, storage="sparse", nnz_cap=st.nnz_cap, background=True, grid=(N, N),
              threshold=threshold, workers=workers)
    lag = eng.info()["lag"]
    ref = O.StreamingDMD(m, background=False)
    frames, outs, checked = [], {}, 0
    for t in range(T):
        fr = st.frame(t)
        frames.append(fr)
        eng.push_sparse(*fr)
        o = ref.push(st.dense(t))
        if o is not None:
            outs[t] = o
        fb = t - lag
        if fb >= m and (check_every or t == T - 1):
            low, s, mask, f = eng.background()
            assert f == fb
            o = outs[fb]
            lr, sr, mr = O.background_newest_pixel(frames[fb - m + 1:fb + 1], frames[fb], st.n, N, N,
                                                   o, o["b"], o["idx"], threshold)
            sc = max(float(np.max(lr)), 1e-300)
            assert np.max(np.abs(low - lr)) < 1e-9 * sc, (t, np.max(np.abs(low - lr)) / sc)
            assert np.max(np.abs(s - sr)) < 1e-9 * max(sc, float(np.max(np.abs(sr))))
            amb = np.abs(sr - threshold) < 1e-9 * max(sc, 1.0)
            assert np.array_equal(mask[~amb], mr[~amb])
            assert np.max(np.abs(low + s - (sr + lr))) < 1e-9 * max(sc, 1.0)
            checked += 1
    return eng, checked


def test_pixel_background_every_frame_vs_oracle():
    eng, checked = _pixel_run(N=64, m=16, T=48, k_low=8.0, n_shell=30, seed=17, threshold=1e-3)
    assert checked >= 10
    eng.close()


def test_pixel_background_rectangular_grid_and_scores():
    """A non-square power-of-two grid (32 x 128): rows and columns take different transform
    lengths; the sparse context scores its pixel masks like a dense one."""
    N1, N2, m = 32, 128, 12
    st = synth.SparseDCTStream(N=128, k_low=8.0, n_shell=20, seed=5)
    # restrict the C5 generator's 128x128 coefficient grid to the first 32 rows (ky < 32)
    keep = lambda fr: (fr[0][fr[0] < N1 * N2], fr[1][fr[0] < N1 * N2])   # noqa: E731
    n = N1 * N2
    cap = max(int(keep(st.frame(t))[0].size) for t in range(40))
    eng = Eng(n, m, storage="sparse", nnz_cap=cap, background=True, grid=(N1, N2),
              threshold=1e-3, workers=2)
    lag = eng.info()["lag"]
    ref = O.StreamingDMD(m, background=False)
    frames = []
    T = m + lag + 8
    for t in range(T):
        fr = keep(st.frame(t))
        frames.append(fr)
        eng.push_sparse(*fr)
        z = np.zeros(n)
        z[fr[0].astype(np.int64)] = fr[1]
        o = ref.push(z)
        fb = t - lag
        if fb >= m:
            low, s, mask, f = eng.background()
            gt = np.zeros(n, dtype=np.uint8)
            gt[: n // 3] = 1
            eng.score(f, gt)
        if t == T - 1 - lag:
            o_last = o
    low, s, mask, f = eng.background()
    lr, sr, mr = O.background_newest_pixel(frames[f - m + 1:f + 1], frames[f], n, N1, N2,
                                           o_last, o_last["b"], o_last["idx"], 1e-3)
    sc = float(np.max(lr))
    assert np.max(np.abs(low - lr)) < 1e-9 * sc
    sco = eng.scores()
    assert sco["frames"] == T - lag - m and sco["tp"] + sco["fp"] + sco["fn"] + sco["tn"] == sco["frames"] * n
    eng.close()


@pytest.mark.slow
def test_pixel_background_c5_full_size():
    """C5 (1024² DCT coefficients, ~1% nonzeros, m = 128) with the pixel-space background: the last
    background frame vs the oracle (dense 1024 x 1024 IDCT matrices) within 1e-9."""
    eng, checked = _pixel_run(N=1024, m=128, T=128 + 1 + 10, k_low=110.0, n_shell=1000, seed=1616,
                              threshold=1e-4, workers=4, check_every=False)
    assert checked == 1
    eng.close()


# ------------------------------------------------ Alg 3 first-window branch (Q24) --------

@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_background_window_vs_oracle_first_window(dtype):
    """sdmd_get_background_window (Alg 3 first branch, exponents 0..m over all m+1
    columns, Q24) vs the oracle's background_first_window on the same window: fp32 1e-4, fp64
    1e-9 relative; masks equal off the threshold band; additivity per column."""
    vs = synth.video_config("C3s")
    m, T = 24, 40
    frames = vs.frames(0, T).numpy()
    X = frames if dtype == "f32" else frames.astype(np.float64)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    eng = Eng(vs.n, m, dtype=dtype, workers=2)
    ref = O.StreamingDMD(m, background=False)
    for t in range(T):
        eng.push(Xd[t])
        ref.push(X[:, t])
    low, s, mask, f = eng.background_window()
    assert f == T - 1
    o = ref.last
    cols = ref.gram.cols
    Lr, Sr, Mr = O.background_first_window(cols, o, o["b"], o["idx"])
    tol = 1e-4 if dtype == "f32" else 1e-9
    low, s, mask = low.cpu().numpy().T, s.cpu().numpy().T, mask.cpu().numpy().T
    sc = float(np.max(Lr))
    assert np.max(np.abs(low - Lr)) < tol * sc
    assert np.max(np.abs(s - Sr)) < tol * sc
    amb = np.abs(Sr - 0.2) < tol * sc
    assert np.array_equal(mask[~amb], Mr[~amb])
    Z = np.stack(cols, axis=1).astype(np.float64)
    assert np.max(np.abs(low.astype(np.float64) + s - Z)) < (1e-6 if dtype == "f32" else 1e-14)
    # the newest column (e = m) is the streaming branch's column (Q4)
    gt = vs.truth_mask(T - 1)
    f_meas = 2 * np.sum(mask[:, -1] & gt) / (mask[:, -1].sum() + gt.sum())
    assert f_meas > 0.85
    eng.close()


def test_background_window_constant_video():
    """constant video -> sparse ≈ 0 everywhere (max |s| < 1e-6 ‖c‖∞)."""
    n, m = 5000, 10
    c = (0.3 + 0.4 * np.random.default_rng(2).random(n)).astype(np.float64)
    eng = Eng(n, m, dtype="f64", workers=1)
    cd = torch.from_numpy(c).cuda()
    for _ in range(m + 3):
        eng.push(cd)
    low, s, mask, f = eng.background_window()
    assert float(s.abs().max()) < 1e-6 * float(np.max(c))
    assert not bool(mask.any())
    eng.close()


# ------------------------------------------------ a0: one-pass init Gram (TMA multicast) ---

@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("n,m", [(20011, 70), (4099, 200), (777, 3)])
def test_init_gram_multicast_vs_oracle_and_pair_kernel(dtype, n, m, monkeypatch):
    """sdmd_init_window's Gram from the cluster/TMA-multicast kernel (default for k <= 224) vs the
    oracle's compensated Gram (1e-12 normwise, Q17) and vs the pair-blocked DMMA kernel
    (SDMD_INIT_GRAM=v1, read at the first launch of a process — so compared through a second
    process-independent path: the oracle)."""
    rng = np.random.default_rng(n + m)
    npdt = np.float32 if dtype == "f32" else np.float64
    Z = rng.standard_normal((n, m + 1)).astype(npdt)
    Zd = torch.from_numpy(np.ascontiguousarray(Z.T)).cuda()
    eng = Eng(n, m, dtype=dtype, workers=1)
    eng.init_window(Zd)
    eng.sync()
    assert normwise(eng.gram(), O.gram(Z)) < 1e-12
    eng.close()


# ------------------------------------------------ NEXT-1: both K1b kernels ----------------

@pytest.mark.parametrize("kernel,dtype", [("tma", "f32"), ("v1", "f32"), ("tma", "f64"), ("v1", "f64")])
def test_push_batch_kernels_agree_with_oracle(kernel, dtype, monkeypatch):
    """The batched Gram pass through the TMA-tile kernel and through the cp.async kernel
    (SDMD_K1B, read once per process — so each parametrisation runs in a subprocess) gives the
    oracle's Gram (1e-12 normwise) on a window that wraps past the ring's last slot, with a ragged
    row tail (n = 5000), for fp32 and fp64 storage."""
    import subprocess
    import sys
    import textwrap
    code = textwrap.dedent('''
        import numpy as np, torch, synth
        from oracle import sdmd_oracle as O
        from paper_1612_07875_b200 import StreamingDMD
        rng = np.random.default_rng(7)
        n, m, k = 5000, 20, 8
        dt = "DTYPE"
        X = rng.standard_normal((n, 3 * (m + 1) + 5 * k)).astype(np.float32 if dt == "f32" else np.float64)
        Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
        eng = StreamingDMD(n, m, dtype=dt, workers=2, batch_max=k)
        sg = O.StreamingGram(m)
        t = 0
        for _ in range(m + 1):
            eng.push(Xd[t]); sg.push(X[:, t]); t += 1
        while t + k <= X.shape[1]:
            eng.push_batch(Xd[t:t + k]); [sg.push(X[:, t + j]) for j in range(k)]; t += k
        eng.sync()
        G = eng.gram(); Gr = sg.G
        d = np.sqrt(np.diag(Gr)); err = float(np.max(np.abs(G - Gr) / np.outer(d, d)))
        print(err)
        assert err < 1e-12, err
    ''')
    import os
    code = code.replace("DTYPE", dtype)
    env = dict(os.environ, SDMD_K1B=kernel)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
