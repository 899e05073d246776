"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): fp64 Gram entries 1e-12 (normwise, reading Q17), fp64
eigenvalues 1e-9 (optimal assignment), fp32 paths 1e-4 relative.  Eigenvectors are compared up
to sign/phase through projectors and scale-free products b_j φ_j (SURVEY §8(c) protocol)."""
import ctypes
import math

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


def dev_cols(X, dtype):
    """(T, n) contiguous device tensor from an (n, T) host array."""
    return torch.from_numpy(np.ascontiguousarray(X.T.astype(dtype))).to("cuda:0")


def _cudart():
    import glob
    import os
    import nvidia.cuda_runtime as cr
    libs = glob.glob(os.path.join(list(cr.__path__)[0], "lib", "libcudart.so*"))
    return ctypes.CDLL(libs[0])


def Eng(*a, **k):
    from paper_1612_07875_b200 import StreamingDMD
    return StreamingDMD(*a, **k)


# ------------------------------------------------------------------------------ C1 --------

def test_c1_every_window_closed_form_and_oracle():
    pm = synth.planted_c1()
    m, T = 16, 81
    X = pm.frames(0, T)
    Xd = dev_cols(X, np.float64)
    eng = Eng(pm.n, m, dtype="f64", workers=3)
    ref = O.StreamingDMD(m, background=False)
    for t in range(T):
        eng.push(Xd[t])
        out = ref.push(X[:, t])
        if t < m and t % 5 == 0:                     # warm-up: partial Gram
            eng.sync()
            assert normwise(eng.gram(), ref.gram.G) < 1e-12
        if out is None:
            continue
        eng.sync()
        assert normwise(eng.gram(), ref.gram.G) < 1e-12
        sp = eng.spectrum()
        assert sp["r"] == 4 and sp["frame"] == t
        e_cf, _ = match(sp["lam"], pm.lambdas)
        e_or, _ = match(sp["lam"], out["lam"])
        assert e_cf < 1e-9 and e_or < 1e-9, (t, e_cf, e_or)
        assert abs(sp["lam"][sp["idx"]] - out["lam"][out["idx"]]) < 1e-9 or \
            abs(sp["lam"][sp["idx"]] - np.conj(out["lam"][out["idx"]])) < 1e-9
    # last window: σ, projector, amplitudes, modes
    sv = eng.svd()
    r = sv["r"]
    assert np.max(np.abs(sv["sigma"][:r] - out["sigma"][:r]) / out["sigma"][:r]) < 1e-10
    P = sv["V"] @ sv["V"].T
    Pr = out["V"][:, :r] @ out["V"][:, :r].T
    assert np.max(np.abs(P - Pr)) < 1e-9
    sp = eng.spectrum(with_b=True)
    err, perm = match(sp["lam"], out["lam"])
    Phi = eng.modes(list(range(r))).cpu().numpy()
    Phi_ref = O.modes(ref.gram.cols[1:], out)
    for j in range(r):
        jr = perm[j]
        a = sp["b"][j] * Phi[:, j]
        b = out["b"][jr] * Phi_ref[:, jr]
        assert np.linalg.norm(a - b) < 1e-8 * np.linalg.norm(b), j
    eng.close()


# ----------------------------------------------------------------- ragged / dtypes --------

@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("n", [1000, 256 * 37 + 13, 70001])
def test_gram_stream_ragged(dtype, n):
    rng = np.random.default_rng(n)
    m, T = 9, 30
    npdt = np.float32 if dtype == "f32" else np.float64
    X = rng.standard_normal((n, T)).astype(npdt)
    Xd = dev_cols(X, npdt)
    eng = Eng(n, m, dtype=dtype, dmd=False, workers=1)
    sg = O.StreamingGram(m)
    for t in range(T):
        eng.push(Xd[t])
        sg.push(X[:, t])
        if t in (0, 3, m, m + 1, T - 1):
            eng.sync()
            assert normwise(eng.gram(), sg.G) < 1e-12
            g = eng.partial_gram_column()
            assert np.max(np.abs(g - sg.G[:, -1]) / np.sqrt(np.diag(sg.G) * sg.G[-1, -1])) < 1e-12
    eng.close()


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("n", [1, 5, 31, 33, 129])
def test_gram_stream_tiny_n(dtype, n):
    """Fewer rows than one warp / one tile; n = 1 makes every Gram entry a plain product."""
    rng = np.random.default_rng(1000 + n)
    m, T = 12, 20
    npdt = np.float32 if dtype == "f32" else np.float64
    X = rng.standard_normal((n, T)).astype(npdt)
    Xd = dev_cols(X, npdt)
    eng = Eng(n, m, dtype=dtype, dmd=False, workers=1)
    sg = O.StreamingGram(m)
    for t in range(T):
        eng.push(Xd[t])
        sg.push(X[:, t])
    eng.sync()
    assert normwise(eng.gram(), sg.G) < 1e-12
    eng.close()


def test_dmd_fewer_rows_than_window():
    """n = 6 < m = 16: the window Gram has rank 4 (two planted complex pairs); the truncation must
    find r = 4 and the eigenvalues must be the planted ones (closed form) and the oracle's."""
    pairs = [(np.exp(1j * np.pi / 8), np.exp(0.3j)), (0.99 * np.exp(1j * np.pi / 5), 0.5 * np.exp(1.1j))]
    pm = synth.PlantedModes(n=6, pairs=pairs, reals=[], seed=3)
    m, T = 16, 40
    X = pm.frames(0, T)
    Xd = dev_cols(X, np.float64)
    eng = Eng(pm.n, m, dtype="f64", workers=2)
    ref = O.StreamingDMD(m, background=False)
    for t in range(T):
        eng.push(Xd[t])
        out = ref.push(X[:, t])
    eng.sync()
    sp = eng.spectrum()
    assert sp["r"] == out["r"] == 4 and sp["frame"] == T - 1
    e_cf, _ = match(sp["lam"], pm.lambdas)
    e_or, _ = match(sp["lam"], out["lam"])
    assert e_cf < 1e-9 and e_or < 1e-9, (e_cf, e_or)
    eng.close()


@pytest.mark.parametrize("which", [0, 1, 2])
@pytest.mark.parametrize("m", [2, 3])
def test_minimum_window_planted_spectra(which, m):
    """The smallest windows the ABI accepts (m = 2, 3) on SPEC.md's planted spectra: the
    eigenvalues are the planted ones wherever the window holds the full rank."""
    pm = synth.planted_spec(which)
    T = 12
    X = pm.frames(0, T)
    Xd = dev_cols(X, np.float64)
    eng = Eng(pm.n, m, dtype="f64", workers=1)
    ref = O.StreamingDMD(m, background=False)
    for t in range(T):
        eng.push(Xd[t])
        out = ref.push(X[:, t])
    eng.sync()
    sp = eng.spectrum()
    assert sp["r"] == out["r"] and sp["frame"] == T - 1
    e_or, _ = match(sp["lam"], out["lam"])
    assert e_or < 1e-9, e_or
    if out["r"] == len(pm.lambdas):
        e_cf, _ = match(sp["lam"], pm.lambdas)
        assert e_cf < 1e-9, e_cf
    eng.close()


def test_host_input_and_zero_copy_slot():
    rng = np.random.default_rng(1)
    n, m, T = 5000, 6, 12
    X = rng.random((n, T)).astype(np.float32)
    eng = Eng(n, m, dtype="f32", dmd=False, workers=1)
    sg = O.StreamingGram(m)
    for t in range(T):
        if t % 2 == 0:
            eng.push(np.ascontiguousarray(X[:, t]))                 # HOST pointer
        else:
            ptr = eng.acquire_slot()                                  # zero-copy ingest
            src = torch.from_numpy(X[:, t].copy()).cuda()
            torch.cuda.synchronize()
            assert _cudart().cudaMemcpy(ctypes.c_void_p(ptr), ctypes.c_void_p(src.data_ptr()),
                                        ctypes.c_size_t(n * 4), 3) == 0
            eng.commit_slot()
        sg.push(X[:, t])
    eng.sync()
    assert normwise(eng.gram(), sg.G) < 1e-12
    eng.close()


def test_device_ready_pushes_with_background_vs_oracle():
    """SDMD_DEVICE_READY pushes (ring copies on the copy stream, overlapping the previous Gram
    pass) mixed with ordered DEVICE and HOST pushes: the Gram and the fused background equal the
    oracle's, frame by frame, across several ring wraps."""
    vs = synth.video_config("C3s")
    m, T = 12, 60
    frames = vs.frames(0, T).numpy()
    pool = torch.from_numpy(np.ascontiguousarray(frames.T)).cuda()
    torch.cuda.synchronize()
    eng = Eng(vs.n, m, dtype="f32", background=True, workers=2)
    lag = eng.info()["lag"]
    ref = O.StreamingDMD(m, background=True)
    outs = {}
    for t in range(T):
        if t % 3 == 2:
            eng.push(np.ascontiguousarray(frames[:, t]))
        else:
            eng.push(pool[t], ready=(t % 3 == 0))
        o = ref.push(frames[:, t].astype(np.float64))
        if o is not None:
            outs[t] = o
        fb = t - lag
        if fb >= m + 1 and t % 4 == 0:
            low, sp_, mask, f = eng.background()
            assert f == fb
            lr = outs[fb]["lowrank"]
            assert np.max(np.abs(low - lr)) / np.max(np.abs(lr)) < 1e-4, t
    eng.sync()
    assert normwise(eng.gram(), ref.gram.G) < 1e-12
    eng.close()


# ------------------------------------------------------------------------------ C2 --------

def test_c2_wake_fp64_rank21():
    pm = synth.cylinder_wake()
    m, T = 150, 158
    X = pm.frames(0, T)
    Xd = dev_cols(X, np.float64)
    eng = Eng(pm.n, m, dtype="f64", workers=2)
    ref = O.StreamingDMD(m, background=False)
    for t in range(T):
        eng.push(Xd[t])
        ref.push(X[:, t])
    eng.sync()
    out = ref.last
    assert normwise(eng.gram(), ref.gram.G) < 1e-12
    sp = eng.spectrum()
    assert sp["r"] == 21 == out["r"]
    lam_cf = np.array([1.0] + [np.exp(s * 1j * k * 2 * np.pi / 30) for k in range(1, 11)
                               for s in (1, -1)])
    assert match(sp["lam"], lam_cf)[0] < 1e-9
    assert match(sp["lam"], out["lam"])[0] < 1e-9
    assert abs(sp["lam"][sp["idx"]] - 1.0) < 1e-9
    sv = eng.svd(with_V=False)
    s_ref = out["sigma"]
    keep = s_ref / s_ref[0] >= 1e-4
    assert np.max(np.abs(sv["sigma"][keep] - s_ref[keep]) / s_ref[keep]) < 1e-9
    eng.close()


# ----------------------------------------------------------------- video background ------

@pytest.mark.parametrize("workers", [1, 3])
def test_video_background_parity(workers):
    vs = synth.video_config("C3s")
    m, T = 30, 48
    frames = vs.frames(0, T).numpy()                 # (n, T) fp32
    Xd = torch.from_numpy(np.ascontiguousarray(frames.T)).cuda()
    eng = Eng(vs.n, m, dtype="f32", background=True, workers=workers)
    lag = eng.info()["lag"]
    ref = O.StreamingDMD(m, background=True)
    outs = {}
    for t in range(T):
        eng.push(Xd[t])
        o = ref.push(frames[:, t])
        if o is not None:
            outs[t] = o
    eng.sync()
    low, sp, mask, fb = eng.background()
    assert fb == T - 1 - lag
    o = outs[fb]
    x = frames[:, fb].astype(np.float64)
    rel = np.max(np.abs(low - o["lowrank"])) / np.max(np.abs(o["lowrank"]))
    assert rel < 1e-4, rel
    assert np.max(np.abs(sp - o["sparse"])) < 1e-4 * np.max(np.abs(x))
    near = np.abs(o["sparse"] - 0.2) < 1e-4
    assert np.all(mask[~near] == o["mask"][~near])
    # additivity on the fp32 outputs (up to one rounding) and F-measure sanity
    assert np.max(np.abs(low.astype(np.float64) + sp - x)) < 1e-6
    gt = vs.truth_mask(fb)
    tp = np.sum(mask & gt)
    f = 2 * tp / (mask.sum() + gt.sum())
    assert f > 0.85, f
    eng.close()


def test_background_async_readback_every_frame():
    """SDMD_HOST_ASYNC read-back after every push (the e2e path): the double-buffered outputs of
    each background pass, copied on the D2H stream while the next Gram pass runs, equal the
    oracle's background of the frame the call reports."""
    vs = synth.video_config("C3s")
    m, T = 30, 52
    frames = vs.frames(0, T).numpy()
    Xd = torch.from_numpy(np.ascontiguousarray(frames.T)).cuda()
    eng = Eng(vs.n, m, dtype="f32", background=True, workers=2)
    ref = O.StreamingDMD(m, background=True)
    outs, bufs = {}, {}
    for t in range(T):
        eng.push(Xd[t])
        o = ref.push(frames[:, t])
        if o is not None:
            outs[t] = o
        low = torch.empty(vs.n, dtype=torch.float32, pin_memory=True)
        mask = torch.empty(vs.n, dtype=torch.uint8, pin_memory=True)
        try:
            fb = eng.background_async(mask=mask, lowrank=low)
        except Exception:
            continue                                    # no background pass enqueued yet
        bufs[fb] = (low, mask)
    eng.sync()
    lag = eng.info()["lag"]
    assert sorted(bufs) == list(range(m, T - lag))
    for fb, (low, mask) in bufs.items():
        o = outs[fb]
        rel = np.max(np.abs(low.numpy() - o["lowrank"])) / np.max(np.abs(o["lowrank"]))
        assert rel < 1e-4, (fb, rel)
        near = np.abs(o["sparse"] - 0.2) < 1e-4
        assert np.all(mask.numpy()[~near] == o["mask"][~near]), fb
    eng.close()


@pytest.mark.parametrize("nb", [2, 3])
def test_multi_mode_background_planted_closed_form(nb):
    """NEXT-2 (reading Q25) on planted C1b (λ = 1 plus two conjugate pairs, fp64): the
    background column built from the mode set B (nb = 2 → {1, e^{±iπ/8}} after conjugate
    closure, nb = 3 → the same) equals the planted contributions of those modes to the frame
    (closed form) and the oracle's multi-mode background."""
    pm = synth.planted_c1(with_unit_mode=True)
    m, T = 16, 40
    X = pm.frames(0, T)
    Xd = dev_cols(X, np.float64)
    eng = Eng(pm.n, m, dtype="f64", background=True, workers=2, bg_modes=nb)
    ref = O.StreamingDMD(m, background=True, bg_modes=nb)
    outs = {}
    for t in range(T):
        eng.push(Xd[t])
        o = ref.push(X[:, t])
        if o is not None:
            outs[t] = o
    eng.sync()
    low, sp, mask, fb = eng.background()
    o = outs[fb]
    assert len(o["bg_set"]) == 3
    prods = pm.mode_products(fb)
    l_cf = sum(v for lam, v in prods.items()
               if abs(lam - 1.0) < 1e-12 or abs(abs(np.angle(lam)) - np.pi / 8) < 1e-12)
    scale = np.max(np.abs(l_cf))
    assert np.max(np.abs(low - np.abs(l_cf))) < 1e-9 * scale
    assert np.max(np.abs(low - o["lowrank"])) < 1e-9 * scale
    eng.close()


def test_single_mode_background_fp64_real_coefficients_closed_form():
    """Alg 3 as written on planted C1b in fp64 (λ_idx = 1 is real, so K1 takes its real-coefficient
    background path with fp64 storage): the background column equals the planted contribution
    of the unit mode to the frame (closed form) and the oracle's background."""
    pm = synth.planted_c1(with_unit_mode=True)
    m, T = 16, 40
    X = pm.frames(0, T)
    Xd = dev_cols(X, np.float64)
    eng = Eng(pm.n, m, dtype="f64", background=True, workers=2)
    ref = O.StreamingDMD(m, background=True)
    outs = {}
    for t in range(T):
        eng.push(Xd[t])
        o = ref.push(X[:, t])
        if o is not None:
            outs[t] = o
    eng.sync()
    low, sp, mask, fb = eng.background()
    prods = pm.mode_products(fb)
    l_cf = sum(v for lam, v in prods.items() if abs(lam - 1.0) < 1e-12)
    scale = np.max(np.abs(l_cf))
    assert np.max(np.abs(low - np.abs(l_cf))) < 1e-9 * scale
    assert np.max(np.abs(low - outs[fb]["lowrank"])) < 1e-9 * scale
    assert np.max(np.abs(low + sp - X[:, fb])) < 1e-12 * np.max(np.abs(X[:, fb]))
    eng.close()


def test_multi_mode_background_video():
    """NEXT-2 on the C3-shaped video (fp32, r ≈ m): background from the 4 slowest modes (plus a
    conjugate partner) against the oracle, same tolerances as the single-mode video test."""
    vs = synth.video_config("C3s")
    m, T = 30, 48
    frames = vs.frames(0, T).numpy()
    Xd = torch.from_numpy(np.ascontiguousarray(frames.T)).cuda()
    eng = Eng(vs.n, m, dtype="f32", background=True, workers=2, bg_modes=4)
    ref = O.StreamingDMD(m, background=True, bg_modes=4)
    outs = {}
    for t in range(T):
        eng.push(Xd[t])
        o = ref.push(frames[:, t])
        if o is not None:
            outs[t] = o
    eng.sync()
    low, sp, mask, fb = eng.background()
    o = outs[fb]
    x = frames[:, fb].astype(np.float64)
    rel = np.max(np.abs(low - o["lowrank"])) / np.max(np.abs(o["lowrank"]))
    assert rel < 1e-4, rel
    near = np.abs(o["sparse"] - 0.2) < 1e-4
    assert np.all(mask[~near] == o["mask"][~near])
    assert np.max(np.abs(low.astype(np.float64) + sp - x)) < 1e-6
    eng.close()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_buildup_dmd_every_window(dtype):
    """NEXT-4: with buildup the DMD runs from the 2nd frame on the growing window.
    Planted C1: from 4 X-columns the spectrum is the planted one (closed form, 1e-9); every
    build-up window's σ and λ match the oracle's; after the window fills, the stream continues
    as without buildup."""
    pm = synth.planted_c1()
    m, T = 16, 24
    npdt = np.float64 if dtype == "f64" else np.float32
    X = pm.frames(0, T).astype(npdt)
    Xd = dev_cols(X, npdt)
    eng = Eng(pm.n, m, dtype=dtype, workers=2, buildup=True)
    ref = O.StreamingDMD(m, background=False, buildup=True)
    for t in range(T):
        eng.push(Xd[t])
        out = ref.push(X[:, t].astype(np.float64))
        if t == 0:
            assert out is None
            continue
        eng.sync()
        sp = eng.spectrum()
        assert sp["frame"] == t and sp["r"] == out["r"], (t, sp["r"], out["r"])
        tol = 1e-9 * max(1.0, np.abs(out["lam"]).max())
        if t >= 4 and dtype == "f64":
            assert match(sp["lam"], pm.lambdas)[0] < 1e-9, t
        assert match(sp["lam"], out["lam"])[0] < tol, t
        sv = eng.svd()
        w = min(t, m)
        r = sv["r"]
        assert np.all(sv["sigma"][w:] == 0.0)
        assert np.max(np.abs(sv["sigma"][:r] - out["sigma"][:r]) / out["sigma"][:r]) < 1e-10, t
        P = sv["V"][:w] @ sv["V"][:w].T
        Pr = out["V"][:, :r] @ out["V"][:, :r].T
        assert np.max(np.abs(P - Pr)) < 1e-9, t
    eng.close()


# ------------------------------------------------------------------- robustness ----------

def test_nonfinite_frame_rejected_atomically():
    from paper_1612_07875_b200 import SDMDError
    rng = np.random.default_rng(2)
    n, m = 3000, 8
    X = rng.standard_normal((n, 30))
    Xd = dev_cols(X, np.float64)
    eng = Eng(n, m, dtype="f64", workers=2)
    ref = O.StreamingDMD(m, background=False)
    for t in range(15):
        eng.push(Xd[t])
        ref.push(X[:, t])
    eng.sync()
    G0 = eng.gram()
    bad = Xd[15].clone()
    bad[123] = float("nan")
    eng.push(bad)
    _push_through_poison(eng, Xd, 16, 1)             # discarded by the poison contract (or refused)
    with pytest.raises(SDMDError) as e:
        eng.sync()
    assert e.value.status == 2 and e.value.failed_frame == 15
    assert np.array_equal(eng.gram(), G0)
    assert eng.info()["frames"] == 15
    for t in range(16, 30):
        eng.push(Xd[t])
        ref.push(X[:, t])
    eng.sync()
    assert normwise(eng.gram(), ref.gram.G) < 1e-12
    assert match(eng.spectrum()["lam"], ref.last["lam"])[0] < 1e-9
    eng.close()


def _push_through_poison(eng, frames_dev, t0, count):
    """Push frames t0 .. t0+count-1 after a rejected frame, before any sync: the first few are
    accepted (their ring slots cannot hold anything the rolled-back state reads), then the ring
    guard refuses further pushes with E_NONFINITE.  Returns how many were accepted."""
    from paper_1612_07875_b200 import SDMDError
    accepted = 0
    for t in range(t0, t0 + count):
        try:
            eng.push(frames_dev[t])
            accepted += 1
        except SDMDError as e:
            assert e.status == 2
    return accepted


def test_nonfinite_then_many_pushes_before_sync_leaves_state_intact():
    """a rejected frame followed by many pushes before sync (more than the ring's
    spare slots) must leave the rolled-back state bit-identical; the resumed stream matches the
    oracle (Gram 1e-12, λ 1e-9)."""
    from paper_1612_07875_b200 import SDMDError
    rng = np.random.default_rng(12)
    n, m = 3000, 8
    X = rng.standard_normal((n, 80))
    Xd = dev_cols(X, np.float64)
    eng = Eng(n, m, dtype="f64", workers=2)
    ref = O.StreamingDMD(m, background=False)
    for t in range(15):
        eng.push(Xd[t])
        ref.push(X[:, t])
    eng.sync()
    G0 = eng.gram()
    bad = Xd[15].clone()
    bad[123] = float("nan")
    eng.push(bad)
    acc = _push_through_poison(eng, Xd, 16, 2 * (m + eng.info()["ring_slots"]))
    assert acc < eng.info()["ring_slots"] - m          # the guard stopped the writes
    with pytest.raises(SDMDError) as e:
        eng.sync()
    assert e.value.status == 2 and e.value.failed_frame == 15
    assert np.array_equal(eng.gram(), G0)
    assert eng.info()["frames"] == 15
    for t in range(16, 80):
        eng.push(Xd[t])
        ref.push(X[:, t])
    eng.sync()
    assert normwise(eng.gram(), ref.gram.G) < 1e-12
    assert match(eng.spectrum()["lam"], ref.last["lam"])[0] < 1e-9
    eng.close()


def test_nonfinite_then_many_pushes_with_background():
    """The same with the fused background (its lag keeps older ring slots live): after the
    rollback and lag + 6 valid frames, the newest background column equals the oracle's."""
    from paper_1612_07875_b200 import SDMDError
    vs = synth.video_config("C3s")
    m = 30
    eng = Eng(vs.n, m, dtype="f32", background=True, workers=2)
    lag = eng.info()["lag"]
    T = m + 2 * lag + 40
    frames = vs.frames(0, T).numpy()
    Xd = torch.from_numpy(np.ascontiguousarray(frames.T)).cuda()
    ref = O.StreamingDMD(m, background=True)
    p = m + lag + 3
    for t in range(p):
        eng.push(Xd[t])
        ref.push(frames[:, t])
    eng.sync()
    bad = Xd[p].clone()
    bad[7] = float("inf")
    eng.push(bad)
    _push_through_poison(eng, Xd, p + 1, T - p - 1)
    with pytest.raises(SDMDError) as e:
        eng.sync()
    assert e.value.failed_frame == p and eng.info()["frames"] == p
    outs = {}
    for t in range(p + 1, T):                         # frame p's data is skipped: the valid
        eng.push(Xd[t])                               # stream continues with frame p+1
        o = ref.push(frames[:, t])
        outs[ref.frames - 1] = o
    eng.sync()
    low, sp, mask, fb = eng.background()
    o = outs[fb]
    rel = np.max(np.abs(low - o["lowrank"])) / np.max(np.abs(o["lowrank"]))
    assert rel < 1e-4, rel
    assert normwise(eng.gram(), ref.gram.G) < 1e-12
    eng.close()


def test_push_batch_flow_control_many_batches_without_sync():
    """hundreds of dmd_every batches with one slow eigen worker and no sync.  The
    batched Gram pass may not run ahead of the eigen work it would overwrite: every K1b pass that
    commits frames up to t_last starts after the eigen tasks of all frames <= t_last - lag - 2
    have finished (device timeline), and the final Gram / spectrum match the closed form."""
    pm = synth.planted_c1()
    m, k, nb = 16, 8, 50                             # t <= 416: 0.99^t stays well resolved
    T = m + 1 + k * nb
    X = pm.frames(0, T)
    Xd = dev_cols(X, np.float64)
    eng = Eng(pm.n, m, dtype="f64", workers=1, batch_max=k)
    L = eng.info()["lag"]
    for t in range(m + 1):
        eng.push(Xd[t])
    eng.sync()
    eng.set_timing(True)
    eng.stats(reset=True)
    t = m + 1
    for _ in range(nb):
        eng.push_batch(Xd[t:t + k], dmd_every=True)
        t += k
    eng.sync()
    tl = eng.timeline()
    k4b_end = {int(f): e for f, kind, s, e in tl if kind == 2}
    passes = [(int(f), s) for f, kind, s, e in tl if kind == 0]
    assert len(passes) == nb and len(k4b_end) == nb * k
    for f_last, start in passes:                      # eigen tasks enqueued before this batch
        done_before = [e for f, e in k4b_end.items() if f <= min(f_last - L - 2, f_last - k)]
        if done_before:
            assert max(done_before) <= start + 1e-3, (f_last, max(done_before), start)
    ref = O.StreamingGram(m)
    for tt in range(T - m - 1, T):
        ref.push(X[:, tt])
    assert normwise(eng.gram(), ref.G) < 1e-12
    sp = eng.spectrum()
    assert sp["frame"] == T - 1 and match(sp["lam"], pm.lambdas)[0] < 1e-9
    eng.close()


def test_zero_window_and_warmup_status():
    from paper_1612_07875_b200 import SDMDError
    n, m = 2048, 5
    eng = Eng(n, m, dtype="f32", workers=1)
    z = torch.zeros(n, device="cuda:0")
    for t in range(m):
        eng.push(z)
    eng.sync()
    with pytest.raises(SDMDError) as e:
        eng.spectrum()
    assert e.value.status == 3                      # window not full
    eng.push(z)
    eng.sync()
    with pytest.raises(SDMDError) as e:
        eng.spectrum()
    assert e.value.status == 4                      # σ₁ == 0
    eng.close()


def test_determinism_bitwise():
    rng = np.random.default_rng(4)
    n, m, T = 50000, 20, 30
    X = rng.random((n, T)).astype(np.float32)
    Xd = dev_cols(X, np.float32)
    res = []
    for _ in range(2):
        eng = Eng(n, m, dtype="f32", workers=2)
        for t in range(T):
            eng.push(Xd[t])
        eng.sync()
        res.append((eng.gram(), eng.spectrum()["lam"], eng.svd()["sigma"]))
        eng.close()
    for a, b in zip(res[0], res[1]):
        assert np.array_equal(a, b)


def test_determinism_bitwise_sparse_batch_background():
    """Every reduction is fixed-order: the sparse Gram (K3 partials), batched pushes (K1b) and the
    fused background pass (K1, 4-mode set) repeat bit for bit across contexts."""
    st = synth.SparseDCTStream(N=96, k_low=10.0, n_shell=40, seed=31)
    frames = [st.frame(t) for t in range(28)]
    rng = np.random.default_rng(6)
    n, m = 40000, 12
    X = rng.random((n, 36)).astype(np.float32)
    Xd = dev_cols(X, np.float32)
    runs = []
    workers = 3
    for _ in range(2):
        sp = Eng(st.n, 10, storage="sparse", nnz_cap=st.nnz_cap, workers=workers)
        for idx, val in frames:
            sp.push_sparse(idx, val)
        sp.sync()
        bt = Eng(n, m, dtype="f32", dmd=False, workers=workers, batch_max=8)
        for t in range(m + 1):                                # batches need a full window
            bt.push(Xd[t])
        for t0 in range(m + 1, 36, 8):
            bt.push_batch(Xd[t0:min(t0 + 8, 36)])
        bt.sync()
        bg = Eng(n, m, dtype="f32", workers=workers, background=True, bg_modes=4, lag=4)
        for t in range(36):
            bg.push(Xd[t])
        bg.sync()
        low, sparse, mask, fr = bg.background()
        runs.append((sp.gram(), sp.spectrum()["lam"], bt.gram(), bg.gram(), low, sparse, mask,
                     np.array([fr])))
        for e in (sp, bt, bg):
            e.close()
    for a, b in zip(runs[0], runs[1]):
        assert np.array_equal(a, b)


# --------------------------------------------------------------- init window (K2) --------

@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_init_window_dmma_gram(dtype):
    rng = np.random.default_rng(5)
    n, m = 20011, 70
    npdt = np.float32 if dtype == "f32" else np.float64
    Z = rng.standard_normal((n, m + 1)).astype(npdt)
    Zd = dev_cols(Z, npdt)                           # (m+1, n) row-major = n x (m+1) col-major
    eng = Eng(n, m, dtype=dtype, workers=1)
    eng.init_window(Zd)
    eng.sync()
    Gr = O.gram(Z)
    assert normwise(eng.gram(), Gr) < 1e-12
    d = O.dmd_window(Z)
    sp = eng.spectrum()
    assert match(sp["lam"], d["lam"])[0] < 1e-9 * max(1.0, np.abs(d["lam"]).max())
    # stream on from the initialised window
    sg = O.StreamingGram(m)
    for t in range(m + 1):
        sg.push(Z[:, t])
    X2 = rng.standard_normal((n, 4)).astype(npdt)
    X2d = dev_cols(X2, npdt)
    for t in range(4):
        eng.push(X2d[t])
        sg.push(X2[:, t])
    eng.sync()
    assert normwise(eng.gram(), sg.G) < 1e-12
    eng.close()


def test_init_window_nonfinite_rejected_whole():
    """A first window with a NaN (or Inf) is rejected: SDMD_E_NONFINITE, 0 frames; the
    stream then starts cleanly from a good window."""
    from paper_1612_07875_b200 import SDMDError
    rng = np.random.default_rng(8)
    n, m = 5000, 12
    Z = rng.standard_normal((n, m + 1))
    eng = Eng(n, m, dtype="f64", workers=1)
    for bad in (float("nan"), float("inf")):
        Zb = Z.copy()
        Zb[777, 5] = bad
        with pytest.raises(SDMDError) as e:
            eng.init_window(dev_cols(Zb, np.float64))
        assert e.value.status == 2
        assert eng.info()["frames"] == 0
    eng.init_window(dev_cols(Z, np.float64))
    eng.sync()
    assert eng.info()["frames"] == m + 1
    assert normwise(eng.gram(), O.gram(Z)) < 1e-12
    assert match(eng.spectrum()["lam"], O.dmd_window(Z)["lam"])[0] < 1e-9
    eng.close()


def test_maximum_workers_every_window_and_limits():
    """The largest worker-stream count the ABI accepts (24): every window's spectrum, read after
    each push, still equals the closed form; 25 workers and batches above batch_max are refused."""
    from paper_1612_07875_b200 import SDMDError
    pm = synth.planted_c1()
    m, T = 16, 60
    X = pm.frames(0, T)
    Xd = dev_cols(X, np.float64)
    with pytest.raises(SDMDError) as e:
        Eng(pm.n, m, dtype="f64", workers=25)
    assert e.value.status == 1
    eng = Eng(pm.n, m, dtype="f64", workers=24, batch_max=4)
    for t in range(T):
        eng.push(Xd[t])
        if t >= m + 1 and t % 3 == 0:
            eng.sync()
            sp = eng.spectrum()
            assert sp["frame"] == t and sp["r"] == 4
            assert match(sp["lam"], pm.lambdas)[0] < 1e-9, t
    with pytest.raises(SDMDError) as e:
        eng.push_batch(dev_cols(pm.frames(T, T + 5), np.float64))
    assert e.value.status == 1
    eng.push_batch(dev_cols(pm.frames(T, T + 4), np.float64))
    eng.sync()
    sp = eng.spectrum()
    assert sp["frame"] == T + 3 and match(sp["lam"], pm.lambdas)[0] < 1e-9
    eng.close()


def _planted_window(n, m, npairs, seed):
    """n x (m+1) window of 2·npairs planted DMD modes x_t = Σ 2 Re(b_j φ_j λ_j^t) (fp64)."""
    rng = np.random.default_rng(seed)
    rho = rng.uniform(0.9, 1.0, npairs)
    th = np.linspace(0.05, 3.0, npairs) + rng.uniform(-0.01, 0.01, npairs)
    lam = rho * np.exp(1j * th)
    phi = (rng.standard_normal((n, npairs)) + 1j * rng.standard_normal((n, npairs))) / np.sqrt(2 * n)
    b = rng.standard_normal(npairs) + 1j * rng.standard_normal(npairs)
    t = np.arange(m + 1)
    return 2.0 * np.real((phi * b[None, :]) @ (lam[:, None] ** t[None, :]))


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_modes_tensor_core_multi_chunk(dtype):
    """K2 (a0 init Gram + a12 modes) on a ragged n with r = 40 > 32 modes (two mode chunks of
    the modes kernel) and k = 71 (two Gram column blocks): b_j φ_j per mode and the
    reconstruction Φ b against the oracle on the same (fp32-rounded) window."""
    n, m, npairs = 20011, 70, 20
    npdt = np.float32 if dtype == "f32" else np.float64
    Z = _planted_window(n, m, npairs, seed=11).astype(npdt)
    eng = Eng(n, m, dtype=dtype, workers=1, r_max=2 * npairs)
    eng.init_window(dev_cols(Z, npdt))
    eng.sync()
    Zr = Z.astype(np.float64)
    Gr = O.gram(Zr)
    assert normwise(eng.gram(), Gr) < 1e-12
    d = O.dmd_from_gram(Gr, r_max=2 * npairs)
    b_ref, _ = O.amplitudes(d)
    sp = eng.spectrum(with_b=True)
    r = sp["r"]
    assert r == d["r"] == 2 * npairs
    err, perm = match(sp["lam"], d["lam"])
    assert err < 1e-9
    Phi = eng.modes(list(range(r))).cpu().numpy()
    Phi_ref = O.modes([Zr[:, k] for k in range(1, m + 1)], d)
    for j in range(r):
        a = sp["b"][j] * Phi[:, j]
        bb = b_ref[perm[j]] * Phi_ref[:, perm[j]]
        assert np.linalg.norm(a - bb) < 1e-8 * np.linalg.norm(bb), j
    rec, rec_ref = Phi @ sp["b"], Phi_ref @ b_ref
    assert np.linalg.norm(rec - rec_ref) < 1e-9 * np.linalg.norm(rec_ref)
    # a subset of columns in a non-contiguous order lands in the requested slots
    cols = [r - 1, 0, 33, 5]
    Ps = eng.modes(cols).cpu().numpy()
    assert np.array_equal(Ps, Phi[:, cols])
    eng.close()


def test_init_window_c4_full_size_sampled():
    """K2 init Gram at BASELINE config 4's full size (n = 24,883,200, m = 200, fp32): sampled
    entries against fp64 dots of CPU-regenerated frames (normwise 1e-12, reading Q17)."""
    vs = synth.video_config("C4")
    m = 200
    Zd = torch.empty((m + 1, vs.n), dtype=torch.float32, device="cuda:0")
    for t in range(m + 1):
        Zd[t] = vs.frame(t, device="cuda:0")
    eng = Eng(vs.n, m, dtype="f32", workers=1)
    eng.init_window(Zd)
    eng.sync()
    del Zd
    G = eng.gram()
    assert np.array_equal(G, G.T)
    cache = {}

    def fr(t):
        if t not in cache:
            cache[t] = vs.frame(t).numpy()
        return cache[t]
    for i, j in ((0, 0), (0, 200), (57, 123), (199, 200), (200, 200), (123, 123)):
        ref = float(O.gram_column([fr(i)], fr(j))[0])         # compensated oracle dot (O1)
        assert abs(G[i, j] - ref) <= 1e-12 * math.sqrt(G[i, i] * G[j, j]), (i, j)
    eng.close()


# ------------------------------------------------------------- batched push (K1b) --------

def test_push_batch_c1_matches_streaming_oracle():
    """K1b (k frames per pass, DMMA) on the planted C1 stream: after every batch the Gram equals
    the oracle's frame-by-frame streamed Gram (normwise 1e-12), and every window's spectrum (DMD
    for each of the k windows) matches the closed-form eigenvalues (1e-9)."""
    pm = synth.planted_c1()
    m = 16
    ks = [4, 3, 8, 1, 5, 8, 2]
    T = m + 1 + sum(ks)
    X = pm.frames(0, T)
    Xd = dev_cols(X, np.float64)
    eng = Eng(pm.n, m, dtype="f64", workers=3, batch_max=8)
    ref = O.StreamingGram(m)
    for t in range(m + 1):
        eng.push(Xd[t])
        ref.push(X[:, t])
    t = m + 1
    for k in ks:
        eng.push_batch(Xd[t:t + k])
        for j in range(k):
            ref.push(X[:, t + j])
        t += k
        eng.sync()
        assert normwise(eng.gram(), ref.G) < 1e-12, (t, k)
        sp = eng.spectrum()
        assert sp["frame"] == t - 1 and sp["r"] == 4
        assert match(sp["lam"], pm.lambdas)[0] < 1e-9
    eng.close()


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("n", [70001, 256 * 9 + 40])
def test_push_batch_ragged_and_catch_up(dtype, n):
    """Ragged n, both storage types, k = 8 and a batch that wraps the ring; catch-up mode
    (dmd_every=False) computes only the newest window's DMD, equal to the oracle's."""
    rng = np.random.default_rng(n % 97)
    m = 40
    npdt = np.float32 if dtype == "f32" else np.float64
    T = m + 1 + 8 * 6 + 3
    X = rng.standard_normal((n, T)).astype(npdt)
    Xd = dev_cols(X, npdt)
    eng = Eng(n, m, dtype=dtype, workers=2, batch_max=8)
    ref = O.StreamingGram(m)
    for t in range(m + 1):
        eng.push(Xd[t])
        ref.push(X[:, t].astype(np.float64))
    t = m + 1
    while t < T:
        k = min(8, T - t)
        eng.push_batch(Xd[t:t + k], dmd_every=False)
        for j in range(k):
            ref.push(X[:, t + j].astype(np.float64))
        t += k
    eng.sync()
    assert normwise(eng.gram(), ref.G) < 1e-12
    d = O.dmd_from_gram(ref.G)
    sp = eng.spectrum()
    assert sp["frame"] == T - 1 and sp["r"] == d["r"]
    sv = eng.svd()
    r = sv["r"]
    big = d["sigma"][:r] >= 1e-4 * d["sigma"][0]
    assert np.max(np.abs(sv["sigma"][:r][big] - d["sigma"][:r][big]) / d["sigma"][:r][big]) < 1e-10
    eng.close()


def test_push_batch_nonfinite_rejected_as_a_whole():
    pm = synth.planted_c1()
    m = 16
    X = pm.frames(0, m + 1 + 8)
    Xd = dev_cols(X, np.float64)
    eng = Eng(pm.n, m, dtype="f64", workers=1, batch_max=8)
    for t in range(m + 1):
        eng.push(Xd[t])
    eng.sync()
    G0 = eng.gram()
    bad = Xd[m + 1:m + 1 + 6].clone()
    bad[3, 17] = float("nan")
    from paper_1612_07875_b200.sdmd import SDMDError
    eng.push_batch(bad)
    with pytest.raises(SDMDError) as ei:
        eng.sync()
    assert ei.value.status == 2 and ei.value.failed_frame == m + 1 + 3
    assert eng.info()["frames"] == m + 1
    assert np.array_equal(eng.gram(), G0)
    # the stream continues from the untouched state
    eng.push_batch(Xd[m + 1:m + 1 + 8])
    eng.sync()
    ref = O.StreamingGram(m)
    for t in range(m + 1 + 8):
        ref.push(X[:, t])
    assert normwise(eng.gram(), ref.G) < 1e-12
    eng.close()


# ---------------------------------------------------------------------- sparse (K3) -------

def test_sparse_dct_gram_and_dmd():
    st = synth.SparseDCTStream(N=128, k_low=14.0, n_shell=60, seed=9)
    m, T = 24, 40
    eng = Eng(st.n, m, storage="sparse", nnz_cap=st.nnz_cap, workers=2)
    ref = O.StreamingDMD(m, background=False)
    for t in range(T):
        idx, val = st.frame(t)
        if t % 2:
            eng.push_sparse(torch.from_numpy(idx).cuda(), torch.from_numpy(val).cuda())
        else:
            eng.push_sparse(idx, val)
        ref.push(st.dense(t))
    eng.sync()
    assert normwise(eng.gram(), ref.gram.G) < 1e-12
    sp = eng.spectrum()
    assert sp["r"] == ref.last["r"]
    lam_ref = ref.last["lam"]
    big = np.abs(lam_ref) > 1e-3
    err, perm = match(sp["lam"], lam_ref)
    assert err < 1e-7 * max(1, np.abs(lam_ref).max())
    eng.close()


def test_sparse_modes_in_coefficient_space_and_host_ingest():
    """NEXT-3 subset: host-side sparse pushes (only the nonzeros cross PCIe, on the copy stream)
    and DMD modes returned in the DCT coefficient space, b_j φ̂_j against the oracle's modes of
    the scattered (dense) coefficient vectors."""
    st = synth.SparseDCTStream(N=96, k_low=10.0, n_shell=40, seed=21)
    m, T = 20, 36
    eng = Eng(st.n, m, storage="sparse", nnz_cap=st.nnz_cap, workers=2)
    ref = O.StreamingDMD(m, background=False)
    for t in range(T):
        idx, val = st.frame(t)
        eng.push_sparse(idx, val)                       # host arrays
        out = ref.push(st.dense(t))
    eng.sync()
    assert normwise(eng.gram(), ref.gram.G) < 1e-12
    sp = eng.spectrum(with_b=True)
    r = sp["r"]
    assert r == out["r"]
    err, perm = match(sp["lam"], out["lam"])
    assert err < 1e-8 * max(1.0, np.abs(out["lam"]).max())
    Phi = eng.modes(list(range(r))).cpu().numpy()
    Phi_ref = O.modes(ref.gram.cols[1:], out)
    lam = out["lam"]
    sep = np.array([np.min(np.abs(np.delete(lam, j) - lam[j])) if r > 1 else 1.0 for j in range(r)])
    checked = 0
    for j in range(r):
        jr = perm[j]
        if sep[jr] < 1e-3:
            continue                                    # near-degenerate pair: not unique
        a = sp["b"][j] * Phi[:, j]
        bb = out["b"][jr] * Phi_ref[:, jr]
        assert np.linalg.norm(a - bb) < 1e-7 * np.linalg.norm(bb), j
        checked += 1
    assert checked >= r // 2
    rec, rec_ref = Phi @ sp["b"], Phi_ref @ out["b"]
    assert np.linalg.norm(rec - rec_ref) < 1e-8 * np.linalg.norm(rec_ref)
    eng.close()


# ---------------------------------------------------------- C4 full size, sampled ---------

@pytest.mark.slow
def test_c4_full_size_sampled():
    """BASELINE config 4 at full size (3840x2160x3, m=200, fp32) in the bench's launch
    configuration; the oracle recomputes sampled Gram entries one by one (fp64 dots of
    CPU-regenerated frames) and the background is checked by properties that hold at any size."""
    vs = synth.video_config("C4")
    m = 200
    eng = Eng(vs.n, m, dtype="f32", background=True, workers=4)
    lag = eng.info()["lag"]
    T = m + lag + 4
    for t in range(T):
        eng.push(vs.frame(t, device="cuda:0"))
    eng.sync()
    G = eng.gram()
    assert np.allclose(G, G.T, rtol=0, atol=0)
    t = T - 1
    x_t = vs.frame(t).numpy()
    for k in (0, 57, 199, 200):
        z = vs.frame(t - m + k).numpy()
        ref = float(O.gram_column([z], x_t)[0])                # compensated oracle dot (O1)
        assert abs(G[k, m] - ref) <= 1e-12 * math.sqrt(G[k, k] * G[m, m]), k
    low, sp, mask, fb = eng.background()
    assert fb == T - 1 - lag
    x = vs.frame(fb).numpy().astype(np.float64)
    assert np.max(np.abs(low.astype(np.float64) + sp - x)) < 1e-6
    assert np.array_equal(mask, sp > np.float32(0.2)) or \
        np.mean(mask != (sp > np.float32(0.2))) < 1e-6
    gt = vs.truth_mask(fb)
    tp = np.sum(mask & gt)
    assert 2 * tp / (mask.sum() + gt.sum()) > 0.85
    eng.close()


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_k1_v2_and_v1_variants_agree(dtype, monkeypatch):
    """The default K1 (v2: one vector per lane, designated-warp background reduction) and the v1
    K1 (SDMD_K1=v1: 8 rows per lane, lockstep reduction) compute the same Gram columns and
    background (different fixed summation orders)."""
    vs = synth.video_config("C3s")
    m, T = 24, 40
    npdt = np.float32 if dtype == "f32" else np.float64
    frames = vs.frames(0, T).numpy().astype(npdt)
    Xd = dev_cols(frames, npdt)
    outs = []
    for mode in ("v2", "v1"):
        if mode == "v1":
            monkeypatch.setenv("SDMD_K1", "v1")
        else:
            monkeypatch.delenv("SDMD_K1", raising=False)
        eng = Eng(vs.n, m, dtype=dtype, background=True, workers=2)
        for t in range(T):
            eng.push(Xd[t])
        eng.sync()
        outs.append((eng.gram(), eng.background()))
        eng.close()
    assert normwise(outs[0][0], outs[1][0]) < 1e-14
    la, lb = outs[0][1][0].astype(np.float64), outs[1][1][0].astype(np.float64)
    assert np.max(np.abs(la - lb)) < 1e-5 * np.max(np.abs(lb))
    assert outs[0][1][3] == outs[1][1][3]


@pytest.mark.parametrize("m", [64, 100])
def test_noisy_video_full_rank_spectrum(m):
    """Noisy video window with r = m (multishift QR path for r > 32): all eigenvalues of Ã vs the
    oracle by optimal assignment (parity of noise eigenvalues is 'unpinned' beyond GPU-vs-oracle,
    DESIGN.md §4), the background eigenvalue to 1e-9, σ to 1e-10 relative."""
    vs = synth.video_config("C3s")
    T = m + 6
    frames = vs.frames(0, T).numpy()
    Xd = torch.from_numpy(np.ascontiguousarray(frames.T)).cuda()
    eng = Eng(vs.n, m, dtype="f32", workers=2)
    ref = O.StreamingDMD(m, background=False)
    for t in range(T):
        eng.push(Xd[t])
        ref.push(frames[:, t])
    eng.sync()
    out = ref.last
    sp = eng.spectrum()
    assert sp["r"] == out["r"] == m
    err, _ = match(sp["lam"], out["lam"])
    assert err < 1e-7, err
    assert abs(sp["lam"][sp["idx"]] - out["lam"][out["idx"]]) < 1e-9
    sv = eng.svd(with_V=False)
    keep = out["sigma"] / out["sigma"][0] >= 1e-4
    assert np.max(np.abs(sv["sigma"][keep] - out["sigma"][keep]) / out["sigma"][keep]) < 1e-10
    eng.close()


@pytest.mark.parametrize("m,cl,chol", [(65, "1", "1"), (128, "1", "1"), (65, "4", "1"), (128, "4", "1"),
                                        (128, "1", "0"), (128, "4", "0")])
def test_k4a_one_cta_and_cluster_vs_oracle(m, cl, chol, monkeypatch):
    """K4a on one CTA (the default for dense 64 < m <= 128: whole S in shared memory, Ã in 64-row
    chunks, one-CTA Hessenberg and Aberth) and on the 4-CTA cluster (SDMD_K4_CL=4, read at create),
    with the Cholesky-preconditioned Jacobi start (default) and the S·Q0 start (SDMD_K4_CHOL=0),
    give the oracle's SVD and spectrum on a noisy full-rank video window at both ends of the
    one-CTA range, every window of the stream (warm starts included), and the same fused
    background: σ 1e-10 relative (σ/σ1 >= 1e-4), λ_idx 1e-9, all λ 1e-7 (assignment), lowrank 1e-4."""
    monkeypatch.setenv("SDMD_K4_CL", cl)
    monkeypatch.setenv("SDMD_K4_CHOL", chol)
    vs = synth.video_config("C3s")
    T = m + 12
    frames = vs.frames(0, T).numpy()
    Xd = torch.from_numpy(np.ascontiguousarray(frames.T)).cuda()
    eng = Eng(vs.n, m, dtype="f32", workers=3, background=True)
    lag = eng.info()["lag"]
    ref = O.StreamingDMD(m, background=True)
    outs = {}
    for t in range(T):
        eng.push(Xd[t])
        o = ref.push(frames[:, t])
        if o is not None:
            outs[t] = o
        if t >= m + 2 and t % 3 == 0:
            eng.sync()
            out = ref.last
            sp = eng.spectrum()
            assert sp["frame"] == t and sp["r"] == out["r"]
            assert abs(sp["lam"][sp["idx"]] - out["lam"][out["idx"]]) < 1e-9, t
            assert match(sp["lam"], out["lam"])[0] < 1e-7, t
            sv = eng.svd(with_V=False)
            keep = out["sigma"] / out["sigma"][0] >= 1e-4
            assert np.max(np.abs(sv["sigma"][keep] - out["sigma"][keep]) / out["sigma"][keep]) < 1e-10
    eng.sync()
    low, sp_, mask, fb = eng.background()
    lr = outs[fb]["lowrank"]
    assert np.max(np.abs(low - lr)) / np.max(np.abs(lr)) < 1e-4
    eng.close()


def test_modes_every_frame_matches_on_demand_and_oracle():
    """NEXT-2 "full Φ every frame": with modes_every_frame the worker stream computes every
    frame's modes (all eigenvectors, then K2); get_modes of the newest frame must equal the
    on-demand path bitwise and b_j φ_j must match the oracle (planted C1, 1e-8)."""
    pm = synth.planted_c1()
    m, T = 16, 60
    X = pm.frames(0, T)
    Xd = dev_cols(X, np.float64)
    a = Eng(pm.n, m, dtype="f64", workers=3, modes_every_frame=True)
    b = Eng(pm.n, m, dtype="f64", workers=3)
    ref = O.StreamingDMD(m, background=False)
    for t in range(T):
        a.push(Xd[t])
        b.push(Xd[t])
        out = ref.push(X[:, t])
    a.sync()
    b.sync()
    r = a.spectrum()["r"]
    Pa = a.modes(list(range(r))).cpu().numpy()
    Pb = b.modes(list(range(r))).cpu().numpy()
    assert np.array_equal(Pa, Pb)
    sp = a.spectrum(with_b=True)
    err, perm = match(sp["lam"], out["lam"])
    Phi_ref = O.modes(ref.gram.cols[1:], out)
    for j in range(r):
        u = sp["b"][j] * Pa[:, j]
        v = out["b"][perm[j]] * Phi_ref[:, perm[j]]
        assert np.linalg.norm(u - v) < 1e-8 * np.linalg.norm(v), j
    a.close()
    b.close()


def test_maximum_sizes_m256_r224_with_background():
    """Edge case at the ABI maxima: m = SDMD_MAX_M = 256 (K1 union m + lag > 256 columns, the
    widest K1 instance), r capped at SDMD_MAX_R = 224 on a full-rank noisy window (largest QR,
    K4 shared memory), background on: Gram, σ, λ and the background against the oracle."""
    vs = synth.video_config("C3s")
    m = 256
    T = m + 1 + 12
    frames = vs.frames(0, T).numpy()
    Xd = torch.from_numpy(np.ascontiguousarray(frames.T)).cuda()
    eng = Eng(vs.n, m, dtype="f32", background=True, workers=2)
    lag = eng.info()["lag"]
    ref = O.StreamingDMD(m, background=True, r_max=224)
    outs = {}
    for t in range(T):
        eng.push(Xd[t])
        o = ref.push(frames[:, t])
        if o is not None:
            outs[t] = o
    eng.sync()
    out = ref.last
    assert normwise(eng.gram(), ref.gram.G) < 1e-12
    sp = eng.spectrum()
    assert sp["r"] == out["r"] == 224
    err, _ = match(sp["lam"], out["lam"])
    assert err < 1e-7, err
    assert abs(sp["lam"][sp["idx"]] - out["lam"][out["idx"]]) < 1e-9
    sv = eng.svd(with_V=False)
    keep = out["sigma"] / out["sigma"][0] >= 1e-4
    assert np.max(np.abs(sv["sigma"][keep] - out["sigma"][keep]) / out["sigma"][keep]) < 1e-10
    low, spv, mask, fb = eng.background()
    assert fb == T - 1 - lag
    o = outs[fb]
    rel = np.max(np.abs(low - o["lowrank"])) / np.max(np.abs(o["lowrank"]))
    assert rel < 1e-4, rel
    eng.close()


def test_empty_sparse_frames():
    """Edge case: sparse snapshots with no nonzeros (nnz = 0) give zero Gram rows/columns and a
    rank-deficient window; the Gram matches the oracle and the DMD still runs."""
    st = synth.SparseDCTStream(N=64, k_low=8.0, n_shell=20, seed=5)
    m, T = 10, 24
    eng = Eng(st.n, m, storage="sparse", nnz_cap=st.nnz_cap, workers=1)
    ref = O.StreamingGram(m)
    for t in range(T):
        if t in (3, 15, 16):
            idx, val = np.zeros(0, dtype=np.int32), np.zeros(0, dtype=np.float64)
            dense = np.zeros(st.n)
        else:
            idx, val = st.frame(t)
            dense = st.dense(t)
        eng.push_sparse(idx, val)
        ref.push(dense)
    eng.sync()
    assert normwise(eng.gram(), ref.G) < 1e-12
    G = eng.gram()
    assert np.all(G[2, :] == 0.0) and np.all(G[:, 3] == 0.0)    # frames 15, 16 of window 13..23
    d = O.dmd_from_gram(ref.G)
    sp = eng.spectrum()
    assert sp["r"] == d["r"]
    eng.close()


def test_sparse_fully_dense_frames_and_rejected_pushes():
    """Edge cases of the sparse ingest: frames with nnz = n = nnz_cap (every coefficient nonzero,
    the maximum size) match the dense oracle; pushes that break the contract (nnz > nnz_cap,
    indices not strictly ascending, out of range) raise and leave the stream unchanged."""
    from paper_1612_07875_b200 import SDMDError
    rng = np.random.default_rng(77)
    n, m, T = 300, 8, 20
    X = rng.standard_normal((n, T))
    eng = Eng(n, m, storage="sparse", nnz_cap=n, workers=1)
    ref = O.StreamingGram(m)
    all_idx = np.arange(n, dtype=np.int32)
    bad = [(np.arange(n + 1, dtype=np.int32) % n, np.ones(n + 1)),            # nnz > nnz_cap
           (np.array([5, 3], dtype=np.int32), np.ones(2)),                     # descending
           (np.array([4, 4], dtype=np.int32), np.ones(2)),                     # duplicate
           (np.array([0, n], dtype=np.int32), np.ones(2))]                     # out of range
    for t in range(T):
        if t in (4, 13):
            for idx, val in bad:
                with pytest.raises(SDMDError):
                    eng.push_sparse(idx, val)
        eng.push_sparse(all_idx, np.ascontiguousarray(X[:, t]))
        ref.push(X[:, t])
    eng.sync()
    assert normwise(eng.gram(), ref.G) < 1e-12
    d = O.dmd_from_gram(ref.G)
    sp = eng.spectrum()
    assert sp["r"] == d["r"] and sp["frame"] == T - 1
    e_or, _ = match(sp["lam"], d["lam"])
    assert e_or < 1e-9, e_or
    eng.close()


def test_constant_stream_fixed_point():
    """S:346, S:353, S:377 on the device: a constant video has σ₁ = √m‖x‖, r = 1, λ_idx = 1 and
    an all-background foreground (sparse ≈ 0, empty mask)."""
    vs = synth.VideoStream(72, 96, 1, seed=5, n_squares=0, noise_sigma=0.0)
    x = vs.frame(0).cuda()
    m = 20
    eng = Eng(vs.n, m, dtype="f32", background=True, workers=2)
    lag = eng.info()["lag"]
    for _ in range(m + lag + 3):
        eng.push(x)
    eng.sync()
    sv = eng.svd(with_V=False)
    xn = float(torch.linalg.norm(x.double()))
    assert sv["r"] == 1
    assert abs(sv["sigma"][0] - math.sqrt(m) * xn) < 1e-10 * sv["sigma"][0]
    sp = eng.spectrum()
    assert abs(sp["lam"][sp["idx"]] - 1.0) < 1e-9
    low, spr, mask, fb = eng.background()
    assert np.max(np.abs(spr)) < 1e-5 and not mask.any()
    eng.close()


@pytest.mark.slow
def test_c3_full_size_sampled():
    """BASELINE config 3 at full size (1920x1080 grey, m=100, fp32): sampled Gram entries vs CPU
    fp64 dots of regenerated frames; background additivity and F-measure sanity."""
    vs = synth.video_config("C3")
    m = 100
    eng = Eng(vs.n, m, dtype="f32", background=True, workers=4)
    T = m + eng.info()["lag"] + 4
    for t in range(T):
        eng.push(vs.frame(t, device="cuda:0"))
    eng.sync()
    G = eng.gram()
    t = T - 1
    x_t = vs.frame(t).numpy()
    for k in (0, 33, 99, 100):
        z = vs.frame(t - m + k).numpy()
        ref = float(O.gram_column([z], x_t)[0])                # compensated oracle dot (O1)
        assert abs(G[k, m] - ref) <= 1e-12 * math.sqrt(G[k, k] * G[m, m]), k
    low, sp, mask, fb = eng.background()
    x = vs.frame(fb).numpy().astype(np.float64)
    assert np.max(np.abs(low.astype(np.float64) + sp - x)) < 1e-6
    gt = vs.truth_mask(fb)
    assert 2 * np.sum(mask & gt) / (mask.sum() + gt.sum()) > 0.85
    eng.close()


# ------------------------------------------- two ranks on one GPU (SDMD_LOCAL_GROUP) ---------

@pytest.mark.parametrize("eigen_shard", [1, 0])
def test_two_ranks_one_gpu_local_group(monkeypatch, eigen_shard):
    """The multi-rank data path on one GPU: two contexts (ranks 0 and 1, half of the rows each)
    driven by two host threads, collectives through the in-process test group (NCCL refuses two
    ranks on one device).  Row sharding + allreduce of g: both ranks hold the same Gram, bitwise,
    equal to one rank's within 1e-12 (summation split only).  Eigen sharding, c_t carried by the
    allreduce of a later frame's Gram column: the background rows of the two ranks form the
    one-rank background; each rank's spectrum is the newest frame it solved.  Exactly ONE
    collective per push (the allreduce of the (m+1)-vector is the only one)."""
    import threading
    from paper_1612_07875_b200 import row_partition
    monkeypatch.setenv("SDMD_LOCAL_GROUP", "1")
    vs = synth.VideoStream(108, 192, 1, seed=31, side=24)
    m, T = 24, 61
    uid = bytes((7 * i + eigen_shard) % 256 for i in range(128))
    res, errs = {}, []

    def run(rank):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                b, e = row_partition(vs.n, 2, rank)
                eng = Eng(e - b, m, dtype="f32", background=True, workers=2, rank=rank, nranks=2,
                          row_begin=b, n_global=vs.n, nccl_uid=uid, eigen_shard=eigen_shard)
                for t in range(T):
                    eng.push(vs.frame(t, "cuda:0", (b, e)))
                eng.sync()
                res[rank] = (eng.gram(), eng.background(), eng.spectrum(), eng.info(), eng.stats())
                eng.close()
        except Exception as ex:                        # surfaced below
            errs.append(repr(ex))
    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=300)
    assert not errs, errs
    one = Eng(vs.n, m, dtype="f32", background=True, workers=2, lag=res[0][3]["lag"])
    for t in range(T):
        one.push(vs.frame(t, "cuda:0"))
    one.sync()
    G1 = one.gram()
    low1, sp1, mask1, fb1 = one.background()
    spec1 = one.spectrum()
    assert np.array_equal(res[0][0], res[1][0])
    assert normwise(res[0][0], G1) < 1e-12
    assert res[0][4]["collectives"] == res[1][4]["collectives"] == T
    low = np.concatenate([res[0][1][0], res[1][1][0]])
    assert res[0][1][3] == res[1][1][3] == fb1
    assert np.max(np.abs(low - low1)) < 1e-4 * np.max(np.abs(low1))
    if eigen_shard:
        assert res[0][2]["frame"] == T - 1 and res[1][2]["frame"] == T - 2   # T-1 = 60 is even
    else:
        assert res[0][2]["frame"] == res[1][2]["frame"] == T - 1
        assert np.array_equal(res[0][2]["lam"], res[1][2]["lam"])
    r0 = res[0][2] if res[0][2]["frame"] == T - 1 else res[1][2]
    assert match(r0["lam"], spec1["lam"])[0] < 1e-8 * max(1.0, np.abs(spec1["lam"]).max())
    one.close()


def test_two_ranks_one_gpu_init_window_and_batches(monkeypatch):
    """The other collectives of the multi-rank path on one GPU (test group): the (m+1)² init
    Gram allreduce of sdmd_init_window and the k(m+1) allreduce of sdmd_push_batch, with eigen
    sharding; both ranks end with the one-rank Gram (1e-12, bitwise equal across ranks)."""
    import threading
    from paper_1612_07875_b200 import row_partition
    monkeypatch.setenv("SDMD_LOCAL_GROUP", "1")
    rng = np.random.default_rng(23)
    n, m, k = 20011, 30, 4
    T = m + 1 + 5 * k
    X = rng.standard_normal((n, T)).astype(np.float32)
    uid = bytes((11 * i + 3) % 256 for i in range(128))
    res, errs = {}, []

    def run(rank):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                b, e = row_partition(n, 2, rank)
                Xd = torch.from_numpy(np.ascontiguousarray(X[b:e].T)).cuda()
                eng = Eng(e - b, m, dtype="f32", workers=2, rank=rank, nranks=2, row_begin=b,
                          n_global=n, nccl_uid=uid, batch_max=k)
                eng.init_window(Xd[: m + 1])
                for t in range(m + 1, T, k):
                    eng.push_batch(Xd[t:t + k])
                eng.sync()
                res[rank] = (eng.gram(), eng.spectrum())
                eng.close()
        except Exception as ex:
            errs.append(repr(ex))
    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=300)
    assert not errs, errs
    ref = O.StreamingGram(m)
    for t in range(T):
        ref.push(X[:, t].astype(np.float64))
    assert np.array_equal(res[0][0], res[1][0])
    assert normwise(res[0][0], ref.G) < 1e-12
    d = O.dmd_from_gram(ref.G)
    last = res[0][1] if res[0][1]["frame"] == T - 1 else res[1][1]
    assert last["frame"] == T - 1
    assert match(last["lam"], d["lam"])[0] < 1e-7 * max(1.0, np.abs(d["lam"]).max())


def test_two_ranks_one_gpu_sparse(monkeypatch):
    """Sparse (K3) pushes on two ranks (test group): each rank holds the coefficient indices of
    its row range; the allreduced Gram equals the one-rank sparse Gram (1e-12)."""
    import threading
    from paper_1612_07875_b200 import row_partition
    monkeypatch.setenv("SDMD_LOCAL_GROUP", "1")
    st = synth.SparseDCTStream(N=96, k_low=10.0, n_shell=40, seed=29)
    m, T = 16, 30
    frames = [st.frame(t) for t in range(T)]
    uid = bytes((13 * i + 5) % 256 for i in range(128))
    res, errs = {}, []

    def run(rank):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                b, e = row_partition(st.n, 2, rank)
                eng = Eng(e - b, m, storage="sparse", nnz_cap=st.nnz_cap, workers=1, rank=rank,
                          nranks=2, row_begin=b, n_global=st.n, nccl_uid=uid)
                for idx, val in frames:
                    sel = (idx >= b) & (idx < e)
                    eng.push_sparse(np.ascontiguousarray(idx[sel]), np.ascontiguousarray(val[sel]))
                eng.sync()
                res[rank] = eng.gram()
                eng.close()
        except Exception as ex:
            errs.append(repr(ex))
    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=300)
    assert not errs, errs
    ref = O.StreamingGram(m)
    for t in range(T):
        ref.push(st.dense(t))
    assert np.array_equal(res[0], res[1])
    assert normwise(res[0], ref.G) < 1e-12


def _sparse_dev(idx, val):
    return (torch.from_numpy(np.ascontiguousarray(idx, dtype=np.int32)).to("cuda:0"),
            torch.from_numpy(np.ascontiguousarray(val, dtype=np.float64)).to("cuda:0"))


def test_sparse_device_indices_checked_on_device():
    """Device-resident sparse frames are validated on the device (the host cannot see them): a
    frame with descending or out-of-range indices is rejected like a non-finite one — nothing is
    scattered, sync reports it and the stream resumes from the last committed frame."""
    from paper_1612_07875_b200 import SDMDError
    st = synth.SparseDCTStream(N=64, k_low=8.0, n_shell=20, seed=41)
    m, T = 10, 30
    bad = {12: lambda i: i[::-1].copy(), 20: lambda i: i + st.n}     # descending, out of range
    eng = Eng(st.n, m, storage="sparse", nnz_cap=st.nnz_cap, workers=1)
    ref = O.StreamingGram(m)
    committed, skip = 0, set()
    for t in range(T):
        if t in skip:
            continue
        if t in bad:
            eng.sync()
            G0 = eng.gram()
            idx, val = st.frame(t)
            eng.push_sparse(*_sparse_dev(bad[t](idx), val))
            try:                                                   # discarded by the poison contract
                eng.push_sparse(*_sparse_dev(*st.frame(t + 1)))    # (or refused if the host
            except SDMDError as e:                                 #  already saw the rejection)
                assert e.status == 2
            skip.add(t + 1)
            with pytest.raises(SDMDError) as e:
                eng.sync()
            assert e.value.status == 2 and e.value.failed_frame == committed
            assert np.array_equal(eng.gram(), G0)
            assert eng.info()["frames"] == committed
            continue
        eng.push_sparse(*_sparse_dev(*st.frame(t)))
        ref.push(st.dense(t))
        committed += 1
    eng.sync()
    assert normwise(eng.gram(), ref.G) < 1e-12
    d = O.dmd_from_gram(ref.G)
    assert eng.spectrum()["r"] == d["r"]
    eng.close()


def test_two_ranks_one_gpu_sparse_bad_indices_rejected_on_every_rank(monkeypatch):
    """Rank 0 pushes a device frame with an index outside its row range: the NaN self product goes through
    the allreduce, so BOTH ranks reject the same frame and resume in step."""
    import threading
    from paper_1612_07875_b200 import SDMDError, row_partition
    monkeypatch.setenv("SDMD_LOCAL_GROUP", "1")
    st = synth.SparseDCTStream(N=64, k_low=8.0, n_shell=20, seed=43)
    m, T, bad_at = 8, 24, 11
    uid = bytes((7 * i + 3) % 256 for i in range(128))
    res, errs, fails = {}, [], {}

    def run(rank):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                b, e = row_partition(st.n, 2, rank)
                eng = Eng(e - b, m, storage="sparse", nnz_cap=st.nnz_cap, workers=1, rank=rank,
                          nranks=2, row_begin=b, n_global=st.n, nccl_uid=uid)

                def push(t, corrupt=False):
                    idx, val = st.frame(t)
                    sel = (idx >= b) & (idx < e)
                    ii = idx[sel].copy()
                    if corrupt and ii.size:
                        ii[-1] = e + 5 if rank == 0 else ii[-1]   # a valid index, but rank 1's
                    eng.push_sparse(*_sparse_dev(ii, val[sel]))
                for t in range(bad_at):
                    push(t)
                push(bad_at, corrupt=True)
                try:
                    eng.sync()
                    fails[rank] = None
                except SDMDError as ex:
                    fails[rank] = (ex.status, ex.failed_frame)
                for t in range(bad_at + 1, T):
                    push(t)
                eng.sync()
                res[rank] = eng.gram()
                eng.close()
        except Exception as ex:
            errs.append(repr(ex))
    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=300)
    assert not errs, errs
    assert fails[0] == fails[1] == (2, bad_at), fails
    ref = O.StreamingGram(m)
    for t in list(range(bad_at)) + list(range(bad_at + 1, T)):
        ref.push(st.dense(t))
    assert np.array_equal(res[0], res[1])
    assert normwise(res[0], ref.G) < 1e-12


# ------------------------------------------------ W_SINGULAR amplitudes (reading Q15) --------

def _planted_zero_mode(n=300, m=6, orth=True, seed=60, T=None):
    """Real modes, λ = {0, 0.9, -0.7, 0.5}: x_t = Σ b_j φ_j λ_j^t (φ_0 appears in x_0 only), so the
    window that starts at t = 0 has an exact zero DMD eigenvalue (WΛ singular)."""
    rng = np.random.default_rng(seed)
    lam = np.array([0.0, 0.9, -0.7, 0.5])
    b = np.array([1.3, 0.8, -0.6, 1.1])
    Phi = rng.standard_normal((n, 4))
    if orth:
        Phi, _ = np.linalg.qr(Phi)
    T = m + 1 if T is None else T
    X = np.stack([Phi @ (b * lam ** t) for t in range(T)], axis=1)
    return X, lam, b, Phi


@pytest.mark.parametrize("orth", [True, False])
def test_singular_amplitudes_least_squares_on_kept_modes(orth):
    """GPU W_SINGULAR semantics = the oracle's (O9): status W_SINGULAR, b = 0 for the zero mode,
    least squares of WΛ's kept columns for the others (compared as b_j φ_j, 1e-9 relative)."""
    m = 6
    X, lam_p, _, _ = _planted_zero_mode(m=m, orth=orth, seed=70 + int(orth))
    ref = O.dmd_window(X)
    assert ref["amp_status"] == O.W_SINGULAR
    eng = Eng(X.shape[0], m, dtype="f64", workers=1)
    eng.init_window(dev_cols(X, np.float64))
    sp = eng.spectrum(with_b=True)
    assert sp["status"] == 6 and sp["r"] == ref["r"] == 4
    err, perm = match(sp["lam"], ref["lam"])
    assert err < 1e-9
    Phi = eng.modes(list(range(4))).cpu().numpy()
    Phi_ref = O.modes(X[:, 1:], ref)
    for j in range(4):
        k = perm[j]
        got, want = sp["b"][j] * Phi[:, j], ref["b"][k] * Phi_ref[:, k]
        scale = max(np.linalg.norm(want), 1e-300)
        if np.all(want == 0):
            assert np.linalg.norm(got) == 0
        else:
            assert np.linalg.norm(got - want) < 1e-9 * scale, (j, np.linalg.norm(got - want) / scale)
    eng.close()


def test_singular_frame_background_uses_least_squares():
    """The per-frame path: the streamed background column of a W_SINGULAR window (built from the
    kept-mode least-squares b_idx on the device) equals the oracle's, 1e-9 relative (fp64)."""
    m = 6
    eng = Eng(300, m, dtype="f64", background=True, workers=1)
    L = eng.info()["lag"]
    X, _, _, _ = _planted_zero_mode(m=m, orth=False, seed=72, T=m + 1 + L)
    X = X + 0.5                                        # an exact constant mode: λ = 1 is idx
    ref = O.StreamingDMD(m, background=True)
    out_m = ref.init_window(X[:, :m + 1])
    assert out_m["amp_status"] == O.W_SINGULAR
    eng.init_window(dev_cols(X[:, :m + 1], np.float64))
    assert eng.spectrum()["status"] == 6
    Xd = dev_cols(X, np.float64)
    for t in range(m + 1, m + 1 + L):
        eng.push(Xd[t])
    eng.sync()
    low, sp_, mask, fb = eng.background()
    assert fb == m
    rel = np.max(np.abs(low - out_m["lowrank"])) / np.max(np.abs(out_m["lowrank"]))
    assert rel < 1e-9, rel
    eng.close()


# ------------------------------------------- the real NCCL data plane on a 1-rank communicator --

def test_nccl_one_rank_communicator_matches_single_rank(monkeypatch):
    """SDMD_FORCE_NCCL=1 runs the multi-rank code path of a 1-rank context through a real NCCL
    communicator (ncclCommInitRank with nranks = 1): the init-Gram allreduce, the per-frame
    allreduce of g with the background coefficients folded in, and the separate commit kernel.
    A 1-rank sum is the identity, so Gram, spectrum and background equal the plain single-rank
    run bitwise, with exactly one NCCL call per push."""
    vs = synth.VideoStream(108, 192, 1, seed=33, side=24)
    m, T = 24, 70
    frames = vs.frames(0, T).numpy()
    Xd = torch.from_numpy(np.ascontiguousarray(frames.T)).cuda()

    def run(force):
        if force:
            monkeypatch.setenv("SDMD_FORCE_NCCL", "1")
        else:
            monkeypatch.delenv("SDMD_FORCE_NCCL", raising=False)
        eng = Eng(vs.n, m, dtype="f32", background=True, workers=2)
        eng.init_window(Xd[:m + 1])
        eng.sync()
        eng.stats(reset=True)
        for t in range(m + 1, T):
            eng.push(Xd[t])
        eng.sync()
        out = (eng.gram(), eng.background(), eng.spectrum(), eng.stats(), eng.partial_gram_column())
        eng.close()
        return out
    plain, nccl = run(False), run(True)
    assert plain[3]["collectives"] == 0
    assert nccl[3]["collectives"] == T - m - 1
    assert np.array_equal(plain[0], nccl[0])
    for a, b in zip(plain[1][:3], nccl[1][:3]):
        assert np.array_equal(a, b)
    assert plain[1][3] == nccl[1][3]
    assert np.array_equal(plain[2]["lam"], nccl[2]["lam"]) and plain[2]["idx"] == nccl[2]["idx"]
    assert np.array_equal(plain[4], nccl[4])


def test_nccl_one_rank_batches_and_sparse(monkeypatch):
    """The batched (k-frame allreduce) and sparse (K3 + allreduce + commit kernel) multi-rank paths
    through a real 1-rank NCCL communicator equal the oracle's streamed Gram (1e-12)."""
    monkeypatch.setenv("SDMD_FORCE_NCCL", "1")
    pm = synth.planted_c1()
    m = 16
    X = pm.frames(0, m + 1 + 24)
    Xd = dev_cols(X, np.float64)
    eng = Eng(pm.n, m, dtype="f64", workers=2, batch_max=8)
    ref = O.StreamingGram(m)
    for t in range(m + 1):
        eng.push(Xd[t])
        ref.push(X[:, t])
    for t0 in (m + 1, m + 9, m + 17):
        eng.push_batch(Xd[t0:t0 + 8])
        for j in range(8):
            ref.push(X[:, t0 + j])
    eng.sync()
    assert normwise(eng.gram(), ref.G) < 1e-12
    assert match(eng.spectrum()["lam"], pm.lambdas)[0] < 1e-9
    eng.close()
    st = synth.SparseDCTStream(N=128, k_low=14.0, n_shell=60, seed=5)
    m, T = 12, 30
    eng = Eng(st.n, m, storage="sparse", nnz_cap=st.nnz_cap, workers=1)
    ref = O.StreamingGram(m)
    for t in range(T):
        eng.push_sparse(*st.frame(t))
        ref.push(st.dense(t))
    eng.sync()
    assert normwise(eng.gram(), ref.G) < 1e-12
    assert eng.stats()["collectives"] == T
    eng.close()


# ------------------------------------------------ parity at the benchmarked instances --------

def test_c5_scale_sparse_multi_chunk_gram_and_lambda_idx():
    """BASELINE config 5 at full size (1024² DCT coefficients, ~1% nonzeros, m = 128): nnz_cap
    ≈ 10.6k takes K3's 6-chunk reduction.  Gram vs the oracle's compensated definition (on the
    window's union support, bitwise equal to the dense definition) normwise 1e-12; r equal; λ_idx
    within 1e-9 (§3.5)."""
    st = synth.SparseDCTStream()                      # C5: N=1024, k_low=110, n_shell=1000
    m, T = 128, 128 + 1 + 12
    assert (st.nnz_cap + 2047) // 2048 >= 5
    eng = Eng(st.n, m, storage="sparse", nnz_cap=st.nnz_cap, workers=4)
    slots = []
    for t in range(T):
        fr = st.frame(t)
        eng.push_sparse(*fr)
        slots = (slots + [fr])[-(m + 1):]
    eng.sync()
    G = eng.gram()
    Gr = O.gram(O.sparse_window_on_support(slots))
    assert normwise(G, Gr) < 1e-12
    d = O.dmd_from_gram(Gr)
    idx_ref = O.background_index(d["lam"])
    sp = eng.spectrum()
    assert sp["r"] == d["r"] and sp["frame"] == T - 1
    assert abs(sp["lam"][sp["idx"]] - d["lam"][idx_ref]) < 1e-9
    eng.close()


def test_c4s_bench_kernel_instance_background_elementwise():
    """The bench's background instance (k1v2_kernel<float, bg, 13>: m = 200, 6 workers, lag 8 →
    208 union columns) on a reduced-n C4-shaped video (384x216x3): low-rank, sparse and mask of the
    streamed background column vs the oracle element by element (fp32 path: 1e-4 relative;
    mask equal away from |s − 0.2| < 1e-4)."""
    vs = synth.video_config("C4s")
    m = 200
    eng = Eng(vs.n, m, dtype="f32", background=True, workers=6)
    info = eng.info()
    assert info["lag"] == 8 and (m + info["lag"]) == 16 * 13
    T = m + info["lag"] + 6
    frames = vs.frames(0, T).numpy()
    Xd = torch.from_numpy(np.ascontiguousarray(frames.T)).cuda()
    for t in range(T):
        eng.push(Xd[t])
    eng.sync()
    low, sp, mask, fb = eng.background()
    assert fb == T - 1 - info["lag"]
    ref = O.StreamingDMD(m, background=True)
    o = ref.init_window([frames[:, k] for k in range(fb - m, fb + 1)])
    x = frames[:, fb].astype(np.float64)
    rel = np.max(np.abs(low - o["lowrank"])) / np.max(np.abs(o["lowrank"]))
    assert rel < 1e-4, rel
    assert np.max(np.abs(sp - o["sparse"])) < 1e-4 * np.max(np.abs(x))
    near = np.abs(o["sparse"] - 0.2) < 1e-4
    assert np.all(mask[~near] == o["mask"][~near])
    eng.close()
