"""CPU model of the one-sided Jacobi sweep counts (round-robin ordering as on the GPU, tol = m·eps)
for the K4a start choices: S itself, the Rᵀ of a pivoted Cholesky S = RᵀR, and their warm-started
forms S·Q0 and Q0ᵀSQ0 = RᵀR (Q0 = previous window's eigenvectors, rows shifted).
Usage: python scripts/proto/jacobi_start_sweeps.py C1|C2|C3|C5 ; ... C4 w / C5 w (warm variants).
Output of the runs quoted in DESIGN.md: profiles/r2/chol_sweeps_cpu_model.txt"""
import sys, numpy as np
sys.path.insert(0, __import__('os').path.join(__import__('os').path.dirname(__import__('os').path.abspath(__file__)), '..', '..'))
import synth
eps = np.finfo(float).eps
def rr(pos, step, mp):
    # round-robin tournament player at position pos in step (circle method)
    if pos == 0: return 0
    return 1 + (pos - 1 + step) % (mp - 1)
def osj_rr(A, tol, maxsw=60):
    A = A.copy(); m = A.shape[1]; mp = m + (m & 1)
    if mp > m: A = np.hstack([A, np.zeros((A.shape[0], 1))])
    for sw in range(1, maxsw + 1):
        rot = 0
        for st in range(mp - 1):
            P = np.array([rr(pp, st, mp) for pp in range(mp // 2)]); Q = np.array([rr(mp - 1 - pp, st, mp) for pp in range(mp // 2)])
            ap, aq = A[:, P], A[:, Q]
            al = (ap * ap).sum(0); be = (aq * aq).sum(0); ga = (ap * aq).sum(0)
            do = (ga != 0) & (ga * ga > tol * tol * al * be)
            if do.any():
                d = be - al; sq = np.sqrt(d * d + 4 * ga * ga)
                t = np.where(d >= 0, 2 * ga, -2 * ga) / np.where(do, np.abs(d) + sq, 1.0)
                c = 1 / np.sqrt(1 + t * t); s = c * t
                c = np.where(do, c, 1.0); s = np.where(do, s, 0.0)
                A[:, P], A[:, Q] = c * ap - s * aq, s * ap + c * aq
                rot += int(do.sum())
        if rot == 0: return sw
    return -1
def pchol_rows(S):
    S = S.copy(); m = S.shape[0]; R = np.zeros((m, m)); used = np.zeros(m, bool)
    d = np.diag(S).copy()
    for k in range(m):
        dd = np.where(used, -np.inf, d); piv = int(np.argmax(dd))
        if dd[piv] <= 0: break
        used[piv] = True; rkk = np.sqrt(dd[piv])
        row = (S[piv] - R[:k, piv] @ R[:k]) / rkk
        row[used] = 0; row[piv] = rkk
        R[k] = row; d = d - row * row
    return R
def test(name, X, m):
    S = X[:, :m].T @ X[:, :m]; tol = max(1e-15, m * eps)
    R = pchol_rows(S)
    print(name, 'S:', osj_rr(S, tol), ' cholRt:', osj_rr(R.T.copy(), tol), flush=True)
which = sys.argv[1]
if which == 'C3':
    vs = synth.video_config('C3'); X = np.stack([vs.frame(t, 'cpu', (0, vs.n // 8)).numpy().astype(np.float64) for t in range(101)], 1); test('C3', X, 100)
if which == 'C2':
    cw = synth.cylinder_wake(); X = cw.frames(0, 151); test('C2', X, 150)
if which == 'C5':
    ss = synth.SparseDCTStream(); X = np.stack([ss.dense(t) for t in range(129)], 1); test('C5', X, 128)
if which == 'C1':
    pm = synth.planted_c1(); X = pm.frames(0, 17); test('C1', X, 16)
def test_warm(name, X, m):
    S0 = X[:, :m].T @ X[:, :m]; S = X[:, 1:m+1].T @ X[:, 1:m+1]; tol = max(1e-15, m * eps)
    w, V0 = np.linalg.eigh(S0); Q0 = np.roll(V0, -1, axis=0)
    Sw = Q0.T @ S @ Q0
    R = pchol_rows(Sw)
    print(name, 'warm S·Q0:', osj_rr(S @ Q0, tol), ' chol(Q0ᵀSQ0):', osj_rr(R.T.copy(), tol), flush=True)
if len(sys.argv) > 2:
    if which == 'C3':
        test_warm('C3', X if False else np.stack([synth.video_config('C3').frame(t, 'cpu', (0, synth.video_config('C3').n // 8)).numpy().astype(np.float64) for t in range(102)], 1), 100)
    if which == 'C5':
        ss = synth.SparseDCTStream(); test_warm('C5', np.stack([ss.dense(t) for t in range(130)], 1), 128)
    if which == 'C4':
        vs = synth.video_config('C4'); X = np.stack([vs.frame(t, 'cpu', (0, vs.n // 64)).numpy().astype(np.float64) for t in range(202)], 1); test('C4', X, 200); test_warm('C4', X, 200)
