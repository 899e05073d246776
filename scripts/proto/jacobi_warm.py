"""Prototype: sweeps of parallel-ordered Hestenes Jacobi on S = XᵀX (m = 200, C4s video frames)
from the identity vs a warm start Q0 = P^k V_{t-k} (cyclic row shift of an earlier frame's V)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth

m = int(sys.argv[1]) if len(sys.argv) > 1 else 200
vs = synth.video_config("C4s")
T = m + 12
X = np.stack([vs.frame(t).numpy().astype(np.float64) for t in range(T)], axis=1)
G = X.T @ X
tol = max(1e-15, m * np.finfo(float).eps)

def pairs_rounds(m):
    n = m + (m % 2)
    pl = list(range(n))
    for rd in range(n - 1):
        P = [pl[i] for i in range(n // 2)]
        Q = [pl[n - 1 - i] for i in range(n // 2)]
        yield [(p, q) for p, q in zip(P, Q) if p < m and q < m]
        pl = [pl[0]] + [pl[-1]] + pl[1:-1]

def hestenes(A):
    A = A.copy()
    for sweep in range(60):
        rot = False
        for prs in pairs_rounds(A.shape[1]):
            P = np.array([p for p, _ in prs]); Q = np.array([q for _, q in prs])
            ap, aq = A[:, P], A[:, Q]
            al = (ap * ap).sum(0); be = (aq * aq).sum(0); ga = (ap * aq).sum(0)
            act = (ga != 0) & (ga * ga > tol * tol * al * be)
            if not act.any():
                continue
            rot = True
            d = be - al
            sq = np.sqrt(d * d + 4 * ga * ga)
            t = np.where(d >= 0, 2 * ga, -2 * ga) / (np.abs(d) + sq)
            t = np.where(act, t, 0.0)
            c = 1 / np.sqrt(1 + t * t); s = c * t
            A[:, P] = c * ap - s * aq
            A[:, Q] = s * ap + c * aq
        if not rot:
            return A, sweep + 1
    return A, 60

def V_of(A):
    mu = np.linalg.norm(A, axis=0)
    return A / mu

t0 = m + 4
S = lambda t: G[t - m:t, t - m:t]
A_cold, sw = hestenes(S(t0))
print("cold sweeps", sw)
ev_ref = np.sort(np.linalg.eigvalsh(S(t0)))[::-1]
for k in (1, 2, 3):
    Ap, _ = hestenes(S(t0 - k))
    Vp = V_of(Ap)
    Q0 = np.roll(Vp, -k, axis=0)        # row i+k of V_{t-k} -> row i
    A0 = S(t0) @ Q0
    A, sw = hestenes(A0)
    mu = np.sort(np.linalg.norm(A, axis=0))[::-1]
    print(f"warm k={k}: sweeps {sw}, max rel eig err {np.max(np.abs(mu - ev_ref) / ev_ref[0]):.2e}")

def hestenes_dt(A, dt, tol_):
    A = A.astype(dt).copy()
    for sweep in range(60):
        rot = False
        for prs in pairs_rounds(A.shape[1]):
            P = np.array([p for p, _ in prs]); Q = np.array([q for _, q in prs])
            ap, aq = A[:, P], A[:, Q]
            al = (ap * ap).sum(0); be = (aq * aq).sum(0); ga = (ap * aq).sum(0)
            act = (ga != 0) & (ga * ga > tol_ * tol_ * al * be)
            if not act.any():
                continue
            rot = True
            d = be - al
            sq = np.sqrt(d * d + 4 * ga * ga)
            t = np.where(d >= 0, 2 * ga, -2 * ga) / (np.abs(d) + sq)
            t = np.where(act, t, 0).astype(dt)
            c = (1 / np.sqrt(1 + t * t)).astype(dt); s = (c * t).astype(dt)
            A[:, P] = c * ap - s * aq
            A[:, Q] = s * ap + c * aq
        if not rot:
            return A, sweep + 1
    return A, 60

Sm = S(t0)
for tol32 in (1e-3, 1e-4, 1e-5, 2e-6):
    A32, sw32 = hestenes_dt(Sm, np.float32, tol32)
    V32 = A32.astype(np.float64); V32 /= np.linalg.norm(V32, axis=0)
    Q, R = np.linalg.qr(V32)                      # re-orthogonalise in fp64
    A, sw = hestenes(Sm @ Q)
    mu = np.sort(np.linalg.norm(A, axis=0))[::-1]
    print(f"fp32 tol {tol32}: {sw32} fp32 sweeps + {sw} fp64 sweeps, err {np.max(np.abs(mu - ev_ref) / ev_ref[0]):.2e}")
print("eig range", ev_ref[0], ev_ref[1], ev_ref[10], ev_ref[-1])
