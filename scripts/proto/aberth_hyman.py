"""Prototype (cost/convergence model, numpy): eigenvalues of the Hessenberg form of Ã by the
Ehrlich-Aberth iteration with Hyman's method (p(z)/p'(z) of det(H - zI) by the Hessenberg
back-recurrence), warm-started from an earlier frame's spectrum.  Not the product path."""
import os
import sys

import numpy as np
import scipy.linalg as sl

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import qr_aed  # noqa: E402


def hyman_ratio(H, z):
    """N(z) = p(z)/p'(z) for p(z) = det(H - zI), H unreduced upper Hessenberg (column-oriented
    back-substitution with x_n = 1, scaled)."""
    n = H.shape[0]
    x = np.zeros(n, complex)
    xd = np.zeros(n, complex)
    s = np.zeros(n, complex)       # s_i = sum_{j>i} h_ij x_j (accumulated column by column)
    sd = np.zeros(n, complex)
    x[n - 1] = 1.0
    xd[n - 1] = 0.0
    for j in range(n - 1, 0, -1):
        # column j contributes to rows < j
        s[:j] += H[:j, j] * x[j]
        sd[:j] += H[:j, j] * xd[j]
        # row j: h_{j,j-1} x_{j-1} + (h_jj - z) x_j + s_j = 0   (s_j excludes column j itself)
        r = (H[j, j] - z) * x[j] + s[j]
        rd = (H[j, j] - z) * xd[j] - x[j] + sd[j]
        x[j - 1] = -r / H[j, j - 1]
        xd[j - 1] = -rd / H[j, j - 1]
        sc = max(abs(x[j - 1]), abs(xd[j - 1]))
        if sc > 1e100 or (0 < sc < 1e-100):
            f = 1.0 / sc
            x *= f; xd *= f; s *= f; sd *= f
    # row 0: (h_00 - z) x_0 + sum_{j>0} h_0j x_j = alpha
    a = (H[0, 0] - z) * x[0] + (s[0] - 0)
    ad = (H[0, 0] - z) * xd[0] - x[0] + sd[0]
    return a / ad


def aberth(H, z0, tol=4 * np.finfo(float).eps, maxit=60, stats=None):
    z = np.array(z0, complex)
    n = len(z)
    done = np.zeros(n, bool)
    evals = 0
    for it in range(1, maxit + 1):
        evals += int((~done).sum())
        if stats is not None:
            stats.append(int((~done).sum()))
        N = np.array([hyman_ratio(H, zk) if not done[k] else 0.0 for k, zk in enumerate(z)])
        D = z[:, None] - z[None, :]
        np.fill_diagonal(D, 1.0)
        S = (1.0 / D).sum(axis=1) - 1.0        # remove the diagonal's 1/1
        step = N / (1 - N * S)
        step[done] = 0
        z = z - step
        done |= np.abs(step) <= tol * np.abs(z)
        if done.all():
            return z, it
    return z, -1


if __name__ == "__main__":
    from scipy.optimize import linear_sum_assignment
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    for t0, lag in [(20, 6), (40, 6), (60, 1), (80, 12)]:
        A = qr_aed.atilde(m, t0)
        Ap = qr_aed.atilde(m, t0 - lag)
        H = sl.hessenberg(A)
        ref = np.linalg.eigvals(A)
        prev = np.linalg.eigvals(Ap)
        # warm start: previous spectrum, real ones nudged off the axis
        z0 = prev.copy()
        real = np.abs(z0.imag) < 1e-14 * np.abs(z0)
        z0[real] += 1e-3j * np.abs(z0[real]) * np.where(np.arange(real.sum()) % 2, 1, -1)
        for tol in (4 * np.finfo(float).eps, 1e-14, 1e-13):
            st = []
            z, its = aberth(H, z0, tol=tol, stats=st)
            C = np.abs(z[:, None] - ref[None, :])
            ri, ci = linear_sum_assignment(C)
            print(f"t0={t0} lag={lag} tol={tol:.1e}: iterations {its}, evals {sum(st)} active/it {st[:12]}, "
                  f"max|Δλ| vs LAPACK {C[ri, ci].max():.2e}, trace err {abs(z.sum() - np.trace(H)):.2e}")
    # cold: circle
    A = qr_aed.atilde(m, 20)
    H = sl.hessenberg(A)
    ref = np.linalg.eigvals(A)
    rad = np.linalg.norm(H, 2)
    z0 = rad * np.exp(2j * np.pi * (np.arange(m) + 0.25) / m)
    z, its = aberth(H, z0)
    C = np.abs(z[:, None] - ref[None, :])
    ri, ci = linear_sum_assignment(C)
    print(f"cold circle: iterations {its}, max|Δλ| {C[ri, ci].max():.2e}")
