"""Prototype: sweep counts of the eigenvalue-only multishift QR on Ã (m = r = 200, C4s video
window) with and without aggressive early deflation (AED, Braman–Byers–Mathias 2002 II).
Cost model only (numpy, fp64): counts sweeps and bulge steps; not the product path."""
import os
import sys

import numpy as np
import scipy.linalg as sl
from scipy.linalg import lapack

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth  # noqa: E402

EPS = np.finfo(float).eps


def atilde(m, t0, name="C4s"):
    vs = synth.video_config(name)
    Z = np.stack([vs.frame(t).numpy().astype(np.float64) for t in range(t0, t0 + m + 1)], axis=1)
    G = Z.T @ Z
    S = G[:m, :m]
    mu, V = np.linalg.eigh(S)
    o = np.argsort(mu)[::-1]
    mu, V = mu[o], V[:, o]
    sig = np.sqrt(np.abs(mu))
    Y = V / sig
    return Y.T @ G[:m, 1:] @ Y


def francis(H, l, nn, st, sd):
    """one double-shift bulge chase on H[l:nn+1, l:nn+1] with shift polynomial x² - st x + sd."""
    n = nn - l + 1
    if n < 3:
        return
    h = H
    x = h[l, l] * h[l, l] - st * h[l, l] + sd + h[l, l + 1] * h[l + 1, l]
    y = h[l + 1, l] * (h[l, l] + h[l + 1, l + 1] - st)
    z = h[l + 1, l] * h[l + 2, l + 1]
    for k in range(l, nn):
        nr = 3 if k < nn - 1 else 2
        v = np.array([x, y, z][:nr])
        a = np.linalg.norm(v)
        if a == 0:
            break
        v[0] += np.copysign(a, v[0])
        v /= np.linalg.norm(v)
        r0 = max(l, k - 1)
        h[k:k + nr, r0:nn + 1] -= 2 * np.outer(v, v @ h[k:k + nr, r0:nn + 1])
        if k > l:
            h[k + 1:k + nr, k - 1] = 0.0
        r1 = min(nn, k + 3)
        h[l:r1 + 1, k:k + nr] -= 2 * np.outer(h[l:r1 + 1, k:k + nr] @ v, v)
        if k + 1 <= nn - 1:
            x = h[k + 1, k]
            y = h[k + 2, k]
            z = h[k + 3, k] if k + 3 <= nn else 0.0


def shifts_from(ev, ns):
    """pair up eigenvalues (conjugate pairs / two reals) into (trace, det) double shifts."""
    ev = list(ev)[:ns]
    out, pend = [], None
    i = 0
    while i < len(ev):
        e = ev[i]
        if abs(e.imag) > 0:
            out.append((2 * e.real, abs(e) ** 2))
            i += 2
            continue
        if pend is None:
            pend = e.real
        else:
            out.append((pend + e.real, pend * e.real))
            pend = None
        i += 1
    return out


def bottom_deflate(H, lo, nn, an):
    for li in range(nn, lo, -1):
        s = abs(H[li - 1, li - 1]) + abs(H[li, li])
        if s == 0:
            s = an
        if abs(H[li, li - 1]) + s == s:
            H[li, li - 1] = 0.0
            return li
    return lo


def ms_qr(H0, ns=16, aed=0, small=32, verbose=False):
    H = H0.copy()
    n = H.shape[0]
    an = np.abs(H).sum()
    nn = n - 1
    sweeps = steps = aed_calls = 0
    ev = []
    pending_shifts = None
    while nn >= 0:
        l = bottom_deflate(H, 0, nn, an)
        if l >= nn - 1:
            ev += list(np.linalg.eigvals(H[l:nn + 1, l:nn + 1]))
            nn = l - 1
            pending_shifts = None
            continue
        nact = nn - l + 1
        if nact <= small:
            ev += list(np.linalg.eigvals(H[l:nn + 1, l:nn + 1]))   # single-bulge (qr_block) tail
            nn = l - 1
            continue
        if aed and nact > aed + 2:
            aed_calls += 1
            w = aed
            kw = nn - w + 1
            T, Q = sl.schur(H[kw:nn + 1, kw:nn + 1], output="real")
            spike = H[kw, kw - 1] * Q[0, :].copy()
            # deflation check from the bottom, moving undeflatable blocks to the top (dtrexc)
            ndef = 0
            ifst_top = 0          # number of undeflatable eigenvalues moved to the top
            kend = w - 1
            while kend >= ifst_top:
                bs = 2 if (kend > 0 and T[kend, kend - 1] != 0) else 1
                if bs == 1:
                    ok = abs(spike[kend]) <= max(EPS * abs(T[kend, kend]), 1e-300)
                else:
                    blk = T[kend - 1:kend + 1, kend - 1:kend + 1]
                    lam = np.sqrt(abs(blk[0, 1])) * np.sqrt(abs(blk[1, 0])) + abs(blk[0, 0])
                    ok = max(abs(spike[kend]), abs(spike[kend - 1])) <= max(EPS * lam, 1e-300)
                if ok:
                    ndef += bs
                    kend -= bs
                    continue
                # move block at kend-bs+1 to position ifst_top (1-based for lapack)
                T, Q, info = lapack.dtrexc(T, Q, kend - bs + 2, ifst_top + 1)
                if info != 0:
                    break
                spike = H[kw, kw - 1] * Q[0, :]
                ifst_top += bs
            ndef = w - ifst_top
            # apply: H[kw:, kw:] <- T, spike in column kw-1, coupling rows/cols transformed
            H[kw:nn + 1, kw:nn + 1] = T
            H[kw:nn + 1, kw - 1] = spike
            H[l:kw, kw:nn + 1] = H[l:kw, kw:nn + 1] @ Q
            if ndef > 0:
                H[nn - ndef + 1, nn - ndef] = 0.0 if nn - ndef >= kw else H[nn - ndef + 1, nn - ndef]
                for j in range(nn - ndef + 1, nn + 1):
                    H[j, kw - 1] = 0.0
            # restore Hessenberg on [kw-1 .. nn-ndef] (Householder on the spike + top block)
            top = nn - ndef
            if top > kw:
                blk = H[kw - 1:top + 1, kw - 1:top + 1]
                Hh, Qh = sl.hessenberg(blk, calc_q=True)
                # apply the similarity to the coupling parts
                H[kw - 1:top + 1, kw - 1:top + 1] = Hh
                # Qh acts on indices kw-1..top; it must fix index kw-1 (first) for a valid similarity
                H[l:kw - 1, kw - 1:top + 1] = H[l:kw - 1, kw - 1:top + 1] @ Qh
                H[kw - 1:top + 1, top + 1:nn + 1] = Qh.T @ H[kw - 1:top + 1, top + 1:nn + 1]
            if ndef > 0:
                ev += list(np.linalg.eigvals(H[top + 1:nn + 1, top + 1:nn + 1]))
                nn = top
                if ndef >= 0.14 * w:          # LAPACK nibble: skip the sweep if AED did well
                    continue
            und = np.linalg.eigvals(T[:ifst_top, :ifst_top]) if ifst_top > 0 else []
            und = sorted(und, key=lambda e: abs(e))     # smallest last -> used first? keep order
            pending_shifts = shifts_from(und[-ns:], ns) if len(und) >= 2 else None
        nact = nn - l + 1
        if nact <= small:
            continue
        if pending_shifts:
            sh = pending_shifts
            pending_shifts = None
        else:
            b0 = nn - ns + 1
            sh = shifts_from(np.linalg.eigvals(H[b0:nn + 1, b0:nn + 1]), ns)
        for st, sd in sh:
            francis(H, l, nn, st, sd)
        sweeps += 1
        steps += (nn - l) + 4 * (len(sh) - 1)
    return np.array(ev), sweeps, steps, aed_calls


if __name__ == "__main__":
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    A = atilde(m, int(sys.argv[2]) if len(sys.argv) > 2 else 8)
    Hh = sl.hessenberg(A)
    ref = np.linalg.eigvals(A)
    for ns, aed in [(16, 0), (16, 24), (16, 32), (24, 36), (32, 48)]:
        ev, sw, stp, ac = ms_qr(Hh, ns=ns, aed=aed)
        # match
        from scipy.optimize import linear_sum_assignment
        C = np.abs(ev[:, None] - ref[None, :])
        ri, ci = linear_sum_assignment(C)
        print(f"ns={ns} aed={aed}: sweeps {sw} bulge-steps {stp} aed calls {ac} "
              f"n_ev {len(ev)} max|Δλ| {C[ri, ci].max():.2e}")


def ms_qr_recycled(H0, prev_ev, ns=16, small=32, fresh_after=None):
    """multishift QR whose first sweeps take their shifts from a previous frame's spectrum
    (pairs of conjugates / reals, ns per sweep); falls back to trailing-block shifts."""
    H = H0.copy()
    n = H.shape[0]
    an = np.abs(H).sum()
    nn = n - 1
    pool = list(shifts_from(sorted(prev_ev, key=lambda e: (abs(e), e.imag)), len(prev_ev)))
    sweeps = steps = fresh = 0
    ev = []
    while nn >= 0:
        l = bottom_deflate(H, 0, nn, an)
        if l >= nn - 1:
            ev += list(np.linalg.eigvals(H[l:nn + 1, l:nn + 1]))
            nn = l - 1
            continue
        nact = nn - l + 1
        if nact <= small:
            ev += list(np.linalg.eigvals(H[l:nn + 1, l:nn + 1]))
            nn = l - 1
            continue
        if pool:
            sh, pool = pool[:ns // 2], pool[ns // 2:]
        else:
            b0 = nn - ns + 1
            sh = shifts_from(np.linalg.eigvals(H[b0:nn + 1, b0:nn + 1]), ns)
            fresh += 1
        for st, sd in sh:
            francis(H, l, nn, st, sd)
        sweeps += 1
        steps += (nn - l) + 4 * (len(sh) - 1)
    return np.array(ev), sweeps, steps, fresh


def recycled_experiment(m=200, t0=8, lag=6):
    from scipy.optimize import linear_sum_assignment
    A = atilde(m, t0)
    Ap = atilde(m, t0 - lag)
    ref = np.linalg.eigvals(A)
    prev = np.linalg.eigvals(Ap)
    C = np.abs(prev[:, None] - ref[None, :])
    ri, ci = linear_sum_assignment(C)
    d = C[ri, ci]
    print(f"lag {lag}: |λ_t - λ_(t-lag)| matched: median {np.median(d):.2e} max {d.max():.2e}")
    Hh = sl.hessenberg(A)
    for ns in (16, 32):
        ev, sw, stp, fr = ms_qr_recycled(Hh, prev, ns=ns)
        C2 = np.abs(ev[:, None] - ref[None, :])
        r2, c2 = linear_sum_assignment(C2)
        print(f"  recycled ns={ns}: sweeps {sw} (fresh-shift sweeps {fr}) steps {stp} max|Δλ| {C2[r2, c2].max():.2e}")
