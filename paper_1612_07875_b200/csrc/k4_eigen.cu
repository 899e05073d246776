// k4_eigen.cu — K4: single-CTA on-device eigen engine of one streamed frame (no CPU fallback).
//
// For the window ending at frame f (Z = [x_{f-m} … x_f]), entirely from the Gram history:
//   a5  S = XᵀX = G[0:m,0:m]; one-sided (Hestenes) Jacobi on S: S J = A with orthogonal columns,
//       so |eig(S)| = ‖a_j‖ and V = a_j/‖a_j‖ (no rotation accumulation)   (§2.1; Alg 1)
//   a6  σ = sqrt(|μ|) sorted desc, V permuted, r = #{σ > τσ₁} (Alg 1; reading Q7),
//       Y = V Σ⁻¹ ("vsi", Alg 2)
//   a7  Ã = Yᵀ (XᵀX') Y with XᵀX' = G[0:m,1:m+1] — zero new n-length dots (Alg 2)
//   a8  eig(Ã): Householder Hessenberg reduction + Francis double-shift QR (eigenvalues) in
//       shared memory (textbook algorithms, Golub–Van Loan §7.4-7.5; the paper only says "eig",
//       P:314); inverse iteration on the Hessenberg form for the right/left eigenvectors needed
//   a9  α₁ = Σ V[0,:]ᵀ (reading Q3), b_idx = y_idxᴴα₁ / (λ_idx y_idxᴴ w_idx)  (§3.3 P:264-273:
//       "only the row corresponding to the … DMD eigenvalue need be calculated")
//   a10 idx = argmin |log λ| (Alg 3; tie rule Q5)
//   a11 (coefficients) c = b_idx λ_idx^m Y w_idx, so that l = X' c = b_idx φ_idx λ_idx^m (Q4)
// The result c is consumed by a later K1 pass (fused background).  Everything is deterministic
// (fixed reduction orders, no atomics), so replicated ranks compute bit-identical factors.
#include <cfloat>
#include <cstdlib>
#include "sdmd_internal.cuh"

namespace sdmd {

constexpr int K4_THREADS = 512;
constexpr int K4_WARPS = K4_THREADS / 32;
constexpr int JACOBI_MAX_SWEEPS = 60;
constexpr int QR_MAXITS = 60;

// ------------------------------------------------------------------ small helpers ------------
static __device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
static __device__ __forceinline__ double wmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
static __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
static __device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
static __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
static __device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
static __device__ __forceinline__ double cabs2(double2 a) { return hypot(a.x, a.y); }
static __device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  // Smith's algorithm
  if (fabs(b.x) >= fabs(b.y)) {
    const double rr = b.y / b.x, den = b.x + b.y * rr;
    return make_double2((a.x + a.y * rr) / den, (a.y - a.x * rr) / den);
  }
  const double rr = b.x / b.y, den = b.x * rr + b.y;
  return make_double2((a.x * rr + a.y) / den, (a.y * rr - a.x) / den);
}
static __device__ __forceinline__ double2 wsum2(double2 v) { return make_double2(wsum(v.x), wsum(v.y)); }

// G_f(i, j), 0 <= i, j <= m, for the window ending at frame f (see sdmd_internal.cuh)
static __device__ __forceinline__ double gram_at(const double* gh, int NH, int mh, int w, long long f,
                                                int i, int j) {
  // window of width w ending at frame f (frames f-w .. f); history rows of stride mh+1
  // (row of frame g: <x_{g-mh+k}, x_g> at k)
  const int a = i < j ? i : j, b = i < j ? j : i;
  const long long fb = f - w + b;
  return __ldcg(gh + (fb % NH) * (mh + 1) + (a - b + mh));   // L2: rows are published by commits
}

static __device__ __forceinline__ int rr_player(int pos, int step, int mp) {
  return pos == 0 ? 0 : 1 + (pos - 1 + step) % (mp - 1);
}

// Packed upper-Hessenberg storage with 3 sub-diagonals of slack for the double-shift bulge:
// row i holds columns max(0, i-3) .. r-1; its offset is computed arithmetically (no lookup table).
__host__ __device__ __forceinline__ long long hs_off(int i, int r) {
  return i <= 4 ? (long long)i * r
                : 4LL * r + (long long)(i - 4) * (r + 3) - ((long long)(i - 1) * i / 2 - 6);
}
struct HsAcc {
  double* hs;
  int r;
  __device__ __forceinline__ double& operator()(int i, int j) const {
    const int lo = i > 3 ? i - 3 : 0;
    return hs[hs_off(i, r) + j - lo];
  }
  __device__ __forceinline__ double* row(int i) const { return hs + (hs_off(i, r) - (i > 3 ? i - 3 : 0)); }
};
// Packed Hessenberg through a per-row offset table in shared memory (one LDS per row access)
struct RowAcc {
  double* hs;
  const int* roff;            // roff[i] = hs_off(i) - max(0, i-3)
  __device__ __forceinline__ double& operator()(int i, int j) const { return hs[roff[i] + j]; }
  __device__ __forceinline__ double* row(int i) const { return hs + roff[i]; }
};
// Dense row-major small block (leading dimension ld)
struct DenseAcc {
  double* a;
  int ld;
  __device__ __forceinline__ double& operator()(int i, int j) const { return a[i * ld + j]; }
  __device__ __forceinline__ double* row(int i) const { return a + i * ld; }
};

__host__ __device__ inline long long hs_elems(int r) { return hs_off(r, r); }

// Eigenvalues of an upper Hessenberg matrix by the Francis double-shift QR iteration with
// deflation on negligible sub-diagonals and ad-hoc exceptional shifts every 10 iterations
// (eigenvalues only: updates restricted to the active block).  Executed by ONE warp: every lane
// runs the scalar recurrences redundantly on identical shared-memory data; lanes split the row
// and column updates of each 3x3 reflector.  Returns 0, or -1 when an eigenvalue needs more than
// QR_MAXITS iterations.
template <class Acc>
static __device__ int qr_block(Acc a, int lo, int hi, double2* wv, int lane, int* total_its,
                               int* cnt) {
  int c_steps = 0, c_scan = 0, c_mscan = 0;
  double an = 0.0;
  for (int i = lo; i <= hi; ++i)
    for (int j = (i > lo ? i - 1 : lo) + lane; j <= hi; j += 32) an += fabs(a(i, j));
  an = wsum(an);
  int nn = hi, tot = 0;
  double t = 0.0;
  while (nn >= lo) {
    int its = 0, l;
    do {
      // largest l in [lo+1, nn] with a negligible sub-diagonal a(l, l-1) (lanes test 32 at a time)
      l = lo;
      for (int base = nn; base >= lo + 1; base -= 32) {
        ++c_scan;
        const int li = base - lane;
        bool neg = false;
        if (li >= lo + 1) {
          double s = fabs(a(li - 1, li - 1)) + fabs(a(li, li));
          if (s == 0.0) s = an;
          neg = (fabs(a(li, li - 1)) + s == s);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, neg);
        if (bal) { l = base - (__ffs(bal) - 1); break; }
      }
      if (l >= lo + 1) {
        __syncwarp();
        if (lane == 0) a(l, l - 1) = 0.0;
        __syncwarp();
      }
      double x = a(nn, nn);
      if (l == nn) {                                   // one root
        if (lane == 0) wv[nn] = make_double2(x + t, 0.0);
        nn -= 1;
      } else {
        double y = a(nn - 1, nn - 1), w = a(nn, nn - 1) * a(nn - 1, nn);
        if (l == nn - 1) {                             // two roots (2x2 block)
          const double p = 0.5 * (y - x), q = p * p + w;
          double z = sqrt(fabs(q));
          x += t;
          if (q >= 0.0) {
            z = p + copysign(z, p);
            const double e1 = x + z, e2 = (z != 0.0) ? x - w / z : e1;
            if (lane == 0) { wv[nn - 1] = make_double2(e1, 0.0); wv[nn] = make_double2(e2, 0.0); }
          } else if (lane == 0) {
            wv[nn - 1] = make_double2(x + p, z);
            wv[nn] = make_double2(x + p, -z);
          }
          nn -= 2;
        } else {                                       // no root yet: one double-shift sweep
          if (its == QR_MAXITS) return -1;
          if (its > 0 && its % 10 == 0) {              // exceptional shift
            t += x;
            __syncwarp();
            for (int i = lo + lane; i <= nn; i += 32) a(i, i) -= x;
            __syncwarp();
            const double s = fabs(a(nn, nn - 1)) + fabs(a(nn - 1, nn - 2));
            y = x = 0.75 * s;
            w = -0.4375 * s * s;
          }
          ++its;
          ++tot;
          // start of the bulge: the largest mm in [l, nn-2] where two consecutive sub-diagonals
          // are negligible relative to the shifted first column (or mm = l); lanes test 32 at a time
          int mm = l;
          for (int base = nn - 2; base >= l; base -= 32) {
            ++c_mscan;
            const int mi = base - lane;
            bool ok = false;
            if (mi >= l) {
              if (mi == l) {
                ok = true;
              } else {
                const double zz = a(mi, mi), rr = x - zz, ss = y - zz;
                double pp = (rr * ss - w) / a(mi + 1, mi) + a(mi, mi + 1);
                double qq = a(mi + 1, mi + 1) - zz - rr - ss;
                double r3 = a(mi + 2, mi + 1);
                const double sc = fabs(pp) + fabs(qq) + fabs(r3);
                pp /= sc; qq /= sc; r3 /= sc;
                const double u = fabs(a(mi, mi - 1)) * (fabs(qq) + fabs(r3));
                const double v = fabs(pp) * (fabs(a(mi - 1, mi - 1)) + fabs(zz) + fabs(a(mi + 1, mi + 1)));
                ok = (u + v == v);
              }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, ok);
            if (bal) { mm = base - (__ffs(bal) - 1); break; }
          }
          double p, q, r, z;
          {
            z = a(mm, mm);
            r = x - z;
            const double s = y - z;
            p = (r * s - w) / a(mm + 1, mm) + a(mm, mm + 1);
            q = a(mm + 1, mm + 1) - z - r - s;
            r = a(mm + 2, mm + 1);
            const double is = 1.0 / (fabs(p) + fabs(q) + fabs(r));
            p *= is; q *= is; r *= is;
          }
          __syncwarp();
          for (int i = mm + 2 + lane; i <= nn; i += 32) {
            a(i, i - 2) = 0.0;
            if (i != mm + 2) a(i, i - 3) = 0.0;
          }
          __syncwarp();
          for (int k = mm; k <= nn - 1; ++k) {          // chase the bulge
            ++c_steps;
            double xs = 1.0;                            // scale of (p, q, r)
            if (k != mm) {
              p = a(k, k - 1);
              q = a(k + 1, k - 1);
              r = (k != nn - 1) ? a(k + 2, k - 1) : 0.0;
              const double ss = p * p + q * q + r * r;
              if (!(ss > 1e-280 && ss < 1e280)) {       // rescale only when squares leave range
                x = fabs(p) + fabs(q) + fabs(r);
                if (x != 0.0) { const double ix = 1.0 / x; p *= ix; q *= ix; r *= ix; xs = x; }
              }
            }
            const double s = copysign(sqrt(p * p + q * q + r * r), p);
            if (s != 0.0) {
              __syncwarp();
              if (k == mm) {
                if (l != mm && lane == 0) a(k, k - 1) = -a(k, k - 1);
              } else if (lane == 0) {
                a(k, k - 1) = -s * xs;
              }
              p += s;
              {                                         // one division for 1/s and 1/p
                const double inv = 1.0 / (s * p);
                const double is = p * inv, ip = s * inv;
                x = p * is; y = q * is; z = r * is;
                q *= ip; r *= ip;
              }
              const bool three = (k != nn - 1);
              __syncwarp();
              {                                         // row modification (2 columns per lane in flight)
                double* r0 = a.row(k);
                double* r1 = a.row(k + 1);
                double* r2 = a.row(three ? k + 2 : k + 1);
                for (int j = k + lane; j <= nn; j += 64) {
                  const int j2 = j + 32;
                  const bool h2 = j2 <= nn;
                  const double a0 = r0[j], a1 = r1[j], a2 = three ? r2[j] : 0.0;
                  const double b0 = h2 ? r0[j2] : 0.0, b1 = h2 ? r1[j2] : 0.0;
                  const double b2 = (h2 && three) ? r2[j2] : 0.0;
                  const double pa = a0 + q * a1 + r * a2, pb = b0 + q * b1 + r * b2;
                  if (three) r2[j] = a2 - pa * z;
                  r1[j] = a1 - pa * y;
                  r0[j] = a0 - pa * x;
                  if (h2) {
                    if (three) r2[j2] = b2 - pb * z;
                    r1[j2] = b1 - pb * y;
                    r0[j2] = b0 - pb * x;
                  }
                }
              }
              __syncwarp();
              const int mmin = nn < k + 3 ? nn : k + 3;
              for (int i = l + lane; i <= mmin; i += 64) { // column modification (2 rows per lane)
                const int i2 = i + 32;
                const bool h2 = i2 <= mmin;
                double* ri = a.row(i);
                double* rj = a.row(h2 ? i2 : i);
                const double c0 = ri[k], c1 = ri[k + 1], c2 = three ? ri[k + 2] : 0.0;
                const double d0 = h2 ? rj[k] : 0.0, d1 = h2 ? rj[k + 1] : 0.0;
                const double d2 = (h2 && three) ? rj[k + 2] : 0.0;
                const double pp = x * c0 + y * c1 + z * c2, pq = x * d0 + y * d1 + z * d2;
                if (three) ri[k + 2] = c2 - pp * r;
                ri[k + 1] = c1 - pp * q;
                ri[k] = c0 - pp;
                if (h2) {
                  if (three) rj[k + 2] = d2 - pq * r;
                  rj[k + 1] = d1 - pq * q;
                  rj[k] = d0 - pq;
                }
              }
              __syncwarp();
            }
          }
        }
      }
    } while (l < nn - 1);
  }
  *total_its += tot;
  if (cnt && lane == 0) { cnt[0] += c_steps; cnt[2] += tot; }
  (void)c_scan; (void)c_mscan;
  return 0;
}

// ---------------------------------------------------------------------------------------------
// Multishift QR (eigenvalues only), CTA-level.  Each sweep takes ns = 2·NB shifts — the
// eigenvalues of the trailing ns x ns block, computed by qr_block on a small copy — and chases NB
// double-shift bulges down the active block in lockstep, bulge b on warp b, 4 positions apart.
// Per global step: (A) every active bulge forms its 3x3 reflector, (B) row updates, (C) column
// updates, each phase followed by a CTA barrier.  Concurrent bulges act on disjoint rows in (B) and
// disjoint columns in (C), and left and right reflections commute, so a sweep is exactly NB
// successive Francis double-shift steps with the given shifts.  Small or stagnating blocks fall
// back to the single-bulge qr_block.  (Golub–Van Loan §7.5; small-bulge multishift idea of
// Braman–Byers–Mathias; no aggressive early deflation.)
constexpr int MS_NB = 8;           // bulges per sweep (2 warps each)
#ifndef K4_MS_SMALL
#define K4_MS_SMALL 32
#endif
constexpr int MS_SMALL = K4_MS_SMALL;   // blocks up to this size use the single-bulge iteration
constexpr int MS_STALL = 30;       // sweeps without deflation before falling back
constexpr int MS_SPACING = 4;
constexpr int MS_DLD = MS_SMALL + 1;   // leading dimension of the dense small-block copy

// 3x3 (or 2x2) Householder reflector of the double-shift chase in the hqr form: applied to
// (a0, a1, a2) as pr = a0 + q a1 + r a2; a0 -= pr x; a1 -= pr y; a2 -= pr z (rows), and with
// (x, y, z) / (1, q, r) swapped for columns; sxs = the new bulge-column head -s·scale.
struct MsRefl {
  double x, y, z, q, r, sxs;
  bool on;
};
static __device__ __forceinline__ MsRefl ms_reflector(double P, double Q, double R) {
  MsRefl f;
  double xs = 1.0;
  const double sc = fabs(P) + fabs(Q) + fabs(R);
  const double ss0 = P * P + Q * Q + R * R;
  if (!(ss0 > 1e-280 && ss0 < 1e280) && sc != 0.0) {     // rescale only when squares leave range
    const double isc = 1.0 / sc;
    P *= isc; Q *= isc; R *= isc;
    xs = sc;
  }
  const double s = copysign(sqrt(P * P + Q * Q + R * R), P);
  f.on = (s != 0.0);
  if (f.on) {
    f.sxs = -s * xs;
    const double pp = P + s;
    const double inv = 1.0 / (s * pp);                  // one division for 1/s and 1/pp
    const double is = pp * inv, ip = s * inv;
    f.x = pp * is; f.y = Q * is; f.z = R * is;
    f.q = Q * ip; f.r = R * ip;
  } else {
    f.x = f.y = f.z = f.q = f.r = f.sxs = 0.0;
  }
  return f;
}

#ifndef K4_JAC_FLAGS
#define K4_JAC_FLAGS 1     // Jacobi rounds 1..6 synchronised by neighbour step counters, not barriers
#endif
#ifndef K4_MS_PIPE
#define K4_MS_PIPE 160     // r >= this: shifts computed one sweep ahead by warp 0 while warps 2..15
                           // chase (0 = never).  Measured QR cycles pipelined vs in place:
                           // r = 100 10.8 M vs 9.4 M, r = 128 12.9 M vs 12.9 M, r = 200 19.9 M vs
                           // 22.3 M (more, staler sweeps; the shift work leaves the critical path)
#endif
struct MsShared {
  double dense[MS_SMALL * MS_DLD]; // dense copy of the shift block (ns x ns) or of a tail block
  double st[MS_NB], sd[MS_NB];
  double stn[MS_NB], sdn[MS_NB];   // pipelined shifts for the next sweep
  double2 sw[MS_SMALL];
  int l, nbe, fail, nbn;
};

// eigenvalues of the dense ns x ns copy (one warp) paired into double shifts (trace, det)
static __device__ int ms_pair_shifts(MsShared* sh, int ns, double* st, double* sd, int lane) {
  int its_s = 0;
  const int rc = qr_block(DenseAcc{sh->dense, MS_DLD}, 0, ns - 1, sh->sw, lane, &its_s, nullptr);
  __syncwarp();
  int nb = 0;
  if (rc == 0) {
    double rl = 0.0;
    bool have_real = false;
    for (int i = 0; i < ns && nb < MS_NB; ++i) {
      const double2 e = sh->sw[i];
      if (e.y != 0.0) {                            // conjugate pair (i, i+1)
        if (lane == 0) { st[nb] = 2.0 * e.x; sd[nb] = e.x * e.x + e.y * e.y; }
        ++nb;
        ++i;
      } else if (have_real) {
        if (lane == 0) { st[nb] = rl + e.x; sd[nb] = rl * e.x; }
        ++nb;
        have_real = false;
      } else {
        rl = e.x;
        have_real = true;
      }
    }
  }
  __syncwarp();
  return nb;
}

static __device__ __forceinline__ void ms_chase_sync(bool pipe) {
  if (pipe) asm volatile("bar.sync 1, %0;" ::"n"(K4_THREADS - 64) : "memory");   // warps 2..15
  else __syncthreads();
}

template <class Acc>
static __device__ void ms_two_roots(Acc a, int nn, double2* wv) {
  const double x = a(nn, nn), y = a(nn - 1, nn - 1), w = a(nn, nn - 1) * a(nn - 1, nn);
  const double p = 0.5 * (y - x), q = p * p + w;
  double z = sqrt(fabs(q));
  if (q >= 0.0) {
    z = p + copysign(z, p);
    const double e1 = x + z, e2 = (z != 0.0) ? x - w / z : e1;
    wv[nn - 1] = make_double2(e1, 0.0);
    wv[nn] = make_double2(e2, 0.0);
  } else {
    wv[nn - 1] = make_double2(x + p, z);
    wv[nn] = make_double2(x + p, -z);
  }
}

// copy the Hessenberg block [b0, b0+nb) of a into the dense small buffer (all threads)
static __device__ void ms_copy_block(RowAcc a, int b0, int nb, double* dense, int tid) {
  for (int e = tid; e < nb * nb; e += K4_THREADS) {
    const int i = e / nb, j = e % nb;
    dense[i * MS_DLD + j] = (j >= i - 1) ? a(b0 + i, b0 + j) : 0.0;
  }
}

// Per global step of the lockstep chase: (AB) the two warps of each active bulge form its 3x3
// reflector redundantly in registers and apply it to rows k..k+2 (columns k..nn, split between
// the warps); CTA barrier; (C) they apply it to columns k..k+2 (rows l..min(nn,k+3)) and write
// the annihilated bulge column k-1; CTA barrier.  Concurrent bulges (MS_SPACING apart) touch
// disjoint rows in (AB) and disjoint columns in (C), and a bulge's reflector input (column k-1)
// is written only by its own warps in the previous (C), so two barriers per step suffice.
static __device__ int multishift_qr(RowAcc a, int n, double2* wv, MsShared* sh, int tid, int warp,
                                    int lane, int* total_its, int* cnt, long long* shift_cycles,
                                    long long* chase_cycles) {
  double an = 0.0;
  if (warp == 0) {
    for (int i = 0; i < n; ++i) {
      const double* ri = a.row(i);
      for (int j = (i > 0 ? i - 1 : 0) + lane; j < n; j += 32) an += fabs(ri[j]);
    }
    an = wsum(an);
  }
  int nn = n - 1, stall = 0, status = 0;
  bool pend = false;                                 // pipelined shifts available (sh->stn/sdn)
  while (nn >= 0) {
    // ---- deflation at the bottom of the active block (warp 0)
    if (warp == 0) {
      int l = 0;
      for (int base = nn; base >= 1; base -= 32) {
        const int li = base - lane;
        bool neg = false;
        if (li >= 1) {
          double s = fabs(a(li - 1, li - 1)) + fabs(a(li, li));
          if (s == 0.0) s = an;
          neg = (fabs(a(li, li - 1)) + s == s);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, neg);
        if (bal) { l = base - (__ffs(bal) - 1); break; }
      }
      if (lane == 0) {
        if (l >= 1) a(l, l - 1) = 0.0;
        sh->l = l;
        if (l == nn) wv[nn] = make_double2(a(nn, nn), 0.0);
        else if (l == nn - 1) ms_two_roots(a, nn, wv);
      }
    }
    __syncthreads();
    const int l = sh->l;
    if (l >= nn - 1) {                                   // 1 or 2 eigenvalues deflated
      nn = l - 1;
      stall = 0;
      __syncthreads();
      continue;
    }
    const int nact = nn - l + 1;
    if (nact <= MS_SMALL || stall >= MS_STALL) {        // single-bulge iteration on [l, nn]
      if (nact <= MS_SMALL) {
        ms_copy_block(a, l, nact, sh->dense, tid);
        __syncthreads();
        if (warp == 0) {
          const int rc = qr_block(DenseAcc{sh->dense, MS_DLD}, 0, nact - 1, wv + l, lane, total_its, cnt);
          if (lane == 0) sh->fail = rc;
        }
      } else if (warp == 0) {
        const int rc = qr_block(a, l, nn, wv, lane, total_its, cnt);
        if (lane == 0) sh->fail = rc;
      }
      __syncthreads();
      if (sh->fail != 0) status = -1;
      nn = l - 1;
      stall = 0;
      __syncthreads();
      if (status) return status;
      continue;
    }
    // ---- shifts: eigenvalues of the trailing ns x ns block (dense copy, warp 0).  Pipelined
    // (K4_MS_PIPE): after the first sweep, the shifts of sweep s come from the trailing block at
    // the START of sweep s-1, computed by warp 0 while warps 2..15 chase sweep s-1 (one sweep
    // stale: more sweeps, but the shift computation leaves the critical path; the numpy model
    // scripts/proto/qr_aed.py counts +25-38 % sweeps).  The first sweep computes them in place.
    int ns = 2 * MS_NB;
    if (ns > ((nact - 2) & ~1)) ns = (nact - 2) & ~1;
    const long long t_sh0 = clock64();
    const bool pipe = K4_MS_PIPE > 0 && n >= K4_MS_PIPE && pend;   // uniform
    if (!pipe) {
      ms_copy_block(a, nn - ns + 1, ns, sh->dense, tid);
      __syncthreads();
      if (warp == 0) {
        const int nb = ms_pair_shifts(sh, ns, sh->st, sh->sd, lane);
        if (lane == 0) {
          sh->nbe = nb;
          for (int q = 0; q < nb; ++q) { sh->stn[q] = sh->st[q]; sh->sdn[q] = sh->sd[q]; }
          sh->nbn = nb;                                   // sweep s+1 reuses them (same state)
        }
      }
    } else {
      if (tid == 0) {
        const int nb = sh->nbn < MS_NB - 1 ? sh->nbn : MS_NB - 1;   // 7 bulges on warps 2..15
        for (int q = 0; q < nb; ++q) { sh->st[q] = sh->stn[q]; sh->sd[q] = sh->sdn[q]; }
        sh->nbe = nb;
      }
      ms_copy_block(a, nn - ns + 1, ns, sh->dense, tid);   // snapshot for sweep s+1's shifts
    }
    __syncthreads();
    if (tid == 0 && shift_cycles) *shift_cycles += clock64() - t_sh0;
    const int nbe = sh->nbe;
    if (nbe == 0) { stall = MS_STALL; pend = false; continue; }
    if (K4_MS_PIPE > 0 && n >= K4_MS_PIPE) pend = true;
    if (pipe && warp == 0) {                                 // next sweep's shifts, concurrently
      const int nb = ms_pair_shifts(sh, ns, sh->stn, sh->sdn, lane);
      if (lane == 0) sh->nbn = nb;
    }
    // ---- chase nbe bulges in lockstep, bulge b on warps 2b (half 0) and 2b+1 (half 1); when
    // pipelined, on warps 2b+2 and 2b+3 with a named barrier over those 14 warps
    const int bw = pipe ? warp - 2 : warp;
    const int b = bw >= 0 ? bw >> 1 : MS_NB, half = warp & 1;
    const double st_b = (b < nbe) ? sh->st[b] : 0.0, sd_b = (b < nbe) ? sh->sd[b] : 0.0;
    const int G = (nn - 1 - l) + MS_SPACING * (nbe - 1);
    const bool chaser = !pipe || warp >= 2;
    MsRefl rf{};                       // reflector of the current step (both halves)
    long long t_ab = 0, t_c = 0;
    for (int g = 0; chaser && g <= G; ++g) {
      const long long t0 = clock64();
      const int k = l + g - MS_SPACING * b;
      const bool act = (b < nbe) && (k >= l && k <= nn - 1);
      const bool three = (k != nn - 1);
      if (act) {
        if (k == l) {                  // introduce the bulge: first column of (H - s1)(H - s2)
          const double* rl0 = a.row(l);
          const double* rl1 = a.row(l + 1);
          const double h00 = rl0[l], h01 = rl0[l + 1], h10 = rl1[l], h11 = rl1[l + 1];
          const double h21 = a(l + 2, l + 1);
          rf = ms_reflector(h00 * (h00 - st_b) + sd_b + h01 * h10, h10 * (h00 + h11 - st_b), h10 * h21);
        } else {                       // both halves, redundantly, from the bulge column k-1
          rf = ms_reflector(a(k, k - 1), a(k + 1, k - 1), three ? a(k + 2, k - 1) : 0.0);
        }
        if (rf.on) {                   // (AB) rows k..k+2, columns k..nn
          double* r0 = a.row(k);
          double* r1 = a.row(k + 1);
          double* r2 = three ? a.row(k + 2) : r1;
          for (int j = k + half * 32 + lane; j <= nn; j += 64) {
            const double a0 = r0[j], a1 = r1[j], a2 = three ? r2[j] : 0.0;
            const double pr = a0 + rf.q * a1 + rf.r * a2;
            if (three) r2[j] = a2 - pr * rf.z;
            r1[j] = a1 - pr * rf.y;
            r0[j] = a0 - pr * rf.x;
          }
        }
      }
      ms_chase_sync(pipe);
      const long long t1 = clock64();
      if (act && rf.on) {
        // (C) columns k..k+2, rows l..min(nn, k+3); bulge column k-1
        if (half == 0 && lane == 0 && k > l) {
          a(k, k - 1) = rf.sxs;
          a(k + 1, k - 1) = 0.0;
          if (three) a(k + 2, k - 1) = 0.0;
        }
        const int mmin = nn < k + 3 ? nn : k + 3;
        for (int i = l + half * 32 + lane; i <= mmin; i += 64) {
          double* ri = a.row(i);
          const double c0 = ri[k], c1 = ri[k + 1], c2 = three ? ri[k + 2] : 0.0;
          const double pc = rf.x * c0 + rf.y * c1 + rf.z * c2;
          if (three) ri[k + 2] = c2 - pc * rf.r;
          ri[k + 1] = c1 - pc * rf.q;
          ri[k] = c0 - pc;
        }
      }
      ms_chase_sync(pipe);
      t_ab += t1 - t0;
      t_c += clock64() - t1;
    }
    __syncthreads();                                           // chase and shift warps join
    if (tid == (pipe ? 64 : 0) && chase_cycles) { chase_cycles[0] += t_ab; chase_cycles[1] += t_c; }
    if (tid == 0) { *total_its += 1; if (cnt) { cnt[1] += G + 1; cnt[3] += 1; } }
    ++stall;
  }
  return status;
}

// ---------------------------------------------------------------------------------------------
// Eigenvalues of the unreduced upper Hessenberg H (r x r) by the Ehrlich–Aberth simultaneous
// iteration (Aberth 1973; Bini–Gemignani–Tisseur's Hessenberg variant), warm-started from an
// earlier frame's spectrum.  For each root z_k the Newton ratio N = p(z)/p'(z), p = det(H − zI),
// comes from Hyman's method: the back-recurrence of (H − zI) x = α e₁ with x_{r-1} = 1,
//     x_{j-1} = −[(h_jj − z) x_j + Σ_{i>j} h_ji x_i] / h_{j,j-1},   α = (h_00 − z) x_0 + Σ h_0i x_i,
// so p(z) ∝ α(z) and p'/p = α'/α (the constant Π h_{j,j-1} cancels; x and its z-derivative x' are
// rescaled together whenever they leave [1e-100, 1e100]).  One warp per root: lanes own rows,
// accumulate the partial sums Σ_{i>j} h_ji x_i column by column (column-packed H in shared memory,
// 1/h_{j,j-1} stored in place of h_{j,j-1}), and the owner lane of row j forms x_{j-1}.  The update
// z_k ← z_k − N_k / (1 − N_k Σ_{j≠k} 1/(z_k − z_j)) is Jacobi-style (every root from the previous
// iterate), so the result is deterministic.  A root is frozen once its correction is below
// 4u|z_k|.  Returns 0 with the spectrum (conjugate pairs made exact, near-real roots snapped to
// the real axis) in lam_out, or −1 (not converged in the budget, a non-finite step, a trace
// mismatch, a reducible H) — the caller then runs the Francis QR.
constexpr int AB_MAXIT = 40;
constexpr int AB_RQ = (kMaxR + 31) / 32;
__host__ __device__ __forceinline__ int ab_cofs(int j) { return j * (j + 5) / 2; }  // column j start

static __device__ double2 hyman_ratio(const double* hc, int r, double2 z, int lane) {
  double2 s[AB_RQ], sd[AB_RQ];
#pragma unroll
  for (int q = 0; q < AB_RQ; ++q) { s[q] = make_double2(0.0, 0.0); sd[q] = make_double2(0.0, 0.0); }
  double2 x = make_double2(1.0, 0.0), xd = make_double2(0.0, 0.0);
  // rows in blocks of 32 (block qb: rows 32qb .. 32qb+31, lane = row mod 32), unrolled over qb so
  // that the owner's partial sums s[qb] and the axpy extents are static: at step j (block qb,
  // jj = j - 32qb) the owner is lane jj; column j updates the full blocks q < qb and lanes < jj
  // of block qb (rows i < j)
#pragma unroll
  for (int qb = AB_RQ - 1; qb >= 0; --qb) {
    if (32 * qb >= r) continue;
    const int jhi = (r - 1 - 32 * qb) < 31 ? (r - 1 - 32 * qb) : 31;
    const int jlo = qb == 0 ? 1 : 0;
    for (int jj = jhi; jj >= jlo; --jj) {
      const int j = 32 * qb + jj;
      const double* cj = hc + ab_cofs(j);
      const double2 dz = make_double2(cj[j] - z.x, -z.y);             // h_jj − z
      const double inv = hc[ab_cofs(j - 1) + j];                        // 1/h_{j,j-1} (in place)
      // owner (lane jj): x_{j-1} = −[(h_jj − z) x_j + s_j] / h_{j,j-1}, and its z-derivative
      const double2 rr = cadd(cmul(dz, x), s[qb]);
      const double2 rd = csub(cadd(cmul(dz, xd), sd[qb]), x);
      const double2 xn = make_double2(-rr.x * inv, -rr.y * inv);
      const double2 xdn = make_double2(-rd.x * inv, -rd.y * inv);
      // column j into the rows above it
#pragma unroll
      for (int q = 0; q < qb; ++q) {
        const double h = cj[lane + 32 * q];
        s[q] = make_double2(fma(h, x.x, s[q].x), fma(h, x.y, s[q].y));
        sd[q] = make_double2(fma(h, xd.x, sd[q].x), fma(h, xd.y, sd[q].y));
      }
      if (lane < jj) {
        const double h = cj[lane + 32 * qb];
        s[qb] = make_double2(fma(h, x.x, s[qb].x), fma(h, x.y, s[qb].y));
        sd[qb] = make_double2(fma(h, xd.x, sd[qb].x), fma(h, xd.y, sd[qb].y));
      }
      x = make_double2(__shfl_sync(0xffffffffu, xn.x, jj), __shfl_sync(0xffffffffu, xn.y, jj));
      xd = make_double2(__shfl_sync(0xffffffffu, xdn.x, jj), __shfl_sync(0xffffffffu, xdn.y, jj));
      if ((jj & 3) == 0) {                                             // warp-uniform rescale
        const double mx = fabs(x.x) + fabs(x.y) + fabs(xd.x) + fabs(xd.y);
        if (mx > 1e100 || (mx < 1e-100 && mx > 0.0)) {
          const double f = 1.0 / mx;
          x = make_double2(x.x * f, x.y * f);
          xd = make_double2(xd.x * f, xd.y * f);
#pragma unroll
          for (int q = 0; q < AB_RQ; ++q) {
            s[q] = make_double2(s[q].x * f, s[q].y * f);
            sd[q] = make_double2(sd[q].x * f, sd[q].y * f);
          }
        }
      }
    }
  }
  // row 0 (owner: lane 0, block 0): α = (h_00 − z) x_0 + s_0, α' = (h_00 − z) x'_0 − x_0 + s'_0
  double2 N = make_double2(0.0, 0.0);
  if (lane == 0) {
    const double2 dz = make_double2(hc[0] - z.x, -z.y);
    const double2 a = cadd(cmul(dz, x), s[0]);
    const double2 ad = csub(cadd(cmul(dz, xd), sd[0]), x);
    N = cdiv(a, ad);
  }
  return make_double2(__shfl_sync(0xffffffffu, N.x, 0), __shfl_sync(0xffffffffu, N.y, 0));
}

// Inverse iteration on the Hessenberg form H (row-major r x r, global) for eigenvalue lam, one
// warp.  Returns the right eigenvector w = Q z and (if yout) the left eigenvector y = Q u of the
// ORIGINAL matrix Ã = Q H Qᵀ, both unit 2-norm; w additionally has its largest entry real > 0.
// (H - λI) = P L U with adjacent-row pivoting is formed in one streaming pass: the pivot row is
// carried in registers (lane j%32 owns column j), the rows of U are written once to the global
// workspace M and read back by the triangular solves; l_k and the swap flags go to shared memory.
// smem: z, rhs (r complex each), lk (r complex), sw (r ints).
constexpr int IV_S = (kMaxR + 31) / 32;            // column slots per lane

static __device__ __forceinline__ double2 iv_pick(const double2 (&v)[IV_S], int slot) {
  double2 out = v[0];
#pragma unroll
  for (int s = 1; s < IV_S; ++s)
    if (s == slot) out = v[s];
  return out;
}
static __device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

static __device__ void iv_normalise(double2* z, int r, int lane) {
  double nrm = 0.0;
  for (int i = lane; i < r; i += 32) nrm = fmax(nrm, cabs2(z[i]));
  nrm = wmax(nrm);
  if (nrm == 0.0) nrm = 1.0;
  const double in = 1.0 / nrm;
  double ss = 0.0;
  for (int i = lane; i < r; i += 32) { const double2 v = z[i]; ss += (v.x * in) * (v.x * in) + (v.y * in) * (v.y * in); }
  ss = wsum(ss);
  const double inv = in / sqrt(ss);
  __syncwarp();
  for (int i = lane; i < r; i += 32) z[i] = make_double2(z[i].x * inv, z[i].y * inv);
  __syncwarp();
}

// The Householder vectors, the U factor and τ live in global memory (L2); every loop below loads
// the NEXT row/vector into registers before it reduces the current one, so the L2 latency
// overlaps the warp reductions instead of serialising with them.
static __device__ void iv_apply_q(const double* Qv, const double* tau, int r, double2* v, int lane) {
  double qc[IV_S], qn[IV_S];                         // v <- P_k v, k = r-3 .. 0  (Q = P_0 … P_{r-3})
  double tc = 0.0, tn = 0.0;
  auto load = [&](int k, double (&q)[IV_S], double& t) {
#pragma unroll
    for (int s = 0; s < IV_S; ++s) {
      const int i = lane + 32 * s;
      q[s] = (k >= 0 && i > k && i < r) ? __ldcg(Qv + (long long)k * r + i) : 0.0;
    }
    t = k >= 0 ? __ldcg(tau + k) : 0.0;
  };
  load(r - 3, qc, tc);
  for (int k = r - 3; k >= 0; --k) {
    load(k - 1, qn, tn);
    if (tc != 0.0) {
      double2 sm = make_double2(0.0, 0.0);
#pragma unroll
      for (int s = 0; s < IV_S; ++s) {
        const int i = lane + 32 * s;
        if (i > k && i < r) { sm.x = fma(qc[s], v[i].x, sm.x); sm.y = fma(qc[s], v[i].y, sm.y); }
      }
      sm = wsum2(sm);
      __syncwarp();
#pragma unroll
      for (int s = 0; s < IV_S; ++s) {
        const int i = lane + 32 * s;
        if (i > k && i < r) v[i] = make_double2(v[i].x - tc * sm.x * qc[s], v[i].y - tc * sm.y * qc[s]);
      }
      __syncwarp();
    }
#pragma unroll
    for (int s = 0; s < IV_S; ++s) qc[s] = qn[s];
    tc = tn;
  }
}

// (H − λI) = P L U (see inverse_iteration); hn_in >= 0: max |h_ij| precomputed by the caller
static __device__ void iv_lu(const double* H, int r, double2 lam, double2* M, double2* lk, int* sw,
                             int lane, double hn_in, double2* Mc = nullptr) {
  double hn = hn_in;
  if (hn < 0.0) {
    hn = 0.0;
    for (int i = 0; i < r; ++i)
      for (int j = (i > 0 ? i - 1 : 0) + lane; j < r; j += 32) hn = fmax(hn, fabs(__ldcg(H + (long long)i * r + j)));
    hn = wmax(hn);
  }
  const double small = (hn > 0.0 ? hn : 1.0) * DBL_EPSILON;
  // ---- streaming LU of (H - λI); U rows -> M (row-major, entries j >= k of row k)
  double2 cur[IV_S], nxt[IV_S];
  double pre[IV_S];
#pragma unroll
  for (int s = 0; s < IV_S; ++s) {
    const int j = lane + 32 * s;
    double h = (j < r) ? __ldcg(H + j) : 0.0;
    cur[s] = make_double2(h - (j == 0 ? lam.x : 0.0), j == 0 ? -lam.y : 0.0);
    pre[s] = (r > 1 && j < r) ? __ldcg(H + r + j) : 0.0;           // row 1, prefetched
  }
  for (int k = 0; k < r - 1; ++k) {
#pragma unroll
    for (int s = 0; s < IV_S; ++s) {                                 // row k+1 of H - λI
      const int j = lane + 32 * s;
      nxt[s] = make_double2(pre[s] - (j == k + 1 ? lam.x : 0.0), j == k + 1 ? -lam.y : 0.0);
      pre[s] = (k + 2 < r && j < r) ? __ldcg(H + (long long)(k + 2) * r + j) : 0.0;
    }
    const double2 a = shfl2(iv_pick(cur, k >> 5), k & 31);
    const double2 b = shfl2(iv_pick(nxt, k >> 5), k & 31);
    const bool swp = cabs2(b) > cabs2(a);
    double2 piv = swp ? b : a;
    const double2 other = swp ? a : b;
    if (cabs2(piv) == 0.0) piv = make_double2(small, 0.0);
    const double2 l = cdiv(other, piv);
#pragma unroll
    for (int s = 0; s < IV_S; ++s) {
      const int j = lane + 32 * s;
      const double2 urow = swp ? nxt[s] : cur[s];
      const double2 crow = swp ? cur[s] : nxt[s];
      if (j >= k && j < r) {
        const double2 u = (j == k) ? piv : urow;
        M[(long long)k * r + j] = u;
        if (Mc) Mc[(long long)j * r + k] = u;            // column-major copy (CTA-group right solve)
      }
      cur[s] = (j > k) ? csub(crow, cmul(l, urow)) : make_double2(0.0, 0.0);
    }
    if (lane == 0) { lk[k] = l; sw[k] = swp ? 1 : 0; }
  }
  {
    const double2 d = shfl2(iv_pick(cur, (r - 1) >> 5), (r - 1) & 31);
    if (lane == ((r - 1) & 31)) {
      const double2 u = (cabs2(d) == 0.0) ? make_double2(small, 0.0) : d;
      M[(long long)(r - 1) * r + r - 1] = u;
      if (Mc) Mc[(long long)(r - 1) * r + r - 1] = u;
    }
  }
  __syncwarp();
}

// w = Q z with the Q12 normalisation (unit norm, largest-|.| entry real > 0), one warp
static __device__ void iv_finish_right(const double* Qv, const double* tau, int r, const double2* z,
                                      double2* wout, int lane) {
  for (int i = lane; i < r; i += 32) wout[i] = z[i];
  __syncwarp();
  iv_apply_q(Qv, tau, r, wout, lane);
  {                                                  // unit norm, largest-|.| entry real > 0 (Q12)
    double best = -1.0;
    int bi = 0;
    double ss = 0.0;
    for (int i = lane; i < r; i += 32) {
      const double av = cabs2(wout[i]);
      ss += av * av;
      if (av > best) { best = av; bi = i; }
    }
    ss = wsum(ss);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const double2 pv = wout[bi];
    const double ap = cabs2(pv);
    const double2 ph = make_double2(pv.x / ap, -pv.y / ap);
    const double inv = 1.0 / sqrt(ss);
    __syncwarp();
    for (int i = lane; i < r; i += 32) {
      const double2 v = cmul(wout[i], ph);
      wout[i] = make_double2(v.x * inv, v.y * inv);
    }
    __syncwarp();
    if (lane == 0) wout[bi] = make_double2(wout[bi].x, 0.0);
    __syncwarp();
  }
}

// right eigenvector from the LU of iv_lu: two solves U z = (L⁻¹P) rhs, w = Q z, Q12 normalisation
static __device__ void iv_right(const double* Qv, const double* tau, int r, const double2* M,
                                const double2* lk, const int* sw, double2* z, double2* rhs,
                                double2* wout, int lane) {
  // ---- right vector: two solves U z = (L⁻¹P) rhs, rhs = e then the normalised z
  for (int i = lane; i < r; i += 32) rhs[i] = make_double2(1.0, 0.0);
  __syncwarp();
  for (int it = 0; it < 2; ++it) {
    if (lane == 0) {
      for (int k = 0; k < r - 1; ++k) {
        if (sw[k]) { const double2 t = rhs[k]; rhs[k] = rhs[k + 1]; rhs[k + 1] = t; }
        rhs[k + 1] = csub(rhs[k + 1], cmul(lk[k], rhs[k]));
      }
    }
    __syncwarp();
    {                                                // U z = rhs, row i of U prefetched one row ahead
      double2 mc[IV_S], mn[IV_S], dc, dn;
      auto load = [&](int i, double2 (&mr)[IV_S], double2& d) {
#pragma unroll
        for (int s = 0; s < IV_S; ++s) {
          const int j = lane + 32 * s;
          mr[s] = (i >= 0 && j > i && j < r) ? __ldcg(M + (long long)i * r + j) : make_double2(0.0, 0.0);
        }
        d = i >= 0 ? __ldcg(M + (long long)i * r + i) : make_double2(1.0, 0.0);
      };
      load(r - 1, mc, dc);
      for (int i = r - 1; i >= 0; --i) {
        load(i - 1, mn, dn);
        double2 s = make_double2(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < IV_S; ++q) {
          const int j = lane + 32 * q;
          if (j > i && j < r) s = cadd(s, cmul(mc[q], z[j]));
        }
        s = wsum2(s);
        if (lane == 0) z[i] = cdiv(csub(rhs[i], s), dc);
        __syncwarp();
#pragma unroll
        for (int q = 0; q < IV_S; ++q) mc[q] = mn[q];
        dc = dn;
      }
    }
    iv_normalise(z, r, lane);
    for (int i = lane; i < r; i += 32) rhs[i] = z[i];
    __syncwarp();
  }
  iv_finish_right(Qv, tau, r, z, wout, lane);
}

// left eigenvector from the LU of iv_lu: Mᴴ u = e (two solves), y = Q u, unit norm
static __device__ void iv_left(const double* Qv, const double* tau, int r, const double2* M,
                               const double2* lk, const int* sw, double2* z, double2* rhs,
                               double2* yout, int lane) {
  // ---- left vector: Mᴴ u = e  →  Uᴴ a = rhs (forward), then a ← S_k E_kᴴ a for k = r-2 … 0
  for (int i = lane; i < r; i += 32) rhs[i] = make_double2(1.0, 0.0);
  __syncwarp();
  for (int it = 0; it < 2; ++it) {
    {                                                // Uᴴ a = rhs, column i of U prefetched ahead
      double2 mc[IV_S], mn[IV_S], dc, dn;
      auto load = [&](int i, double2 (&mr)[IV_S], double2& d) {
#pragma unroll
        for (int s = 0; s < IV_S; ++s) {
          const int j = lane + 32 * s;
          mr[s] = (i < r && j < i) ? __ldcg(M + (long long)j * r + i) : make_double2(0.0, 0.0);
        }
        d = i < r ? __ldcg(M + (long long)i * r + i) : make_double2(1.0, 0.0);
      };
      load(0, mc, dc);
      for (int i = 0; i < r; ++i) {
        load(i + 1, mn, dn);
        double2 s = make_double2(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < IV_S; ++q) {
          const int j = lane + 32 * q;
          if (j < i) s = cadd(s, cmul(cconj(mc[q]), z[j]));
        }
        s = wsum2(s);
        if (lane == 0) z[i] = cdiv(csub(rhs[i], s), cconj(dc));
        __syncwarp();
#pragma unroll
        for (int q = 0; q < IV_S; ++q) mc[q] = mn[q];
        dc = dn;
      }
    }
    if (lane == 0) {
      for (int k = r - 2; k >= 0; --k) {
        z[k] = csub(z[k], cmul(cconj(lk[k]), z[k + 1]));
        if (sw[k]) { const double2 t = z[k]; z[k] = z[k + 1]; z[k + 1] = t; }
      }
    }
    __syncwarp();
    iv_normalise(z, r, lane);
    for (int i = lane; i < r; i += 32) rhs[i] = z[i];
    __syncwarp();
  }
  for (int i = lane; i < r; i += 32) yout[i] = z[i];
  __syncwarp();
  iv_apply_q(Qv, tau, r, yout, lane);
}

// ---- CTA-group triangular solves of the per-frame inverse iteration (K4b, single background
// mode).  A group of IV_GT threads (8 warps) owns one row each (thread j <-> row j, r <= 224 <
// IV_GT): after the owner of row i forms its unknown and publishes it in shared memory, one named
// barrier, and every other thread updates its own right-hand side in a register — one barrier
// per row instead of a warp reduction.  The U entries a thread needs do not depend on the solve,
// so each thread streams them IV_PD rows/columns ahead through a register shift queue (the L2
// latency hides behind the solve).  Same arithmetic as the row-oriented warp solves up to the
// summation order of each row.
constexpr int IV_GT = 256;                           // threads per group
constexpr int IV_PD = 8;                             // prefetch depth
static __device__ __forceinline__ void grp_bar(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(IV_GT) : "memory");
}

// U z = rhs (backward), U column-major: column i at Uc[i*r + (0..i)]; rhs[j] in, z[] out (smem)
static __device__ __noinline__ void grp_solve_upper(const double2* Uc, int r, const double2* rhs, double2* z, int j,
                                       int bar) {
  double2 b = j < r ? rhs[j] : make_double2(0.0, 0.0);
  double2 q[IV_PD];
#pragma unroll
  for (int d = 0; d < IV_PD; ++d) {
    const int i = r - 1 - d;
    q[d] = (j < r && i >= j) ? __ldcg(Uc + (long long)i * r + j) : make_double2(0.0, 0.0);
  }
  for (int i = r - 1; i >= 0; --i) {
    const double2 u = q[0];
#pragma unroll
    for (int d = 0; d < IV_PD - 1; ++d) q[d] = q[d + 1];
    {
      const int in = i - IV_PD;
      q[IV_PD - 1] = (j < r && in >= j) ? __ldcg(Uc + (long long)in * r + j) : make_double2(0.0, 0.0);
    }
    if (j == i) z[i] = cdiv(b, u);
    grp_bar(bar);
    if (j < i) b = csub(b, cmul(u, z[i]));
  }
  grp_bar(bar);
}

// Uᴴ a = rhs (forward), U row-major: row i at Ur[i*r + (i..r-1)]
static __device__ __noinline__ void grp_solve_upper_h(const double2* Ur, int r, const double2* rhs, double2* a, int k,
                                         int bar) {
  double2 b = k < r ? rhs[k] : make_double2(0.0, 0.0);
  double2 q[IV_PD];
#pragma unroll
  for (int d = 0; d < IV_PD; ++d)
    q[d] = (k < r && d <= k) ? __ldcg(Ur + (long long)d * r + k) : make_double2(0.0, 0.0);
  for (int i = 0; i < r; ++i) {
    const double2 u = q[0];
#pragma unroll
    for (int d = 0; d < IV_PD - 1; ++d) q[d] = q[d + 1];
    {
      const int in = i + IV_PD;
      q[IV_PD - 1] = (k < r && in <= k) ? __ldcg(Ur + (long long)in * r + k) : make_double2(0.0, 0.0);
    }
    if (k == i) a[i] = cdiv(b, cconj(u));
    grp_bar(bar);
    if (k > i) b = csub(b, cmul(cconj(u), a[i]));
  }
  grp_bar(bar);
}

// right eigenvector by the group (gt = thread in the group, gw = warp in the group): two inverse
// iterations U z = L⁻¹P rhs, then w = Q z with the Q12 normalisation (as iv_right)
static __device__ void iv_right_grp(const double* Qv, const double* tau, int r, const double2* Uc,
                                    const double2* lk, const int* sw, double2* z, double2* rhs,
                                    double2* wout, int gt, int gw, int lane, int bar) {
  for (int i = gt; i < r; i += IV_GT) rhs[i] = make_double2(1.0, 0.0);
  grp_bar(bar);
  for (int it = 0; it < 2; ++it) {
    if (gt == 0) {
      for (int k = 0; k < r - 1; ++k) {
        if (sw[k]) { const double2 t = rhs[k]; rhs[k] = rhs[k + 1]; rhs[k + 1] = t; }
        rhs[k + 1] = csub(rhs[k + 1], cmul(lk[k], rhs[k]));
      }
    }
    grp_bar(bar);
    grp_solve_upper(Uc, r, rhs, z, gt, bar);
    if (gw == 0) {
      iv_normalise(z, r, lane);
      for (int i = lane; i < r; i += 32) rhs[i] = z[i];
    }
    grp_bar(bar);
  }
  if (gw == 0) iv_finish_right(Qv, tau, r, z, wout, lane);
}

static __device__ void iv_left_grp(const double* Qv, const double* tau, int r, const double2* Ur,
                                   const double2* lk, const int* sw, double2* z, double2* rhs,
                                   double2* yout, int gt, int gw, int lane, int bar) {
  for (int i = gt; i < r; i += IV_GT) rhs[i] = make_double2(1.0, 0.0);
  grp_bar(bar);
  for (int it = 0; it < 2; ++it) {
    grp_solve_upper_h(Ur, r, rhs, z, gt, bar);
    if (gt == 0) {
      for (int k = r - 2; k >= 0; --k) {
        z[k] = csub(z[k], cmul(cconj(lk[k]), z[k + 1]));
        if (sw[k]) { const double2 t = z[k]; z[k] = z[k + 1]; z[k + 1] = t; }
      }
    }
    grp_bar(bar);
    if (gw == 0) {
      iv_normalise(z, r, lane);
      for (int i = lane; i < r; i += 32) rhs[i] = z[i];
    }
    grp_bar(bar);
  }
  if (gw == 0) {
    for (int i = lane; i < r; i += 32) yout[i] = z[i];
    __syncwarp();
    iv_apply_q(Qv, tau, r, yout, lane);
  }
}

static __device__ void inverse_iteration(const double* H, const double* Qv, const double* tau, int r,
                                         double2 lam, double2* M, double2* z, double2* rhs,
                                         double2* lk, int* sw, double2* wout, double2* yout,
                                         int lane, double hn = -1.0) {
  iv_lu(H, r, lam, M, lk, sw, lane, hn);
  __syncwarp();
  iv_right(Qv, tau, r, M, lk, sw, z, rhs, wout, lane);
  if (yout != nullptr) iv_left(Qv, tau, r, M, lk, sw, z, rhs, yout, lane);
}

// ------------------------------------------------------------------ the per-frame kernel ------
// One thread-block cluster of K4_CLUSTER CTAs per frame (= per eigen worker).  The parallel phases
// (Gram gather, one-sided Jacobi, sort, VΣ⁻¹, the two small GEMMs, Householder-Hessenberg) are
// spread over all warps of the cluster with cluster barriers between dependent steps; the
// workspace lives in global memory (L2-resident, read with ld.global.cg so that no SM sees stale
// L1 lines).  The inherently sequential Francis QR, the eigenvector solves and the background
// coefficients then run on CTA 0.
constexpr int K4_CLUSTER = 4;
constexpr int K4_SMALL_M = 64;                         // single-CTA Jacobi up to this window width
constexpr int K4_SOLO_M = 128;                         // K4a on one CTA (CL = 1) up to this width
constexpr int K4_JAC_DSM_M = 216;                      // block Jacobi kept in DSMEM up to this width
constexpr int K4_GW = K4_WARPS * K4_CLUSTER;           // warps in the cluster
constexpr int K4_GT = K4_THREADS * K4_CLUSTER;         // threads in the cluster

static __device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
static __device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// One Hestenes rotation of the column pair (cp, cq) of length m by a half-warp (lane hl holds rows
// hl + 16e, e < EH; EH = ceil(m/16) rounded to an instantiated size, so the unrolled loops carry
// no dead predicated rows).  Returns true if the pair was rotated.
template <int EH>
static __device__ __forceinline__ bool jacobi_pair(double* cp, double* cq, int m, int hl, bool act,
                                                   double tol, unsigned mask = 0xffffffffu) {
  double ap[EH], aq[EH];
  double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
  for (int e = 0; e < EH; ++e) {
    const int i = hl + 16 * e;
    const bool ok = act && i < m;
    ap[e] = ok ? cp[i] : 0.0;
    aq[e] = ok ? cq[i] : 0.0;
  }
#pragma unroll
  for (int e = 0; e < EH; ++e) {
    al = fma(ap[e], ap[e], al);
    be = fma(aq[e], aq[e], be);
    ga = fma(ap[e], aq[e], ga);
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {                 // reduce within the half-warp
    al += __shfl_xor_sync(mask, al, o);
    be += __shfl_xor_sync(mask, be, o);
    ga += __shfl_xor_sync(mask, ga, o);
  }
  if (act && ga != 0.0 && ga * ga > tol * tol * (al * be)) {
    // t = tan θ = sign(ζ)/(|ζ| + sqrt(1+ζ²)), ζ = (β-α)/(2γ), written with one sqrt and
    // one division: t = sign(β-α)·2γ / (|β-α| + sqrt((β-α)² + 4γ²))
    const double d = be - al;
    const double sq = sqrt(fma(d, d, 4.0 * ga * ga));
    const double t = (d >= 0.0 ? 2.0 * ga : -2.0 * ga) / (fabs(d) + sq);
    const double c = rsqrt(fma(t, t, 1.0)), sn = c * t;
#pragma unroll
    for (int e = 0; e < EH; ++e) {
      const int i = hl + 16 * e;
      if (i < m) {
        cp[i] = c * ap[e] - sn * aq[e];
        cq[i] = sn * ap[e] + c * aq[e];
      }
    }
    return true;
  }
  return false;
}

// ---- a8 on the K4a cluster: the Ehrlich–Aberth iteration of aberth_eigs with the active roots
// spread over all K4_CLUSTER CTAs (root q of the active list on CTA q mod 4, warp (q / 4) mod 16),
// so four SMs' shared-memory bandwidth and fp64 pipes share the Hyman evaluations.  Every CTA
// holds the column-packed H and the full iterate; each writes the new iterate of its roots (and
// its freeze / failure marks) into every CTA's shared memory (DSMEM), then one cluster barrier
// publishes them and a second one keeps the next iteration's remote writes behind every CTA's
// publish.  All CTAs therefore hold identical state and leave the loop together; CTA 0 then runs
// the trace check and the conjugate pairing (as aberth_eigs) and returns 0 with lam_out filled, or
// −1 (the caller falls back to the Francis QR).  CTAs other than 0 return 1 after the loop.
static __device__ __forceinline__ unsigned dsm_addr(const void* p, unsigned cta) {
  unsigned a = (unsigned)__cvta_generic_to_shared(p), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(cta));
  return ra;
}
static __device__ __forceinline__ void dsm_st(double2* p, unsigned cta, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(dsm_addr(p, cta)), "d"(v.x), "d"(v.y) : "memory");
}
static __device__ __forceinline__ void dsm_st(double* p, unsigned cta, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(dsm_addr(p, cta)), "d"(v) : "memory");
}
static __device__ __forceinline__ void dsm_st(float* p, unsigned cta, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(dsm_addr(p, cta)), "f"(v) : "memory");
}
static __device__ __forceinline__ void dsm_st(int* p, unsigned cta, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(dsm_addr(p, cta)), "r"(v) : "memory");
}

template <int CL>
static __device__ int aberth_eigs_cluster(const double* Hg, int r, double* hc, const double2* z0,
                                          int n0, double2* z, double2* zn, int* act, double2* lam_out,
                                          int crank, int tid, int warp, int lane, int* its_out,
                                          int* evals_out) {
  constexpr int K4_CLUSTER = CL;                             // CTAs sharing the roots
  __shared__ int sh_na, sh_bad;
  __shared__ float prv[kMaxR];                               // |correction| of each root's last step
  if (n0 != r || z0 == nullptr || r < 2) return crank == 0 ? -1 : 1;
  for (int j = warp; j < r; j += K4_WARPS) {
    const int len = j + 2 < r ? j + 2 : r;
    for (int i = lane; i < len; i += 32) hc[ab_cofs(j) + i] = __ldcg(Hg + (long long)i * r + j);
  }
  if (tid == 0) sh_bad = 0;
  __syncthreads();
  for (int j = tid + 1; j < r; j += K4_THREADS) {
    const double sub = hc[ab_cofs(j - 1) + j];
    const double sc = fabs(hc[ab_cofs(j - 1) + j - 1]) + fabs(hc[ab_cofs(j) + j]);
    if (!(fabs(sub) > DBL_EPSILON * sc) || !isfinite(sub)) atomicOr(&sh_bad, 1);   // reducible
  }
  __syncthreads();
  if (sh_bad) return crank == 0 ? -2 : 1;                    // reducible (same data everywhere)
  for (int j = tid + 1; j < r; j += K4_THREADS) hc[ab_cofs(j - 1) + j] = 1.0 / hc[ab_cofs(j - 1) + j];
  for (int k = tid; k < r; k += K4_THREADS) {
    double2 g = z0[k];
    const double a = hypot(g.x, g.y);
    const double sc = a > 0.0 ? a : 1.0;
    if (g.y == 0.0) g.y = ((k & 1) ? 1e-3 : -1e-3) * sc;
    g.x *= 1.0 + 1e-9 * (k + 1);
    z[k] = g;
    act[k] = k;
    prv[k] = INFINITY;
  }
  if (tid == 0) sh_na = r;
  cl_sync();                                                 // every CTA initialised before remote writes
  int its = 0, evals = 0;
  const double tol = 4.0 * DBL_EPSILON;
  while (sh_na > 0) {
    if (its == AB_MAXIT) return crank == 0 ? -3 : 1;
    ++its;
    const int na = sh_na;
    evals += na;
    for (int q = crank + K4_CLUSTER * warp; q < na; q += K4_CLUSTER * K4_WARPS) {
      const int k = act[q];
      const double2 zk = z[k];
      const double2 N = hyman_ratio(hc, r, zk, lane);
      double2 S = make_double2(0.0, 0.0);                    // Σ_{j≠k} 1/(z_k − z_j)
      for (int jj = lane; jj < r; jj += 32)
        if (jj != k) {
          const double2 d = csub(zk, z[jj]);
          const double id = 1.0 / fma(d.x, d.x, d.y * d.y);
          S = make_double2(fma(d.x, id, S.x), fma(-d.y, id, S.y));
        }
      S = wsum2(S);
      if (lane < K4_CLUSTER) {                               // lane c writes CTA c's copy
        const double2 den = csub(make_double2(1.0, 0.0), cmul(N, S));
        const double2 step = cdiv(N, den);
        double2 nz = csub(zk, step);
        const bool bad = !isfinite(nz.x) || !isfinite(nz.y);
        if (bad) nz = zk;
        dsm_st(zn + k, (unsigned)lane, nz);
        if (bad) dsm_st(&sh_bad, (unsigned)lane, 1);
        // frozen at rounding level, or stagnating at the evaluation's noise floor: a correction
        // below 1e-11|z| that no longer shrinks by half (cubic convergence shrinks it far more;
        // an ill-conditioned or clustered root hovers there instead, as accurate as QR would be)
        const double as = hypot(step.x, step.y), az = hypot(nz.x, nz.y);
        if (as <= tol * az || (as <= 1e-11 * az && as > 0.5 * (double)prv[k]))
          dsm_st(act + q, (unsigned)lane, -1 - k);
        dsm_st(prv + k, (unsigned)lane, (float)as);
      }
    }
    cl_sync();                                               // the new iterate everywhere
    if (sh_bad) return crank == 0 ? -4 : 1;
    for (int q = tid; q < na; q += K4_THREADS) {
      const int a = act[q];
      const int k = a >= 0 ? a : -1 - a;
      z[k] = zn[k];
    }
    __syncthreads();
    if (tid == 0) {
      int c = 0;
      for (int q = 0; q < na; ++q)
        if (act[q] >= 0) act[c++] = act[q];
      sh_na = c;
    }
    cl_sync();                                               // publish done before new remote writes
  }
  if (its_out) *its_out = its;
  if (evals_out) *evals_out = evals;
  if (crank != 0) return 1;
  // CTA 0: trace check and exact conjugate symmetry, as in aberth_eigs
  if (warp == 0) {
    double2 sz = make_double2(0.0, 0.0);
    double tr = 0.0, ta = 0.0;
    for (int k = lane; k < r; k += 32) {
      sz = cadd(sz, z[k]);
      tr += hc[ab_cofs(k) + k];
      ta += fabs(hc[ab_cofs(k) + k]) + hypot(z[k].x, z[k].y);
    }
    sz = wsum2(sz);
    tr = wsum(tr);
    ta = wsum(ta);
    if (lane == 0 && (fabs(sz.x - tr) > 1e-10 * ta || fabs(sz.y) > 1e-10 * ta)) sh_bad = 1;
  }
  __syncthreads();
  if (sh_bad) return -5;                                     // trace mismatch
  int* partner = reinterpret_cast<int*>(zn);
  int* chosen = partner + kMaxR;
  for (int k = tid; k < r; k += K4_THREADS) {
    act[k] = 0;
    chosen[k] = 0;
    partner[k] = -1;
    if (fabs(z[k].y) <= 1e-10 * hypot(z[k].x, z[k].y)) { z[k].y = 0.0; act[k] = 1; }
  }
  __syncthreads();
  for (int k = tid; k < r; k += K4_THREADS) {
    if (act[k] || z[k].y < 0.0) continue;
    int best = -1;
    double bd = 0.0;
    for (int j = 0; j < r; ++j) {
      if (act[j] || z[j].y >= 0.0) continue;
      const double d = hypot(z[j].x - z[k].x, z[j].y + z[k].y);
      if (best < 0 || d < bd) { best = j; bd = d; }
    }
    if (best < 0 || bd > 1e-8 * hypot(z[k].x, z[k].y)) { atomicOr(&sh_bad, 1); continue; }
    partner[k] = best;
    atomicAdd(&chosen[best], 1);
  }
  __syncthreads();
  for (int j = tid; j < r; j += K4_THREADS)
    if (!act[j] && z[j].y < 0.0 && chosen[j] != 1) atomicOr(&sh_bad, 1);
  __syncthreads();
  if (sh_bad) return -6;                                     // conjugate pairing failed
  for (int k = tid; k < r; k += K4_THREADS) {
    const int b = partner[k];
    if (b < 0) continue;
    const double re = 0.5 * (z[k].x + z[b].x), im = 0.5 * (z[k].y - z[b].y);
    z[k] = make_double2(re, im);
    z[b] = make_double2(re, -im);
  }
  __syncthreads();
  for (int k = tid; k < r; k += K4_THREADS) lam_out[k] = z[k];
  __syncthreads();
  return 0;
}

// ---- a7 tiles: out[i0+ii][j] (rows [i0, i0+ni), columns j < r) = Σ_k A[i0+ii][k] Bm[k][j] over
// k < m, with A read by `ga(i, k)` and Bm by `gb(k, j)`, staged through shared memory in k-chunks of
// 32 (A chunk [32][mb], B chunk [32][r]); thread (ti, tj) of the 16 x 32 grid accumulates rows
// ti + 16a, columns tj + 32b (a < 4, b < 7) as fixed-order fma chains over k.  Kept out of line so
// that its register tile does not raise the pressure of the Jacobi phase.
// mode 0: A = XᵀX' (gathered from the Gram history of the window ending at f), Bm = Y, out = B
//         (column-major, ld m);  mode 1: A = Yᵀ, Bm = B, out = Ã (row-major, ld r, into H)
static __device__ __noinline__ void k4_tiled_product(int mode, int m, int r, int i0, int ni, int mb,
                                                     int tid, double* t0, const double* gh, int NH,
                                                     int mh, long long f, const double* Y, double* B,
                                                     double* H) {
  auto ga = [&](int i, int k) -> double {
    return mode == 0 ? gram_at(gh, NH, mh, m, f, i, k + 1) : __ldcg(Y + (long long)i * m + k);
  };
  auto gb = [&](int k, int j) -> double {
    return __ldcg((mode == 0 ? Y : B) + (long long)j * m + k);
  };
  auto st = [&](int i, int j, double v) {
    if (mode == 0) B[(long long)j * m + i] = v;
    else H[(long long)i * r + j] = v;
  };
  constexpr int KC = 32, RA = 4, RB = (kMaxR + 31) / 32;
  const int ti = tid >> 5, tj = tid & 31;
  double* As = t0;                                           // [KC][mb]
  double* Bs = t0 + KC * mb;                                 // [KC][r]
  double acc[RA][RB];
#pragma unroll
  for (int a = 0; a < RA; ++a)
#pragma unroll
    for (int b = 0; b < RB; ++b) acc[a][b] = 0.0;
  for (int k0 = 0; k0 < m; k0 += KC) {
    const int nk = min(KC, m - k0);
    for (int e = tid; e < KC * mb; e += K4_THREADS) {
      const int ii = e / KC, kk = e % KC;
      As[kk * mb + ii] = (kk < nk && ii < ni) ? ga(i0 + ii, k0 + kk) : 0.0;
    }
    for (int e = tid; e < KC * r; e += K4_THREADS) {
      const int j = e / KC, kk = e % KC;
      Bs[kk * r + j] = kk < nk ? gb(k0 + kk, j) : 0.0;
    }
    __syncthreads();
    for (int kk = 0; kk < nk; ++kk) {
      double g[RA], y[RB];
#pragma unroll
      for (int a = 0; a < RA; ++a) g[a] = (ti + 16 * a < mb) ? As[kk * mb + ti + 16 * a] : 0.0;
#pragma unroll
      for (int b = 0; b < RB; ++b) y[b] = (tj + 32 * b < r) ? Bs[kk * r + tj + 32 * b] : 0.0;
#pragma unroll
      for (int a = 0; a < RA; ++a)
#pragma unroll
        for (int b = 0; b < RB; ++b) acc[a][b] = fma(g[a], y[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < RA; ++a)
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int ii = ti + 16 * a, j = tj + 32 * b;
      if (ii < ni && j < r) st(i0 + ii, j, acc[a][b]);
    }
}

// C[i][j] = Σ_{k<K} X(i,k)·Y(k,j) for rows i in [i0, i0+ni) (ni <= 64) and all N <= kMaxR columns,
// tiled through shared memory t0 (32 x (64 + N) doubles); X, Y element accessors, st(i, j, v) the
// store.  CTA-wide (K4_THREADS threads: 16 row groups x 32 column lanes, 4 x 7 outputs each).
template <class FX, class FY, class FS>
static __device__ __forceinline__ void k4_gemm_rows(int K, int N, int i0, int ni, int tid, double* t0,
                                                    FX X, FY Y, FS st) {
  constexpr int KC = 32, RA = 4, RB = (kMaxR + 31) / 32, MB = 64;
  const int ti = tid >> 5, tj = tid & 31;
  double* As = t0;                                           // [KC][MB]
  double* Bs = t0 + KC * MB;                                 // [KC][N]
  double acc[RA][RB];
#pragma unroll
  for (int a = 0; a < RA; ++a)
#pragma unroll
    for (int b = 0; b < RB; ++b) acc[a][b] = 0.0;
  for (int k0 = 0; k0 < K; k0 += KC) {
    const int nk = min(KC, K - k0);
    for (int e = tid; e < KC * MB; e += K4_THREADS) {
      const int ii = e / KC, kk = e % KC;
      As[kk * MB + ii] = (kk < nk && ii < ni) ? X(i0 + ii, k0 + kk) : 0.0;
    }
    for (int e = tid; e < KC * N; e += K4_THREADS) {
      const int j = e / KC, kk = e % KC;
      Bs[kk * N + j] = kk < nk ? Y(k0 + kk, j) : 0.0;
    }
    __syncthreads();
    for (int kk = 0; kk < nk; ++kk) {
      double g[RA], y[RB];
#pragma unroll
      for (int a = 0; a < RA; ++a) g[a] = As[kk * MB + ti + 16 * a];
#pragma unroll
      for (int b = 0; b < RB; ++b) y[b] = (tj + 32 * b < N) ? Bs[kk * N + tj + 32 * b] : 0.0;
#pragma unroll
      for (int a = 0; a < RA; ++a)
#pragma unroll
        for (int b = 0; b < RB; ++b) acc[a][b] = fma(g[a], y[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < RA; ++a)
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int ii = ti + 16 * a, j = tj + 32 * b;
      if (ii < ni && j < N) st(i0 + ii, j, acc[a][b]);
    }
}

constexpr int K4_CHOL_SMEM_M = 157;                    // R (m² fp64) in shared memory up to this m

// Pivoted Cholesky (largest remaining diagonal first, lowest index on ties) of the symmetric
// positive semidefinite Sw (column-major m x m in Ag), rows kept in the ORIGINAL column order:
// step k writes R[k][j] to Rg[k*m + j], so that RᵀR = Sw without a permutation.  Stops at the
// first non-positive pivot (the numerical null space); the remaining rows are zero.  One CTA;
// returns the number of steps taken.
//  - Ts != nullptr (m <= K4_CHOL_SMEM_M): the rows of R (and Sw itself for m <= 110) in shared
//    memory: per step one warp picks the pivot, then each unused column forms its entry of row k
//    from the k previous rows — two barriers and no L2 round trip per step (a right-looking rank-1
//    update of the Schur complement in shared memory measured slower: smem-bandwidth bound);
//  - else the same from L2 (row k from Sw and the previous rows, four loads in flight).
static __device__ __noinline__ int k4_pchol(const double* Ag, double* Rg, int m, int tid, int warp, int lane,
                                            double* Ts) {
  __shared__ double dg[kMaxM];
  __shared__ double rp[kMaxM];                               // R[0..k-1][piv] (left-looking) / row k (right-looking)
  __shared__ unsigned char used[kMaxM];
  __shared__ double wb[K4_WARPS];
  __shared__ int wi[K4_WARPS];
  __shared__ int sh_piv;
  __shared__ double sh_d;
  if (Ts) {
    // left-looking with R (and, for m <= 110, Sw) in shared memory: per step warp 0 picks the pivot
    // from the running diagonal, then every unused column j forms R[k][j] from k shared-memory rows
    // (four partial sums) — two barriers per step
    const bool sw_s = m <= 110;
    double* Ss = Ts + (size_t)m * m;                         // Sw copy (sw_s)
    for (int j = tid; j < m; j += K4_THREADS) { dg[j] = __ldcg(Ag + (long long)j * m + j); used[j] = 0; }
    if (sw_s)
      for (int e = tid; e < m * m; e += K4_THREADS) Ss[e] = __ldcg(Ag + e);
    __syncthreads();
    int k = 0;
    for (; k < m; ++k) {
      if (warp == 0) {
        double b = -INFINITY;
        int bi = m;
        for (int j = lane; j < m; j += 32)
          if (!used[j] && dg[j] > b) { b = dg[j]; bi = j; }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, b, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > b || (ob == b && oi < bi)) { b = ob; bi = oi; }
        }
        if (lane == 0) { sh_piv = bi; sh_d = b; }
      }
      __syncthreads();
      const int piv = sh_piv;
      const double d = sh_d;
      if (!(d > 0.0) || piv >= m) break;                     // uniform
      const double rkk = sqrt(d), irk = 1.0 / rkk;
      for (int j = tid; j < m; j += K4_THREADS) {
        double v = 0.0;
        if (j == piv) {
          v = rkk;
          used[j] = 1;                                       // only this thread reads used[piv] now
        } else if (!used[j]) {
          double sacc = sw_s ? Ss[piv * m + j] : __ldcg(Ag + (long long)piv * m + j);   // Sw[j][piv]
          double s1 = 0.0, s2 = 0.0, s3 = 0.0;
          int l = 0;
          for (; l + 4 <= k; l += 4) {
            sacc = fma(-Ts[l * m + piv], Ts[l * m + j], sacc);
            s1 = fma(-Ts[(l + 1) * m + piv], Ts[(l + 1) * m + j], s1);
            s2 = fma(-Ts[(l + 2) * m + piv], Ts[(l + 2) * m + j], s2);
            s3 = fma(-Ts[(l + 3) * m + piv], Ts[(l + 3) * m + j], s3);
          }
          for (; l < k; ++l) sacc = fma(-Ts[l * m + piv], Ts[l * m + j], sacc);
          sacc += (s1 + s2) + s3;
          v = sacc * irk;
          dg[j] -= v * v;
        }
        Ts[k * m + j] = v;
      }
      __syncthreads();
    }
    for (int e = tid; e < k * m; e += K4_THREADS) Rg[e] = Ts[e];
    for (long long e = (long long)k * m + tid; e < (long long)m * m; e += K4_THREADS) Rg[e] = 0.0;
    return k;
  }
  for (int j = tid; j < m; j += K4_THREADS) { dg[j] = __ldcg(Ag + (long long)j * m + j); used[j] = 0; }
  __syncthreads();
  int k = 0;
  for (; k < m; ++k) {
    double b = -INFINITY;
    int bi = m;
    for (int j = tid; j < m; j += K4_THREADS)
      if (!used[j] && dg[j] > b) { b = dg[j]; bi = j; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, b, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > b || (ob == b && oi < bi)) { b = ob; bi = oi; }
    }
    if (lane == 0) { wb[warp] = b; wi[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      double bb = wb[0];
      int ii = wi[0];
      for (int w = 1; w < K4_WARPS; ++w)
        if (wb[w] > bb || (wb[w] == bb && wi[w] < ii)) { bb = wb[w]; ii = wi[w]; }
      sh_piv = ii;
      sh_d = bb;
    }
    __syncthreads();
    const int piv = sh_piv;
    const double d = sh_d;
    if (!(d > 0.0) || piv >= m) break;                       // uniform
    for (int l = tid; l < k; l += K4_THREADS) rp[l] = __ldcg(Rg + (long long)l * m + piv);
    __syncthreads();
    const double rkk = sqrt(d), irk = 1.0 / rkk;
    for (int j = tid; j < m; j += K4_THREADS) {
      double v = 0.0;
      if (j == piv) {
        v = rkk;
        used[j] = 1;                                         // only this thread reads used[piv] now
      } else if (!used[j]) {
        double sacc = __ldcg(Ag + (long long)piv * m + j);   // Sw[j][piv]
        double s1 = 0.0, s2 = 0.0, s3 = 0.0;                 // four loads in flight per step
        int l = 0;
        for (; l + 4 <= k; l += 4) {
          const double r0 = __ldcg(Rg + (long long)l * m + j), r1 = __ldcg(Rg + (long long)(l + 1) * m + j);
          const double r2 = __ldcg(Rg + (long long)(l + 2) * m + j), r3 = __ldcg(Rg + (long long)(l + 3) * m + j);
          sacc = fma(-rp[l], r0, sacc);
          s1 = fma(-rp[l + 1], r1, s1);
          s2 = fma(-rp[l + 2], r2, s2);
          s3 = fma(-rp[l + 3], r3, s3);
        }
        for (; l < k; ++l) sacc = fma(-rp[l], __ldcg(Rg + (long long)l * m + j), sacc);
        sacc += (s1 + s2) + s3;
        v = sacc * irk;
        dg[j] -= v * v;
      }
      Rg[(long long)k * m + j] = v;
    }
    __syncthreads();
  }
  for (long long e = (long long)k * m + tid; e < (long long)m * m; e += K4_THREADS) Rg[e] = 0.0;
  return k;
}

// CL = CTAs per cluster: 4 (the cluster path above), or 1 for windows up to K4_SOLO_M: the whole
// K4a on one SM (Jacobi with S in shared memory, Ã, Hessenberg and the Aberth iteration on one
// CTA) — about half the SM-cycles of the 4-CTA cluster per frame at m = 100-128, at a longer
// latency that the background lag absorbs; more worker streams then run concurrently.
template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(K4_THREADS, 1)
k4a_kernel(const K4Params p) {
  constexpr int K4_CLUSTER = CL;
  constexpr int K4_GW = K4_WARPS * CL;                      // warps in the cluster
  constexpr int K4_GT = K4_THREADS * CL;                    // threads in the cluster
  extern __shared__ __align__(16) unsigned char k4_smem[];
  __shared__ double mu[kMaxM];
  __shared__ double sig[kMaxM];
  __shared__ int perm[kMaxM];
  __shared__ int sh_r, sh_status;
  __shared__ long long ph[8];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int crank = (int)cl_rank();
  const int gtid = crank * K4_THREADS + tid, gwarp = crank * K4_WARPS + warp;
  const int m = p.m;
  const long long f = p.f;
  K4Result* res = p.res;
  {
    volatile DevState* st = p.st;
    // frame discarded by the poison contract.  K4a is released by the commit of frame f-1, so only
    // poison from frames < f is settled (uniform across the cluster) here; frame f's own outcome
    // is decided uniformly before the Ã stage
    if (st->status != 0 && st->failed_frame < f) return;
  }
  if (tid == 0) ph[0] = clock64();
  // ---- a5: S = G[0:m,0:m] and XᵀX' = G[0:m,1:m+1] from the Gram history
  for (int idx = gtid; idx < m * m; idx += K4_GT) {
    const int i = idx % m, j = idx / m;
    p.A[idx] = gram_at(p.ghist, p.NH, p.mh, m, f, i, j);
  }
  if (gtid < JACOBI_MAX_SWEEPS) p.flags[gtid] = 0;
  cl_sync();
  // ---- warm start (one-sided Jacobi is applied to S·Q0 for any orthogonal Q0: its converged
  // columns are still V·Λ).  Q0 = the previous frame's eigenvectors with rows shifted by the k
  // frames the window moved (Q0[i][j] = V_prev[(i + k) mod m][j]), which leaves far fewer
  // rotations to do than Q0 = I.
  __shared__ int sh_chol_full;                // CTA 0: the Cholesky start ran all m steps
  __shared__ int sh_nc;                       // CTA 0: columns of A that can be nonzero (Cholesky steps)
  __shared__ long long ch_cyc[2];             // CTA 0: Cholesky start/end (diagnostics)
  if (tid == 0) { sh_chol_full = 1; sh_nc = m; ch_cyc[0] = ch_cyc[1] = 0; }
  {
    __shared__ int sh_warm;
    if (tid == 0) {
      const volatile K4Result* rp = p.res_prev;
      sh_warm = (p.Vprev != nullptr && rp != nullptr && p.warm_k > 0 && rp->vframe == f - p.warm_k) ? 1 : 0;
    }
    __syncthreads();
    if (p.chol) {
      // ---- Cholesky-preconditioned start (Veselić–Hari): S = Q0 Sw Q0ᵀ with Sw = Q0ᵀ S Q0, and
      // Sw = RᵀR by pivoted Cholesky, so S = A Aᵀ for A = Q0 Rᵀ; one-sided Jacobi on A then gives
      // A J = U Σ with U the eigenvectors of S and Σ² its eigenvalues (σ = column norms).  The rows
      // of a pivoted Cholesky factor are graded, and with the warm Q0 the Jacobi needs ~7 sweeps
      // where S·Q0 needed 9–21 (C4, C5; profiles/r2 …).  Q0 = the previous frame's eigenvectors of
      // this stream with rows shifted by the window move (as below), or I.
      const int wk = sh_warm ? p.warm_k : 0;
      const double* Vp = p.Vprev;
      double* t0 = reinterpret_cast<double*>(k4_smem);
      const int mb = (m + K4_CLUSTER - 1) / K4_CLUSTER;
      const int i0 = crank * mb, ni = max(0, min(m, i0 + mb) - i0);
      if (sh_warm) {
        // B = S·Q0, then Sw = Q0ᵀ·B into A (rows of each split over the cluster, 64-row chunks)
        for (int s0 = 0; s0 < ni; s0 += 64)
          k4_gemm_rows(m, m, i0 + s0, min(64, ni - s0), tid, t0,
                       [&](int i, int k) { return __ldcg(p.A + (long long)k * m + i); },
                       [&](int k, int j) { return __ldcg(Vp + (long long)j * m + (k + wk) % m); },
                       [&](int i, int j, double v) { p.B[(long long)j * m + i] = v; });
        cl_sync();
        for (int s0 = 0; s0 < ni; s0 += 64)
          k4_gemm_rows(m, m, i0 + s0, min(64, ni - s0), tid, t0,
                       [&](int i, int k) { return __ldcg(Vp + (long long)i * m + (k + wk) % m); },
                       [&](int k, int j) { return __ldcg(p.B + (long long)j * m + k); },
                       [&](int i, int j, double v) { p.A[(long long)j * m + i] = v; });
        cl_sync();
      }
      // (a breakdown before step m leaves zero columns in A, hence zero columns of V beyond the
      // numerical rank: such a V is not orthogonal, so it must not seed a later warm start)
      if (tid == 0) ch_cyc[0] = clock64();
      if (crank == 0) {
        const int ks = k4_pchol(p.A, p.B, m, tid, warp, lane,   // R rows -> columns of B
                                m <= K4_CHOL_SMEM_M ? reinterpret_cast<double*>(k4_smem) : nullptr);
        if (tid == 0) { sh_chol_full = ks == m ? 1 : 0; sh_nc = ks; }
      }
      cl_sync();
      if (tid == 0) ch_cyc[1] = clock64();
      if (sh_warm) {                                         // A = Q0·Rᵀ
        for (int s0 = 0; s0 < ni; s0 += 64)
          k4_gemm_rows(m, m, i0 + s0, min(64, ni - s0), tid, t0,
                       [&](int i, int k) { return __ldcg(Vp + (long long)k * m + (i + wk) % m); },
                       [&](int k, int j) { return __ldcg(p.B + (long long)j * m + k); },
                       [&](int i, int j, double v) { p.A[(long long)j * m + i] = v; });
      } else {
        for (int e = crank * K4_THREADS + tid; e < m * m; e += K4_GT) p.A[e] = __ldcg(p.B + e);
      }
      cl_sync();
    } else if (sh_warm) {                       // uniform across the cluster (same inputs)
      const int cb = (m + K4_CLUSTER - 1) / K4_CLUSTER;
      const int j0 = crank * cb, j1 = min(m, j0 + cb);
      const int nj = j1 > j0 ? j1 - j0 : 0;
      double* q0 = reinterpret_cast<double*>(k4_smem);        // [nj][m]: Q0 columns j0..j1
      for (int e = tid; e < nj * m; e += K4_THREADS) {
        const int jj = e / m, i = e % m;
        const int src = (i + p.warm_k) % m;                  // any orthogonal Q0 is valid
        q0[e] = __ldcg(p.Vprev + (long long)(j0 + jj) * m + src);
      }
      __syncthreads();
      for (int e = tid; e < nj * m; e += K4_THREADS) {        // B[:, j] = S Q0[:, j]
        const int jj = e / m, i = e % m;
        const double* qj = q0 + jj * m;
        double acc = 0.0;
        for (int kk = 0; kk < m; ++kk) acc = fma(__ldcg(p.A + (long long)kk * m + i), qj[kk], acc);
        p.B[(long long)(j0 + jj) * m + i] = acc;
      }
      cl_sync();
      for (int e = tid; e < nj * m; e += K4_THREADS) p.A[(long long)j0 * m + e] = __ldcg(p.B + (long long)j0 * m + e);
      cl_sync();
    }
  }
  if (tid == 0) ph[1] = clock64();
  // the columns of A past the Cholesky steps are zero and never rotate: the Jacobi tournament runs
  // over the first nc columns only (rank-deficient windows: C2's rank-21 S breaks down after ~31
  // steps, so 31 instead of 150 columns).  nc is CTA 0's (read over DSMEM: uniform).
  int nc = m;
  if (p.chol) {
    cl_sync();
    unsigned a = (unsigned)__cvta_generic_to_shared(&sh_nc), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(ra) : "r"(a));
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(nc) : "r"(ra) : "memory");
    cl_sync();
    nc = nc < 2 ? (m < 2 ? m : 2) : nc;
  }

  // ---- a5 (small windows, m <= K4_SMALL_M): the whole S fits one CTA's shared memory, so CTA 0
  // runs the cyclic one-sided Jacobi alone (round-robin tournament of the m columns, one column
  // pair per half-warp, a CTA barrier per round) instead of the cluster's block tournament, whose
  // per-round cluster barriers and L2 staging dominate at small m (C1: m = 16).
  constexpr int EL = kMaxM / 32;
  int sweeps = 0;
  bool converged = false;
  if (CL == 1 || m <= K4_SMALL_M) {
    if (crank == 0) {
      const int mp = (nc + 1) & ~1;                         // tournament over the nc live columns
      double* sA = reinterpret_cast<double*>(k4_smem);       // mp columns x m, column-major
      for (int e = tid; e < mp * m; e += K4_THREADS) sA[e] = e < nc * m ? __ldcg(p.A + e) : 0.0;
      __syncthreads();
      const double tol = fmax(1e-15, (double)m * DBL_EPSILON);
      const int hw = warp * 2 + (lane >> 4), hl = lane & 15;
      const int np = mp / 2;                                 // column pairs per step (<= 64)
      const int eh = m <= 64 ? 4 : m <= 112 ? 7 : 8;         // rows per lane: ceil(m / 16)
      for (int sweep = 0; sweep < JACOBI_MAX_SWEEPS; ++sweep) {
        int rot = 0;
        for (int st = 0; st < mp - 1; ++st) {
          // pairs hw, hw + 32 (m > 64): every half-warp runs the same number of passes, so the
          // half-warp shuffles of both halves of a warp stay converged
          for (int pb = 0; pb < np; pb += 2 * K4_WARPS) {
            const int pp = pb + hw;
            int P = 0, Q = 0;
            bool act = false;
            if (pp < np) {
              P = rr_player(pp, st, mp);
              Q = rr_player(mp - 1 - pp, st, mp);
              act = P < nc && Q < nc;
            }
            bool r_;
            switch (eh) {
              case 4: r_ = jacobi_pair<4>(sA + P * m, sA + Q * m, m, hl, act, tol); break;
              case 7: r_ = jacobi_pair<7>(sA + P * m, sA + Q * m, m, hl, act, tol); break;
              default: r_ = jacobi_pair<8>(sA + P * m, sA + Q * m, m, hl, act, tol); break;
            }
            if (r_) rot = 1;
          }
          __syncthreads();
        }
        ++sweeps;
        if (!__syncthreads_or(rot)) { converged = true; break; }
      }
      for (int e = tid; e < nc * m; e += K4_THREADS) p.A[e] = sA[e];   // (columns >= nc stay zero)
      if (tid == 0) { p.flags[0] = converged ? 1 : 0; p.flags[1] = sweeps; }
    }
    cl_sync();
    converged = *(volatile int*)(p.flags) != 0;
    sweeps = *(volatile int*)(p.flags + 1);
  } else {
  // ---- a5: one-sided (Hestenes) block Jacobi on S.  The m columns form 8 blocks; a block sweep
  // is the round-robin tournament of the 8 blocks (7 rounds).  In each round CTA c of the cluster
  // holds block pair c in shared memory and rotates every column pair that crosses the two
  // blocks (round 0 also the pairs inside each block), so every pair of columns meets once per
  // block sweep.  Only the round boundaries need cluster barriers.
  // With m <= K4_JAC_DSM_M the blocks stay in the cluster's shared memory for the whole sweep:
  // each CTA keeps two buffers of its block pair and, at a round boundary, copies the two blocks of
  // its next pair out of the previous round's owners' buffers over DSMEM — no L2/HBM round trip
  // per round (the Gram pass streams at full HBM bandwidth meanwhile) and still one cluster
  // barrier per round (a CTA only overwrites the buffer the others read one round earlier).
  const int bs = (nc + 7) / 8;                    // block size (columns; the nc live ones)
  __shared__ volatile int jdone[32];
  const int ehs = m <= 64 ? 4 : m <= 112 ? 7 : m <= 160 ? 10 : m <= 208 ? 13 : kMaxM / 16;
  const double tol = fmax(1e-15, (double)m * DBL_EPSILON);
  const bool dsm = m <= K4_JAC_DSM_M;
  double* sbuf0 = reinterpret_cast<double*>(k4_smem);   // 2*bs columns x m, column-major
  double* sbuf1 = sbuf0 + (size_t)2 * bs * m;
  double* sA = sbuf0;
  int rounds = 0;                                 // rounds done (buffer of round q: q & 1)
  for (int sweep = 0; sweep < JACOBI_MAX_SWEEPS; ++sweep) {
    int rot = 0;
    for (int rd = 0; rd < 7; ++rd) {
      const int PB = rr_player(crank, rd, 8), QB = rr_player(7 - crank, rd, 8);
      if (tid < 32) jdone[tid] = -1;                   // per-half-warp step counters (flags mode)
      // local column lc in [0, 2bs): global column gc(lc)
      auto gcol = [&](int lc) { return lc < bs ? PB * bs + lc : QB * bs + (lc - bs); };
      if (dsm && rounds > 0) {
        sA = (rounds & 1) ? sbuf1 : sbuf0;
        const double* prev = (rounds & 1) ? sbuf0 : sbuf1;
        const int prd = rd == 0 ? 6 : rd - 1;
        for (int lc = warp; lc < 2 * bs; lc += K4_WARPS) {
          const int blk = lc < bs ? PB : QB, cb = lc < bs ? lc : lc - bs;
          int own = 0, slot = 0;
          for (int o = 0; o < K4_CLUSTER; ++o) {
            if (rr_player(o, prd, 8) == blk) { own = o; slot = 0; }
            if (rr_player(7 - o, prd, 8) == blk) { own = o; slot = 1; }
          }
          const unsigned src = dsm_addr(prev + (size_t)(slot * bs + cb) * m, (unsigned)own);
          double* dst = sA + (size_t)lc * m;
          for (int i = lane; i < m; i += 32) {
            double v;
            asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(src + 8u * (unsigned)i) : "memory");
            dst[i] = v;
          }
        }
      } else {
        for (int lc = warp; lc < 2 * bs; lc += K4_WARPS) {     // warp per column: no divisions
          const int gc = gcol(lc);
          double* dst = sA + lc * m;
          if (gc < nc) {
            const double* src = p.A + (long long)gc * m;
            for (int i = lane; i < m; i += 32) dst[i] = __ldcg(src + i);
          } else {
            for (int i = lane; i < m; i += 32) dst[i] = 0.0;
          }
        }
      }
      __syncthreads();
      const int nsteps = (rd == 0) ? 2 * bs - 1 : bs;
      if (K4_JAC_FLAGS && rd > 0) {
        // Rounds 1..6: half-warp hw keeps column P = hw and takes over column Q from half-warp
        // hw+1 (mod bs) each step, so it only has to wait for that neighbour's previous step
        // (a per-half-warp step counter in shared memory) instead of a CTA barrier per step.
        const int hw = warp * 2 + (lane >> 4), hl = lane & 15;
        const unsigned hmask = (lane >> 4) ? 0xffff0000u : 0x0000ffffu;
        if (hw < bs) {
          const int nb = hw + 1 == bs ? 0 : hw + 1;
          for (int st = 0; st < bs; ++st) {
            if (st > 0) {
              while (jdone[nb] < st - 1) { }
              __threadfence_block();
            }
            const int hs = hw + st, P = hw, Q = bs + (hs >= bs ? hs - bs : hs);
            const bool act = gcol(P) < nc && gcol(Q) < nc;
            bool r_;
            switch (ehs) {
              case 4: r_ = jacobi_pair<4>(sA + P * m, sA + Q * m, m, hl, act, tol, hmask); break;
              case 7: r_ = jacobi_pair<7>(sA + P * m, sA + Q * m, m, hl, act, tol, hmask); break;
              case 10: r_ = jacobi_pair<10>(sA + P * m, sA + Q * m, m, hl, act, tol, hmask); break;
              case 13: r_ = jacobi_pair<13>(sA + P * m, sA + Q * m, m, hl, act, tol, hmask); break;
              default: r_ = jacobi_pair<kMaxM / 16>(sA + P * m, sA + Q * m, m, hl, act, tol, hmask); break;
            }
            if (r_) rot = 1;
            __syncwarp(hmask);
            if (hl == 0) { __threadfence_block(); jdone[hw] = st; }
          }
        }
        __syncthreads();
      } else
      for (int st = 0; st < nsteps; ++st) {
        {
          // one column pair per half-warp (bs <= 32 pairs, 32 half-warps): 16 lanes x <=16 rows
          const int hw = warp * 2 + (lane >> 4), hl = lane & 15;
          int P = 0, Q = 0;
          bool act = false;
          if (hw < bs) {
            if (rd == 0) { P = rr_player(hw, st, 2 * bs); Q = rr_player(2 * bs - 1 - hw, st, 2 * bs); }
            else { const int hs = hw + st; P = hw; Q = bs + (hs >= bs ? hs - bs : hs); }   // hw, st < bs
            act = gcol(P) < nc && gcol(Q) < nc;
          }
          bool r_;
          switch (ehs) {                                    // per-lane rows: ceil(m / 16)
            case 4: r_ = jacobi_pair<4>(sA + P * m, sA + Q * m, m, hl, act, tol); break;
            case 7: r_ = jacobi_pair<7>(sA + P * m, sA + Q * m, m, hl, act, tol); break;
            case 10: r_ = jacobi_pair<10>(sA + P * m, sA + Q * m, m, hl, act, tol); break;
            case 13: r_ = jacobi_pair<13>(sA + P * m, sA + Q * m, m, hl, act, tol); break;
            default: r_ = jacobi_pair<kMaxM / 16>(sA + P * m, sA + Q * m, m, hl, act, tol); break;
          }
          if (r_) rot = 1;
        }
        __syncthreads();
      }
      if (!dsm) {
        for (int lc = warp; lc < 2 * bs; lc += K4_WARPS) {
          const int gc = gcol(lc);
          if (gc < nc) {
            const double* src = sA + lc * m;
            double* dst = p.A + (long long)gc * m;
            for (int i = lane; i < m; i += 32) dst[i] = src[i];
          }
        }
      }
      ++rounds;
      cl_sync();
    }
    ++sweeps;
    // rotations happen per half-warp: vote over the whole warp (lane 0 alone would miss a sweep
    // whose only rotations were on the upper half-warp)
    if (__any_sync(0xffffffffu, rot) && lane == 0) atomicOr(p.flags + sweep, 1);
    cl_sync();
    if (*(volatile int*)(p.flags + sweep) == 0) { converged = true; break; }
  }
  if (dsm) {                                      // the final blocks back to p.A for the a6 stage
    const int rd = 6;                             // every sweep ends with round 6
    const int PB = rr_player(crank, rd, 8), QB = rr_player(7 - crank, rd, 8);
    for (int lc = warp; lc < 2 * bs; lc += K4_WARPS) {
      const int gc = lc < bs ? PB * bs + lc : QB * bs + (lc - bs);
      if (gc < nc) {
        const double* src = sA + (size_t)lc * m;
        double* dst = p.A + (long long)gc * m;
        for (int i = lane; i < m; i += 32) dst[i] = src[i];
      }
    }
    cl_sync();
  }
  }
  if (tid == 0) ph[2] = clock64();

  // ---- a6: μ_j = ‖a_j‖ = |eig_j(S)|, σ = sqrt(|μ|) sorted desc, rank r, V (sign-normalised)
  for (int j = gwarp; j < m; j += K4_GW) {
    const double* cj = p.A + (long long)j * m;
    double s = 0.0;
    for (int i = lane; i < m; i += 32) { const double v = __ldcg(cj + i); s = fma(v, v, s); }
    s = wsum(s);
    if (lane == 0) p.mu[j] = p.chol ? s : sqrt(s);             // μ = σ² in both starts
  }
  cl_sync();
  for (int j = tid; j < m; j += K4_THREADS) mu[j] = __ldcg(p.mu + j);
  __syncthreads();
  for (int j = tid; j < m; j += K4_THREADS) {                // every CTA: identical permutation
    int rk = 0;
    const double mj = mu[j];
    for (int i = 0; i < m; ++i) rk += (mu[i] > mj || (mu[i] == mj && i < j)) ? 1 : 0;
    perm[rk] = j;
  }
  __syncthreads();
  for (int i = tid; i < m; i += K4_THREADS) {
    sig[i] = sqrt(mu[perm[i]]);
    if (crank == 0) p.sigma[i] = sig[i];
  }
  __syncthreads();
  if (tid == 0) {
    int r = 0;
    const double thr = p.rank_tol * sig[0];
    for (int i = 0; i < m; ++i) r += (sig[i] > thr) ? 1 : 0;
    if (r > p.r_max) r = p.r_max;
    sh_r = r;
    sh_status = (sig[0] == 0.0 || r == 0) ? 4 /*SDMD_E_ZERO_MATRIX*/ : (converged ? 0 : 5);
  }
  __syncthreads();
  const int r = sh_r;
  if (sh_status == 4) {                                     // uniform across the cluster
    if (crank == 0) {
      for (int i = tid; i < m; i += K4_THREADS) p.cout[i] = make_double2(0.0, 0.0);
      if (tid == 0) {
        res->frame = f; res->status = 4; res->r = 0; res->idx = -1; res->sweeps = sweeps; res->vframe = -1;
        res->nkeep = 0; res->nB = 0;
        res->qr_its = 0; res->sigma1 = sig[0];
      }
    }
    return;
  }
  for (int i = gwarp; i < m; i += K4_GW) {
    const int src = perm[i];
    // ‖a_j‖ = σ_j (Cholesky start) or |μ_j| = σ_j² (S·Q0 start)
    const double inv = mu[src] > 0.0 ? (p.chol ? 1.0 / sqrt(mu[src]) : 1.0 / mu[src]) : 0.0;
    const double* cj = p.A + (long long)src * m;
    double v[EL];
    double best = -1.0;
    int bi = 0;
#pragma unroll
    for (int e = 0; e < EL; ++e) {
      const int k = lane + 32 * e;
      v[e] = k < m ? __ldcg(cj + k) : 0.0;
      if (k < m && fabs(v[e]) > best) { best = fabs(v[e]); bi = k; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const double sgn_src = __ldcg(cj + bi);
    const double sgn = (sgn_src < 0.0) ? -inv : inv;        // reading Q6
#pragma unroll
    for (int e = 0; e < EL; ++e) {
      const int k = lane + 32 * e;
      if (k < m) {
        const double vv = v[e] * sgn;
        p.V[(long long)i * m + k] = vv;
        if (i < r) p.Y[(long long)i * m + k] = vv / sig[i];  // Y = V Σ⁻¹ ("vsi")
      }
    }
    if (lane == 0 && i < r) p.alpha1[i] = sig[i] * (v[0] * sgn);   // α₁ = σ ⊙ V[0,:] (Q3)
  }
  cl_sync();
  if (tid == 0) ph[3] = clock64();
  long long t_wait0 = 0;

  // ---- XᵀX' = G[0:m,1:m+1] needs the Gram column of frame f itself.  S = G[0:m,0:m] only needs
  // frames up to f-1, so K4a is released by the commit of frame f-1 and the Jacobi above overlaps
  // the Gram pass of frame f; here it waits for that pass's commit (device counter, published
  // after the history row) — or for the stream to be poisoned.
  // Frame f either gets committed, or the stream is poisoned before it is (a rejected frame <= f,
  // or a rejected batch containing f — whose failed_frame may be > f).  The poison flag is read
  // BEFORE the counter: a poison raised after f's commit (a later frame) is causally after the
  // commit, so seeing it and then an uncommitted f proves f will never commit.  CTA 0 of the
  // cluster decides (with a ~35 s bound so that a broken invariant can never hang the device) and
  // the other CTAs read its decision through distributed shared memory: uniform by construction.
  {
    __shared__ int sh_go;
    if (crank == 0 && tid == 0) {
      volatile DevState* vs = p.st;
      int go = -1;
      const long long t_start = clock64();
      while (go < 0) {
        const int poisoned = vs->status;
        __threadfence();
        if (vs->committed >= f + 1) go = 1;
        else if (poisoned != 0) go = 0;
        else if (clock64() - t_start > (1LL << 36)) go = 0;
        else __nanosleep(256);
      }
      sh_go = go;
    }
    cl_sync();
    int go;
    {
      unsigned a = (unsigned)__cvta_generic_to_shared(&sh_go), ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(ra) : "r"(a));
      asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(go) : "r"(ra) : "memory");
    }
    cl_sync();                                               // rank 0's flag read by everyone
    if (!go) return;                                         // frame f rejected: discard
  }
  if (tid == 0) t_wait0 = clock64() - ph[3];                 // commit wait (diagnostics)
  __threadfence();
  if (p.atilde_v1) {                                        // A/B: the untiled L2 version
    for (int idx = gtid; idx < m * m; idx += K4_GT) {
      const int i = idx % m, j = idx / m;
      p.Gxy[idx] = gram_at(p.ghist, p.NH, p.mh, m, f, i, j + 1);
    }
    cl_sync();
    for (int idx = gtid; idx < m * r; idx += K4_GT) {
      const int i = idx % m, j = idx / m;
      const double* yj = p.Y + (long long)j * m;
      double s = 0.0;
      for (int k = 0; k < m; ++k) s = fma(__ldcg(p.Gxy + (long long)k * m + i), __ldcg(yj + k), s);
      p.B[idx] = s;
    }
    cl_sync();
    for (int idx = gwarp; idx < r * r; idx += K4_GW) {
      const int i = idx / r, j = idx % r;
      const double* yi = p.Y + (long long)i * m;
      const double* bj = p.B + (long long)j * m;
      double s = 0.0;
      for (int k = lane; k < m; k += 32) s = fma(__ldcg(yi + k), __ldcg(bj + k), s);
      s = wsum(s);
      if (lane == 0) p.H[(long long)i * r + j] = s;
    }
    cl_sync();
  } else {
  // ---- a7: B = (XᵀX') Y (m x r), then Ã = Yᵀ B (r x r, row-major into H) — zero n-length dots.
  // Two fp64 products tiled through shared memory (k4_tiled_product), split over the cluster by
  // output rows (CTA c: rows [c·mb, (c+1)·mb) of B, then rows [c·rb, (c+1)·rb) of Ã); XᵀX' =
  // G[0:m,1:m+1] is gathered from the Gram history straight into the tiles.
  {
    double* t0 = reinterpret_cast<double*>(k4_smem);
    // (one call covers at most 64 output rows: 16 warps x 4 rows per thread)
    const int mb = (m + K4_CLUSTER - 1) / K4_CLUSTER;
    const int i0 = crank * mb, ni = max(0, min(m, i0 + mb) - i0);
    for (int s0 = 0; s0 < ni; s0 += 64)
      k4_tiled_product(0, m, r, i0 + s0, min(64, ni - s0), min(64, mb), tid, t0, p.ghist, p.NH, p.mh, f,
                       p.Y, p.B, p.H);
    cl_sync();                                               // all of B visible cluster-wide
    const int rb = (r + K4_CLUSTER - 1) / K4_CLUSTER;
    const int i1 = crank * rb, n1 = max(0, min(r, i1 + rb) - i1);
    for (int s0 = 0; s0 < n1; s0 += 64)
      k4_tiled_product(1, m, r, i1 + s0, min(64, n1 - s0), min(64, rb), tid, t0, p.ghist, p.NH, p.mh, f,
                       p.Y, p.B, p.H);
  }
  cl_sync();
  }
  if (tid == 0) ph[4] = clock64();

  // ---- a8: Householder reduction to upper Hessenberg form.  The rows of Ã are distributed over
  // the cluster's shared memory (CTA c owns rows [c·rb, (c+1)·rb)); per reflector only the pivot
  // column and the partial row-sums wᵀ = vᵀH cross CTAs, written straight into every CTA's shared
  // memory (DSMEM; two cluster barriers per step, no global round trips).  The partial sums are
  // added in CTA order on every CTA, so all hold the same reflector and the same τw.
  {
    const int rb = (r + K4_CLUSTER - 1) / K4_CLUSTER;
    const int r0 = crank * rb, r1 = min(r, r0 + rb);
    const int nr = r1 > r0 ? r1 - r0 : 0;
    double* sH = reinterpret_cast<double*>(k4_smem);        // nr x r, row-major
    double* sv = sH + (size_t)rb * r;                        // v  (kMaxR)
    double* sw = sv + kMaxR;                                 // τw (kMaxR)
    double* colk = sw + kMaxR;                               // pivot column (kMaxR, every CTA's rows)
    double* wpart = colk + kMaxR;                            // [K4_CLUSTER][kMaxR] partial wᵀ
    __shared__ double sh_tk, sh_beta;
    for (int e = tid; e < nr * r; e += K4_THREADS) sH[e] = __ldcg(p.H + (long long)r0 * r + e);
    __syncthreads();
    for (int k = 0; k < r - 2; ++k) {
      const int L = r - k - 1;
      const int i0 = r0 > k + 1 ? r0 : k + 1;                // my rows taking part in the reflector
      for (int e = tid; e < (r1 - i0) * K4_CLUSTER; e += K4_THREADS) {
        const int i = i0 + e / K4_CLUSTER;
        dsm_st(colk + i, (unsigned)(e % K4_CLUSTER), sH[(size_t)(i - r0) * r + k]);
      }
      cl_sync();
      if (warp == 0) {                                       // identical on every CTA
        double s2 = 0.0;
        for (int i = 1 + lane; i < L; i += 32) { const double x = colk[k + 1 + i]; s2 = fma(x, x, s2); }
        s2 = wsum(s2);
        const double x0 = colk[k + 1];
        double tauk = 0.0, beta = x0, v0 = 1.0;
        if (s2 != 0.0) {
          const double mu_ = sqrt(x0 * x0 + s2);
          v0 = (x0 <= 0.0) ? x0 - mu_ : -s2 / (x0 + mu_);
          tauk = 2.0 * v0 * v0 / (s2 + v0 * v0);
          beta = mu_;
        }
        for (int i = lane; i < L; i += 32) {
          const double v = (i == 0) ? 1.0 : (tauk != 0.0 ? colk[k + 1 + i] / v0 : 0.0);
          sv[i] = v;
          if (crank == 0) p.Qv[(long long)k * r + k + 1 + i] = v;
        }
        if (lane == 0) {
          sh_tk = tauk;
          sh_beta = beta;
          if (crank == 0) p.tau[k] = tauk;
        }
      }
      __syncthreads();
      const double tk = sh_tk;
      for (int i = i0 + tid; i < r1; i += K4_THREADS)
        sH[(size_t)(i - r0) * r + k] = (i == k + 1) ? sh_beta : 0.0;
      if (tk != 0.0) {
        for (int j = k + 1 + tid; j < r; j += K4_THREADS) {  // partial wᵀ = vᵀ H over my rows
          double s = 0.0;
          for (int i = i0; i < r1; ++i) s = fma(sv[i - k - 1], sH[(size_t)(i - r0) * r + j], s);
#pragma unroll
          for (int c = 0; c < K4_CLUSTER; ++c) dsm_st(wpart + crank * kMaxR + j, (unsigned)c, s);
        }
        cl_sync();
        for (int j = k + 1 + tid; j < r; j += K4_THREADS) {
          double s = 0.0;
          for (int c = 0; c < K4_CLUSTER; ++c) s += wpart[c * kMaxR + j];
          sw[j] = s * tk;
        }
        __syncthreads();
        if (r1 > i0) {                                       // left: H[i][j] -= v_i (τw)_j
          const int nrow = r1 - i0;
          for (int e = tid; e < nrow * L; e += K4_THREADS) {
            const int i = i0 + e / L, j = k + 1 + e % L;
            sH[(size_t)(i - r0) * r + j] -= sv[i - k - 1] * sw[j];
          }
        }
        __syncthreads();
        for (int i = r0 + warp; i < r1; i += K4_WARPS) {     // right: H[i][:] -= (τ H v)_i vᵀ
          double* hi = sH + (size_t)(i - r0) * r + k + 1;
          double s = 0.0;
          for (int jj = lane; jj < L; jj += 32) s = fma(hi[jj], sv[jj], s);
          s = wsum(s) * tk;
          for (int jj = lane; jj < L; jj += 32) hi[jj] -= s * sv[jj];
        }
        __syncthreads();
      } else {
        cl_sync();                                           // keep the barrier sequence uniform
      }
    }
    for (int e = tid; e < nr * r; e += K4_THREADS) p.H[(long long)r0 * r + e] = sH[e];
    cl_sync();
  }
  if (tid == 0) ph[5] = clock64();

  // ---- a8: eigenvalues of Ã (unsorted, into p.lam; K4b orders them).  Ehrlich–Aberth with Hyman's
  // method on all CTAs of the cluster (aberth_eigs_cluster), warm-started from the previous frame
  // of this cluster stream; the Francis multishift QR on CTA 0 when there is no warm spectrum of
  // the same size, H is reducible, or the iteration does not certify.
  __shared__ MsShared ms_sh;
  __shared__ int qr_st;
  {
    double* hs = reinterpret_cast<double*>(k4_smem);
    double2* lam_raw = reinterpret_cast<double2*>(hs + ((hs_elems(r) + 1) & ~1LL));
    int ab_rc = -1, ab_its = 0, ab_ev = 0;
    bool ab_tried = false;
    if (r > K4_MS_SMALL && p.r_warm != nullptr) {
      const int n0 = *(volatile const int*)p.r_warm;       // written by this stream's previous K4a
      if (n0 == r) {
        ab_tried = true;
        double2* zz = reinterpret_cast<double2*>(ms_sh.dense);
        double2* zn = zz + kMaxR;
        int* act = reinterpret_cast<int*>(zn + kMaxR);
        ab_rc = aberth_eigs_cluster<CL>(p.H, r, hs, p.lam_warm, n0, zz, zn, act, lam_raw, crank, tid, warp,
                                    lane, &ab_its, &ab_ev);
      }
    }
    if (crank != 0) return;                                  // the rest is CTA 0's
    if (tid == 0) qr_st = 0;
    if (ab_rc != 0) {
      for (int i = warp; i < r; i += K4_WARPS) {
        const int lo = i > 3 ? i - 3 : 0;
        const long long o = hs_off(i, r);
        for (int j = lo + lane; j < r; j += 32)
          hs[o + j - lo] = (j >= i - 1) ? __ldcg(p.H + (long long)i * r + j) : 0.0;
      }
      for (int i = tid; i < r; i += K4_THREADS) lam_raw[i] = make_double2(0.0, 0.0);
      __syncthreads();
      __shared__ int qc_sh[4];
      __shared__ int its_sh;
      __shared__ int roff_sh[kMaxR];
      if (tid < 4) qc_sh[tid] = 0;
      if (tid == 0) its_sh = 0;
      for (int i = tid; i < r; i += K4_THREADS) roff_sh[i] = (int)(hs_off(i, r) - (i > 3 ? i - 3 : 0));
      __syncthreads();
      int its_local = 0;
      long long shift_cyc = 0, chase_cyc[2] = {0, 0};
      const int rc = multishift_qr(RowAcc{hs, roff_sh}, r, lam_raw, &ms_sh, tid, warp, lane, &its_local,
                                   warp == 0 ? qc_sh : nullptr, &shift_cyc, chase_cyc);
      if (warp == 0 && lane == 0) atomicAdd(&its_sh, its_local);
      __syncthreads();
      if (tid == 0) {
        if (rc != 0) qr_st = 5;
        res->qr_its = its_sh;
        res->qr_cnt[0] = qc_sh[0]; res->qr_cnt[1] = qc_sh[1]; res->qr_cnt[2] = qc_sh[2];
        res->qr_cnt[3] = qc_sh[3];
        res->phase[7] = shift_cyc;
        res->qr_dbg[0] = chase_cyc[0];
        res->qr_dbg[1] = chase_cyc[1];
      }
    } else if (tid == 0) {
      res->qr_its = 0;
      res->qr_cnt[0] = res->qr_cnt[1] = res->qr_cnt[2] = res->qr_cnt[3] = 0;
      res->phase[7] = 0;
      res->qr_dbg[0] = ch_cyc[1] - ch_cyc[0];    // (Aberth path) diagnostics: pivoted-Cholesky cycles
      res->qr_dbg[1] = 0;
    }
    __syncthreads();
    for (int k = tid; k < r; k += K4_THREADS) {
      p.lam[k] = lam_raw[k];
      if (p.r_warm != nullptr) p.lam_warm[k] = lam_raw[k];  // the next frame of this stream starts here
    }
    if (tid == 0) {
      if (p.r_warm != nullptr) *p.r_warm = qr_st ? 0 : r;
      // its, or the failure: −1 no warm start tried... −2 reducible, −3 no convergence in AB_MAXIT,
      // −4 non-finite step, −5 trace mismatch, −6 conjugate pairing
      res->aberth_its = ab_rc == 0 ? ab_its : (ab_tried ? ab_rc : 0);
      res->aberth_evals = ab_ev;
    }
  }
  // K4a done: publish the factors' summary for K4b (same stream order via events)
  if (tid == 0) {
    if (r >= 2) p.tau[r - 2] = 0.0;
    p.tau[r > 0 ? r - 1 : 0] = 0.0;
    ph[6] = clock64();
    res->frame = f; res->status = (sh_status == 0 && qr_st) ? 5 : sh_status; res->r = r; res->idx = -1;
    res->sweeps = sweeps; res->sigma1 = sig[0]; res->nkeep = r; res->nB = 0;
    res->vframe = (converged && sh_chol_full) ? f : -1;   // V usable as the next warm start
    for (int q = 0; q < 6; ++q) res->phase[q] = ph[q + 1] - ph[q];
    res->commit_wait = t_wait0;
    res->phase[6] = 0;
  }
}

// ------------------------------------------------------------------ K4b: eigen(Ã) and c -------
// Single CTA: Francis multishift QR on the Hessenberg form (shared memory), ordering of λ, the
// background index, inverse iteration for w_idx / y_idx, b_idx and the background coefficients.
__global__ void __launch_bounds__(K4_THREADS, 1) k4b_kernel(const K4Params p) {
  extern __shared__ __align__(16) unsigned char k4_smem[];
  __shared__ int sh_status, sh_idx, sh_its, sh_go, sh_nkeep;
  __shared__ long long ph[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = p.m;
  const long long f = p.f;
  K4Result* res = p.res;
  {
    volatile DevState* st = p.st;
    if (st->status != 0 && st->failed_frame <= f) return;
  }
  if (tid == 0) {
    const volatile K4Result* vr = res;
    sh_go = (vr->frame == f && vr->status != 4 && vr->r > 0) ? 1 : 0;
    sh_status = vr->status;
    ph[5] = clock64();
  }
  __syncthreads();
  if (!sh_go) return;                                      // K4a found a zero window (c = 0)
  const int r = res->r;
  const int sweeps = res->sweeps;
  const double sigma1 = res->sigma1;
  double* H = p.H;

  // ---- a8: the eigenvalues of Ã were computed by K4a's cluster (unsorted in p.lam, see k4a_kernel)
  double* hs = reinterpret_cast<double*>(k4_smem);
  const long long hsz = hs_elems(r);
  double2* lam_raw = reinterpret_cast<double2*>(hs + ((hsz + 1) & ~1LL));
  for (int k = tid; k < r; k += K4_THREADS) lam_raw[k] = __ldcg(p.lam + k);
  if (tid == 0) sh_its = res->qr_its;
  __syncthreads();
  if (tid == 0) ph[6] = clock64();

  // ---- sort λ: |λ| desc, Re desc, Im desc (reading Q12)
  for (int j = tid; j < r; j += K4_THREADS) {
    const double2 lj = lam_raw[j];
    const double aj = hypot(lj.x, lj.y);
    int rk = 0;
    for (int i = 0; i < r; ++i) {
      const double2 li = lam_raw[i];
      const double ai = hypot(li.x, li.y);
      const bool before = (ai > aj) || (ai == aj && (li.x > lj.x || (li.x == lj.x && (li.y > lj.y ||
                          (li.y == lj.y && i < j)))));
      rk += before ? 1 : 0;
    }
    p.lam[rk] = lj;
  }
  __syncthreads();

  // ---- a10: idx = argmin |log λ| (principal branch), λ = 0 excluded; ties (Q5).  Warp 0: each
  // lane the lexicographic minimum (|log λ|, |arg λ|, Im λ < 0, index) of its strided subset, then
  // a shuffle reduction with the same order — the result equals the sequential scan's.
  if (warp == 0) {
    int best = -1;
    double k1 = 0, k2 = 0;
    int k3 = 0;
    for (int i = lane; i < r; i += 32) {
      const double2 l = p.lam[i];
      if (l.x == 0.0 && l.y == 0.0) continue;
      const double lr = log(hypot(l.x, l.y)), li = atan2(l.y, l.x);
      const double a1 = hypot(lr, li), a2 = fabs(li);
      const int a3 = (l.y >= 0.0) ? 0 : 1;
      if (best < 0 || a1 < k1 || (a1 == k1 && (a2 < k2 || (a2 == k2 && a3 < k3)))) {
        best = i; k1 = a1; k2 = a2; k3 = a3;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int ob = __shfl_xor_sync(0xffffffffu, best, o);
      const double o1 = __shfl_xor_sync(0xffffffffu, k1, o), o2 = __shfl_xor_sync(0xffffffffu, k2, o);
      const int o3 = __shfl_xor_sync(0xffffffffu, k3, o);
      const bool take = ob >= 0 && (best < 0 || o1 < k1 ||
                        (o1 == k1 && (o2 < k2 || (o2 == k2 && (o3 < k3 || (o3 == k3 && ob < best))))));
      if (take) { best = ob; k1 = o1; k2 = o2; k3 = o3; }
    }
    if (lane == 0) sh_idx = best;
  }
  if (tid == 0) {
    const int best = sh_idx;
    if (best < 0 && sh_status == 0) sh_status = 7;
    // reading Q15: WΛ is singular when some |λ_j| < rank_tol·max|λ|; those
    // modes form a suffix of the sorted λ.  Flag W_SINGULAR; the kept-mode least squares of b
    // (and c) is redone by k4s_kernel right after this kernel on the same stream.
    const double a0 = r > 0 ? cabs2(p.lam[0]) : 0.0;
    int nk = 0;
    if (a0 > 0.0) {
      nk = r;
      while (nk > 0 && !(cabs2(p.lam[nk - 1]) >= p.rank_tol * a0)) --nk;
    }
    sh_nkeep = nk;
    if (nk < r && sh_status == 0) sh_status = 6;
  }
  __syncthreads();
  const int idx = sh_idx;

  // ---- NEXT-2 (reading Q25): background from the mode set B = the nb smallest |log λ| in Q5's
  // order, closed under conjugation; one warp per mode runs the inverse iteration (its own
  // scratch and LU workspace), and c = Σ_{p∈B} b_p λ_p^m Y w_p is summed in B order
  if (idx >= 0 && p.bg_modes > 1) {
    __shared__ int bset[kMaxBgModes + 1];
    __shared__ int nB;
    __shared__ double2 bq_sh[kMaxBgModes + 1];
    __shared__ unsigned char chosen[kMaxR];
    for (int i = tid; i < r; i += K4_THREADS) chosen[i] = 0;
    __syncthreads();
    if (tid == 0) {
      auto key_less = [&](int i, int j) {     // Q5 key of λ_i < key of λ_j
        const double2 a = p.lam[i], b2 = p.lam[j];
        const double ar = log(hypot(a.x, a.y)), ai = atan2(a.y, a.x);
        const double br = log(hypot(b2.x, b2.y)), bi = atan2(b2.y, b2.x);
        const double a1 = hypot(ar, ai), b1 = hypot(br, bi);
        if (a1 != b1) return a1 < b1;
        if (fabs(ai) != fabs(bi)) return fabs(ai) < fabs(bi);
        const int a3 = a.y >= 0.0 ? 0 : 1, b3 = b2.y >= 0.0 ? 0 : 1;
        if (a3 != b3) return a3 < b3;
        return i < j;
      };
      auto next_best = [&]() {
        int best = -1;
        for (int i = 0; i < r; ++i) {
          const double2 l = p.lam[i];
          if ((l.x == 0.0 && l.y == 0.0) || chosen[i]) continue;
          if (best < 0 || key_less(i, best)) best = i;
        }
        return best;
      };
      int cnt = 0;
      const int nb = p.bg_modes < kMaxBgModes ? p.bg_modes : kMaxBgModes;
      while (cnt < nb) {
        const int bi = next_best();
        if (bi < 0) break;
        bset[cnt++] = bi;
        chosen[bi] = 1;
      }
      if (cnt == nb) {                          // conjugate closure of the last mode
        const double2 l = p.lam[bset[cnt - 1]];
        const int nx = next_best();
        if (l.y != 0.0 && nx >= 0 && p.lam[nx].x == l.x && p.lam[nx].y == -l.y) bset[cnt++] = nx;
      }
      nB = cnt;
    }
    __syncthreads();
    const int nb_eff = nB;
    constexpr size_t SCR = 3 * (size_t)kMaxR * sizeof(double2) + (size_t)kMaxR * sizeof(int);
    double2* cpart = reinterpret_cast<double2*>(k4_smem + (size_t)nb_eff * SCR);   // [nB][m]
    if (warp < nb_eff) {
      unsigned char* base = k4_smem + (size_t)warp * SCR;
      double2* zq = reinterpret_cast<double2*>(base);
      double2* rq = zq + kMaxR;
      double2* lq = rq + kMaxR;
      int* sq = reinterpret_cast<int*>(lq + kMaxR);
      double2* wq = p.w + (size_t)warp * kMaxR;
      double2* yq = p.y + (size_t)warp * kMaxR;
      const double2 lam = p.lam[bset[warp]];
      inverse_iteration(H, p.Qv, p.tau, r, lam, p.M + (size_t)warp * kMaxR * kMaxR, zq, rq, lq, sq, wq, yq, lane);
      double2 ya = make_double2(0, 0), yw = make_double2(0, 0);
      for (int i = lane; i < r; i += 32) {
        const double2 yc = cconj(yq[i]);
        ya = cadd(ya, make_double2(yc.x * p.alpha1[i], yc.y * p.alpha1[i]));
        yw = cadd(yw, cmul(yc, wq[i]));
      }
      ya = wsum2(ya);
      yw = wsum2(yw);
      const double2 den = cmul(lam, yw);
      const double2 b = cabs2(den) > 1e-300 ? cdiv(ya, den) : make_double2(0.0, 0.0);
      double2 pw = make_double2(1.0, 0.0), bs_ = lam;        // λ^m by binary powering
      for (int e = m; e > 0; e >>= 1) {
        if (e & 1) pw = cmul(pw, bs_);
        bs_ = cmul(bs_, bs_);
      }
      const double2 coef = cmul(b, pw);
      for (int i = lane; i < m; i += 32) {
        double2 s = make_double2(0.0, 0.0);
        for (int j = 0; j < r; ++j) {
          const double yv = p.Y[(long long)j * m + i];
          s = cadd(s, make_double2(yv * wq[j].x, yv * wq[j].y));
        }
        cpart[(size_t)warp * m + i] = cmul(coef, s);
      }
      if (lane == 0) bq_sh[warp] = (cabs2(den) > 1e-300) ? b : make_double2(NAN, 0.0);
    }
    __syncthreads();
    for (int i = tid; i < m; i += K4_THREADS) {
      double2 s = make_double2(0.0, 0.0);
      for (int q = 0; q < nb_eff; ++q) s = cadd(s, cpart[(size_t)q * m + i]);
      p.cout[i] = s;
    }
    if (tid == 0) {
      int st = sh_status;
      for (int q = 0; q < nb_eff; ++q)
        if (isnan(bq_sh[q].x) && st == 0) st = 6;
      const double2 lam = p.lam[idx];
      const double2 b0 = isnan(bq_sh[0].x) ? make_double2(0.0, 0.0) : bq_sh[0];
      ph[7] = clock64();
      res->phase[6] = ph[7] - ph[6];
      res->frame = f; res->status = st; res->r = r; res->idx = idx; res->sweeps = sweeps;
      res->qr_its = sh_its; res->lam_idx[0] = lam.x; res->lam_idx[1] = lam.y;
      res->b_idx[0] = b0.x; res->b_idx[1] = b0.y; res->sigma1 = sigma1;
      res->nkeep = sh_nkeep; res->nB = nb_eff;
      for (int q = 0; q < nb_eff; ++q) res->bset[q] = bset[q];
    }
    return;
  }

  // ---- a8/a9: eigenvectors of the background mode (LU on warp 0, then the right solve on warp 0
  // and the left solve on warp 1 concurrently), b_idx, and c (all threads); scratch aliases the
  // (now free) packed Hessenberg area
  double2* z = reinterpret_cast<double2*>(k4_smem);
  double2* rhs = z + kMaxR;
  double2* lk = rhs + kMaxR;
  double2* z2 = lk + kMaxR;
  double2* rhs2 = z2 + kMaxR;
  double2* wsm = rhs2 + kMaxR;
  int* swk = reinterpret_cast<int*>(wsm + kMaxR);
  __shared__ double hn_sh;
  __shared__ double2 coef_sh;
  __shared__ int st_sh;
  if (idx >= 0) {
    {                                                    // max |h_ij| of the Hessenberg form
      double hn = 0.0;
      for (int e = tid; e < r * r; e += K4_THREADS) {
        const int i = e / r, j = e % r;
        if (j >= i - 1) hn = fmax(hn, fabs(__ldcg(H + e)));
      }
      hn = wmax(hn);
      if (tid == 0) hn_sh = 0.0;
      __syncthreads();
      if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&hn_sh), __double_as_longlong(hn));
      __syncthreads();
    }
    const double2 lam = p.lam[idx];
    if (warp == 0) iv_lu(H, r, lam, p.M, lk, swk, lane, hn_sh, p.Mc);
    __syncthreads();
    // right vector on threads 0..255, left vector on 256..511 (named barriers 1 and 2)
    if (tid < IV_GT) iv_right_grp(p.Qv, p.tau, r, p.Mc, lk, swk, z, rhs, p.w, tid, warp, lane, 1);
    else iv_left_grp(p.Qv, p.tau, r, p.M, lk, swk, z2, rhs2, p.y, tid - IV_GT, warp - IV_GT / 32, lane, 2);
    __syncthreads();
    if (warp == 0) {
      double2 ya = make_double2(0, 0), yw = make_double2(0, 0);
      for (int i = lane; i < r; i += 32) {
        const double2 yc = cconj(p.y[i]);
        ya = cadd(ya, make_double2(yc.x * p.alpha1[i], yc.y * p.alpha1[i]));
        yw = cadd(yw, cmul(yc, p.w[i]));
      }
      ya = wsum2(ya);
      yw = wsum2(yw);
      if (lane == 0) {
        const double2 den = cmul(lam, yw);
        double2 b = make_double2(0.0, 0.0);
        int st = sh_status;
        if (cabs2(den) > 1e-300) b = cdiv(ya, den);
        else if (st == 0) st = 6;
        double2 pw = make_double2(1.0, 0.0), base = lam;   // λ^m by binary powering
        for (int e = m; e > 0; e >>= 1) {
          if (e & 1) pw = cmul(pw, base);
          base = cmul(base, base);
        }
        coef_sh = cmul(b, pw);
        st_sh = st;
        res->b_idx[0] = b.x; res->b_idx[1] = b.y;
      }
    }
    for (int j = tid; j < r; j += K4_THREADS) wsm[j] = p.w[j];
    __syncthreads();
    const double2 coef = coef_sh;
    for (int i = tid; i < m; i += K4_THREADS) {          // c = b_idx λ^m Y w_idx, one row per thread
      double2 sacc = make_double2(0.0, 0.0);
      for (int j = 0; j < r; ++j) {
        const double yv = __ldcg(p.Y + (long long)j * m + i);
        sacc = make_double2(fma(yv, wsm[j].x, sacc.x), fma(yv, wsm[j].y, sacc.y));
      }
      p.cout[i] = cmul(coef, sacc);
    }
    if (tid == 0) {
      ph[7] = clock64();
      res->phase[6] = ph[7] - ph[6];
      res->frame = f; res->status = st_sh; res->r = r; res->idx = idx; res->sweeps = sweeps;
      res->qr_its = sh_its; res->lam_idx[0] = lam.x; res->lam_idx[1] = lam.y;
      res->sigma1 = sigma1;
      res->nkeep = sh_nkeep; res->nB = 1; res->bset[0] = idx;
    }
  } else if (idx < 0) {
    for (int i = tid; i < m; i += K4_THREADS) p.cout[i] = make_double2(0.0, 0.0);
    if (tid == 0) {
      res->frame = f; res->status = sh_status; res->r = r; res->idx = -1; res->sweeps = sweeps;
      res->qr_its = sh_its; res->sigma1 = sigma1; res->nkeep = sh_nkeep; res->nB = 0;
    }
  }
}

size_t k4_smem_bytes(int r_max, int m, int bg_modes, int cl) {
  const long long hs = hs_elems(r_max);
  const size_t a = (size_t)((hs + 1) & ~1LL) * sizeof(double) + (size_t)kMaxR * sizeof(double2);
  const size_t b = 6 * (size_t)kMaxR * sizeof(double2) + (size_t)kMaxR * sizeof(int);   // eigvec scratch (K4b)
  const size_t c = (cl == 1 || m <= K4_SMALL_M) ? (size_t)((m + 1) & ~1) * m * sizeof(double)   // whole S
                   : (m <= K4_JAC_DSM_M ? 4 : 2) * (size_t)((m + 7) / 8) * m * sizeof(double);  // block pair (x2 buffers)
  const size_t d = ((size_t)((r_max + cl - 1) / cl) * r_max + (3 + cl) * kMaxR) * sizeof(double);  // Hessenberg rows + exchange
  // Ã tiles (K4a a7): 32 x (ceil(max(m, r)/4) + r) doubles
  const int rows2 = ((m > r_max ? m : r_max) + cl - 1) / cl;
  const int cols2 = m <= kMaxR && m > r_max ? m : r_max;            // Cholesky-start GEMMs: N = m
  const size_t d2 = (size_t)32 * (64 + cols2) * sizeof(double);
  // multi-mode background: per-mode inverse-iteration scratch (one warp each) + coefficient parts
  const size_t b3 = 3 * (size_t)kMaxR * sizeof(double2) + (size_t)kMaxR * sizeof(int);   // per mode
  const size_t e = bg_modes > 1 ? (size_t)(bg_modes + 1) * (b3 + (size_t)m * sizeof(double2)) : 0;
  size_t s = a > b ? a : b;
  s = s > c ? s : c;
  s = s > e ? s : e;
  s = s > d2 ? s : d2;
  return s > d ? s : d;
}

void preload_k4_kernels() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k4a_kernel<K4_CLUSTER>);
  cudaFuncGetAttributes(&a, k4a_kernel<1>);
  cudaFuncGetAttributes(&a, k4b_kernel);
}

cudaError_t launch_k4a(const K4Params& p, cudaStream_t s, int cl) {
  size_t smem = k4_smem_bytes(p.r_max, p.m, p.bg_modes, cl);
  if (p.chol && p.m <= K4_CHOL_SMEM_M) {                     // the Cholesky factor (and Sw) in shared memory
    const size_t need = (size_t)p.m * p.m * sizeof(double) * (p.m <= 110 ? 2 : 1);
    if (smem < need) smem = need;
  }
  const void* fn = cl == 1 ? (const void*)k4a_kernel<1> : (const void*)k4a_kernel<K4_CLUSTER>;
  cudaError_t e = set_max_dyn_smem(fn, (int)smem);
  if (e != cudaSuccess) return e;
  if (cl == 1) k4a_kernel<1><<<1, K4_THREADS, smem, s>>>(p);
  else k4a_kernel<K4_CLUSTER><<<K4_CLUSTER, K4_THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_k4b(const K4Params& p, cudaStream_t s) {
  const size_t smem = k4_smem_bytes(p.r_max, p.m, p.bg_modes, K4_CLUSTER);
  cudaError_t e = set_max_dyn_smem((const void*)k4b_kernel, (int)smem);
  if (e != cudaSuccess) return e;
  k4b_kernel<<<1, K4_THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

// CTAs per K4a launch: one for dense windows with K4_SMALL_M < m <= K4_SOLO_M (the Gram pass needs
// the SMs: about half the K4a SM-cycles of the cluster, at a latency the background lag absorbs),
// else the 4-CTA cluster (sparse contexts are eigen-bound and latency-bound by the stream count;
// small windows are launch-bound).  SDMD_K4_CL=1|4 overrides (A/B).
int k4_cluster_size(int m, bool sparse) {
  const char* ev = std::getenv("SDMD_K4_CL");
  const int env = ev ? std::atoi(ev) : 0;
  if (env == 4 || m > K4_SOLO_M) return K4_CLUSTER;
  if (env == 1) return 1;
  return (!sparse && m > K4_SMALL_M) ? 1 : K4_CLUSTER;
}
int k4_small_m() { return K4_SMALL_M; }

// ------------------------------------------------------- on-demand eigenvectors and b --------
__global__ void __launch_bounds__(32) k4_vecs_kernel(const K4VecParams p) {
  extern __shared__ __align__(16) unsigned char vs_smem[];
  const int r = p.res ? ((volatile const K4Result*)p.res)->r : p.r;   // p.r: r_max when p.res
  double2* z = reinterpret_cast<double2*>(vs_smem);
  double2* rhs = z + r;
  double2* lk = rhs + r;
  double2* wv = lk + r;
  double2* yv = wv + r;
  int* swk = reinterpret_cast<int*>(yv + r);
  const int j = p.j0 + blockIdx.x;
  if (j >= r) return;
  const int lane = threadIdx.x;
  const double2 lam = p.lam[j];
  double2* M = p.Mws + (long long)blockIdx.x * r * r;
  inverse_iteration(p.H, p.Qv, p.tau, r, lam, M, z, rhs, lk, swk, wv, yv, lane);
  double2 ya = make_double2(0, 0), yw = make_double2(0, 0);
  for (int i = lane; i < r; i += 32) {
    const double2 yc = cconj(yv[i]);
    ya = cadd(ya, make_double2(yc.x * p.alpha1[i], yc.y * p.alpha1[i]));
    yw = cadd(yw, cmul(yc, wv[i]));
  }
  ya = wsum2(ya);
  yw = wsum2(yw);
  for (int i = lane; i < r; i += 32) p.W[(long long)j * r + i] = wv[i];
  if (lane == 0) {
    const double2 den = cmul(lam, yw);
    p.b[j] = (cabs2(den) > 1e-300) ? cdiv(ya, den) : make_double2(0.0, 0.0);
  }
}

cudaError_t launch_k4_vecs(const K4VecParams& p, int count, cudaStream_t s) {
  const size_t smem = 5 * (size_t)p.r * sizeof(double2) + (size_t)p.r * sizeof(int) + 16;
  k4_vecs_kernel<<<count, 32, smem, s>>>(p);
  return cudaGetLastError();
}

// ------------------------------------------------ W_SINGULAR amplitudes (reading Q15) --------
// One warp per CTA.  (1) The CTAs compute the right eigenvectors of the kept modes j < nkeep by
// inverse iteration on the Hessenberg form (CTA c: j = c, c + grid, …; its own LU workspace).
// (2) The last CTA to finish solves min ‖A b − α₁‖, A = W_K diag(λ_K) (r x nkeep), by complex
// Householder QR (reflector H = I − 2 v vᴴ / vᴴv, v = x + e^{i arg x₀}‖x‖e₁) and back-
// substitution; b_j = 0 for j >= nkeep.  (3) Per frame it rewrites the background coefficients
// c = Σ_{q∈B} b_q λ_q^m Y w_q and b_idx.  Per frame the kernel returns at once unless this frame's
// K4b flagged W_SINGULAR with nkeep < r.
__global__ void __launch_bounds__(32) k4s_kernel(const K4SingParams p, int vecs) {
  extern __shared__ __align__(16) unsigned char ss_smem[];
  __shared__ int am_last;
  const int lane = threadIdx.x;
  int r, nk, m = p.m;
  if (p.res) {
    const volatile K4Result* vr = p.res;
    if (vr->frame != p.f || vr->status != 6) return;
    r = vr->r;
    nk = vr->nkeep;
    if (nk >= r) return;
  } else {
    r = p.r;
    nk = p.nkeep;
  }
  const int R = p.r;                                  // workspace stride (r_max per frame)
  double2* z = reinterpret_cast<double2*>(ss_smem);
  double2* rhs = z + R;
  double2* lk = rhs + R;
  double2* bsh = lk + R;
  int* swk = reinterpret_cast<int*>(bsh + R);
  if (vecs) {
    double2* M = p.Mws + (long long)blockIdx.x * R * R;
    for (int j = blockIdx.x; j < nk; j += gridDim.x)
      inverse_iteration(p.H, p.Qv, p.tau, r, p.lam[j], M, z, rhs, lk, swk, p.W + (long long)j * r,
                        nullptr, lane);
    __threadfence();
    if (lane == 0) am_last = (atomicAdd(p.counter, 1u) == gridDim.x - 1);
    __syncwarp();
    if (!am_last) return;
    __threadfence();
    if (lane == 0) *p.counter = 0u;
  }
  // (2) least squares on A = W_K Λ_K
  double2* A = p.A;
  for (int e = lane; e < r * nk; e += 32) {
    const int i = e % r, j = e / r;
    A[(long long)j * r + i] = cmul(__ldcg(p.W + (long long)j * r + i), p.lam[j]);
  }
  for (int i = lane; i < r; i += 32) rhs[i] = make_double2(p.alpha1[i], 0.0);
  __syncwarp();
  for (int k = 0; k < nk; ++k) {
    double s2 = 0.0;
    for (int i = k + lane; i < r; i += 32) { const double2 a = A[(long long)k * r + i]; s2 += a.x * a.x + a.y * a.y; }
    s2 = wsum(s2);
    const double nrm = sqrt(s2);
    if (nrm == 0.0) continue;                          // R_kk = 0: b_k = 0 below
    const double2 x0 = A[(long long)k * r + k];
    const double ax0 = cabs2(x0);
    const double2 ph = ax0 > 0.0 ? make_double2(x0.x / ax0, x0.y / ax0) : make_double2(1.0, 0.0);
    const double vv = 2.0 * nrm * (nrm + ax0);
    for (int i = k + lane; i < r; i += 32)           // v in z[k..r)
      z[i] = (i == k) ? cadd(x0, make_double2(ph.x * nrm, ph.y * nrm)) : A[(long long)k * r + i];
    __syncwarp();
    for (int j = k; j <= nk; ++j) {                    // columns k..nk-1, then the right-hand side
      double2* col = (j < nk) ? A + (long long)j * r : rhs;
      double2 d = make_double2(0.0, 0.0);
      for (int i = k + lane; i < r; i += 32) d = cadd(d, cmul(cconj(z[i]), col[i]));
      d = wsum2(d);
      d = make_double2(2.0 * d.x / vv, 2.0 * d.y / vv);
      __syncwarp();
      for (int i = k + lane; i < r; i += 32) col[i] = csub(col[i], cmul(z[i], d));
      __syncwarp();
    }
  }
  for (int i = nk - 1; i >= 0; --i) {                  // R b = (Qᴴα₁)[0:nk]
    double2 sacc = make_double2(0.0, 0.0);
    for (int j = i + 1 + lane; j < nk; j += 32) sacc = cadd(sacc, cmul(A[(long long)j * r + i], bsh[j]));
    sacc = wsum2(sacc);
    if (lane == 0) {
      const double2 d = A[(long long)i * r + i];
      bsh[i] = cabs2(d) > 0.0 ? cdiv(csub(rhs[i], sacc), d) : make_double2(0.0, 0.0);
    }
    __syncwarp();
  }
  for (int j = lane; j < r; j += 32) p.b[j] = j < nk ? bsh[j] : make_double2(0.0, 0.0);
  __syncwarp();
  if (p.cout && p.res) {                              // (3) background coefficients of the set B
    const int nB = p.res->nB;
    for (int i = lane; i < m; i += 32) {
      double2 cc = make_double2(0.0, 0.0);
      for (int q = 0; q < nB; ++q) {
        const int jq = p.res->bset[q];
        if (jq < 0 || jq >= nk) continue;
        double2 pw = make_double2(1.0, 0.0), base = p.lam[jq];
        for (int e = m; e > 0; e >>= 1) {
          if (e & 1) pw = cmul(pw, base);
          base = cmul(base, base);
        }
        const double2 coef = cmul(bsh[jq], pw);
        double2 sacc = make_double2(0.0, 0.0);
        for (int j = 0; j < r; ++j) {
          const double yv = p.Y[(long long)j * m + i];
          const double2 wv = __ldcg(p.W + (long long)jq * r + j);
          sacc = cadd(sacc, make_double2(yv * wv.x, yv * wv.y));
        }
        cc = cadd(cc, cmul(coef, sacc));
      }
      p.cout[i] = cc;
    }
    if (lane == 0) {
      const int idx = p.res->idx;
      const double2 bi = (idx >= 0 && idx < nk) ? bsh[idx] : make_double2(0.0, 0.0);
      p.res_out->b_idx[0] = bi.x;
      p.res_out->b_idx[1] = bi.y;
    }
  }
}

cudaError_t launch_k4_singular(const K4SingParams& p, bool vecs, cudaStream_t s) {
  const size_t smem = 4 * (size_t)p.r * sizeof(double2) + (size_t)p.r * sizeof(int) + 16;
  k4s_kernel<<<vecs ? kSingVecGrid : 1, 32, smem, s>>>(p, vecs ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace sdmd
