/* sdmd_oracle.c — ORACLE, test infrastructure, NOT part of the product.
 *
 * Plain, slow, fp64 CPU arithmetic of the streaming method-of-snapshots SVD / DMD of
 * arXiv 1612.07875 (reference: /root/reference/PAPER.md, cited P:<line>; SPEC.md cited S:<line>;
 * readings Qk = DESIGN.md §3 / SURVEY.md §8(c)).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library (through
 * oracle/sdmd_oracle.py).  It shares no code, header, table or helper with the CUDA path
 * (paper_1612_07875_b200/) and never includes or links it.
 *
 * Every routine is a textbook algorithm written out with explicit loops, in the order of the
 * definition it follows; no BLAS, no LAPACK, no blocking beyond a row-block loop that keeps the
 * per-entry summation order (increasing row index) intact:
 *   O1  orc_gram / orc_dots      G_ij = sum_l z_i[l] z_j[l], Neumaier-compensated fp64 sum of
 *                                exact products (fp32 inputs are exact in fp64; fp64 products
 *                                carry their rounding error via fma into the compensation)
 *                                (§3.1, Alg 1)
 *   O3  orc_jacobi               cyclic-by-row Jacobi with the stable rotation of Golub & Van Loan
 *                                §8.5 (t = sgn(th)/(|th|+sqrt(1+th^2))) (Alg 1 "eig(xtx)" P:297)
 *   O6  orc_eig_real             Householder reduction to Hessenberg form (GVL Alg 7.4.2), Francis
 *                                double-shift QR to real Schur form (GVL Alg 7.5.1/7.5.2), eigen-
 *                                vectors by back-substitution on the quasi-triangular factor and
 *                                back-transformation (GVL §7.6.4) (Alg 2 "eig(atilde)" P:314)
 *   O7  orc_modes                Phi = X' T, T = V S^-1 W (complex), compensated (Eq. Phi)
 *   O9  orc_csolve               complex Gaussian elimination with partial pivoting (b = (W L)^-1
 *                                alpha_1, Alg 3)
 *       orc_clstsq               complex Householder QR least squares with column pivoting (the
 *                                "lstsq" of Alg 3 P:330 on the kept modes)
 * Status codes (redefined here, no shared header): 0 OK, 5 no convergence, 6 singular.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_NO_CONVERGENCE 5
#define ORC_SINGULAR 6

/* ------------------------------------------------------------------ Neumaier summation -- */
typedef struct { double s, c; } nsum;

static inline void nadd(nsum* a, double x) {
  const double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
  else a->c += (x - t) + a->s;
  a->s = t;
}
static inline double nval(nsum a) { return a.s + a.c; }

/* product a*b added to the compensated sum: p = fl(a*b) plus its exact rounding error
 * e = a*b - p (fma), which goes into the compensation term */
static inline void nadd_prod(nsum* acc, double a, double b, int exact) {
  const double p = a * b;
  nadd(acc, p);
  if (!exact) acc->c += fma(a, b, -p);
}

static inline double ld_elem(const void* base, int dtype, int64_t i) {
  return dtype == 0 ? (double)((const float*)base)[i] : ((const double*)base)[i];
}

#define ORC_ROWBLK 2048

static int nthreads_of(int threads) {
  if (threads <= 0) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
  }
  return threads;
}

/* O1, streaming form (Alg 1 else-branch P:294 "xtx[:, -1] = X.T * X[:, -1]"):
 * out[i] = <a_i, x> for the ka columns a_i of A (column i at A + i*lda), length n each.
 * threads > 1: the row range is split into `threads` contiguous chunks, each summed in row order
 * with its own compensated accumulator; the chunk sums are then combined in chunk order
 * (compensated).  threads == 1 is the single row-order sum. */
void orc_dots(const void* A, int64_t lda, int ka, const void* x, int64_t n, int dtype, int threads,
              double* out) {
  const int T = nthreads_of(threads);
  const int exact = dtype == 0;
  nsum* part = (nsum*)calloc((size_t)T * (ka > 0 ? ka : 1), sizeof(nsum));
#pragma omp parallel for num_threads(T) schedule(static, 1)
  for (int th = 0; th < T; ++th) {
    const int64_t l0 = n * th / T, l1 = n * (th + 1) / T;
    nsum* acc = part + (size_t)th * ka;
    for (int64_t b0 = l0; b0 < l1; b0 += ORC_ROWBLK) {
      const int64_t b1 = b0 + ORC_ROWBLK < l1 ? b0 + ORC_ROWBLK : l1;
      for (int i = 0; i < ka; ++i) {
        const char* col = (const char*)A + (size_t)i * lda * (dtype == 0 ? 4 : 8);
        for (int64_t l = b0; l < b1; ++l)
          nadd_prod(&acc[i], ld_elem(col, dtype, l), ld_elem(x, dtype, l), exact);
      }
    }
  }
  for (int i = 0; i < ka; ++i) {
    nsum tot = {0.0, 0.0};
    for (int th = 0; th < T; ++th) {
      nadd(&tot, part[(size_t)th * ka + i].s);
      nadd(&tot, part[(size_t)th * ka + i].c);
    }
    out[i] = nval(tot);
  }
  free(part);
}

/* O1, batch form (Alg 1 first branch P:291 "xtx = X.T * X"): G (k x k, row-major) = Z^T Z of the
 * k columns of Z (column j at Z + j*ldz), every entry G_ij (i <= j) a compensated row-order sum,
 * mirrored to G_ji. */
void orc_gram(const void* Z, int64_t ldz, int k, int64_t n, int dtype, int threads, double* G) {
  const int T = nthreads_of(threads);
  const int exact = dtype == 0;
  const size_t np = (size_t)k * (k + 1) / 2;
  nsum* part = (nsum*)calloc((size_t)T * (np > 0 ? np : 1), sizeof(nsum));
  const size_t es = dtype == 0 ? 4 : 8;
#pragma omp parallel for num_threads(T) schedule(static, 1)
  for (int th = 0; th < T; ++th) {
    const int64_t l0 = n * th / T, l1 = n * (th + 1) / T;
    nsum* acc = part + (size_t)th * np;
    for (int64_t b0 = l0; b0 < l1; b0 += ORC_ROWBLK) {
      const int64_t b1 = b0 + ORC_ROWBLK < l1 ? b0 + ORC_ROWBLK : l1;
      size_t q = 0;
      for (int i = 0; i < k; ++i) {
        const char* ci = (const char*)Z + (size_t)i * ldz * es;
        for (int j = i; j < k; ++j, ++q) {
          const char* cj = (const char*)Z + (size_t)j * ldz * es;
          for (int64_t l = b0; l < b1; ++l)
            nadd_prod(&acc[q], ld_elem(ci, dtype, l), ld_elem(cj, dtype, l), exact);
        }
      }
    }
  }
  size_t q = 0;
  for (int i = 0; i < k; ++i)
    for (int j = i; j < k; ++j, ++q) {
      nsum tot = {0.0, 0.0};
      for (int th = 0; th < T; ++th) {
        nadd(&tot, part[(size_t)th * np + q].s);
        nadd(&tot, part[(size_t)th * np + q].c);
      }
      G[(size_t)i * k + j] = G[(size_t)j * k + i] = nval(tot);
    }
  free(part);
}

/* ------------------------------------------------------------- O3 cyclic Jacobi (sym) -- */
/* Eigen-decomposition of the symmetric m x m matrix S (row-major; symmetrised here as
 * (S + S^T)/2) by cyclic-by-row Jacobi (Golub & Van Loan Alg 8.5.3 with the
 * stable rotation of Alg 8.5.1).  A rotation in the (p, q) plane is applied when
 * |s_pq| > eps * sqrt(|s_pp s_qq|) (eps = 2^-52, the relative-accuracy threshold of Demmel &
 * Veselic); the iteration stops after a sweep that applies none (reading R1 in DESIGN.md: the
 * norm test off(S) <= 1e-15 ||S||_F can stall at rounding level for m >= 100).
 * Output: mu (m eigenvalues, unsorted), V (m x m column-major, V[:, j] the eigenvector of mu_j),
 * *sweeps.  Returns ORC_NO_CONVERGENCE after max_sweeps sweeps. */
int orc_jacobi(int m, const double* S_in, double* mu, double* V, int max_sweeps, int* sweeps) {
  double* A = (double*)malloc(sizeof(double) * (size_t)m * m + 8);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) A[(size_t)i * m + j] = 0.5 * (S_in[(size_t)i * m + j] + S_in[(size_t)j * m + i]);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) V[(size_t)i + (size_t)j * m] = i == j ? 1.0 : 0.0;
  const double eps = ldexp(1.0, -52);
  int sw = 0, status = ORC_NO_CONVERGENCE;
  for (sw = 1; sw <= max_sweeps; ++sw) {
    int rotated = 0;
    for (int p = 0; p < m - 1; ++p)
      for (int q = p + 1; q < m; ++q) {
        const double apq = A[(size_t)p * m + q];
        const double app = A[(size_t)p * m + p], aqq = A[(size_t)q * m + q];
        if (apq == 0.0 || fabs(apq) <= eps * sqrt(fabs(app) * fabs(aqq))) continue;
        rotated = 1;
        const double th = (aqq - app) / (2.0 * apq);
        double t;
        if (fabs(th) > 1e150) t = 0.5 / th;                 /* 1/(2 th): sqrt(1+th^2) overflows */
        else t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(1.0 + th * th));
        const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
        /* A <- A J (columns p, q), J = [[c, s], [-s, c]] in the (p, q) plane */
        for (int k = 0; k < m; ++k) {
          const double akp = A[(size_t)k * m + p], akq = A[(size_t)k * m + q];
          A[(size_t)k * m + p] = c * akp - s * akq;
          A[(size_t)k * m + q] = s * akp + c * akq;
        }
        /* A <- J^T A (rows p, q) */
        for (int k = 0; k < m; ++k) {
          const double apk = A[(size_t)p * m + k], aqk = A[(size_t)q * m + k];
          A[(size_t)p * m + k] = c * apk - s * aqk;
          A[(size_t)q * m + k] = s * apk + c * aqk;
        }
        A[(size_t)p * m + q] = A[(size_t)q * m + p] = 0.0;   /* annihilated by construction */
        /* V <- V J */
        for (int k = 0; k < m; ++k) {
          const double vkp = V[(size_t)k + (size_t)p * m], vkq = V[(size_t)k + (size_t)q * m];
          V[(size_t)k + (size_t)p * m] = c * vkp - s * vkq;
          V[(size_t)k + (size_t)q * m] = s * vkp + c * vkq;
        }
      }
    if (!rotated) { status = ORC_OK; break; }
  }
  for (int i = 0; i < m; ++i) mu[i] = A[(size_t)i * m + i];
  if (sweeps) *sweeps = sw;
  free(A);
  return status;
}

/* ------------------------------------------------ O6 real non-symmetric eigenproblem -- */
/* Householder vector (GVL Alg 5.1.1): for x (length len), v with v[0] = 1 and beta such that
 * (I - beta v v^T) x = -sgn(x0) ||x|| e_1.  Returns beta (0 if x is already a multiple of e_1). */
static double house(const double* x, int len, double* v) {
  double sig = 0.0;
  for (int i = 1; i < len; ++i) sig += x[i] * x[i];
  v[0] = 1.0;
  for (int i = 1; i < len; ++i) v[i] = x[i];
  if (sig == 0.0) return 0.0;
  const double mu = sqrt(x[0] * x[0] + sig);
  const double v0 = x[0] <= 0.0 ? x[0] - mu : -sig / (x[0] + mu);
  const double beta = 2.0 * v0 * v0 / (sig + v0 * v0);
  for (int i = 1; i < len; ++i) v[i] /= v0;
  return beta;
}

#define H_(i, j) H[(size_t)(i) * r + (j)]
#define Z_(i, j) Zm[(size_t)(i) * r + (j)]

/* apply the reflector P = I - beta v v^T (v of length len, rows/cols k..k+len-1):
 * H <- P H on rows k.., columns c0..r-1;  H <- H P on columns k.., rows 0..r1;  Z <- Z P. */
static void refl_left(double* H, int r, int k, int len, const double* v, double beta, int c0) {
  for (int j = c0; j < r; ++j) {
    double s = 0.0;
    for (int i = 0; i < len; ++i) s += v[i] * H_(k + i, j);
    s *= beta;
    for (int i = 0; i < len; ++i) H_(k + i, j) -= s * v[i];
  }
}
static void refl_right(double* H, int r, int k, int len, const double* v, double beta, int r1) {
  for (int i = 0; i <= r1; ++i) {
    double s = 0.0;
    for (int j = 0; j < len; ++j) s += H_(i, k + j) * v[j];
    s *= beta;
    for (int j = 0; j < len; ++j) H_(i, k + j) -= s * v[j];
  }
}

/* rotation G = [[c, -s], [s, c]] in the plane (k, k+1): H <- G^T H (rows), H <- H G (cols),
 * Z <- Z G */
static void rot_apply(double* H, double* Zm, int r, int k, double c, double s, int c0, int r1) {
  for (int j = c0; j < r; ++j) {
    const double a = H_(k, j), b = H_(k + 1, j);
    H_(k, j) = c * a + s * b;
    H_(k + 1, j) = -s * a + c * b;
  }
  for (int i = 0; i <= r1; ++i) {
    const double a = H_(i, k), b = H_(i, k + 1);
    H_(i, k) = c * a + s * b;
    H_(i, k + 1) = -s * a + c * b;
  }
  for (int i = 0; i < r; ++i) {
    const double a = Z_(i, k), b = Z_(i, k + 1);
    Z_(i, k) = c * a + s * b;
    Z_(i, k + 1) = -s * a + c * b;
  }
}

typedef struct { double re, im; } cplx;
static inline cplx cmk(double a, double b) { cplx z = {a, b}; return z; }
static inline cplx cadd(cplx a, cplx b) { return cmk(a.re + b.re, a.im + b.im); }
static inline cplx csub(cplx a, cplx b) { return cmk(a.re - b.re, a.im - b.im); }
static inline cplx cmul(cplx a, cplx b) { return cmk(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
static inline double cabs_(cplx a) { return hypot(a.re, a.im); }
static inline cplx cdiv(cplx a, cplx b) {            /* Smith's algorithm */
  if (fabs(b.re) >= fabs(b.im)) {
    const double q = b.im / b.re, d = b.re + b.im * q;
    return cmk((a.re + a.im * q) / d, (a.im - a.re * q) / d);
  }
  const double q = b.re / b.im, d = b.im + b.re * q;
  return cmk((a.re * q + a.im) / d, (a.im * q - a.re) / d);
}

/* Eigenvalues and right eigenvectors of the real r x r matrix A (row-major).
 * Steps (Golub & Van Loan): (1) H = Q^T A Q upper Hessenberg by Householder reflectors, Q
 * accumulated (Alg 7.4.2); (2) Francis double-shift QR steps on the active unreduced block with
 * deflation when |h_{l,l-1}| <= u (|h_{l-1,l-1}| + |h_{l,l}|), exceptional shifts after 10 and 20
 * iterations without deflation, every transform applied to the whole matrix and accumulated into
 * Z = Q ... (Alg 7.5.1/7.5.2) -> real Schur form T = Z^T A Z; a deflated 2x2 block with real
 * eigenvalues is split by one rotation whose first column is its eigenvector; (3) for each
 * eigenvalue lam_k, y solving (T - lam_k I) y = 0 with y_j = 0 below its block, by block
 * back-substitution in complex arithmetic; w_k = Z y (GVL §7.6.4).
 * Output: wr, wi (eigenvalues in Schur-form order), Wre, Wim (r x r column-major, unnormalised
 * right eigenvectors), *its (QR iterations).  Budget 100 r iterations, else ORC_NO_CONVERGENCE. */
int orc_eig_real(int r, const double* A, double* wr, double* wi, double* Wre, double* Wim, int* its_out) {
  double* H = (double*)malloc(sizeof(double) * (size_t)r * r + 8);
  double* Zm = (double*)malloc(sizeof(double) * (size_t)r * r + 8);
  double* v = (double*)malloc(sizeof(double) * (size_t)(r + 3));
  double* x = (double*)malloc(sizeof(double) * (size_t)(r + 3));
  int* blk = (int*)malloc(sizeof(int) * (size_t)(r + 1));    /* 1: 1x1 block start, 2: 2x2 block start, 0: second row of a 2x2 */
  memcpy(H, A, sizeof(double) * (size_t)r * r);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) Z_(i, j) = i == j ? 1.0 : 0.0;
  /* (1) Hessenberg reduction */
  for (int k = 0; k + 2 < r; ++k) {
    const int len = r - k - 1;
    for (int i = 0; i < len; ++i) x[i] = H_(k + 1 + i, k);
    const double beta = house(x, len, v);
    if (beta == 0.0) continue;
    refl_left(H, r, k + 1, len, v, beta, k);
    refl_right(H, r, k + 1, len, v, beta, r - 1);
    /* Z <- Z P */
    for (int i = 0; i < r; ++i) {
      double s = 0.0;
      for (int j = 0; j < len; ++j) s += Z_(i, k + 1 + j) * v[j];
      s *= beta;
      for (int j = 0; j < len; ++j) Z_(i, k + 1 + j) -= s * v[j];
    }
    for (int i = k + 2; i < r; ++i) H_(i, k) = 0.0;
  }
  /* (2) Francis double-shift QR */
  const double u = ldexp(1.0, -53);
  int hi = r - 1, its = 0, since = 0, status = ORC_OK;
  const int budget = 100 * (r > 0 ? r : 1);
  for (int i = 0; i <= r; ++i) blk[i] = 1;
  while (hi >= 0) {
    int l = hi;
    while (l > 0) {
      const double s = fabs(H_(l - 1, l - 1)) + fabs(H_(l, l));
      if (fabs(H_(l, l - 1)) <= u * s || H_(l, l - 1) == 0.0) { H_(l, l - 1) = 0.0; break; }
      --l;
    }
    if (l == hi) {                                   /* 1x1 block */
      wr[hi] = H_(hi, hi); wi[hi] = 0.0; blk[hi] = 1;
      --hi; since = 0;
      continue;
    }
    if (l == hi - 1) {                               /* 2x2 block */
      const double a = H_(hi - 1, hi - 1), b = H_(hi - 1, hi), c = H_(hi, hi - 1), d = H_(hi, hi);
      const double p = 0.5 * (a - d), q = p * p + b * c;
      if (q >= 0.0) {                                /* real pair: split by a rotation */
        const double zz = p + (p >= 0.0 ? sqrt(q) : -sqrt(q));
        const double lam = d + zz;                   /* one eigenvalue of the block */
        /* eigenvector of [[a,b],[c,d]] for lam: (b, lam - a) or (lam - d, c) */
        double e0 = b, e1 = lam - a;
        const double f0 = lam - d, f1 = c;
        if (hypot(f0, f1) > hypot(e0, e1)) { e0 = f0; e1 = f1; }
        const double nr = hypot(e0, e1);
        double cs = 1.0, sn = 0.0;
        if (nr > 0.0) { cs = e0 / nr; sn = e1 / nr; }
        rot_apply(H, Zm, r, hi - 1, cs, sn, hi - 1, hi);
        H_(hi, hi - 1) = 0.0;
        wr[hi - 1] = H_(hi - 1, hi - 1); wi[hi - 1] = 0.0;
        wr[hi] = H_(hi, hi); wi[hi] = 0.0;
        blk[hi - 1] = 1; blk[hi] = 1;
      } else {
        const double re = 0.5 * (a + d), im = sqrt(-q);
        wr[hi - 1] = re; wi[hi - 1] = im;
        wr[hi] = re; wi[hi] = -im;
        blk[hi - 1] = 2; blk[hi] = 0;
      }
      hi -= 2; since = 0;
      continue;
    }
    if (its >= budget) { status = ORC_NO_CONVERGENCE; break; }
    ++its; ++since;
    /* shifts: eigenvalues of the trailing 2x2 (s = trace, t = det), exceptional after 10/20 */
    double s, t;
    if (since == 10 || since == 20) {
      /* exceptional shift pair: the conjugate pair (h_hh + e) +- i e, e the size of the two
         trailing subdiagonal entries (breaks a cycle of the standard shift) */
      const double e = fabs(H_(hi, hi - 1)) + fabs(H_(hi - 1, hi - 2));
      const double c0 = H_(hi, hi) + e;
      s = 2.0 * c0;
      t = c0 * c0 + e * e;
    } else {
      s = H_(hi - 1, hi - 1) + H_(hi, hi);
      t = H_(hi - 1, hi - 1) * H_(hi, hi) - H_(hi - 1, hi) * H_(hi, hi - 1);
    }
    /* first column of (H - s1 I)(H - s2 I) = H^2 - s H + t I on the active block [l, hi] */
    double xx = H_(l, l) * H_(l, l) + H_(l, l + 1) * H_(l + 1, l) - s * H_(l, l) + t;
    double yy = H_(l + 1, l) * (H_(l, l) + H_(l + 1, l + 1) - s);
    double zz = (l + 2 <= hi) ? H_(l + 1, l) * H_(l + 2, l + 1) : 0.0;
    for (int k = l; k <= hi - 2; ++k) {
      double xv[3] = {xx, yy, zz};
      const double beta = house(xv, 3, v);
      if (beta != 0.0) {
        refl_left(H, r, k, 3, v, beta, k > l ? k - 1 : l);
        const int r1 = k + 3 < hi ? k + 3 : hi;
        refl_right(H, r, k, 3, v, beta, r1);
        for (int i = 0; i < r; ++i) {
          double sm = 0.0;
          for (int j = 0; j < 3; ++j) sm += Z_(i, k + j) * v[j];
          sm *= beta;
          for (int j = 0; j < 3; ++j) Z_(i, k + j) -= sm * v[j];
        }
      }
      /* rows above the active block also belong to T: refl_right covered rows 0..r1 */
      xx = H_(k + 1, k);
      yy = H_(k + 2, k);
      zz = (k + 3 <= hi) ? H_(k + 3, k) : 0.0;
      if (k > l) H_(k + 1, k - 1) = 0.0, H_(k + 2, k - 1) = 0.0;
    }
    /* final 2x2 Givens on (hi-1, hi) for (xx, yy) */
    {
      double xv[2] = {xx, yy};
      const double beta = house(xv, 2, v);
      if (beta != 0.0) {
        const int k = hi - 1;
        refl_left(H, r, k, 2, v, beta, k - 1 >= l ? k - 1 : l);
        refl_right(H, r, k, 2, v, beta, hi);
        for (int i = 0; i < r; ++i) {
          double sm = Z_(i, k) * v[0] + Z_(i, k + 1) * v[1];
          sm *= beta;
          Z_(i, k) -= sm * v[0];
          Z_(i, k + 1) -= sm * v[1];
        }
      }
      if (hi - 2 >= l) H_(hi, hi - 2) = 0.0;
    }
  }
  if (its_out) *its_out = its;
  if (status != ORC_OK) {
    free(H); free(Zm); free(v); free(x); free(blk);
    return status;
  }
  /* (3) eigenvectors of T by back-substitution, then W = Z y */
  double tnorm = 0.0;
  for (int i = 0; i < r; ++i)
    for (int j = (i > 0 ? i - 1 : 0); j < r; ++j) tnorm = fmax(tnorm, fabs(H_(i, j)));
  const double smin = fmax(tnorm * ldexp(1.0, -52), 1e-300);
  cplx* y = (cplx*)malloc(sizeof(cplx) * (size_t)(r + 1));
  for (int k = 0; k < r; ++k) {
    const cplx lam = cmk(wr[k], wi[k]);
    for (int i = 0; i < r; ++i) y[i] = cmk(0.0, 0.0);
    int top;                                         /* first row of this eigenvalue's block */
    if (wi[k] == 0.0) {
      y[k] = cmk(1.0, 0.0);
      top = k;
    } else {
      const int k0 = wi[k] > 0.0 ? k : k - 1;        /* block rows k0, k0+1 */
      const double a = H_(k0, k0), b = H_(k0, k0 + 1), c = H_(k0 + 1, k0), d = H_(k0 + 1, k0 + 1);
      /* (T_blk - lam I) y = 0: y = (b, lam - a) or (lam - d, c) */
      cplx e0 = cmk(b, 0.0), e1 = csub(lam, cmk(a, 0.0));
      const cplx f0 = csub(lam, cmk(d, 0.0)), f1 = cmk(c, 0.0);
      if (cabs_(f0) + cabs_(f1) > cabs_(e0) + cabs_(e1)) { e0 = f0; e1 = f1; }
      y[k0] = e0;
      y[k0 + 1] = e1;
      top = k0;
    }
    /* block back-substitution for rows top-1 .. 0 */
    int i = top - 1;
    while (i >= 0) {
      if (i >= 1 && blk[i - 1] == 2) {               /* 2x2 block rows i-1, i */
        const int i0 = i - 1;
        cplx r0 = cmk(0.0, 0.0), r1 = cmk(0.0, 0.0);
        for (int j = i + 1; j < r; ++j) {
          r0 = csub(r0, cmul(cmk(H_(i0, j), 0.0), y[j]));
          r1 = csub(r1, cmul(cmk(H_(i, j), 0.0), y[j]));
        }
        const cplx m00 = csub(cmk(H_(i0, i0), 0.0), lam), m01 = cmk(H_(i0, i), 0.0);
        const cplx m10 = cmk(H_(i, i0), 0.0), m11 = csub(cmk(H_(i, i), 0.0), lam);
        cplx det = csub(cmul(m00, m11), cmul(m01, m10));
        if (cabs_(det) < smin * smin) det = cmk(smin * smin, 0.0);
        y[i0] = cdiv(csub(cmul(m11, r0), cmul(m01, r1)), det);
        y[i] = cdiv(csub(cmul(m00, r1), cmul(m10, r0)), det);
        i -= 2;
      } else {                                       /* 1x1 block */
        cplx rr = cmk(0.0, 0.0);
        for (int j = i + 1; j < r; ++j) rr = csub(rr, cmul(cmk(H_(i, j), 0.0), y[j]));
        cplx dd = csub(cmk(H_(i, i), 0.0), lam);
        if (cabs_(dd) < smin) dd = cmk(smin, 0.0);
        y[i] = cdiv(rr, dd);
        i -= 1;
      }
      /* rescale against overflow (the vector is normalised by the caller) */
      double mx = 0.0;
      for (int j = 0; j < r; ++j) mx = fmax(mx, cabs_(y[j]));
      if (mx > 1e100)
        for (int j = 0; j < r; ++j) y[j] = cmk(y[j].re / mx, y[j].im / mx);
    }
    /* w_k = Z y */
    for (int row = 0; row < r; ++row) {
      double sr = 0.0, si = 0.0;
      for (int j = 0; j < r; ++j) { sr += Z_(row, j) * y[j].re; si += Z_(row, j) * y[j].im; }
      Wre[(size_t)row + (size_t)k * r] = sr;
      Wim[(size_t)row + (size_t)k * r] = si;
    }
  }
  free(y); free(H); free(Zm); free(v); free(x); free(blk);
  return ORC_OK;
}
#undef H_
#undef Z_

/* ------------------------------------------------------------- O9 complex linear algebra -- */
/* x = A^-1 b for complex A (r x r, column-major, interleaved re/im) by Gaussian elimination with
 * partial pivoting (GVL Alg 3.4.1).  Returns ORC_SINGULAR if a pivot has modulus
 * <= r * u * max|a_ij| (x is then undefined). */
int orc_csolve(int r, const double* A_in, const double* b_in, double* x_out) {
  cplx* A = (cplx*)malloc(sizeof(cplx) * (size_t)r * r + 16);
  cplx* b = (cplx*)malloc(sizeof(cplx) * (size_t)r + 16);
  double amax = 0.0;
  for (int j = 0; j < r; ++j)
    for (int i = 0; i < r; ++i) {
      A[(size_t)i + (size_t)j * r] = cmk(A_in[2 * ((size_t)i + (size_t)j * r)], A_in[2 * ((size_t)i + (size_t)j * r) + 1]);
      amax = fmax(amax, cabs_(A[(size_t)i + (size_t)j * r]));
    }
  for (int i = 0; i < r; ++i) b[i] = cmk(b_in[2 * i], b_in[2 * i + 1]);
  const double tol = (double)r * ldexp(1.0, -53) * amax;
  int status = ORC_OK;
  for (int k = 0; k < r; ++k) {
    int p = k;
    for (int i = k + 1; i < r; ++i)
      if (cabs_(A[(size_t)i + (size_t)k * r]) > cabs_(A[(size_t)p + (size_t)k * r])) p = i;
    if (!(cabs_(A[(size_t)p + (size_t)k * r]) > tol)) { status = ORC_SINGULAR; break; }
    if (p != k) {
      for (int j = 0; j < r; ++j) {
        const cplx t = A[(size_t)k + (size_t)j * r];
        A[(size_t)k + (size_t)j * r] = A[(size_t)p + (size_t)j * r];
        A[(size_t)p + (size_t)j * r] = t;
      }
      const cplx t = b[k]; b[k] = b[p]; b[p] = t;
    }
    for (int i = k + 1; i < r; ++i) {
      const cplx l = cdiv(A[(size_t)i + (size_t)k * r], A[(size_t)k + (size_t)k * r]);
      for (int j = k + 1; j < r; ++j)
        A[(size_t)i + (size_t)j * r] = csub(A[(size_t)i + (size_t)j * r], cmul(l, A[(size_t)k + (size_t)j * r]));
      b[i] = csub(b[i], cmul(l, b[k]));
    }
  }
  if (status == ORC_OK)
    for (int i = r - 1; i >= 0; --i) {
      cplx s = b[i];
      for (int j = i + 1; j < r; ++j) s = csub(s, cmul(A[(size_t)i + (size_t)j * r], cmk(x_out[2 * j], x_out[2 * j + 1])));
      const cplx xi = cdiv(s, A[(size_t)i + (size_t)i * r]);
      x_out[2 * i] = xi.re;
      x_out[2 * i + 1] = xi.im;
    }
  free(A); free(b);
  return status;
}

/* Least squares min ||A x - b|| for complex A (rows x cols, column-major interleaved) by
 * Householder QR with column pivoting (GVL Alg 5.4.1, complex reflectors).  Columns beyond the
 * numerical rank (|R_kk| <= max(rows,cols) * u * |R_00|) get x = 0 (the basic solution).
 * Returns the numerical rank. */
int orc_clstsq(int rows, int cols, const double* A_in, const double* b_in, double* x_out) {
  cplx* A = (cplx*)malloc(sizeof(cplx) * (size_t)rows * cols + 16);
  cplx* b = (cplx*)malloc(sizeof(cplx) * (size_t)rows + 16);
  cplx* v = (cplx*)malloc(sizeof(cplx) * (size_t)rows + 16);
  int* perm = (int*)malloc(sizeof(int) * (size_t)cols + 4);
  double* cn = (double*)malloc(sizeof(double) * (size_t)cols + 8);
  for (int j = 0; j < cols; ++j)
    for (int i = 0; i < rows; ++i)
      A[(size_t)i + (size_t)j * rows] = cmk(A_in[2 * ((size_t)i + (size_t)j * rows)], A_in[2 * ((size_t)i + (size_t)j * rows) + 1]);
  for (int i = 0; i < rows; ++i) b[i] = cmk(b_in[2 * i], b_in[2 * i + 1]);
  for (int j = 0; j < cols; ++j) perm[j] = j;
  const int kmax = rows < cols ? rows : cols;
  int rank = 0;
  double r00 = 0.0;
  const double u = ldexp(1.0, -53);
  for (int k = 0; k < kmax; ++k) {
    /* pivot: the remaining column of largest norm (rows k..) */
    int p = k;
    double best = -1.0;
    for (int j = k; j < cols; ++j) {
      double s = 0.0;
      for (int i = k; i < rows; ++i) { const cplx a = A[(size_t)i + (size_t)j * rows]; s += a.re * a.re + a.im * a.im; }
      cn[j] = sqrt(s);
      if (cn[j] > best) { best = cn[j]; p = j; }
    }
    if (p != k) {
      for (int i = 0; i < rows; ++i) {
        const cplx t = A[(size_t)i + (size_t)k * rows];
        A[(size_t)i + (size_t)k * rows] = A[(size_t)i + (size_t)p * rows];
        A[(size_t)i + (size_t)p * rows] = t;
      }
      const int t = perm[k]; perm[k] = perm[p]; perm[p] = t;
    }
    const double nrm = best;
    if (k == 0) r00 = nrm;
    if (!(nrm > (double)(rows > cols ? rows : cols) * u * r00) || nrm == 0.0) break;
    /* complex Householder: v = x + e^{i arg x0} ||x|| e_1, H = I - 2 v v^H / (v^H v) */
    const cplx x0 = A[(size_t)k + (size_t)k * rows];
    const double ax0 = cabs_(x0);
    const cplx ph = ax0 > 0.0 ? cmk(x0.re / ax0, x0.im / ax0) : cmk(1.0, 0.0);
    for (int i = k; i < rows; ++i) v[i] = A[(size_t)i + (size_t)k * rows];
    v[k] = cadd(v[k], cmk(ph.re * nrm, ph.im * nrm));
    double vv = 0.0;
    for (int i = k; i < rows; ++i) vv += v[i].re * v[i].re + v[i].im * v[i].im;
    for (int j = k; j < cols; ++j) {                /* A[:, j] -= v (2 v^H a / vv) */
      cplx s = cmk(0.0, 0.0);
      for (int i = k; i < rows; ++i) s = cadd(s, cmul(cmk(v[i].re, -v[i].im), A[(size_t)i + (size_t)j * rows]));
      s = cmk(2.0 * s.re / vv, 2.0 * s.im / vv);
      for (int i = k; i < rows; ++i) A[(size_t)i + (size_t)j * rows] = csub(A[(size_t)i + (size_t)j * rows], cmul(v[i], s));
    }
    {
      cplx s = cmk(0.0, 0.0);
      for (int i = k; i < rows; ++i) s = cadd(s, cmul(cmk(v[i].re, -v[i].im), b[i]));
      s = cmk(2.0 * s.re / vv, 2.0 * s.im / vv);
      for (int i = k; i < rows; ++i) b[i] = csub(b[i], cmul(v[i], s));
    }
    rank = k + 1;
  }
  /* back-substitution R[0:rank,0:rank] z = (Q^H b)[0:rank]; x[perm] = z, the rest 0 */
  cplx* z = (cplx*)calloc((size_t)cols + 1, sizeof(cplx));
  for (int i = rank - 1; i >= 0; --i) {
    cplx s = b[i];
    for (int j = i + 1; j < rank; ++j) s = csub(s, cmul(A[(size_t)i + (size_t)j * rows], z[j]));
    z[i] = cdiv(s, A[(size_t)i + (size_t)i * rows]);
  }
  for (int j = 0; j < cols; ++j) { x_out[2 * j] = 0.0; x_out[2 * j + 1] = 0.0; }
  for (int j = 0; j < rank; ++j) { x_out[2 * perm[j]] = z[j].re; x_out[2 * perm[j] + 1] = z[j].im; }
  free(z); free(A); free(b); free(v); free(perm); free(cn);
  return rank;
}

/* ----------------------------------------------------------------------- O7 modes ------ */
/* Phi (n x nc complex, column-major interleaved, column j at Phi + 2*j*ldp) = X' T with X' the m
 * real columns (column k at X + k*ldx, dtype 0 f32 / 1 f64) and T (m x nc complex, column-major
 * interleaved): Phi[l, j] = sum_k X'[l, k] T[k, j], real and imaginary parts each a compensated
 * sum over k in increasing order ("vsiw = vsi * w; phi = X[:, 1:] * vsiw", Alg 2). */
void orc_modes(const void* X, int64_t ldx, int m, int64_t n, int dtype, const double* T, int nc,
               double* Phi, int64_t ldp, int threads) {
  const int TT = nthreads_of(threads);
  const size_t es = dtype == 0 ? 4 : 8;
#pragma omp parallel for num_threads(TT) schedule(static)
  for (int64_t l = 0; l < n; ++l) {
    for (int j = 0; j < nc; ++j) {
      nsum sr = {0.0, 0.0}, si = {0.0, 0.0};
      for (int k = 0; k < m; ++k) {
        const double xv = ld_elem((const char*)X + (size_t)k * ldx * es, dtype, l);
        const double tr = T[2 * ((size_t)k + (size_t)j * m)], ti = T[2 * ((size_t)k + (size_t)j * m) + 1];
        nadd_prod(&sr, xv, tr, 0);
        nadd_prod(&si, xv, ti, 0);
      }
      Phi[2 * ((size_t)l + (size_t)j * ldp)] = nval(sr);
      Phi[2 * ((size_t)l + (size_t)j * ldp) + 1] = nval(si);
    }
  }
}

int orc_abi(void) { return 1; }
