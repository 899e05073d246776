// k6_background.cu — background outputs beyond the fused per-frame column of K1:
//   * NEXT-3 pixel-space background of a sparse-DCT context,
//   * Alg 3's first-window branch (all m+1 columns of the newest DMD window, reading Q24),
//   * NEXT-4 mask scoring.
//
// Pixel-space background (SURVEY §8(f) NEXT-3 "an inverse-DCT kernel for pixel-space background";
// P:357-360 "transfer the compressed DMD from the GPU back"): the window lives as sparse orthonormal
// DCT-II coefficient vectors (K3), so Alg 3's streaming branch is evaluated as
//   l̂ = X̂' c  (c = b_idx λ_idx^m V Σ⁻¹ w_idx, the m complex coefficients K4b writes, Q4),
//   l = IDCT2(l̂) (real transform applied to Re and Im),  x = IDCT2(x̂_newest),
//   s = x − |l|,  mask = s > threshold                       (Q8; the paper's ".2")
// in three steps:
//   (1) pix_lincomb_kernel: each CTA owns 1024 consecutive coefficient indices; for k = 0..m-1 IN
//       ORDER it adds c_k · val over the nonzeros of window column k that fall in its range
//       (indices are unique within a column, a CTA barrier separates columns, so every element is
//       a fixed-order fma chain); the newest column is also copied out as x̂.  Output: 3 dense
//       planes (Re l̂, Im l̂, x̂) of grid_rows x grid_cols.
//   (2) idct_lines_kernel (twice: along rows, then along columns): the orthonormal DCT-III of
//       length N by Makhoul's N-point complex FFT, two real lines packed into one complex FFT
//       (V = V_a + i V_b, both Hermitian, so the inverse DFT returns line a in Re and line b in
//       Im).  One CTA per line pair; radix-2 DIT in shared memory with an exact twiddle table.
//   (3) pix_epilogue_kernel: |l|, s, mask per pixel (fp64).
// Each plane is 8 MB at 1024² — the whole pipeline is L2-resident (126 MB).
//
// Scoring (NEXT-4; Table 2, reading Q26): TP/FP/FN of the mask against
// a ground-truth mask, block-reduced and added to device counters (pooled over frames).
#include "sdmd_internal.cuh"

namespace sdmd {

constexpr int PIX_R = 1024;        // coefficient indices per lincomb CTA (3 fp64 planes: 24 KB smem)
constexpr int PIX_THREADS = 256;
constexpr int PIX_PER_T = PIX_R / PIX_THREADS;

__global__ void __launch_bounds__(PIX_THREADS) pix_lincomb_kernel(const PixBgParams p) {
  if (*(volatile int*)&p.st->status != 0) return;
  __shared__ double acc_re[PIX_R];
  __shared__ double acc_im[PIX_R];
  __shared__ double acc_x[PIX_R];
  __shared__ int lo[kMaxM], hi[kMaxM];
  const long long n = (long long)p.rows * p.cols;
  const long long a = (long long)blockIdx.x * PIX_R;
  const int tid = threadIdx.x;
  const long long f0 = p.f_bg - p.m + 1;
  for (int k = tid; k < p.m; k += PIX_THREADS) {       // this CTA's slice of each column
    const int slot = (int)((f0 + k) % p.NS);
    const int nz = p.nnz[slot];
    const int* ix = p.idx + (long long)slot * p.nnz_cap;
    int l = 0, h = nz > 0 ? nz : 0;
    while (l < h) { const int md = (l + h) >> 1; if (ix[md] < a) l = md + 1; else h = md; }
    const int lo_k = l;
    h = nz > 0 ? nz : 0;
    while (l < h) { const int md = (l + h) >> 1; if (ix[md] < a + PIX_R) l = md + 1; else h = md; }
    lo[k] = lo_k;
    hi[k] = l;
  }
  for (int i = tid; i < PIX_R; i += PIX_THREADS) { acc_re[i] = 0.0; acc_im[i] = 0.0; acc_x[i] = 0.0; }
  __syncthreads();
  // software pipeline: the nonzeros of column k+1 are loaded into registers while column k is
  // accumulated (the loads do not depend on the accumulation order, only the adds do)
  int ci[PIX_PER_T], ni[PIX_PER_T];
  double cv[PIX_PER_T], nv[PIX_PER_T];
  auto load = [&](int k, int* ii, double* vv) {
    const int slot = (int)((f0 + k) % p.NS);
    const int* ix = p.idx + (long long)slot * p.nnz_cap;
    const double* vx = p.val + (long long)slot * p.nnz_cap;
#pragma unroll
    for (int j = 0; j < PIX_PER_T; ++j) {
      const int e = lo[k] + tid + j * PIX_THREADS;
      if (e < hi[k]) { ii[j] = (int)(ix[e] - a); vv[j] = vx[e]; } else { ii[j] = -1; vv[j] = 0.0; }
    }
  };
  load(0, ci, cv);
  for (int k = 0; k < p.m; ++k) {
    if (k + 1 < p.m) load(k + 1, ni, nv);
    const double2 c = p.c[k];
    const bool newest = (k == p.m - 1);
#pragma unroll
    for (int j = 0; j < PIX_PER_T; ++j) {
      if (ci[j] >= 0) {
        acc_re[ci[j]] = fma(cv[j], c.x, acc_re[ci[j]]);
        acc_im[ci[j]] = fma(cv[j], c.y, acc_im[ci[j]]);
        if (newest) acc_x[ci[j]] = cv[j];
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < PIX_PER_T; ++j) { ci[j] = ni[j]; cv[j] = nv[j]; }
  }
  for (int i = tid; i < PIX_R; i += PIX_THREADS) {
    const long long g = a + i;
    if (g < n) {
      p.planes[g] = acc_re[i];
      p.planes[n + g] = acc_im[i];
      p.planes[2 * n + g] = acc_x[i];
    }
  }
}

// Orthonormal DCT-III (inverse DCT-II) of two real lines a, b of length N = 2^logN at once.
// Makhoul: y_k = X_k / w_k (w_0 = √(1/N), w_k = √(2/N)), V_k = e^{iπk/2N} (y_k − i y_{N−k}),
// V_0 = y_0; v = IDFT(V) (1/N folded into the input scale); x_{2n} = v_n, x_{2n+1} = v_{N−1−n}.
// Lines: line l = plane (l / lpp), index r = l % lpp; element e of it at
// base + plane·pe + r·ls + e·es (same geometry for in and out).
__global__ void __launch_bounds__(256) idct_lines_kernel(const double* __restrict__ in,
                                                         double* __restrict__ out, int logN, int lpp,
                                                         long long pe, long long ls, long long es,
                                                         const DevState* st) {
  if (*(volatile const int*)&st->status != 0) return;
  extern __shared__ double2 sm[];
  const int N = 1 << logN;
  double2* d = sm;                 // N
  double2* tw = sm + N;            // N/2: e^{+2πi j/N}
  const int la = 2 * blockIdx.x, lb = la + 1;
  const long long ba = (long long)(la / lpp) * pe + (long long)(la % lpp) * ls;
  const long long bb = (long long)(lb / lpp) * pe + (long long)(lb % lpp) * ls;
  for (int j = threadIdx.x; j < N / 2; j += blockDim.x) {
    double sn, cs;
    sincospi(2.0 * j / N, &sn, &cs);
    tw[j] = make_double2(cs, sn);
  }
  const double s0 = rsqrt((double)N), s1 = rsqrt(2.0 * N);       // (1/w_k)/N
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const double ya = in[ba + k * es] * (k == 0 ? s0 : s1);
    const double yb = in[bb + k * es] * (k == 0 ? s0 : s1);
    double2 V;
    if (k == 0) {
      V = make_double2(ya, yb);                                    // V_a + i V_b, both real
    } else {
      const double yan = in[ba + (N - k) * es] * s1;
      const double ybn = in[bb + (N - k) * es] * s1;
      double sn, cs;
      sincospi((double)k / (2.0 * N), &sn, &cs);
      // V_a = (cs + i sn)(ya − i yan),  V_b likewise;  V = V_a + i V_b
      const double ar = fma(cs, ya, sn * yan), ai = fma(sn, ya, -cs * yan);
      const double br = fma(cs, yb, sn * ybn), bi = fma(sn, yb, -cs * ybn);
      V = make_double2(ar - bi, ai + br);
    }
    d[__brev((unsigned)k) >> (32 - logN)] = V;
  }
  __syncthreads();
  for (int s = 1; s <= logN; ++s) {
    const int half = 1 << (s - 1);
    const int tstep = N >> s;
    for (int b = threadIdx.x; b < N / 2; b += blockDim.x) {
      const int j = b & (half - 1);
      const int i0 = ((b >> (s - 1)) << s) + j, i1 = i0 + half;
      const double2 w = tw[j * tstep];
      const double2 u = d[i0], v = d[i1];
      const double tr = fma(w.x, v.x, -w.y * v.y), ti = fma(w.x, v.y, w.y * v.x);
      d[i0] = make_double2(u.x + tr, u.y + ti);
      d[i1] = make_double2(u.x - tr, u.y - ti);
    }
    __syncthreads();
  }
  for (int q = threadIdx.x; q < N; q += blockDim.x) {
    const int src = (q & 1) ? N - ((q + 1) >> 1) : (q >> 1);
    const double2 v = d[src];
    out[ba + q * es] = v.x;
    out[bb + q * es] = v.y;
  }
}

__global__ void __launch_bounds__(256) pix_epilogue_kernel(const PixBgParams p) {
  if (*(volatile int*)&p.st->status != 0) return;
  const long long n = (long long)p.rows * p.cols;
  const double thr = (double)p.thr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double lr = p.planes[i], li = p.planes[n + i], x = p.planes[2 * n + i];
    const double low = hypot(lr, li);
    const double s = x - low;
    p.lowrank[i] = low;
    p.sparse[i] = s;
    p.mask[i] = s > thr ? 1 : 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) p.st->bg_frame = p.f_bg;
}

static int ilog2(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return l;
}

cudaError_t launch_pixel_background(const PixBgParams& p, cudaStream_t s) {
  const long long n = (long long)p.rows * p.cols;
  const int g1 = (int)((n + PIX_R - 1) / PIX_R);
  pix_lincomb_kernel<<<g1, PIX_THREADS, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // rows: 3 planes x rows lines of length cols (contiguous); columns: 3 x cols lines of length rows
  const int lr = ilog2(p.cols), lc = ilog2(p.rows);
  size_t sm_r = (size_t)(p.cols + p.cols / 2) * sizeof(double2);
  size_t sm_c = (size_t)(p.rows + p.rows / 2) * sizeof(double2);
  const size_t smax = sm_r > sm_c ? sm_r : sm_c;
  if (smax > 48 * 1024) {
    e = set_max_dyn_smem((const void*)idct_lines_kernel, (int)smax);
    if (e != cudaSuccess) return e;
  }
  idct_lines_kernel<<<3 * p.rows / 2, 256, sm_r, s>>>(p.planes, p.tmp, lr, p.rows, n, p.cols, 1, p.st);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  idct_lines_kernel<<<3 * p.cols / 2, 256, sm_c, s>>>(p.tmp, p.planes, lc, p.cols, n, 1, p.cols, p.st);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  pix_epilogue_kernel<<<4 * 148, 256, 0, s>>>(p);
  return cudaGetLastError();
}

// ------------------------------------------------ Alg 3 first-window branch (Q24) --------
// l_e = b_idx φ_idx λ_idx^e for e = 0..m over the window columns z_e ("lambdaPow =
// pow(lambda[idx], [0:X.shape[1]])", "s = X - abs(l)"), for the newest DMD frame f.  Its stored
// background coefficients c_f = b_idx λ^m V Σ⁻¹ w_idx (K4b, the same vector the streaming branch
// uses) give X'c_f = b_idx φ_idx λ^m, so l_e = λ^{e-m} · (X'c_f): one fp64 complex accumulation
// per row over the m columns of X', then m+1 scaled outputs.  λ^{e-m} = (1/λ)^{m-e} by binary
// powering (|λ_idx| is the eigenvalue nearest the unit circle, Q5).  Columns are read coalesced
// (consecutive rows per thread); outputs column-major with leading dimension ldo.
template <typename T>
__global__ void __launch_bounds__(256) window_bg_kernel(const T* __restrict__ ring, long long ld, int NS,
                                                        long long n, long long f, int m,
                                                        const double2* __restrict__ cf,
                                                        const K4Result* __restrict__ res,
                                                        T* __restrict__ low, T* __restrict__ sparse,
                                                        unsigned char* __restrict__ mask, long long ldo,
                                                        float thr) {
  __shared__ double2 c[kMaxM];
  __shared__ double2 pw[kMaxM + 1];
  const double2 lam = make_double2(res->lam_idx[0], res->lam_idx[1]);
  for (int k = threadIdx.x; k < m; k += blockDim.x) c[k] = cf[k];
  for (int e = threadIdx.x; e <= m; e += blockDim.x) {
    const double d = lam.x * lam.x + lam.y * lam.y;
    double2 base = make_double2(lam.x / d, -lam.y / d), q = make_double2(1.0, 0.0);
    for (int k = m - e; k > 0; k >>= 1) {
      if (k & 1) q = make_double2(q.x * base.x - q.y * base.y, q.x * base.y + q.y * base.x);
      base = make_double2(base.x * base.x - base.y * base.y, 2.0 * base.x * base.y);
    }
    pw[e] = q;
  }
  __syncthreads();
  const long long f0 = f - m;                           // frame of window column 0
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double ax = 0.0, ay = 0.0;
    for (int k = 0; k < m; ++k) {                       // X' column k = frame f0 + 1 + k
      const double x = (double)__ldg(ring + ((f0 + 1 + k) % NS) * ld + i);
      ax = fma(c[k].x, x, ax);
      ay = fma(c[k].y, x, ay);
    }
    for (int e = 0; e <= m; ++e) {
      const double z = (double)__ldg(ring + ((f0 + e) % NS) * ld + i);
      const double lx = pw[e].x * ax - pw[e].y * ay, ly = pw[e].x * ay + pw[e].y * ax;
      const double l = sqrt(lx * lx + ly * ly);          // |l| (Q8)
      const double sv = z - l;                           // s = x - |l|
      if (low) low[e * ldo + i] = (T)l;
      if (sparse) sparse[e * ldo + i] = (T)sv;
      if (mask) mask[e * ldo + i] = (sv > (double)thr) ? 1 : 0;
    }
  }
}

cudaError_t launch_window_background(const void* ring, long long ld, int NS, int dtype, long long n,
                                     long long f, int m, const double2* cf, const K4Result* res,
                                     void* low, void* sparse, unsigned char* mask, long long ldo,
                                     float thr, cudaStream_t s) {
  long long blocks = (n + 255) / 256;
  if (blocks > 8 * 148) blocks = 8 * 148;
  if (dtype == 0)
    window_bg_kernel<float><<<(int)blocks, 256, 0, s>>>((const float*)ring, ld, NS, n, f, m, cf, res,
                                                        (float*)low, (float*)sparse, mask, ldo, thr);
  else
    window_bg_kernel<double><<<(int)blocks, 256, 0, s>>>((const double*)ring, ld, NS, n, f, m, cf, res,
                                                         (double*)low, (double*)sparse, mask, ldo, thr);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- NEXT-4: scoring --------
__global__ void __launch_bounds__(256) score_kernel(const unsigned char* __restrict__ mask,
                                                   const unsigned char* __restrict__ gt, long long n,
                                                   int vec, unsigned long long* __restrict__ cnt) {
  unsigned long long tp = 0, fp = 0, fn = 0;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long done = 0;
  if (vec) {                                   // 16-byte vectors (both buffers 16-B aligned)
    const long long nv = n >> 4;
    const uint4* mv = reinterpret_cast<const uint4*>(mask);
    const uint4* gv = reinterpret_cast<const uint4*>(gt);
    for (long long i = tid; i < nv; i += stride) {
      const uint4 a = __ldcs(mv + i), b = __ldcs(gv + i);
      const unsigned aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int w = 0; w < 4; ++w) {
#pragma unroll
        for (int by = 0; by < 4; ++by) {
          const unsigned ma = (aw[w] >> (8 * by)) & 0xffu, gb = (bw[w] >> (8 * by)) & 0xffu;
          tp += (ma != 0u) & (gb != 0u);
          fp += (ma != 0u) & (gb == 0u);
          fn += (ma == 0u) & (gb != 0u);
        }
      }
    }
    done = nv << 4;
  }
  for (long long i = done + tid; i < n; i += stride) {
    const bool ma = mask[i] != 0, gb = gt[i] != 0;
    tp += ma & gb;
    fp += ma & !gb;
    fn += !ma & gb;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    tp += __shfl_xor_sync(0xffffffffu, tp, o);
    fp += __shfl_xor_sync(0xffffffffu, fp, o);
    fn += __shfl_xor_sync(0xffffffffu, fn, o);
  }
  __shared__ unsigned long long red[3][8];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[0][w] = tp; red[1][w] = fp; red[2][w] = fn; }
  __syncthreads();
  if (threadIdx.x < 3) {
    unsigned long long t = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[threadIdx.x][q];
    atomicAdd(cnt + threadIdx.x, t);           // integer sums: order-independent, exact
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(cnt + 3, 1ull);
}

cudaError_t launch_score(const unsigned char* mask, const unsigned char* gt, long long n,
                         unsigned long long* cnt, cudaStream_t s) {
  const int vec = ((((uintptr_t)mask) | ((uintptr_t)gt)) & 15) == 0;
  long long blocks = (n / 16 + 255) / 256;
  if (blocks > 4 * 148) blocks = 4 * 148;
  if (blocks < 1) blocks = 1;
  score_kernel<<<(int)blocks, 256, 0, s>>>(mask, gt, n, vec, cnt);
  return cudaGetLastError();
}

}  // namespace sdmd
