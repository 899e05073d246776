// k2_dmma.cu — K2: dense fp64 contractions on the tensor pipe (DMMA, mma.sync m8n8k4 f64).
//
//  (a0) batch Gram of the first window, G = Zᵀ Z  (Alg 1 first branch "xtx = X.T * X"):
//       split-K over rows, 64x64 output blocks (upper triangle only), fp32 data converted exactly
//       to fp64 when staged in shared memory; per-split partial blocks reduced in fixed order.
//  (a12) DMD modes on demand, Φ = X' (V Σ⁻¹ W)  (Eq. Phi; "phi = X[:, 1:] * vsiw",
//       Alg 2): a real n x m by complex m x nc product, computed as one real GEMM against
//       the interleaved (re, im) columns of T = Y W.
// tcgen05 has no f64 kind; the fp64 tensor path on sm_100a is DMMA (HMMA-class SASS "DMMA").
#include "sdmd_internal.cuh"

namespace sdmd {

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

template <typename T>
__device__ __forceinline__ double ld_as_double(const T* p) { return (double)*p; }

// ---------------------------------------------------------------------- (a0) Gram ------------
constexpr int G_BLK = 64;          // output block edge
constexpr int G_KC = 32;           // rows staged per step
constexpr int G_THREADS = 256;     // 8 warps; warp w owns output rows 8w..8w+7 of the block

template <typename T>
__global__ void __launch_bounds__(G_THREADS) gram_dmma_kernel(const T* __restrict__ Z, long long ldz,
                                                              long long n, int k, int nbk,
                                                              long long rows_per_split,
                                                              double* __restrict__ work) {
  __shared__ double As[G_KC][G_BLK + 1];   // As[l][i] = Z[row0 + l][bi*64 + i]
  __shared__ double Bs[G_KC][G_BLK + 1];
  // upper-triangular block index -> (bi, bj)
  int bidx = blockIdx.x, bi = 0;
  while (bidx >= nbk - bi) { bidx -= nbk - bi; ++bi; }
  const int bj = bi + bidx;
  const long long r0 = (long long)blockIdx.y * rows_per_split;
  long long r1 = r0 + rows_per_split;
  if (r1 > n) r1 = n;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  double acc[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) acc[t][0] = acc[t][1] = 0.0;
  for (long long row = r0; row < r1; row += G_KC) {
    __syncthreads();
    for (int e = tid; e < G_KC * G_BLK; e += G_THREADS) {
      const int l = e % G_KC, c = e / G_KC;              // coalesced along rows
      const long long rr = row + l;
      const int ci = bi * G_BLK + c, cj = bj * G_BLK + c;
      As[l][c] = (rr < r1 && ci < k) ? ld_as_double(Z + (long long)ci * ldz + rr) : 0.0;
      Bs[l][c] = (rr < r1 && cj < k) ? ld_as_double(Z + (long long)cj * ldz + rr) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < G_KC; kk += 4) {
      const double a = As[kk + tig][warp * 8 + g];        // A[i][l] = Z[l][i], row-major frag
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const double b = Bs[kk + tig][t * 8 + g];         // B[l][j] = Z[l][j], col-major frag
        dmma_8x8x4(acc[t][0], acc[t][1], a, b);
      }
    }
  }
  double* out = work + ((long long)blockIdx.y * gridDim.x + blockIdx.x) * G_BLK * G_BLK;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int i = warp * 8 + g, j = t * 8 + tig * 2;
    out[i * G_BLK + j] = acc[t][0];
    out[i * G_BLK + j + 1] = acc[t][1];
  }
}

__global__ void gram_reduce_kernel(const double* __restrict__ work, int nblk, int nsplit, int nbk,
                                   int k, double* __restrict__ G) {
  const int b = blockIdx.x;
  int bidx = b, bi = 0;
  while (bidx >= nbk - bi) { bidx -= nbk - bi; ++bi; }
  const int bj = bi + bidx;
  for (int e = threadIdx.x; e < G_BLK * G_BLK; e += blockDim.x) {
    double s = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) s += work[((long long)sp * nblk + b) * G_BLK * G_BLK + e];
    const int i = bi * G_BLK + e / G_BLK, j = bj * G_BLK + e % G_BLK;
    if (i < k && j < k) {
      G[(long long)j * k + i] = s;
      G[(long long)i * k + j] = s;
    }
  }
}

static int g_nsplit(long long n) {
  long long s = (n + 8191) / 8192;
  if (s > 64) s = 64;
  if (s < 1) s = 1;
  return (int)s;
}

size_t init_gram_work_elems(long long n, int k) {
  const int nbk = (k + G_BLK - 1) / G_BLK;
  const int nblk = nbk * (nbk + 1) / 2;
  return (size_t)g_nsplit(n) * nblk * G_BLK * G_BLK;
}

cudaError_t launch_init_gram(const void* Z, long long ldz, int dtype, long long n, int k,
                             double* Gout, double* work, cudaStream_t s) {
  const int nbk = (k + G_BLK - 1) / G_BLK;
  const int nblk = nbk * (nbk + 1) / 2;
  const int nsplit = g_nsplit(n);
  long long rps = (n + nsplit - 1) / nsplit;
  rps = (rps + G_KC - 1) / G_KC * G_KC;
  dim3 grid(nblk, nsplit);
  if (dtype == 0)
    gram_dmma_kernel<float><<<grid, G_THREADS, 0, s>>>((const float*)Z, ldz, n, k, nbk, rps, work);
  else
    gram_dmma_kernel<double><<<grid, G_THREADS, 0, s>>>((const double*)Z, ldz, n, k, nbk, rps, work);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  gram_reduce_kernel<<<nblk, 256, 0, s>>>(work, nblk, nsplit, nbk, k, Gout);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------- (a12) modes ----------
constexpr int M_ROWS = 64;         // rows per CTA (8 warps x 8 rows)
constexpr int M_COLS = 64;         // real output columns per pass (32 complex modes)
constexpr int M_KC = 32;

// T: m x nc complex, column-major (T[(j*m + k)] = (re, im)); phi: n x nc complex, column-major ld.
template <typename T>
__global__ void __launch_bounds__(256) modes_dmma_kernel(const T* __restrict__ ring, long long ld,
                                                         int NS, long long n, long long first_frame,
                                                         int m, const double2* __restrict__ Tm,
                                                         int nc, int c0, double2* __restrict__ phi,
                                                         long long ldphi) {
  __shared__ double As[M_ROWS][M_KC + 1];   // As[row][k] = X'[row0+row][k0+k]
  __shared__ double Bs[M_KC][M_COLS + 1];   // Bs[k][2q+c] = (re|im) T[k0+k][c0+q]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  const long long row0 = (long long)blockIdx.x * M_ROWS;
  double acc[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) acc[t][0] = acc[t][1] = 0.0;
  for (int k0 = 0; k0 < m; k0 += M_KC) {
    __syncthreads();
    for (int e = tid; e < M_ROWS * M_KC; e += 256) {
      const int rr = e % M_ROWS, kk = e / M_ROWS;
      const long long row = row0 + rr;
      const int k = k0 + kk;
      double v = 0.0;
      if (row < n && k < m) {
        const long long f = first_frame + k;
        v = (double)ring[(f % NS) * ld + row];
      }
      As[rr][kk] = v;
    }
    for (int e = tid; e < M_KC * M_COLS; e += 256) {
      const int kk = e / M_COLS, c = e % M_COLS;
      const int k = k0 + kk, q = c0 + c / 2;
      double v = 0.0;
      if (k < m && q < nc) {
        const double2 t = Tm[(long long)q * m + k];
        v = (c & 1) ? t.y : t.x;
      }
      Bs[kk][c] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < M_KC; kk += 4) {
      const double a = As[warp * 8 + g][kk + tig];
#pragma unroll
      for (int t = 0; t < 8; ++t) dmma_8x8x4(acc[t][0], acc[t][1], a, Bs[kk + tig][t * 8 + g]);
    }
  }
  const long long row = row0 + warp * 8 + g;
  if (row < n) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int q = c0 + (t * 8 + tig * 2) / 2;          // columns (2q, 2q+1) = (re, im)
      if (q < nc) phi[(long long)q * ldphi + row] = make_double2(acc[t][0], acc[t][1]);
    }
  }
}

cudaError_t launch_modes(const void* ring, long long ld, int NS, int dtype, long long n,
                         long long first_frame, int m, const double* T, int nc, double* phi,
                         long long ldphi, cudaStream_t s) {
  const int grid = (int)((n + M_ROWS - 1) / M_ROWS);
  for (int c0 = 0; c0 < nc; c0 += M_COLS / 2) {
    if (dtype == 0)
      modes_dmma_kernel<float><<<grid, 256, 0, s>>>((const float*)ring, ld, NS, n, first_frame, m,
                                                    (const double2*)T, nc, c0, (double2*)phi, ldphi);
    else
      modes_dmma_kernel<double><<<grid, 256, 0, s>>>((const double*)ring, ld, NS, n, first_frame, m,
                                                     (const double2*)T, nc, c0, (double2*)phi, ldphi);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// T = Y W[:, cols]  (m x nc complex): the "vsiw" product of Alg 2 P:315 for selected modes.
__global__ void make_T_kernel(const double* Y, int m, int r, const double2* W, const int* cols, int nc,
                              double2* T) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= m * nc) return;
  const int k = idx % m, q = idx / m;
  const int j = cols[q];
  double2 s = make_double2(0.0, 0.0);
  for (int i = 0; i < r; ++i) {
    const double y = Y[(long long)i * m + k];
    const double2 w = W[(long long)j * r + i];
    s.x = fma(y, w.x, s.x);
    s.y = fma(y, w.y, s.y);
  }
  T[idx] = s;
}

cudaError_t launch_make_T(const double* Y, int m, int r, const double2* W, const int* cols, int nc,
                          double* T, cudaStream_t s) {
  const int n = m * nc;
  make_T_kernel<<<(n + 255) / 256, 256, 0, s>>>(Y, m, r, W, cols, nc, (double2*)T);
  return cudaGetLastError();
}

}  // namespace sdmd
