// k3_sparse.cu — K3: Gram column over natively compressed (sparse orthonormal-DCT) snapshots.
//
// §3.5: SVD and DMD are invariant under unitary transforms, so the window may be kept
// in a sparse transform basis and "many of the core steps … performed on sparse data matrices"
// — the paper did not implement this.  Each ring slot holds (idx int32 ascending,
// val fp64, nnz).  Per push: (1) scatter x̂_new into a dense fp64 scratch vector that stays
// L2-resident (8 MB for 1024²), (2) for every window column, gather-multiply its nonzeros against
// the scratch (g_k = <ẑ_k, x̂_new>), partial sums per (column, chunk) reduced in fixed order by the
// last block, which also (3) clears the scattered positions and commits the column.
#include "sdmd_internal.cuh"

namespace sdmd {

constexpr int K3_THREADS = 256;
constexpr int K3_CHUNK = 2048;     // nonzeros per block

__global__ void k3_scatter_kernel(const K3Params p) {
  if (*(volatile int*)&p.st->status != 0) return;
  const int slot = (int)(p.f_new % p.NS);
  const int nnz = p.nnz[slot];
  const int* idx = p.idx + (long long)slot * p.nnz_cap;
  const double* val = p.val + (long long)slot * p.nnz_cap;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += gridDim.x * blockDim.x)
    p.scratch[idx[e] - p.row_begin] = val[e];
}

__global__ void __launch_bounds__(K3_THREADS) k3_dot_kernel(const K3Params p) {
  __shared__ double red[K3_THREADS / 32];
  __shared__ int am_last;
  if (*(volatile int*)&p.st->status != 0) return;
  const int kd = blockIdx.y;                          // dot column (frame f_new - nd + 1 + kd)
  const int c = blockIdx.x;                           // chunk of its nonzeros
  const long long f = p.f_new - p.nd + 1 + kd;
  const int slot = (int)(f % p.NS);
  const int nnz = p.nnz[slot];
  const int* idx = p.idx + (long long)slot * p.nnz_cap;
  const double* val = p.val + (long long)slot * p.nnz_cap;
  double s = 0.0;
  const int e0 = c * K3_CHUNK, e1 = min(nnz, e0 + K3_CHUNK);
  for (int e = e0 + threadIdx.x; e < e1; e += K3_THREADS)
    s = fma(val[e], __ldcg(&p.scratch[idx[e] - p.row_begin]), s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < K3_THREADS / 32; ++w) t += red[w];
    p.partials[(long long)kd * p.chunks + c] = t;
    __threadfence();
    const unsigned prev = atomicAdd(&p.st->k3_done, 1u);
    am_last = (prev == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  for (int k = threadIdx.x; k < p.nd; k += K3_THREADS) {
    double t = 0.0;
    for (int cc = 0; cc < p.chunks; ++cc) t += __ldcg(&p.partials[(long long)k * p.chunks + cc]);
    p.gout[k] = t;
  }
  // clear the scatter positions of the new frame (scratch stays all-zero between pushes)
  const int sl = (int)(p.f_new % p.NS);
  const int nn = p.nnz[sl];
  const int* ix = p.idx + (long long)sl * p.nnz_cap;
  __syncthreads();
  for (int e = threadIdx.x; e < nn; e += K3_THREADS) p.scratch[ix[e] - p.row_begin] = 0.0;
  // a device-pushed frame whose indices failed the check (nnz recorded as -1, nothing scattered):
  // a NaN self inner product, so that the commit rejects the frame — after the allreduce when
  // rows are sharded, i.e. on every rank alike
  if (nn < 0 && threadIdx.x == 0) p.gout[p.nd - 1] = __longlong_as_double(0x7ff8000000000000LL);
  if (threadIdx.x == 0) p.st->k3_done = 0;
  if (p.do_commit) {
    __syncthreads();
    commit_block(p.gout, p.nd, p.m, p.f_new, p.ghist, p.NH, p.st);
  }
}

cudaError_t launch_k3(const K3Params& p, cudaStream_t s) {
  k3_scatter_kernel<<<64, 256, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 grid(p.chunks, p.nd);
  k3_dot_kernel<<<grid, K3_THREADS, 0, s>>>(p);
  return cudaGetLastError();
}

// Record the nonzero count of a device-pushed sparse frame after checking its indices on the
// device (the host cannot see them): strictly ascending and inside [lo, hi).  A violation records
// nnz = -1, which makes the scatter, gather and clear loops empty (no out-of-range access) and the
// Gram pass reject the frame (see k3_dot_kernel).
__global__ void __launch_bounds__(256) sparse_nnz_checked_kernel(const int* __restrict__ idx, int nnz,
                                                                 long long lo, long long hi,
                                                                 int* __restrict__ nnz_slot) {
  int bad = 0;
  for (int e = threadIdx.x; e < nnz; e += blockDim.x) {
    const int i = idx[e];
    bad |= (i < lo) | (i >= hi) | (e > 0 && i <= idx[e - 1]);
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) *nnz_slot = bad ? -1 : nnz;
}

cudaError_t launch_sparse_nnz_checked(const int* idx, int nnz, long long lo, long long hi,
                                      int* nnz_slot, cudaStream_t s) {
  sparse_nnz_checked_kernel<<<1, 256, 0, s>>>(idx, nnz, lo, hi, nnz_slot);
  return cudaGetLastError();
}

// Record the nonzero count of a ring slot (stream-ordered, no host staging).
__global__ void set_int_kernel(int* p, int v) { *p = v; }

cudaError_t launch_set_int(int* p, int v, cudaStream_t s) {
  set_int_kernel<<<1, 1, 0, s>>>(p, v);
  return cudaGetLastError();
}

// ---- NEXT-3: DMD modes in coefficient space, Φ̂ = X̂'(Y W) over the sparse window (P:355-361:
// the modes of the transformed data are the transformed modes, by unitary invariance).  Block q
// owns mode column q; it zeroes Φ̂[:, q] and then walks the m window columns IN ORDER, its threads
// scattering val_e · T[k][q] into the column's nonzero rows (indices are unique within a column,
// and a block barrier separates columns): every element is accumulated in fixed k order.
__global__ void __launch_bounds__(256) modes_sparse_kernel(const int* __restrict__ idx,
                                                          const double* __restrict__ val,
                                                          const int* __restrict__ nnz, int nnz_cap,
                                                          int NS, long long row_begin, long long n,
                                                          long long first_frame, int m,
                                                          const double2* __restrict__ T, int nc,
                                                          double2* __restrict__ phi, long long ldphi) {
  const int q = blockIdx.x;
  if (q >= nc) return;
  double2* col = phi + (long long)q * ldphi;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) col[i] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int k = 0; k < m; ++k) {
    const int slot = (int)((first_frame + k) % NS);
    const int nz = nnz[slot];
    const int* ik = idx + (long long)slot * nnz_cap;
    const double* vk = val + (long long)slot * nnz_cap;
    const double2 t = T[(long long)q * m + k];
    for (int e = threadIdx.x; e < nz; e += blockDim.x) {
      const long long row = ik[e] - row_begin;
      const double v = vk[e];
      double2 c = col[row];
      c.x = fma(v, t.x, c.x);
      c.y = fma(v, t.y, c.y);
      col[row] = c;
    }
    __syncthreads();
  }
}

cudaError_t launch_modes_sparse(const int* idx, const double* val, const int* nnz, int nnz_cap, int NS,
                                long long row_begin, long long n, long long first_frame, int m,
                                const double* T, int nc, double* phi, long long ldphi, cudaStream_t s) {
  modes_sparse_kernel<<<nc, 256, 0, s>>>(idx, val, nnz, nnz_cap, NS, row_begin, n, first_frame, m,
                                         (const double2*)T, nc, (double2*)phi, ldphi);
  return cudaGetLastError();
}

}  // namespace sdmd
