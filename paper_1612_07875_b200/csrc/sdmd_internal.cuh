// sdmd_internal.cuh — device-side data layout and kernel interfaces of libsdmd (sm_100a).
// Layout (DESIGN.md §"Data layout in HBM"):
//   ring   : NS slots x ld elements (fp32|fp64), slot of frame f = f mod NS, ld = n_local rounded
//            up to 256 elements (padding rows are zero, so vector loads need no row guards)
//   ghist  : NH x (m+1) fp64; ghist[f mod NH][k] = <x_{f-m+k}, x_f>   (the Gram column of frame f)
//            G of the window ending at t:  G[i][j] (i<=j) = ghist[(t-m+j) mod NH][i-j+m]
//            (the paper's "xtx[:-1,:-1] = xtx[1:,1:]" copy, Alg 1, becomes pure indexing)
//   cbuf   : NC x m complex; background coefficients c_t = b_idx λ_idx^m V Σ⁻¹ w_idx of frame t
//   DevState: poison status word + frame counters (device-authoritative)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <map>
#include <mutex>
#include <utility>

namespace sdmd {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device, size increase): the
// per-push launch paths call this on every launch, and the runtime call is not free on the host
// (C1's push is host-bound).
inline cudaError_t set_max_dyn_smem(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> set;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  int& have = set[{func, dev}];
  if (bytes <= have) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

constexpr int kMaxM = 256;
constexpr int kMaxR = 224;
constexpr int kMaxWorkers = 24;
constexpr int kMaxBatch = 8;
constexpr int kMaxBgModes = 8;           // background modes (NEXT-2); +1 for the conjugate partner             // frames per batched push (K1b)
constexpr int kMaxLag = 64;              // background lag cap (frames); union columns m + lag
constexpr int kK1MaxWaves = 32;           // K1 grid <= kK1MaxWaves x SM count
constexpr int kSuperTile = 256;           // K1 rows per CTA iteration (32 lanes x 8 rows)

struct DevState {
  int status;                 // 0 = OK, else SDMD_E_NONFINITE (stream poisoned until sync)
  int pad0;
  long long failed_frame;     // rejected frame index
  long long committed;        // frames committed (device authoritative)
  long long bg_frame;         // frame index of the newest background column written
  unsigned int k1_done;       // last-block counter of K1
  unsigned int k3_done;       // last-block counter of K3
  unsigned int pad1[2];
  int* hpoison;               // device alias of a mapped pinned host word, set to 1 by every rejection
                              // (the host reads it to refuse ring-slot writes while poisoned)
};

// Record a rejection (the caller already set status / failed_frame) in the host-visible mirror.
static __device__ __forceinline__ void poison_mirror(DevState* st) {
  if (st->hpoison) {
    *(volatile int*)st->hpoison = 1;
    __threadfence_system();
  }
}

struct K1Params {
  const void* ring;
  long long ld;               // slot stride (elements)
  int NS;                     // ring slots
  int m;
  long long n;                // local rows (valid rows; ld >= n)
  long long f_new;            // frame being pushed (slot f_new % NS)
  int nd;                     // dot columns: frames f_new-nd+1 .. f_new
  int bg;                     // compute the background column of frame f_bg in this pass
  long long f_bg;
  const double2* cbg;         // m coefficients of frame f_bg (column k <-> frame f_bg-m+1+k)
  void* lowrank;              // n (dtype)
  void* sparse;               // n (dtype)
  unsigned char* mask;        // n
  float thr;
  double* partials;           // K1: [nd][pgrid] (column-major, coalesced reduction)
  int pgrid;                  // partials stride of K1 (>= gridDim.x)
  int dbg;                    // microbenchmark knob (SDMD_K1_DBG): 1 skip bg reduction, 2 skip bg FMAs
  int v1;                     // 1: the v1 K1 (8 rows per lane, lockstep background reduction), A/B only
  double* gout;               // nd reduced values (pre-allreduce)
  int do_commit;              // nranks == 1: commit inside the kernel's last block
  double* ghist;
  int NH;
  DevState* st;
  // commit kernel (multi-rank): background coefficients carried by the same allreduce (one
  // collective per frame): copy cfold_n doubles from cfold_src (after the g part) to cfold_dst
  const double* cfold_src;
  double* cfold_dst;
  int cfold_n;
};

struct K1bParams {             // K1b: Gram columns of k frames f0..f0+k-1 in one pass
  const void* ring;
  long long ld;
  int NS;
  int m;
  long long n;
  long long f0;
  int k;
  double* partials;           // [U][kMaxBatch][grid]
  double* gout;               // k x (m+1): column j = Gram column of frame f0+j
  int do_commit;
  double* ghist;
  int NH;
  DevState* st;
};

struct K4Result {
  long long frame;
  int status;                 // 0 OK or sdmd_status of this frame's DMD
  int r;
  int idx;
  int sweeps;
  int qr_its;
  int pad;
  double lam_idx[2];
  double b_idx[2];
  double sigma1;
  long long phase[8];         // SM cycles per K4 phase: build S, Jacobi, sort/V, Ã, Hessenberg (K4a), QR, eigvec+c (K4b)
  int qr_cnt[4];              // QR: single-bulge steps, multishift steps, single-bulge its, multishift sweeps
  int aberth_its;             // Ehrlich–Aberth iterations (0: not used), < 0: failed → QR fallback
  int aberth_evals;           // Hyman evaluations
  long long qr_dbg[2];        // SM cycles of the multishift chase: (AB) phase + barrier, (C) phase + barrier (warp 0)
  long long vframe;           // frame whose converged eigenvectors V this workspace holds (K4a), or -1
  int nkeep;                  // modes with |λ_j| >= rank_tol·max|λ| (a prefix of the sorted λ); < r → W_SINGULAR
  int nB;                     // background mode set of this frame (B[0] = idx)
  long long commit_wait;      // K4a SM cycles spent waiting for frame f's commit (inside phase[3])
  int bset[kMaxBgModes + 1];
};

// W_SINGULAR amplitudes (reading Q15): the modes j >= nkeep get b_j = 0, the
// kept ones the least-squares solution of min ‖W_K Λ_K b − α₁‖ (K = 0..nkeep-1).  Per frame
// (res != null) both kernels return at once unless the frame's K4b flagged it singular; then
// they recompute b over the kept modes and the background coefficients c.
struct K4SingParams {
  int r;                      // r (on-demand) or r_max (per frame: r, nkeep read from res)
  int m;                      // window width (per frame)
  long long f;                // frame (per frame)
  const K4Result* res;        // per frame: the frame's summary (else null)
  K4Result* res_out;          // per frame: b_idx updated here
  int nkeep;                  // on demand
  const double* H;
  const double* Qv;
  const double* tau;
  const double2* lam;
  const double* alpha1;
  const double* Y;            // m x r (per frame: for c)
  double2* Mws;               // [grid][r_max^2] inverse-iteration LU workspaces
  double2* W;                 // r x r column-major: kept right eigenvectors (ld r)
  double2* A;                 // r x r workspace of the least squares
  double2* b;                 // r amplitudes (output)
  double2* cout;              // m background coefficients (per frame) or null
  unsigned int* counter;      // last-block counter (zero between launches)
};

struct K4Params {
  const double* ghist;
  int NH;
  int m;                      // window width w of this frame's DMD (= cfg.m, or t during build-up)
  int mh;                     // history row stride - 1 (= cfg.m)
  long long f;                // frame whose window is decomposed
  int r_max;
  double rank_tol;
  DevState* st;
  // per-worker workspace
  double* A;                  // m*m  (one-sided Jacobi, column-major)
  double* Gxy;                // m*m  (XᵀX', column-major)
  double* V;                  // m*m  (eigenvectors of S, sorted, column-major)
  double* sigma;              // m
  double* Y;                  // m*kMaxR  V Σ⁻¹ (column-major, ld m)
  double* B;                  // m*kMaxR  Gxy Y
  double* H;                  // kMaxR*kMaxR row-major: Ã, then its Hessenberg form
  double* Qv;                 // kMaxR*kMaxR row-major: Householder vector k in row k
  double* tau;                // kMaxR
  double2* M;                 // kMaxR*kMaxR complex row-major (inverse-iteration LU)
  double2* Mc;                // kMaxR*kMaxR complex: the same U factor column-major (K4b group solve)
  double2* lam;               // kMaxR sorted eigenvalues of Ã
  double2* w;                 // kMaxR right eigenvector (background mode)
  double2* y;                 // kMaxR left eigenvector
  double* alpha1;             // kMaxR
  K4Result* res;
  double2* cout;              // m background coefficients (cbuf slot), zero on failure
  int* flags;                 // per-sweep "rotated" flags (cluster-wide OR)
  double* mu;                 // m column norms
  int bg_modes;               // nb > 1: background from the mode set B (reading Q25), M/w/y hold
                              // nb+1 slots (strides kMaxR*kMaxR and kMaxR)
  double* wv;                 // kMaxR Householder scratch
  double* uv;                 // kMaxR Householder scratch
  // Jacobi warm start: eigenvectors of frame f - warm_k (same cluster stream, so complete), used
  // when res_prev->vframe == f - warm_k; else cold start from S
  const double* Vprev;
  const K4Result* res_prev;
  int warm_k;
  // eig(Ã) warm start: the spectrum of the previous frame solved on the same cluster stream
  // (stream-ordered: read at the start of K4a's eigenvalue stage, rewritten at its end)
  double2* lam_warm;          // kMaxR
  int* r_warm;                // its r (0: none yet)
  int atilde_v1;              // SDMD_ATILDE=v1: the untiled Ã stage (A/B only)
  int chol;                   // Jacobi on Q0·Rᵀ (pivoted Cholesky of Q0ᵀSQ0) instead of S·Q0 (m <= kMaxR)
};

// per-eigenvalue on-demand eigenvectors (right W[:, j], left, amplitude b_j)
struct K4VecParams {
  int r;
  const double* H;
  const double* Qv;
  const double* tau;
  const double2* lam;
  const double* alpha1;
  double2* Mws;               // chunk x r*r complex workspace
  double2* W;                 // r*r column-major (output)
  double2* b;                 // r (output)
  int j0;                     // first eigenvalue of this launch
  const K4Result* res;        // non-null: r (and the W stride) read on the device (per-frame modes)
};

struct K3Params {             // sparse Gram column
  const int* idx;             // NS x nnz_cap
  const double* val;          // NS x nnz_cap
  const int* nnz;             // NS (device)
  int nnz_cap;
  int NS;
  int m;
  long long f_new;
  int nd;
  double* scratch;            // dense n_local fp64 (double2 for the Fourier bases) scatter target,
                              // kept zero between pushes
  long long row_begin;
  int cplx;                   // 1: Fourier bases, val holds interleaved complex (double2) values
  long long half_h;           // RFFT: grid_cols/2 + 1 (weights 2 off the self-conjugate columns), else 0
  int half_even;              // RFFT: grid_cols even (column half_h - 1 is self-conjugate too)
  double* partials;           // [nd][chunks]
  int chunks;
  double* gout;
  int do_commit;
  double* ghist;
  int NH;
  DevState* st;
};

// Commit (Alg 1 else-branch P:293-295, rejection S:285): called by one whole block.
static __device__ __forceinline__ void commit_block(const double* gout, int nd, int m, long long f_new, double* ghist,
                             int NH, DevState* st) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < nd; k += blockDim.x)
    if (!isfinite(gout[k])) bad = 1;
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) { st->status = 2 /*SDMD_E_NONFINITE*/; st->failed_frame = f_new; poison_mirror(st); }
    return;
  }
  double* row = ghist + (long long)(f_new % NH) * (m + 1);
  const int off = m + 1 - nd;
  for (int k = threadIdx.x; k < m + 1; k += blockDim.x) row[k] = (k >= off) ? gout[k - off] : 0.0;
  // publish: the history row must be visible GPU-wide before the counter (K4a of frame f_new
  // polls it to start its Ã stage, see k4_eigen.cu)
  __syncthreads();
  __threadfence();
  if (threadIdx.x == 0) *(volatile long long*)&st->committed = f_new + 1;
}


// kernels (defined in k1_gram.cu, k3_sparse.cu, k4_eigen.cu, k2_dmma.cu)
cudaError_t launch_k1(const K1Params& p, int dtype, int grid, cudaStream_t s);
void preload_k1_kernels();
void preload_k4_kernels();
cudaError_t launch_commit(const K1Params& p, cudaStream_t s);
cudaError_t launch_k1b(const K1bParams& p, int dtype, int grid, cudaStream_t s);
cudaError_t launch_commit_batch(const K1bParams& p, cudaStream_t s);
int k1b_grid(int nsm, long long n, int dtype);
size_t k1b_partials_elems(int grid);
cudaError_t launch_k3(const K3Params& p, cudaStream_t s);
cudaError_t launch_sparse_nnz_checked(const int* idx, int nnz, long long lo, long long hi,
                                      int* nnz_slot, cudaStream_t s);
cudaError_t launch_k4a(const K4Params& p, cudaStream_t s, int cl);   // cl: k4_cluster_size(m)
cudaError_t launch_k4b(const K4Params& p, cudaStream_t s);
size_t k4_smem_bytes(int r_max, int m, int bg_modes, int cl);
int k4_cluster_size(int m, bool sparse);   // CTAs per K4a launch (1 or 4)
int k4_small_m();                  // K4a runs its Jacobi on one CTA up to this window width
cudaError_t launch_k4_vecs(const K4VecParams& p, int count, cudaStream_t s);
cudaError_t launch_k4_singular(const K4SingParams& p, bool vecs, cudaStream_t s);
constexpr int kSingVecGrid = 16;          // CTAs (one warp each) of the singular-path eigenvectors
cudaError_t launch_init_gram(const void* Z, long long ldz, int dtype, long long n, int k,
                             double* Gout, double* work, cudaStream_t s);
size_t init_gram_work_elems(long long n, int k);
cudaError_t launch_modes(const void* ring, long long ld, int NS, int dtype, long long n,
                         long long first_frame, int m, const double* T /*m x nc complex*/,
                         int nc, double* phi, long long ldphi, cudaStream_t s);
cudaError_t launch_modes_sparse(const int* idx, const double* val, const int* nnz, int nnz_cap, int NS,
                                long long row_begin, long long n, long long first_frame, int m,
                                const double* T /*m x nc complex*/, int nc, double* phi, long long ldphi,
                                int cplx, cudaStream_t s);
// NEXT-3 pixel-space background of a sparse DCT context (k6_background.cu)
struct PixBgParams {
  const int* idx;             // sparse ring (NS x nnz_cap), DCT values
  const double* val;
  const int* nnz;
  int nnz_cap;
  int NS;
  int m;
  long long f_bg;             // background frame: X' = frames f_bg-m+1 .. f_bg, x = frame f_bg
  const double2* c;           // m coefficients (column k <-> frame f_bg-m+1+k)
  int rows, cols;             // coefficient / pixel grid (powers of two)
  double* planes;             // 3 x rows x cols: Re l̂, Im l̂, x̂ (then the transforms, in place)
  double* tmp;                // 3 x rows x cols
  double* lowrank;            // rows x cols fp64 outputs
  double* sparse;
  unsigned char* mask;
  float thr;
  DevState* st;
};
cudaError_t launch_pixel_background(const PixBgParams& p, cudaStream_t s);
// Alg 3 first-window branch over the newest DMD window (reading Q24)
cudaError_t launch_window_background(const void* ring, long long ld, int NS, int dtype, long long n,
                                     long long f, int m, const double2* cf, const K4Result* res,
                                     void* low, void* sparse, unsigned char* mask, long long ldo,
                                     float thr, cudaStream_t s);
// NEXT-4 scoring: TP/FP/FN counts of mask vs gt accumulated into cnt[0..2], cnt[3] += 1 (frames)
cudaError_t launch_score(const unsigned char* mask, const unsigned char* gt, long long n,
                         unsigned long long* cnt, cudaStream_t s);
cudaError_t launch_ghist_from_gram(const double* G, int k, double* ghist, int NH, int m,
                                   long long first_frame, cudaStream_t s);
cudaError_t launch_gather_gram(const double* ghist, int NH, int m, long long f_last, int k,
                               double* Gout, cudaStream_t s);
cudaError_t launch_set_int(int* p, int v, cudaStream_t s);
cudaError_t launch_make_T_all(const double* Y, int m, const K4Result* res, int r_max,
                              const double2* W, double* T, cudaStream_t s);
cudaError_t launch_make_T(const double* Y, int m, int r, const double2* W, const int* cols,
                          int nc, double* T, cudaStream_t s);

}  // namespace sdmd
