// k2_dmma.cu — K2: dense fp64 contractions on the tensor pipe (DMMA, mma.sync m8n8k4 f64).
//
//  (a0) batch Gram of the first window, G = Zᵀ Z  (Alg 1 first branch "xtx = X.T * X"):
//       64x64 upper-triangular column-block pairs, rows split per block in proportion to its
//       active warp tiles (one balanced wave), per-split partial blocks reduced in fixed order.
//  (a12) DMD modes on demand, Φ = X' (V Σ⁻¹ W)  (Eq. Phi; "phi = X[:, 1:] * vsiw",
//       Alg 2): a real n x m by complex m x nc product, computed as one real GEMM against
//       the interleaved (re, im) columns of T = Y W.
// tcgen05 has no f64 kind; the fp64 tensor path on sm_100a is DMMA (HMMA-class SASS "DMMA").
#include <cuda.h>            // CUtensorMap (the encode entry point is fetched from the runtime)
#include <cudaTypedefs.h>

#include "sdmd_internal.cuh"

#include <cstdlib>
#include <cstring>

namespace sdmd {

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}


// Both contractions: raw (fp32|fp64) tiles staged in shared memory by a 3-stage cp.async pipeline
// (16-byte chunks, zero-fill outside the operand), fragments converted to fp64 when they are
// loaded from shared memory (fp32 x fp32 products are exact in fp64, reading Q9), 32x32 warp tiles
// = 4x4 DMMA m8n8k4 per 4-deep k step (16 DMMA per 8 fragment loads).  Shared-memory strides are
// padded so that every fragment load is bank-conflict free (lane l reads row l%4, element l/4).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---- (a0) G = Zᵀ Z: 64x64 upper-triangular output blocks, 4 warps (2x2 warp tiles of 32x32);
// warp tiles entirely below the diagonal or entirely past column k are skipped, and the rows are
// split per block in proportion to its active warp tiles so that every CTA carries the same work
// (one balanced wave).  Per-split partial blocks are reduced in fixed order (deterministic).
constexpr int G2_KC = 32;                 // rows per stage
constexpr int G2_ST = 3;                  // pipeline stages
constexpr int G2_LDS = G2_KC + 4;         // staged column stride (elements): conflict-free frags
constexpr int G2_THREADS = 128;
constexpr int G2_MAXB = 21;               // upper-triangular 64-blocks for k <= 384
constexpr int G2_MAXCTA_PER_SM = 8;

struct GramPlan {
  int nbk, nblk;
  int split0[G2_MAXB + 1];                // CTA prefix per block
  long long rps[G2_MAXB];                 // rows per split of each block (multiple of G2_KC)
};

template <typename T>
__global__ void __launch_bounds__(G2_THREADS) gram_tc_kernel(const T* __restrict__ Z, long long ldz,
                                                            long long nrows, int k, const GramPlan plan,
                                                            double* __restrict__ work) {
  extern __shared__ __align__(16) unsigned char g2_smem[];
  T* sm = reinterpret_cast<T*>(g2_smem);  // [G2_ST][2 operands][64 columns][G2_LDS]
  int b = 0;
  while ((int)blockIdx.x >= plan.split0[b + 1]) ++b;
  const long long sp = (long long)blockIdx.x - plan.split0[b];
  int bi = 0, bidx = b;
  while (bidx >= plan.nbk - bi) { bidx -= plan.nbk - bi; ++bi; }
  const int bj = bi + bidx;
  const bool diag = bi == bj;
  const long long r0 = sp * plan.rps[b];
  long long r1 = r0 + plan.rps[b];
  if (r1 > nrows) r1 = nrows;
  const int nsteps = r1 > r0 ? (int)((r1 - r0) / G2_KC) : 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wi = warp >> 1, wj = warp & 1;
  const int ci0 = bi * 64 + wi * 32, cj0 = bj * 64 + wj * 32;
  const bool active = !(diag && wi > wj) && ci0 < k && cj0 < k;
  constexpr int EPC = 16 / (int)sizeof(T);     // elements per 16-byte chunk
  constexpr int CPC = G2_KC / EPC;             // chunks per column per stage
  const int nops = diag ? 1 : 2;               // a diagonal block stages its columns once
  auto load = [&](int step, int buf) {
    const long long row = r0 + (long long)step * G2_KC;
    for (int o = 0; o < nops; ++o) {
      const int cb = (o == 0 ? bi : bj) * 64;
      T* dst = sm + (size_t)(buf * 2 + o) * 64 * G2_LDS;
      for (int e = tid; e < 64 * CPC; e += G2_THREADS) {
        const int c = e / CPC, ch = e % CPC;
        const bool ok = cb + c < k;
        const T* src = ok ? Z + (long long)(cb + c) * ldz + row + ch * EPC : Z;
        cp_async16(dst + c * G2_LDS + ch * EPC, src, ok);
      }
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int s = 0; s < G2_ST - 1; ++s) {
    if (s < nsteps) load(s, s);
    cp_async_commit();
  }
  const int fr = (lane >> 2) * G2_LDS + (lane & 3);   // this lane's fragment offset
  for (int step = 0; step < nsteps; ++step) {
    cp_async_wait<G2_ST - 2>();
    __syncthreads();
    const int nx = step + G2_ST - 1;
    if (nx < nsteps) load(nx, nx % G2_ST);
    cp_async_commit();
    if (active) {
      const int buf = step % G2_ST;
      const T* sa = sm + ((size_t)(buf * 2) * 64 + wi * 32) * G2_LDS + fr;
      const T* sb = sm + ((size_t)(buf * 2 + (diag ? 0 : 1)) * 64 + wj * 32) * G2_LDS + fr;
#pragma unroll
      for (int kk = 0; kk < G2_KC; kk += 4) {
        double a[4], bb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = (double)sa[i * 8 * G2_LDS + kk];
#pragma unroll
        for (int j = 0; j < 4; ++j) bb[j] = (double)sb[j * 8 * G2_LDS + kk];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
      }
    }
  }
  cp_async_wait<0>();
  double* out = work + (size_t)blockIdx.x * 4096;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = wi * 32 + i * 8 + (lane >> 2), c = wj * 32 + j * 8 + 2 * (lane & 3);
      *reinterpret_cast<double2*>(out + r * 64 + c) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

// ---- (a0) G = Zᵀ Z, Blackwell-native variant (k <= 224; the default): one pass over Z.
// Measured at C4 (n = 24.9M fp32, k = 201): 51.6 ms = 19.6 TF/s useful (0.53 of the 37.1 TF/s
// DMMA peak), 20.0 GB DRAM read = the algorithmic bytes; the pair-blocked kernel below
// (SDMD_INIT_GRAM=v1): 72.3 ms, 79.2 GB (profiles/r2/r6f…).  A 4-CTA cluster owns a
// contiguous row range; per stage of R rows (128 bytes of each column: 32 fp32 / 16 fp64 rows) the
// k columns arrive as ceil(k/32) TMA boxes of 32 columns x R rows with the 128-byte swizzle, each
// CTA fetching a quarter of the boxes and MULTICASTING them into all four CTAs' shared memory, so
// every element of Z crosses HBM once (the pair-blocked kernel above re-reads each column block
// per pair).  The 28 (k = 201) upper-triangular 32x32 output tiles are spread one per warp over the
// 32 compute warps of the cluster (warp tile = 4x4 DMMA m8n8k4, lower 8x8 blocks of diagonal tiles
// skipped); a producer warp per CTA drives the TMA ring (full barriers with transaction counts,
// empty barriers that every consuming warp of the cluster releases remotely).  Per-cluster tiles
// are reduced in fixed order (deterministic).
static int g2_sm_count_early() {
  int d = 0, v = 148;
  cudaGetDevice(&d);
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
  return v;
}
constexpr int GM_CL = 4;                  // CTAs per cluster
constexpr int GM_WPC = 14;                // compute warps per CTA (two per output tile: k split; 7 tiles per CTA, 28 per cluster)
constexpr int GM_THREADS = (GM_WPC + 1) * 32;   // + one producer warp
constexpr int GM_ST = 3;                  // pipeline stages
constexpr int GM_RB = 2;                  // 128-byte row boxes per column tile per stage
constexpr int GM_MAXB = 7;                // column boxes (k <= 224)
constexpr int GM_BOX = 4096;              // bytes per box (32 columns x 128 bytes)

__device__ __forceinline__ unsigned gm_cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void gm_cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void gm_mbar_init(unsigned long long* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void gm_mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
               ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void gm_mbar_wait(unsigned long long* b, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(a), "r"(parity) : "memory");
}
// arrive on the barrier at the same offset in CTA `cta` of the cluster
__device__ __forceinline__ void gm_mbar_arrive_remote(unsigned long long* b, unsigned cta) {
  unsigned a = (unsigned)__cvta_generic_to_shared(b), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void gm_tma_multicast(void* dst, const CUtensorMap* tm, int c0, int c1,
                                                 unsigned long long* bar, unsigned short mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(tm), "r"(c0), "r"(c1),
        "r"((unsigned)__cvta_generic_to_shared(bar)), "h"(mask) : "memory");
}

// element (row r, column c) of a 32-column box with the 128-byte swizzle (16-byte chunk index
// XOR column mod 8)
template <typename T>
__device__ __forceinline__ T gm_ld(const unsigned char* box, int r, int c) {
  constexpr int EPC = 16 / (int)sizeof(T);
  const int chunk = (r / EPC) ^ (c & 7);
  return *reinterpret_cast<const T*>(box + c * 128 + chunk * 16 + (r % EPC) * (int)sizeof(T));
}

template <typename T>
__global__ void __cluster_dims__(GM_CL, 1, 1) __maxnreg__(128)
gram_mc_kernel(const __grid_constant__ CUtensorMap tm, long long nrows, int k, long long rpc,
               double* __restrict__ work) {
  extern __shared__ __align__(1024) unsigned char gm_raw[];
  unsigned char* gm = reinterpret_cast<unsigned char*>(((uintptr_t)gm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) unsigned long long full[GM_ST], empty[GM_ST];
  constexpr int R = 128 / (int)sizeof(T);           // rows per box (one 128-byte swizzle line)
  constexpr int RS = R * GM_RB;                      // rows per stage
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int crank = (int)gm_cl_rank();
  const long long cid = blockIdx.x / GM_CL;
  const int nb = (k + 31) / 32;                      // column boxes
  const int ntiles = nb * (nb + 1) / 2;
  const long long r0 = cid * rpc;
  long long r1 = r0 + rpc;
  if (r1 > nrows) r1 = nrows;
  const int nsteps = r1 > r0 ? (int)((r1 - r0) / RS) : 0;
  const unsigned stage_bytes = (unsigned)nb * GM_RB * GM_BOX;
  if (tid == 0) {
    for (int s = 0; s < GM_ST; ++s) {
      gm_mbar_init(&full[s], 1);
      gm_mbar_init(&empty[s], (unsigned)ntiles);       // the warp of each tile that consumed it
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  gm_cl_sync();
  if (warp == GM_WPC) {                              // producer
    if (lane == 0) {
      for (int st = 0; st < nsteps; ++st) {
        const int slot = st % GM_ST;
        if (st >= GM_ST) gm_mbar_wait(&empty[slot], (unsigned)(((st / GM_ST) - 1) & 1));
        gm_mbar_expect_tx(&full[slot], stage_bytes);
        const int row = (int)(r0 + (long long)st * RS);
        for (int b = crank; b < nb; b += GM_CL)
          for (int rb = 0; rb < GM_RB; ++rb)
            gm_tma_multicast(gm + (size_t)slot * stage_bytes + (size_t)(b * GM_RB + rb) * GM_BOX, &tm,
                             row + rb * R, b * 32, &full[slot], (unsigned short)((1u << GM_CL) - 1));
      }
    }
  } else {
    // warps w and w + GM_WPC/2 of a CTA share one output tile; half h consumes the stages st ≡ h
    // (mod 2) — 2·R rows, 16·GM_RB/2 DMMA k steps per barrier round trip
    const int half = warp / (GM_WPC / 2);
    const int gw = crank * (GM_WPC / 2) + warp % (GM_WPC / 2);
    int ti = 0, tj = 0;
    {
      int t = gw;
      while (ti < nb && t >= nb - ti) { t -= nb - ti; ++ti; }
      tj = ti + t;
    }
    const bool active = gw < ntiles;
    const bool diag = ti == tj;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int fr = lane & 3, fc = lane >> 2;          // fragment row (k) / column (m, n) of this lane
    // 128-byte swizzle: element (r, c) of a box at c·128 + ((chunk(r) ^ (c & 7)) << 4) + byte(r);
    // the fragment columns are i·8 + fc, so c & 7 = fc for every i
    auto frag_off = [&](int kk) -> int {
      const int rb = kk / R, kl = kk % R;
      if (sizeof(T) == 4) return rb * GM_BOX + ((((kl >> 2) ^ fc)) << 4) + fr * 4;
      return rb * GM_BOX + ((((kl + fr) >> 1) ^ fc) << 4) + ((fr & 1) << 3);
    };
    if (active) {
      for (int st = half; st < nsteps; st += 2) {
        const int slot = st % GM_ST;
        gm_mbar_wait(&full[slot], (unsigned)((st / GM_ST) & 1));
        const unsigned char* pa = gm + (size_t)slot * stage_bytes + (size_t)ti * GM_RB * GM_BOX + fc * 128;
        const unsigned char* pb = gm + (size_t)slot * stage_bytes + (size_t)tj * GM_RB * GM_BOX + fc * 128;
        double a[4], b[4], an[4], bn[4];
        {
          const int o = frag_off(0);
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = (double)*reinterpret_cast<const T*>(pa + i * 1024 + o);
#pragma unroll
          for (int j = 0; j < 4; ++j) b[j] = (double)*reinterpret_cast<const T*>(pb + j * 1024 + o);
        }
#pragma unroll
        for (int kk = 0; kk < RS; kk += 4) {
          if (kk + 4 < RS) {                             // next k step's fragments in flight
            const int o = frag_off(kk + 4);
#pragma unroll
            for (int i = 0; i < 4; ++i) an[i] = (double)*reinterpret_cast<const T*>(pa + i * 1024 + o);
#pragma unroll
            for (int j = 0; j < 4; ++j) bn[j] = (double)*reinterpret_cast<const T*>(pb + j * 1024 + o);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (!diag || i <= j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
#pragma unroll
          for (int i = 0; i < 4; ++i) { a[i] = an[i]; b[i] = bn[i]; }
        }
        __syncwarp();
        if (lane < GM_CL) gm_mbar_arrive_remote(&empty[slot], (unsigned)lane);   // release in every CTA
      }
    }
    // the two halves of a tile meet in shared memory (the ring is drained: every TMA write was
    // consumed before the last full-barrier wait), half 0 + half 1 in that order
    asm volatile("bar.sync 1, %0;" ::"r"(GM_WPC * 32) : "memory");
    double* tilebuf = reinterpret_cast<double*>(gm) + (size_t)(warp % (GM_WPC / 2)) * 32 * 32;
    if (active && half == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int li = i * 8 + (lane >> 2), lj = j * 8 + 2 * (lane & 3);
          tilebuf[li * 32 + lj] = acc[i][j][0];
          tilebuf[li * 32 + lj + 1] = acc[i][j][1];
        }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(GM_WPC * 32) : "memory");
    if (active && half == 1) {
      double* out = work + (size_t)cid * k * k;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int li = i * 8 + (lane >> 2), lj = j * 8 + 2 * (lane & 3);
          const int gi = ti * 32 + li, gj = tj * 32 + lj;
          if ((diag && i > j) || gi >= k) continue;
          if (gj < k) out[(size_t)gi * k + gj] = tilebuf[li * 32 + lj] + acc[i][j][0];
          if (gj + 1 < k) out[(size_t)gi * k + gj + 1] = tilebuf[li * 32 + lj + 1] + acc[i][j][1];
        }
    }
  }
  gm_cl_sync();                                       // no CTA leaves while others may arrive on it
}

// fixed-order sum of the per-cluster tiles; only entries i <= j were written (diagonal tiles:
// their upper 8x8 blocks, which cover every i <= j of the tile)
__global__ void gram_mc_reduce_kernel(const double* __restrict__ work, int ncl, int k, double* __restrict__ G) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)k * k;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / k), j = (int)(e % k);
    if (i > j) continue;
    double s = 0.0;
    for (int c = 0; c < ncl; ++c) s += work[(size_t)c * k * k + e];
    G[(long long)j * k + i] = s;
    G[(long long)i * k + j] = s;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 gm_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

static int gm_clusters() { return g2_sm_count_early() / GM_CL; }

__global__ void gram_tc_reduce_kernel(const double* __restrict__ work, const GramPlan plan, int k,
                                      double* __restrict__ G) {
  const int b = blockIdx.x;
  int bi = 0, bidx = b;
  while (bidx >= plan.nbk - bi) { bidx -= plan.nbk - bi; ++bi; }
  const int bj = bi + bidx;
  const int s0 = plan.split0[b], s1 = plan.split0[b + 1];
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) {
    const int i = bi * 64 + e / 64, j = bj * 64 + e % 64;
    if (i > j || j >= k) continue;             // upper triangle only; mirrored below
    double s = 0.0;
    for (int q = s0; q < s1; ++q) s += work[(size_t)q * 4096 + e];
    G[(long long)j * k + i] = s;
    G[(long long)i * k + j] = s;
  }
}

static int g2_sm_count() {
  static int nsm = [] {
    int d = 0, v = 148;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    return v;
  }();
  return nsm;
}

template <typename T>
static size_t g2_smem() { return (size_t)G2_ST * 2 * 64 * G2_LDS * sizeof(T); }

// Row splits per block proportional to the block's active warp tiles (equal work per CTA).
static bool g2_plan(long long nrows, int k, int max_ctas, GramPlan& pl) {
  pl.nbk = (k + 63) / 64;
  pl.nblk = pl.nbk * (pl.nbk + 1) / 2;
  if (pl.nblk > G2_MAXB) return false;
  int act[G2_MAXB];
  long long tot = 0;
  for (int b = 0, bi = 0, bj = 0; b < pl.nblk; ++b) {
    int a = 0;
    for (int wi = 0; wi < 2; ++wi)
      for (int wj = 0; wj < 2; ++wj)
        if (!(bi == bj && wi > wj) && bi * 64 + wi * 32 < k && bj * 64 + wj * 32 < k) ++a;
    act[b] = a;
    tot += a;
    if (++bj == pl.nbk) { ++bi; bj = bi; }
  }
  const long long steps = nrows / G2_KC;
  // work per CTA (warp-tile steps), at least 8 steps of a full block
  long long per = (tot * steps + max_ctas - 1) / max_ctas;
  if (per < 32) per = 32;
  // per-block rounding can exceed max_ctas (a partial second wave doubles the time): grow the
  // per-CTA work until the whole grid is one wave
  for (;;) {
    pl.split0[0] = 0;
    for (int b = 0; b < pl.nblk; ++b) {
      long long sps = act[b] > 0 ? (per + act[b] - 1) / act[b] : steps;   // steps per split
      if (sps < 1) sps = 1;
      pl.rps[b] = sps * G2_KC;
      const long long ns = act[b] > 0 ? (steps + sps - 1) / sps : 0;
      pl.split0[b + 1] = pl.split0[b] + (int)ns;
    }
    if (pl.split0[pl.nblk] <= max_ctas) break;
    per += per / 128 + 1;
  }
  for (int b = pl.nblk; b < G2_MAXB; ++b) pl.rps[b] = 0;
  return true;
}

static int g2_max_ctas() { return g2_sm_count() * G2_MAXCTA_PER_SM + G2_MAXB; }

size_t init_gram_work_elems(long long n, int k) {
  (void)n;
  const size_t a = (size_t)g2_max_ctas() * 4096, b = (size_t)gm_clusters() * k * k;
  return a > b ? a : b;
}

// the one-pass cluster/TMA-multicast kernel: k <= 224 (one 32x32 tile per compute warp), a tensor
// map over the ring's first k slots; SDMD_INIT_GRAM=v1 selects the pair-blocked kernel (A/B)
static cudaError_t launch_init_gram_mc(const void* Z, long long ldz, int dtype, long long n, int k,
                                       double* Gout, double* work, cudaStream_t s, bool* used) {
  *used = false;
  static const bool v1 = [] { const char* e = std::getenv("SDMD_INIT_GRAM"); return e && std::strcmp(e, "v1") == 0; }();
  if (v1 || k > GM_MAXB * 32 || k < 2) return cudaSuccess;
  PFN_cuTensorMapEncodeTiled_v12000 enc = gm_encode();
  if (!enc) return cudaSuccess;
  const int es = dtype == 0 ? 4 : 8;
  const int R = 128 / es * GM_RB;                    // rows per stage
  const long long nrows = (n + R - 1) / R * R;
  if (nrows > ldz || (ldz * es) % 16 != 0 || ((uintptr_t)Z & 15) != 0) return cudaSuccess;
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)ldz, (cuuint64_t)k};
  const cuuint64_t strides[1] = {(cuuint64_t)ldz * es};
  const cuuint32_t box[2] = {(cuuint32_t)(128 / es), 32u};
  const cuuint32_t estr[2] = {1u, 1u};
  if (enc(&tm, dtype == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
          const_cast<void*>(Z), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaSuccess;                              // fall back to the pair-blocked kernel
  const int nb = (k + 31) / 32;
  size_t smem = (size_t)GM_ST * nb * GM_RB * GM_BOX;
  if (smem < (size_t)(GM_WPC / 2) * 32 * 32 * sizeof(double)) smem = (size_t)(GM_WPC / 2) * 32 * 32 * sizeof(double);
  smem += 1024;                                      // alignment slack (128-byte swizzle: 1024 B)
  const void* kfn = dtype == 0 ? (const void*)gram_mc_kernel<float> : (const void*)gram_mc_kernel<double>;
  cudaError_t e;
  if ((e = set_max_dyn_smem(kfn, (int)smem)) != cudaSuccess) return e;
  // one wave: only as many 4-CTA clusters as fit the GPCs at once (measured: 33 of the 37 that 148
  // SMs would suggest; a 38th..37th cluster would run as a second wave and double the time)
  int ncl = 0;
  {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(GM_CL * gm_clusters());
    lc.blockDim = dim3(GM_THREADS);
    lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = GM_CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&ncl, kfn, &lc) != cudaSuccess) { cudaGetLastError(); ncl = 0; }
  }
  if (ncl > gm_clusters()) ncl = gm_clusters();
  if (ncl < 1) return cudaSuccess;
  long long rpc = (nrows + ncl - 1) / ncl;
  rpc = (rpc + R - 1) / R * R;
  if (dtype == 0)
    gram_mc_kernel<float><<<ncl * GM_CL, GM_THREADS, smem, s>>>(tm, nrows, k, rpc, work);
  else
    gram_mc_kernel<double><<<ncl * GM_CL, GM_THREADS, smem, s>>>(tm, nrows, k, rpc, work);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  gram_mc_reduce_kernel<<<148, 256, 0, s>>>(work, ncl, k, Gout);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  *used = true;
  return cudaSuccess;
}

// Z: ld-strided columns whose rows [n, roundup(n, 32)) are zero (the ring's padding).
cudaError_t launch_init_gram(const void* Z, long long ldz, int dtype, long long n, int k,
                             double* Gout, double* work, cudaStream_t s) {
  {
    bool used = false;
    const cudaError_t e = launch_init_gram_mc(Z, ldz, dtype, n, k, Gout, work, s, &used);
    if (e != cudaSuccess || used) return e;
  }
  const long long nrows = (n + G2_KC - 1) / G2_KC * G2_KC;
  if (nrows > ldz) return cudaErrorInvalidValue;
  int occ = 1;
  cudaError_t e;
  const size_t smem = dtype == 0 ? g2_smem<float>() : g2_smem<double>();
  if (dtype == 0) {
    if ((e = set_max_dyn_smem((const void*)gram_tc_kernel<float>, (int)smem)) != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gram_tc_kernel<float>, G2_THREADS, smem);
  } else {
    if ((e = set_max_dyn_smem((const void*)gram_tc_kernel<double>, (int)smem)) != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gram_tc_kernel<double>, G2_THREADS, smem);
  }
  if (occ < 1) occ = 1;
  if (occ > G2_MAXCTA_PER_SM) occ = G2_MAXCTA_PER_SM;
  GramPlan pl{};
  if (!g2_plan(nrows, k, g2_sm_count() * occ, pl)) return cudaErrorInvalidValue;
  const int grid = pl.split0[pl.nblk];
  if (grid > g2_max_ctas()) return cudaErrorInvalidValue;
  if (grid > 0) {
    if (dtype == 0)
      gram_tc_kernel<float><<<grid, G2_THREADS, smem, s>>>((const float*)Z, ldz, nrows, k, pl, work);
    else
      gram_tc_kernel<double><<<grid, G2_THREADS, smem, s>>>((const double*)Z, ldz, nrows, k, pl, work);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  gram_tc_reduce_kernel<<<pl.nblk, 256, 0, s>>>(work, pl, k, Gout);
  return cudaGetLastError();
}

// ---- (a12) Φ = X'(Y W): CTA = 128 rows x 32 complex modes (64 real columns), 8 warps (4x2 warp
// tiles of 32x32), k = the m window columns of X' staged 16 at a time.  1-D grid, the mode
// chunks of one row tile adjacent (they re-read the same X' rows from L2).
constexpr int M2_ROWS = 128, M2_COLS = 64, M2_KC = 16, M2_ST = 3, M2_THREADS = 256;
constexpr int M2_LDB = M2_COLS + 4;       // staged T stride (doubles)
template <typename T> struct M2L { static constexpr int A = sizeof(T) == 4 ? M2_ROWS + 8 : M2_ROWS + 4; };

template <typename T>
static size_t m2_smem() { return (size_t)M2_ST * (M2_KC * M2L<T>::A * sizeof(T) + M2_KC * M2_LDB * sizeof(double)); }

template <typename T>
__global__ void __launch_bounds__(M2_THREADS) modes_tc_kernel(const T* __restrict__ ring, long long ld,
                                                             int NS, long long n, long long first_frame,
                                                             int m, const double2* __restrict__ Tm,
                                                             int nc, double2* __restrict__ phi,
                                                             long long ldphi, int nchunks) {
  extern __shared__ __align__(16) unsigned char m2_smem_raw[];
  constexpr int LDA = M2L<T>::A;
  constexpr int ABYTES = M2_KC * LDA * (int)sizeof(T);
  constexpr int SBYTES = ABYTES + M2_KC * M2_LDB * (int)sizeof(double);
  const long long rt = blockIdx.x / nchunks;
  const int q0 = (int)(blockIdx.x % nchunks) * (M2_COLS / 2);
  const long long row0 = rt * M2_ROWS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wi = warp >> 1, wj = warp & 1;
  constexpr int EPC = 16 / (int)sizeof(T);
  constexpr int CPR = M2_ROWS / EPC;           // chunks per window column
  const int nsteps = (m + M2_KC - 1) / M2_KC;
  auto load = [&](int step, int buf) {
    unsigned char* base = m2_smem_raw + (size_t)buf * SBYTES;
    T* sA = reinterpret_cast<T*>(base);
    double* sB = reinterpret_cast<double*>(base + ABYTES);
    const int k0 = step * M2_KC;
    for (int e = tid; e < M2_KC * CPR; e += M2_THREADS) {
      const int kk = e / CPR, ch = e % CPR, kc = k0 + kk;
      const bool ok = kc < m;
      const T* src = ok ? ring + ((first_frame + kc) % NS) * ld + row0 + ch * EPC : ring;
      cp_async16(sA + kk * LDA + ch * EPC, src, ok);
    }
    for (int e = tid; e < M2_KC * (M2_COLS / 2); e += M2_THREADS) {
      const int kk = e / (M2_COLS / 2), q = e % (M2_COLS / 2), kc = k0 + kk;
      const bool ok = kc < m && q0 + q < nc;
      const double2* src = ok ? Tm + (long long)(q0 + q) * m + kc : Tm;
      cp_async16(sB + kk * M2_LDB + 2 * q, src, ok);
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int s = 0; s < M2_ST - 1; ++s) {
    if (s < nsteps) load(s, s);
    cp_async_commit();
  }
  for (int step = 0; step < nsteps; ++step) {
    cp_async_wait<M2_ST - 2>();
    __syncthreads();
    const int nx = step + M2_ST - 1;
    if (nx < nsteps) load(nx, nx % M2_ST);
    cp_async_commit();
    const unsigned char* base = m2_smem_raw + (size_t)(step % M2_ST) * SBYTES;
    const T* sa = reinterpret_cast<const T*>(base) + (lane & 3) * LDA + wi * 32 + (lane >> 2);
    const double* sb = reinterpret_cast<const double*>(base + ABYTES) + (lane & 3) * M2_LDB + wj * 32 + (lane >> 2);
#pragma unroll
    for (int kk = 0; kk < M2_KC; kk += 4) {
      double a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = (double)sa[kk * LDA + i * 8];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = sb[kk * M2_LDB + j * 8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long row = row0 + wi * 32 + i * 8 + (lane >> 2);
    if (row >= n) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int q = q0 + (wj * 32 + j * 8) / 2 + (lane & 3);      // columns (2q, 2q+1) = (re, im)
      if (q < nc) phi[(long long)q * ldphi + row] = make_double2(acc[i][j][0], acc[i][j][1]);
    }
  }
}

cudaError_t launch_modes(const void* ring, long long ld, int NS, int dtype, long long n,
                         long long first_frame, int m, const double* T, int nc, double* phi,
                         long long ldphi, cudaStream_t s) {
  const int nchunks = (nc + M2_COLS / 2 - 1) / (M2_COLS / 2);
  const long long rts = (n + M2_ROWS - 1) / M2_ROWS;
  if (rts * M2_ROWS > ld) return cudaErrorInvalidValue;
  const long long grid = rts * nchunks;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
  cudaError_t e;
  if (dtype == 0) {
    const size_t sm = m2_smem<float>();
    if ((e = set_max_dyn_smem((const void*)modes_tc_kernel<float>, (int)sm)) != cudaSuccess) return e;
    modes_tc_kernel<float><<<(unsigned)grid, M2_THREADS, sm, s>>>((const float*)ring, ld, NS, n, first_frame, m,
                                                                  (const double2*)T, nc, (double2*)phi, ldphi, nchunks);
  } else {
    const size_t sm = m2_smem<double>();
    if ((e = set_max_dyn_smem((const void*)modes_tc_kernel<double>, (int)sm)) != cudaSuccess) return e;
    modes_tc_kernel<double><<<(unsigned)grid, M2_THREADS, sm, s>>>((const double*)ring, ld, NS, n, first_frame, m,
                                                                   (const double2*)T, nc, (double2*)phi, ldphi, nchunks);
  }
  return cudaGetLastError();
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

// T = Y W for every mode (per-frame modes, NEXT-2): r read on the device; columns r..r_max-1 = 0.
__global__ void make_T_all_kernel(const double* Y, int m, const K4Result* res, int r_max,
                                  const double2* W, double2* T) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= m * r_max) return;
  const int r = ((volatile const K4Result*)res)->r;
  const int k = idx % m, q = idx / m;
  double2 s = make_double2(0.0, 0.0);
  if (q < r) {
    for (int i = 0; i < r; ++i) {
      const double y = Y[(long long)i * m + k];
      const double2 w = W[(long long)q * r + i];
      s.x = fma(y, w.x, s.x);
      s.y = fma(y, w.y, s.y);
    }
  }
  T[idx] = s;
}

cudaError_t launch_make_T_all(const double* Y, int m, const K4Result* res, int r_max,
                              const double2* W, double* T, cudaStream_t s) {
  const int n = m * r_max;
  make_T_all_kernel<<<(n + 255) / 256, 256, 0, s>>>(Y, m, res, r_max, W, (double2*)T);
  return cudaGetLastError();
}

cudaError_t launch_make_T(const double* Y, int m, int r, const double2* W, const int* cols, int nc,
                          double* T, cudaStream_t s) {
  const int n = m * nc;
  make_T_kernel<<<(n + 255) / 256, 256, 0, s>>>(Y, m, r, W, cols, nc, (double2*)T);
  return cudaGetLastError();
}

}  // namespace sdmd
