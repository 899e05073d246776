// k1b_batch.cu — K1b: the Gram columns of k ≤ 8 newly arrived frames in ONE pass over the window
// (the paper's future-work item "dynamic updating with more than one column
// at a time; when data inputs slow down, the number of new columns processed may be increased to
// catch up").
//
// For new frames f0 .. f0+k-1 the union of their windows is U = m + k ring columns (frames
// f0-m .. f0+k-1).  The pass forms the thin product D = Z_Uᵀ X_new (U x k, fp64 accumulation of
// exact fp32/fp64 products, reading Q9) on the tensor pipe: DMMA m8n8k4 with the union columns as
// M (8-column groups), the new frames as N (k ≤ 8, zero-padded) and the rows as K.  The row tiles
// of all U columns are staged in shared memory by a cp.async pipeline (each window element is read
// from HBM once per batch instead of once per frame), the new frames' B fragments come from the
// same staged tile.  Frame f0+j's Gram column is g_j[i] = D[j+i][j] = <x_{f0+j-m+i}, x_{f0+j}>,
// i = 0..m (Alg 1 P:294 per frame, reading Q1/Q2).  Per-CTA partial blocks are reduced in fixed
// order by the last CTA (bitwise reproducible), which then commits the k columns atomically: a
// batch containing a non-finite value is rejected as a whole (S:285 extended to batches).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "sdmd_internal.cuh"

namespace sdmd {

constexpr int KB_WARPS = 16;
constexpr int KB_THREADS = KB_WARPS * 32;
constexpr int KB_CSETS = 8;                                     // column sets (warp & 7)
constexpr int KB_RHALF = KB_WARPS / KB_CSETS;                   // row parts of a stage (warp >> 3)
constexpr int KB_MAXU = kMaxM + kMaxBatch;                      // union columns
constexpr int KB_GPW = ((KB_MAXU + 7) / 8 + KB_CSETS - 1) / KB_CSETS;   // 8-column groups per warp

template <typename T> struct KbShape {
  static constexpr int ROWS = sizeof(T) == 4 ? 64 : 32;         // rows per stage
  static constexpr int ST = sizeof(T) == 4 ? 3 : 2;             // stages
  static constexpr int LDS = ROWS + 4;                          // conflict-free fragment loads
};

static __device__ __forceinline__ void kb_cp16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
static __device__ __forceinline__ void kb_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
static __device__ __forceinline__ void kb_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
static __device__ __forceinline__ void kb_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
static __device__ __forceinline__ double kb_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Atomic commit of the k Gram columns gout[j*(m+1) .. +m] (frame f0+j) into the history.
static __device__ void commit_batch(const double* gout, int k, int m, long long f0, double* ghist,
                                    int NH, DevState* st) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0x7fffffff;
  __syncthreads();
  for (int e = threadIdx.x; e < k * (m + 1); e += blockDim.x)
    if (!isfinite(gout[e])) atomicMin(&bad, e / (m + 1));
  __syncthreads();
  if (bad != 0x7fffffff) {
    if (threadIdx.x == 0) { st->status = 2 /*SDMD_E_NONFINITE*/; st->failed_frame = f0 + bad; poison_mirror(st); }
    return;
  }
  for (int e = threadIdx.x; e < k * (m + 1); e += blockDim.x) {
    const int j = e / (m + 1), i = e % (m + 1);
    ghist[((f0 + j) % NH) * (m + 1) + i] = gout[e];
  }
  __syncthreads();
  __threadfence();
  if (threadIdx.x == 0) *(volatile long long*)&st->committed = f0 + k;
}

template <typename T>
__global__ void __launch_bounds__(KB_THREADS, 1) k1b_kernel(const K1bParams p) {
  using S = KbShape<T>;
  extern __shared__ __align__(16) unsigned char kb_smem[];
  T* sm = reinterpret_cast<T*>(kb_smem);                        // [ST][U][LDS]
  __shared__ long long col_base[KB_MAXU];
  __shared__ int am_last;
  if (*(volatile int*)&p.st->status != 0) return;              // stream poisoned: discard
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = p.m, k = p.k, U = m + k, G = (U + 7) / 8;
  const long long F0 = p.f0 - m;
  for (int u = tid; u < U; u += KB_THREADS) col_base[u] = ((F0 + u) % p.NS) * p.ld;
  __syncthreads();
  const long long NT = (p.n + S::ROWS - 1) / S::ROWS;          // row tiles (ld ≥ NT·ROWS)
  const long long per = (NT + gridDim.x - 1) / gridDim.x;      // contiguous tiles per CTA
  const long long t0 = (long long)blockIdx.x * per;
  const long long t1 = t0 + per < NT ? t0 + per : NT;
  const int nsteps = t1 > t0 ? (int)(t1 - t0) : 0;
  constexpr int EPC = 16 / (int)sizeof(T);
  constexpr int CPC = S::ROWS / EPC;                            // 16-byte chunks per column
  const T* ring = reinterpret_cast<const T*>(p.ring);
  auto load = [&](int s, int buf) {
    const long long row0 = (t0 + s) * S::ROWS;
    T* dst = sm + (size_t)buf * U * S::LDS;
    for (int e = tid; e < U * CPC; e += KB_THREADS) {
      const int u = e / CPC, ch = e % CPC;
      kb_cp16(dst + u * S::LDS + ch * EPC, ring + col_base[u] + row0 + ch * EPC);
    }
  };
  double acc[KB_GPW][2];
#pragma unroll
  for (int g = 0; g < KB_GPW; ++g) acc[g][0] = acc[g][1] = 0.0;
  const int jb = lane >> 2;                                     // B fragment: new frame jb, row lane&3
  const bool bok = jb < k;
  const int ub = m + (bok ? jb : 0);
  // warp = (row part wr, column set wc): groups wc, wc+8, … over rows [wr·R/2, (wr+1)·R/2) of
  // each stage; the two row parts' partial sums are reduced with the CTA partials
  const int wr = warp / KB_CSETS, wc = warp % KB_CSETS;
  constexpr int RP = S::ROWS / KB_RHALF;                        // rows of a stage per warp
#pragma unroll
  for (int s = 0; s < S::ST - 1; ++s) {
    if (s < nsteps) load(s, s);
    kb_commit();
  }
  for (int step = 0; step < nsteps; ++step) {
    kb_wait<S::ST - 2>();
    __syncthreads();
    const int nx = step + S::ST - 1;
    if (nx < nsteps) load(nx, nx % S::ST);
    kb_commit();
    const T* Sb = sm + (size_t)(step % S::ST) * U * S::LDS + wr * RP + (lane & 3);
    // all fragments of the warp's RP rows first (independent shared-memory loads in flight),
    // then the conversions and DMMAs
    T bf[RP / 4], af[RP / 4][KB_GPW];
#pragma unroll
    for (int q = 0; q < RP / 4; ++q) {
      bf[q] = bok ? Sb[ub * S::LDS + 4 * q] : (T)0;
#pragma unroll
      for (int g = 0; g < KB_GPW; ++g) {
        const int u = (wc + g * KB_CSETS) * 8 + (lane >> 2);
        af[q][g] = u < U ? Sb[u * S::LDS + 4 * q] : (T)0;
      }
    }
#pragma unroll
    for (int q = 0; q < RP / 4; ++q) {
      const double b = (double)bf[q];
#pragma unroll
      for (int g = 0; g < KB_GPW; ++g)
        if (wc + g * KB_CSETS < G) kb_dmma(acc[g][0], acc[g][1], (double)af[q][g], b);   // warp-uniform
    }
  }
  kb_wait<0>();
  // per-CTA partial block D[u][j] (u < U, j < k): lane holds rows u = grp·8 + lane/4, columns
  // j = 2(lane%4) + {0, 1}
  const int np = gridDim.x * KB_RHALF;                          // partial sums per output
  const int pc = blockIdx.x * KB_RHALF + wr;
#pragma unroll
  for (int g = 0; g < KB_GPW; ++g) {
    const int grp = wc + g * KB_CSETS;
    const int u = grp * 8 + (lane >> 2), j = 2 * (lane & 3);
    if (grp < G && u < U) {
      if (j < k) p.partials[((long long)u * kMaxBatch + j) * np + pc] = acc[g][0];
      if (j + 1 < k) p.partials[((long long)u * kMaxBatch + j + 1) * np + pc] = acc[g][1];
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) am_last = (atomicAdd(&p.st->k1_done, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  // fixed-order reduction (warp per output), then g_j[i] = D[j+i][j]
  for (int o = warp; o < k * (m + 1); o += KB_WARPS) {
    const int j = o / (m + 1), i = o % (m + 1), u = j + i;
    const double* pk = p.partials + ((long long)u * kMaxBatch + j) * np;
    double s = 0.0;
    for (int b = lane; b < np; b += 32) s += __ldcg(pk + b);
    s = kb_warp_sum(s);
    if (lane == 0) p.gout[o] = s;
  }
  __syncthreads();
  if (tid == 0) p.st->k1_done = 0;
  if (p.do_commit) {
    __threadfence_block();
    commit_batch(p.gout, k, m, p.f0, p.ghist, p.NH, p.st);
  }
}

// ---- K1b with TMA tiles (default for rings <= 2 GB): the v1 kernel above moves each stage with
// ~3.3k 16-byte cp.async per CTA and reaches ~0.5 of the HBM rate (ncu at C4: the DMMA sub-pipe is
// the limiter, 54.5 % active under math-pipe throttle, profiles/r2/k1bn…; 256-byte cp.async.bulk
// per column was slower still, profiles/r2/r6l…).  Here a producer
// warp fetches a stage as 2-D TMA boxes of 16 ring slots x 128 bytes of rows (128-byte swizzle:
// conflict-free DMMA fragment loads) — 2·ceil(U/16) boxes per stage, plus two into a scratch region
// when a 16-slot group wraps past the ring's last slot (the out-of-range slots of the first box are
// zero-filled) — completing on the stage's full barrier; the 16 compute warps wait, load fragments,
// convert, issue DMMA and release the stage on its empty barrier.  Same partial layout, reduction
// and commit as v1.
__device__ __forceinline__ void kbt_mbar_init(unsigned long long* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void kbt_mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
               ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void kbt_mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void kbt_mbar_wait(unsigned long long* b, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "KBTW_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra KBTW_%=;\n}" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void kbt_tma2d(void* dst, const CUtensorMap* tm, int c0, int c1, unsigned long long* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(tm), "r"(c0), "r"(c1),
                 "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}

constexpr int KBT_THREADS = KB_THREADS + 32;                   // + the producer warp
constexpr int KBT_BOX = 2048;                                  // 16 slots x 128 bytes
constexpr int KBT_MAXG = (KB_MAXU + 15) / 16;                  // 16-slot groups

template <typename T>
__global__ void __maxnreg__(96) k1b_tma_kernel(const __grid_constant__ CUtensorMap tm, const K1bParams p) {
  constexpr int R = 128 / (int)sizeof(T);                       // rows per box (= rows per warp part)
  constexpr int RS = 2 * R;                                     // rows per stage (two row parts)
  constexpr int ST = 3;
  extern __shared__ __align__(1024) unsigned char kbt_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(((uintptr_t)kbt_raw + 1023) & ~(uintptr_t)1023);
  __shared__ int g_s0[KBT_MAXG];
  __shared__ __align__(8) unsigned long long full[ST], empty[ST];
  __shared__ int am_last;
  if (*(volatile int*)&p.st->status != 0) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = p.m, k = p.k, U = m + k, G = (U + 7) / 8, NG = (U + 15) / 16;
  const long long F0 = p.f0 - m;
  for (int g = tid; g < NG; g += KBT_THREADS) g_s0[g] = (int)((F0 + 16LL * g) % p.NS);
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) { kbt_mbar_init(&full[s], 1); kbt_mbar_init(&empty[s], KB_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int wg = -1;                                                  // the group that wraps (at most one)
  for (int g = 0; g < NG; ++g)
    if (g_s0[g] + 16 > p.NS) wg = g;
  const unsigned stage_bytes = (unsigned)(NG + 1) * 2 * KBT_BOX;
  const long long NT = (p.n + RS - 1) / RS;
  const long long per = (NT + gridDim.x - 1) / gridDim.x;
  const long long t0 = (long long)blockIdx.x * per;
  const long long t1 = t0 + per < NT ? t0 + per : NT;
  const int nsteps = t1 > t0 ? (int)(t1 - t0) : 0;
  double acc[KB_GPW][2];
#pragma unroll
  for (int g = 0; g < KB_GPW; ++g) acc[g][0] = acc[g][1] = 0.0;
  const int wr = warp / KB_CSETS, wc = warp % KB_CSETS;
  if (warp == KB_WARPS) {                                       // producer
    if (lane == 0) {
      const unsigned bytes = (unsigned)(NG + (wg >= 0 ? 1 : 0)) * 2 * KBT_BOX;
      for (int st = 0; st < nsteps; ++st) {
        const int slot = st % ST;
        if (st >= ST) kbt_mbar_wait(&empty[slot], (unsigned)(((st / ST) - 1) & 1));
        kbt_mbar_expect_tx(&full[slot], bytes);
        const int row0 = (int)((t0 + st) * RS);
        unsigned char* base = sm + (size_t)slot * stage_bytes;
        for (int g = 0; g < NG; ++g)
          for (int rb = 0; rb < 2; ++rb)
            kbt_tma2d(base + (size_t)(g * 2 + rb) * KBT_BOX, &tm, row0 + rb * R, g_s0[g], &full[slot]);
        if (wg >= 0)
          for (int rb = 0; rb < 2; ++rb)
            kbt_tma2d(base + (size_t)(NG * 2 + rb) * KBT_BOX, &tm, row0 + rb * R, 0, &full[slot]);
      }
    }
  } else {
    // byte offset (within a stage) of column u's line in this warp's row box, and its swizzle key
    auto col_off = [&](int u, int& key) -> int {
      const int g = u >> 4, c = u & 15, s0 = g_s0[g];
      int region = g, cc = c;
      if (s0 + c >= p.NS) { region = NG; cc = s0 + c - p.NS; }
      key = cc & 7;
      return (region * 2 + wr) * KBT_BOX + cc * 128;
    };
    const int jb = lane >> 2, fr = lane & 3;
    const bool bok = jb < k;
    int bkey, akey[KB_GPW];
    const int boff = col_off(m + (bok ? jb : 0), bkey);
    int aoff[KB_GPW];
    bool aok[KB_GPW];
#pragma unroll
    for (int g = 0; g < KB_GPW; ++g) {
      const int u = (wc + g * KB_CSETS) * 8 + (lane >> 2);
      aok[g] = u < U;
      aoff[g] = col_off(aok[g] ? u : 0, akey[g]);
    }
    // element (row rl of the box, line with key) inside the 128-byte swizzled line
    auto ld = [&](const unsigned char* st_base, int off, int key, int q) -> T {
      const int rl = 4 * q + fr;
      const int byte = rl * (int)sizeof(T);
      return *reinterpret_cast<const T*>(st_base + off + ((((byte >> 4) ^ key)) << 4) + (byte & 15));
    };
    for (int st = 0; st < nsteps; ++st) {
      const int slot = st % ST;
      kbt_mbar_wait(&full[slot], (unsigned)((st / ST) & 1));
      const unsigned char* sb = sm + (size_t)slot * stage_bytes;
#pragma unroll
      for (int q = 0; q < R / 4; ++q) {
        const double b = bok ? (double)ld(sb, boff, bkey, q) : 0.0;
#pragma unroll
        for (int g = 0; g < KB_GPW; ++g)
          if (wc + g * KB_CSETS < G) {
            const double a = aok[g] ? (double)ld(sb, aoff[g], akey[g], q) : 0.0;
            kb_dmma(acc[g][0], acc[g][1], a, b);
          }
      }
      __syncwarp();
      if (lane == 0) kbt_mbar_arrive(&empty[slot]);
    }
  }
  const int np = gridDim.x * KB_RHALF;
  const int pc = blockIdx.x * KB_RHALF + wr;
  if (warp < KB_WARPS) {
#pragma unroll
    for (int g = 0; g < KB_GPW; ++g) {
      const int grp = wc + g * KB_CSETS;
      const int u = grp * 8 + (lane >> 2), j = 2 * (lane & 3);
      if (grp < G && u < U) {
        if (j < k) p.partials[((long long)u * kMaxBatch + j) * np + pc] = acc[g][0];
        if (j + 1 < k) p.partials[((long long)u * kMaxBatch + j + 1) * np + pc] = acc[g][1];
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) am_last = (atomicAdd(&p.st->k1_done, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  for (int o = warp; o < k * (m + 1); o += KB_WARPS + 1) {
    const int j = o / (m + 1), i = o % (m + 1), u = j + i;
    const double* pk = p.partials + ((long long)u * kMaxBatch + j) * np;
    double s = 0.0;
    for (int b = lane; b < np; b += 32) s += __ldcg(pk + b);
    s = kb_warp_sum(s);
    if (lane == 0) p.gout[o] = s;
  }
  __syncthreads();
  if (tid == 0) p.st->k1_done = 0;
  if (p.do_commit) {
    __threadfence_block();
    commit_batch(p.gout, k, m, p.f0, p.ghist, p.NH, p.st);
  }
}

// tensor map over the ring (rows x slots), one per (ring, ld, NS, dtype)
static bool kbt_tensor_map(const K1bParams& p, int dtype, CUtensorMap* out) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, long long, int, int>, CUtensorMap> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(p.ring, p.ld, p.NS, dtype);
  auto it = cache.find(key);
  if (it != cache.end()) { *out = it->second; return true; }
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  if (!enc) return false;
  const int es = dtype == 0 ? 4 : 8;
  const cuuint64_t dims[2] = {(cuuint64_t)p.ld, (cuuint64_t)p.NS};
  const cuuint64_t strides[1] = {(cuuint64_t)p.ld * es};
  const cuuint32_t box[2] = {(cuuint32_t)(128 / es), 16u};
  const cuuint32_t estr[2] = {1u, 1u};
  CUtensorMap tm;
  if (enc(&tm, dtype == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
          const_cast<void*>(p.ring), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  cache[key] = tm;
  *out = tm;
  return true;
}

__global__ void commit_batch_kernel(const K1bParams p) {
  if (*(volatile int*)&p.st->status != 0) return;
  commit_batch(p.gout, p.k, p.m, p.f0, p.ghist, p.NH, p.st);
}

template <typename T>
static cudaError_t launch_k1b_t(const K1bParams& p, int grid, cudaStream_t s) {
  using S = KbShape<T>;
  // measured (profiles/r2/r6m…): the TMA kernel wins while the ring is small (C3 ring 0.85 GB: 0.87
  // vs 1.26 ms per 8-frame batch; C2: 0.21 vs 0.32 ms) and loses on the 21 GB C4 ring (10.8 vs
  // 8.1 ms: every 16-slot box touches 16 far-apart 2 MB pages); SDMD_K1B=v1|tma forces one.
  // (DMMA fragments loaded straight from the ring — one 16-byte load per lane, 64 contiguous bytes
  // per column and warp — measured 16.5 ms at C4: profiles/r2/r8k…, rejected)
  static const int force = [] {
    const char* e = std::getenv("SDMD_K1B");
    return !e ? 0 : std::strcmp(e, "v1") == 0 ? 1 : std::strcmp(e, "tma") == 0 ? 2 : 0;
  }();
  const double ring_bytes = (double)p.NS * (double)p.ld * (double)sizeof(T);
  const bool use_tma = force == 2 || (force == 0 && ring_bytes <= 2.0 * (1 << 30));
  CUtensorMap tm;
  if (use_tma && kbt_tensor_map(p, sizeof(T) == 4 ? 0 : 1, &tm)) {
    const int NG = (p.m + p.k + 15) / 16;
    const int smem = 3 * (NG + 1) * 2 * KBT_BOX + 1024;
    cudaError_t e = set_max_dyn_smem((const void*)k1b_tma_kernel<T>, smem);
    if (e != cudaSuccess) return e;
    k1b_tma_kernel<T><<<grid, KBT_THREADS, smem, s>>>(tm, p);
    return cudaGetLastError();
  }
  const int smem = S::ST * (p.m + p.k) * S::LDS * (int)sizeof(T);
  cudaError_t e = set_max_dyn_smem((const void*)k1b_kernel<T>, smem);
  if (e != cudaSuccess) return e;
  k1b_kernel<T><<<grid, KB_THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

int k1b_grid(int nsm, long long n, int dtype) {
  const int rows = dtype == 0 ? KbShape<float>::ROWS : KbShape<double>::ROWS;
  const long long nt = (n + rows - 1) / rows;
  long long g = (long long)nsm * 4;                             // 4 short waves (room for K4 CTAs)
  if (g > nt / 8) g = nt / 8 > nsm ? nt / 8 : nsm;              // small n: >= 8 tiles per CTA
  if (g > nt) g = nt;
  return g < 1 ? 1 : (int)g;
}

size_t k1b_partials_elems(int grid) { return (size_t)KB_MAXU * kMaxBatch * grid * KB_RHALF; }

cudaError_t launch_k1b(const K1bParams& p, int dtype, int grid, cudaStream_t s) {
  if (p.k < 1 || p.k > kMaxBatch || p.m + p.k > KB_MAXU) return cudaErrorInvalidValue;
  return dtype == 0 ? launch_k1b_t<float>(p, grid, s) : launch_k1b_t<double>(p, grid, s);
}

cudaError_t launch_commit_batch(const K1bParams& p, cudaStream_t s) {
  commit_batch_kernel<<<1, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace sdmd
