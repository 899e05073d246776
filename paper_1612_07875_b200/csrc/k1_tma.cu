// k1_tma.cu — K1 (hot kernel): streaming Gram column + fused background column, TMA-pipelined.
//
// Same mathematics as described in k1_gram.cu's header (§3.1; Alg 1; Alg 3
// P:337-339), organised B200-first:
//   * one persistent CTA per SM (grid = #SMs − eigen workers), 15 consumer warps + 1 producer warp (512 threads, <= 128 registers);
//   * the producer's elected lane streams 1 KB column chunks of the current row tile from the HBM
//     ring into a 5-stage shared-memory ring with cp.async.bulk (TMA bulk copies, L2 evict-first),
//     15 chunks (one per consumer warp) per stage, completion tracked by mbarrier transaction
//     counts — ~80 KB in flight per SM without spending registers on it;
//   * consumer warp w owns union positions p ≡ w (mod 15): its per-lane fp64 dot accumulators stay
//     in registers for the whole kernel (one warp reduction per column at the end, fixed order);
//   * the background partial sums of a tile are reduced across warps through a double-buffered
//     shared array behind a consumer-only named barrier, so the producer keeps prefetching the next
//     tile while consumers reduce (no pipeline drain at tile boundaries);
//   * position 0 of every tile is the new frame x_t itself (its chunk doubles as the x operand).
#include "sdmd_internal.cuh"

namespace sdmd {

constexpr int KT_CONSUMERS = 15;                       // consumer warps (= chunks per stage); +1 producer = 512 threads
constexpr int KT_THREADS = (KT_CONSUMERS + 1) * 32;    // + 1 producer warp
constexpr int KT_STAGES = 5;
constexpr int KT_CHUNK = 1024;                         // bytes per column chunk
constexpr int KT_STAGE_BYTES = KT_CONSUMERS * KT_CHUNK;
constexpr int KT_MAXU = kMaxM + kMaxLag;
constexpr int KT_MAXG = (KT_MAXU + KT_CONSUMERS - 1) / KT_CONSUMERS;
constexpr int KT_PSTRIDE = kMaxM + 16;

// ---------------------------------------------------------------- PTX helpers ---------------
static __device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
static __device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
static __device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
static __device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
static __device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
static __device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                                unsigned long long* bar, unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
static __device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
static __device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(KT_CONSUMERS * 32) : "memory");
}

static __device__ __forceinline__ double kt_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// lane's 8 (f32) or 4 (f64) elements of a 1 KB chunk: bytes [16 lane, +16) and [512 + 16 lane, +16)
template <typename T> struct Chunk;
template <> struct Chunk<float> {
  static constexpr int E = 8;
  static constexpr int ROWS = 256;
  static __device__ __forceinline__ void load(const unsigned char* c, int lane, double* d) {
    const float4 a = *reinterpret_cast<const float4*>(c + 16 * lane);
    const float4 b = *reinterpret_cast<const float4*>(c + 512 + 16 * lane);
    d[0] = a.x; d[1] = a.y; d[2] = a.z; d[3] = a.w; d[4] = b.x; d[5] = b.y; d[6] = b.z; d[7] = b.w;
  }
  static __device__ __forceinline__ int row(int lane, int e) { return (e >> 2) * 128 + lane * 4 + (e & 3); }
};
template <> struct Chunk<double> {
  static constexpr int E = 4;
  static constexpr int ROWS = 128;
  static __device__ __forceinline__ void load(const unsigned char* c, int lane, double* d) {
    const double2 a = *reinterpret_cast<const double2*>(c + 16 * lane);
    const double2 b = *reinterpret_cast<const double2*>(c + 512 + 16 * lane);
    d[0] = a.x; d[1] = a.y; d[2] = b.x; d[3] = b.y;
  }
  static __device__ __forceinline__ int row(int lane, int e) { return (e >> 1) * 64 + lane * 2 + (e & 1); }
};

size_t k1_tma_smem_bytes(int dtype, int bg) {
  const int rows = dtype == 0 ? 256 : 128;
  size_t s = (size_t)KT_STAGES * KT_STAGE_BYTES;
  if (bg) s += 2 * (size_t)KT_CONSUMERS * rows * sizeof(double2) + (size_t)kMaxM * sizeof(double2);
  s += 2 * KT_STAGES * sizeof(unsigned long long) + 64;
  return s;
}

template <typename T, bool BG>
__global__ void __launch_bounds__(KT_THREADS, 1) k1_tma_kernel(const K1Params p) {
  using CH = Chunk<T>;
  constexpr int E = CH::E, ROWS = CH::ROWS;
  extern __shared__ __align__(128) unsigned char kt_smem[];
  unsigned char* stages = kt_smem;
  double2* red = reinterpret_cast<double2*>(kt_smem + KT_STAGES * KT_STAGE_BYTES);
  double2* c_s = red + (BG ? 2 * KT_CONSUMERS * ROWS : 0);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(c_s + (BG ? kMaxM : 0));
  unsigned long long* empty = full + KT_STAGES;
  __shared__ int am_last;

  if (*(volatile int*)&p.st->status != 0) return;      // stream poisoned (header contract)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long f_dot0 = p.f_new - p.nd + 1;
  const long long f_bg0 = p.f_bg - p.m + 1;
  const long long F0 = BG ? (f_dot0 < f_bg0 ? f_dot0 : f_bg0) : f_dot0;
  const int U = (int)(p.f_new - F0 + 1);                // union columns (x_new included)
  const int G = (U + KT_CONSUMERS - 1) / KT_CONSUMERS;  // stages per tile
  const long long NT = p.ld / ROWS;
  if (tid == 0) {
    for (int s = 0; s < KT_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], KT_CONSUMERS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (BG)
    for (int k = tid; k < p.m; k += KT_THREADS) c_s[k] = p.cbg[k];
  __syncthreads();

  // union position -> frame: position 0 is the new frame, then oldest .. f_new-1
  auto frame_of = [&](int pos) -> long long { return pos == 0 ? p.f_new : F0 + pos - 1; };
  const T* ring = (const T*)p.ring;

  double accv[KT_MAXG];
#pragma unroll
  for (int g = 0; g < KT_MAXG; ++g) accv[g] = 0.0;

  if (warp == KT_CONSUMERS) {
    // ------------------------------------------------------------ producer warp -------------
    if (lane == 0) {
      const unsigned long long pol = evict_first_policy();
      int stage = 0;
      unsigned phase = 0;
      for (long long tile = blockIdx.x; tile < NT; tile += gridDim.x) {
        const long long row0 = tile * ROWS;
        for (int g = 0; g < G; ++g) {
          mbar_wait(&empty[stage], phase ^ 1u);
          const int ncol = min(KT_CONSUMERS, U - g * KT_CONSUMERS);
          mbar_arrive_expect_tx(&full[stage], (unsigned)(ncol * KT_CHUNK));
          unsigned char* dst = stages + stage * KT_STAGE_BYTES;
          for (int c = 0; c < ncol; ++c) {
            const long long f = frame_of(g * KT_CONSUMERS + c);
            const T* src = ring + (f % p.NS) * p.ld + row0;
            bulk_g2s(dst + c * KT_CHUNK, src, KT_CHUNK, &full[stage], pol);
          }
          if (++stage == KT_STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ consumer warps ------------
    int stage = 0;
    unsigned phase = 0;
    int buf = 0;
    for (long long tile = blockIdx.x; tile < NT; tile += gridDim.x) {
      const long long row0 = tile * ROWS;
      double xd[E];
      double bre[BG ? E : 1], bim[BG ? E : 1];
      if (BG) {
#pragma unroll
        for (int e = 0; e < E; ++e) { bre[e] = 0.0; bim[e] = 0.0; }
      }
#pragma unroll
      for (int g = 0; g < KT_MAXG; ++g) {
        if (g < G) {
          mbar_wait(&full[stage], phase);
          const unsigned char* sb = stages + stage * KT_STAGE_BYTES;
          if (g == 0) CH::load(sb, lane, xd);                      // chunk 0 = x_t
          const int pos = g * KT_CONSUMERS + warp;
          if (pos < U) {
            double zd[E];
            CH::load(sb + warp * KT_CHUNK, lane, zd);
            const long long f = frame_of(pos);
            if (f >= f_dot0) {
              double s0 = 0.0, s1 = 0.0;
#pragma unroll
              for (int e = 0; e < E; e += 2) { s0 = fma(xd[e], zd[e], s0); s1 = fma(xd[e + 1], zd[e + 1], s1); }
              accv[g] += s0 + s1;
            }
            if (BG) {
              const long long kb = f - f_bg0;
              if (kb >= 0 && kb < p.m) {
                const double2 c = c_s[kb];
#pragma unroll
                for (int e = 0; e < E; ++e) { bre[e] = fma(c.x, zd[e], bre[e]); bim[e] = fma(c.y, zd[e], bim[e]); }
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stage]);
          if (++stage == KT_STAGES) { stage = 0; phase ^= 1u; }
        }
      }
      if (BG) {
        double2* rb = red + buf * (KT_CONSUMERS * ROWS);
#pragma unroll
        for (int e = 0; e < E; ++e) rb[warp * ROWS + CH::row(lane, e)] = make_double2(bre[e], bim[e]);
        consumer_bar();
        if (tid < ROWS) {
          double sx = 0.0, sy = 0.0;
#pragma unroll
          for (int w = 0; w < KT_CONSUMERS; ++w) { const double2 v = rb[w * ROWS + tid]; sx += v.x; sy += v.y; }
          const long long row = row0 + tid;
          if (row < p.n) {
            const double l = hypot(sx, sy);                           // |l| (Q8)
            const double xv = (double)__ldcg(ring + (p.f_bg % p.NS) * p.ld + row);
            const double sp = xv - l;                                 // s = x - |l|
            ((T*)p.lowrank)[row] = (T)l;
            ((T*)p.sparse)[row] = (T)sp;
            p.mask[row] = (sp > (double)p.thr) ? 1 : 0;               // strict '>'
          }
        }
        buf ^= 1;
      }
    }
    // per-column reduction of the lane accumulators (fixed order) -> this CTA's partials
#pragma unroll
    for (int g = 0; g < KT_MAXG; ++g) {
      const int pos = g * KT_CONSUMERS + warp;
      if (g < G && pos < U) {
        const double s = kt_warp_sum(accv[g]);
        const long long f = frame_of(pos);
        if (lane == 0 && f >= f_dot0) p.partials[(long long)blockIdx.x * KT_PSTRIDE + (f - f_dot0)] = s;
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned prev = atomicAdd(&p.st->k1_done, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  for (int k = tid; k < p.nd; k += KT_THREADS) {
    double s = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) s += __ldcg(&p.partials[(long long)b * KT_PSTRIDE + k]);
    p.gout[k] = s;
  }
  if (tid == 0) {
    p.st->k1_done = 0;
    if (BG) p.st->bg_frame = p.f_bg;
  }
  if (p.do_commit) {
    __syncthreads();
    commit_block(p.gout, p.nd, p.m, p.f_new, p.ghist, p.NH, p.st);
  }
}

template <typename T, bool BG>
static cudaError_t launch_tma_t(const K1Params& p, int grid, cudaStream_t s) {
  const size_t smem = k1_tma_smem_bytes(sizeof(T) == 4 ? 0 : 1, BG ? 1 : 0);
  cudaError_t e = cudaFuncSetAttribute(k1_tma_kernel<T, BG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  k1_tma_kernel<T, BG><<<grid, KT_THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_k1_tma(const K1Params& p, int dtype, int grid, cudaStream_t s) {
  if (dtype == 0) return p.bg ? launch_tma_t<float, true>(p, grid, s) : launch_tma_t<float, false>(p, grid, s);
  return p.bg ? launch_tma_t<double, true>(p, grid, s) : launch_tma_t<double, false>(p, grid, s);
}

}  // namespace sdmd
