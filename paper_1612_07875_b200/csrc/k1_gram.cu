// k1_gram.cu — K1: streaming Gram column over the HBM ring (+ fused background column).
//
// Computes g_k = <x_{t-m+k}, x_t> for the nd newest window columns (§3.1: "only the
// last row or column will need to be recalculated"; Alg 1) in ONE pass over the ring, with
// fp64 accumulation of exact fp32/fp64 products (reading Q9).  When a background coefficient
// vector c_{t'} of an earlier frame t' = t - lag is ready, the same pass also forms
// l = X'_{t'} c_{t'} = b_idx φ_idx λ_idx^m (Alg 3, reading Q4) and s = x_{t'} - |l|,
// mask = s > threshold: the columns of X'_{t'} are streamed anyway, so the
// background costs no extra HBM reads beyond lag-1 columns.
//
// Two implementations of the same pass (bitwise-deterministic, different fixed summation orders):
//  * k1v2_kernel (default): 512-thread CTAs (one per SM), 128-row tiles, one 16-byte vector per
//    lane per column, warp w owns union columns j ≡ w (mod 16) and walks exactly NQ of them
//    (branch-free: columns past the union read the L1-resident x_t tile with a zero coefficient),
//    column batches double-buffered in registers across tiles, 32-bit slot offsets.  Background
//    partials are published per tile to shared memory and summed over the 16 warps by ONE
//    designated warp per tile, K1V2_LAGR tiles later (no lockstep reduction).
//  * k1_gram_kernel (v1, SDMD_K1=v1, A/B only): 8 rows per lane, all warps reduce every tile.
// Per-column partial dots stay in registers for the whole pass, are warp-reduced once, written
// per CTA, and the last CTA reduces the CTA partials in fixed order and commits the column into
// the Gram history (nranks == 1).  No floating-point atomics: results are bitwise reproducible.
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "sdmd_internal.cuh"

namespace sdmd {

#ifndef K1_NSLOT
#define K1_NSLOT 2        // background partial slots (tiles in flight between warps)
#endif
#ifndef K1_LAGR
#define K1_LAGR 1         // tiles between publishing and reducing
#endif
#ifndef K1_CB32
#define K1_CB32 4         // fp32 background LDG path: columns (2 LDG.128 each) in flight per lane
#endif
#ifndef K1V2_NBDIV
#define K1V2_NBDIV 16     // v2: batches per tile = 2·ceil(NQ / K1V2_NBDIV) (register budget)
#endif
#ifndef K1V2_LAGR
#define K1V2_LAGR 3       // v2: tiles between publishing background partials and reducing them
#endif
#ifndef K1V2_SLACK
#define K1V2_SLACK 1      // v2: extra reduction slots beyond the lag
#endif
#ifndef K1V2_SKIP
#define K1V2_SKIP 0       // v2 A/B: 1 = warps skip (warp-uniform branch) the dummy slots past their
                          // column count.  Measured slower (C4 pipeline pass 3.69 -> 4.78 ms at lag 9:
                          // the predicated loads defeat the register double-buffering), so off.
#endif
#ifndef K1V2_NORC
#define K1V2_NORC 0       // v2 A/B: 1 = always accumulate the complex background (no real fast path)
#endif
#ifndef K1V2_PF
#define K1V2_PF 0         // v2: L2 bulk-prefetch distance in tiles (0 = off)
#endif
#ifndef K1V2_DBG
#define K1V2_DBG 0        // v2 experiments: 1 = skip the background reduction, 2 = skip its FMAs
#endif
constexpr int K1_THREADS = 512;
constexpr int K1_WARPS = K1_THREADS / 32;
constexpr int K1_MAXU = kMaxM + kMaxLag;          // union columns: m + lag
constexpr int K1_NQMAX = (K1_MAXU + K1_WARPS - 1) / K1_WARPS;

template <typename T> struct VecOf;
template <> struct VecOf<float> { using type = float4; static constexpr int E = 4; };
template <> struct VecOf<double> { using type = double2; static constexpr int E = 2; };

__device__ __forceinline__ void to_double(const float4& v, double* d) {
  d[0] = (double)v.x; d[1] = (double)v.y; d[2] = (double)v.z; d[3] = (double)v.w;
}
__device__ __forceinline__ void to_double(const double2& v, double* d) { d[0] = v.x; d[1] = v.y; }

static __device__ __forceinline__ unsigned k1_smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
static __device__ __forceinline__ void k1_mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(k1_smem_u32(bar)), "r"(count));
}
static __device__ __forceinline__ void k1_mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(k1_smem_u32(bar)) : "memory");
}
#ifndef K1_MBAR_HINT
#define K1_MBAR_HINT 0    // ns: suspend-time hint of the mbarrier waits (0 = the default policy)
#endif
static __device__ __forceinline__ void k1_mbar_wait(unsigned long long* bar, unsigned parity) {
#if K1_MBAR_HINT > 0
  // the waiting warp is suspended (not spinning on issue slots) until the phase completes or the
  // hint expires
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "K1_WAIT:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra K1_DONE;\n\t"
      "bra K1_WAIT;\n"
      "K1_DONE:\n\t}" ::"r"(k1_smem_u32(bar)),
      "r"(parity), "n"(K1_MBAR_HINT)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "K1_WAIT:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra K1_DONE;\n\t"
      "bra K1_WAIT;\n"
      "K1_DONE:\n\t}" ::"r"(k1_smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}


// Background partial-sum slots: [K1_WARPS][8 elements x 40 lanes(32 + 8 pad)], conflict-free for
// both the per-warp writes (lanes contiguous) and the per-row reads of the reduction.
template <typename T> struct BgLayout { static constexpr int L = sizeof(T) == 4 ? 40 : 36; static constexpr int W = 8 * L; };

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

static __device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}

template <typename T> struct BgAcc;     // per-lane background accumulators of 8 rows (re, im)
template <> struct BgAcc<float> {
  // fp32 with packed FFMA2 on natural register pairs: re/im of rows (e, e+1); per-warp sums of
  // ~m/16 terms, then an fp64 cross-warp sum: error ~1e-6 relative, inside the fp32-path
  // tolerance (1e-4)
  using C2 = float2;                   // reduction-slot element (re, im) of one row
  using CW = float4;                   // per-column coefficient entry (c.x, c.x, c.y, c.y)
  float2 re[4], im[4];
  static __device__ __forceinline__ CW make(double2 c) {
    return make_float4((float)c.x, (float)c.x, (float)c.y, (float)c.y);
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < 4; ++i) { re[i] = make_float2(0.f, 0.f); im[i] = make_float2(0.f, 0.f); }
  }
  __device__ __forceinline__ void add(const CW c, const float* z) {
    const float2 cr = make_float2(c.x, c.y), ci = make_float2(c.z, c.w);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 zz = make_float2(z[2 * i], z[2 * i + 1]);
      re[i] = ffma2(cr, zz, re[i]);
      im[i] = ffma2(ci, zz, im[i]);
    }
  }
  __device__ __forceinline__ C2 get(int e) const {
    return (e & 1) ? make_float2(re[e >> 1].y, im[e >> 1].y) : make_float2(re[e >> 1].x, im[e >> 1].x);
  }
};
template <> struct BgAcc<double> {
  using C2 = double2;
  using CW = double2;
  double2 v[8];
  static __device__ __forceinline__ CW make(double2 c) { return c; }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = make_double2(0.0, 0.0);
  }
  __device__ __forceinline__ void add(const CW c, const double* z) {
#pragma unroll
    for (int e = 0; e < 8; ++e) { v[e].x = fma(c.x, z[e], v[e].x); v[e].y = fma(c.y, z[e], v[e].y); }
  }
  __device__ __forceinline__ C2 get(int e) const { return v[e]; }
};

template <typename T, bool BG, int NQ>
// One 512-thread CTA per SM (<= 128 registers).  Without the background: register streaming,
// 16 warps x CB columns x 2 LDG.128 per lane in flight, with or without the background.  (A
// bulk-copy ring variant of the background path measured slower: its 210 KB of shared memory
// starves L1 and couples the warps — removed.)
__global__ void __launch_bounds__(K1_THREADS, 1) k1_gram_kernel(const K1Params p) {
  using VT = typename VecOf<T>::type;
  using BT2 = typename BgAcc<T>::C2;
  using CW = typename BgAcc<T>::CW;
  constexpr int EPV = VecOf<T>::E;          // elements per 16-byte vector
  constexpr int VPL = 8 / EPV;              // vectors per lane per column (8 rows per lane)
  constexpr int CB = sizeof(T) == 4 ? (BG ? K1_CB32 : 4) : 2;   // columns in flight per batch (LDG)
  constexpr int MAXQ = NQ;                  // columns per warp (union U <= 16·NQ, host-checked)
  // BG: NSLOT slots of per-warp partials; warps publish tile i into slot i % NSLOT and reduce
  // their 16-row share of tile i - LAGR, synchronised only by per-slot mbarriers (no CTA barrier)
  constexpr int NSLOT = K1_NSLOT;
  constexpr int LAGR = K1_LAGR;
  static_assert(LAGR >= 1 && LAGR < NSLOT, "reduction lag must leave a free slot");

  __shared__ __align__(16) CW cw_s[BG ? K1_WARPS : 1][BG ? MAXQ : 1];   // coefficient per warp column
  __shared__ long long col_off[K1_WARPS][MAXQ];   // ring offset (slot * ld) of each warp column
  __shared__ int col_kd[K1_WARPS][MAXQ];          // Gram-column index, or -1
  extern __shared__ __align__(128) unsigned char red_raw[];
  BT2* red = reinterpret_cast<BT2*>(red_raw);
  __shared__ unsigned long long fullb[NSLOT], emptyb[NSLOT];
  __shared__ int am_last;

  if (*(volatile int*)&p.st->status != 0) return;   // stream poisoned: discard (header contract)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long f_dot0 = p.f_new - p.nd + 1;
  const long long f_bg0 = p.f_bg - p.m + 1;         // first column of X'_{f_bg}
  const long long F0 = BG ? (f_dot0 < f_bg0 ? f_dot0 : f_bg0) : f_dot0;
  const int U = (int)(p.f_new - F0 + 1);
  for (int e = tid; e < K1_WARPS * MAXQ; e += K1_THREADS) {
    const int w = e / MAXQ, q = e % MAXQ, j = w + K1_WARPS * q;
    const long long f = F0 + j;
    col_off[w][q] = (j < U) ? (f % p.NS) * p.ld : 0;
    col_kd[w][q] = (j < U && f >= f_dot0) ? (int)(f - f_dot0) : -1;
    if (BG) {
      const bool inb = j < U && f >= f_bg0 && f - f_bg0 < p.m;
      cw_s[w][q] = BgAcc<T>::make(inb ? p.cbg[f - f_bg0] : make_double2(0.0, 0.0));
    }
  }
  if (BG) {
    if (tid == 0)
      for (int s = 0; s < NSLOT; ++s) { k1_mbar_init(&fullb[s], K1_WARPS); k1_mbar_init(&emptyb[s], K1_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int cnt = (U > warp) ? (U - warp + K1_WARPS - 1) / K1_WARPS : 0;
  const T* __restrict__ ring = (const T*)p.ring;
  const long long NT = p.ld / kSuperTile;
  const T* xslot = ring + (p.f_new % p.NS) * p.ld;

  // per-lane fp64 partial dots of this warp's columns, kept in registers for the whole pass
  double accv[MAXQ];
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) accv[q] = 0.0;

  long long it = 0;
  if constexpr (!BG) {
    // ---- no background: register streaming, CB columns (VPL LDG.128 each) in flight per lane
    for (long long tile = blockIdx.x; tile < NT; tile += gridDim.x, ++it) {
      const long long row0 = tile * kSuperTile;
      double xd[8];
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        VT xv = __ldg(reinterpret_cast<const VT*>(xslot + row0 + v * 32 * EPV) + lane);
        to_double(xv, xd + v * EPV);
      }
      const T* base = ring + row0;
#pragma unroll
      for (int q0 = 0; q0 < MAXQ; q0 += CB) {
        if (q0 < cnt) {
          VT z[CB][VPL];
#pragma unroll
          for (int b = 0; b < CB; ++b) {
            const int q = q0 + b;
            if (q < MAXQ && q < cnt) {
              const VT* zp = reinterpret_cast<const VT*>(base + col_off[warp][q]);
#pragma unroll
              for (int v = 0; v < VPL; ++v) z[b][v] = __ldcs(zp + v * 32 + lane);
            }
          }
#pragma unroll
          for (int b = 0; b < CB; ++b) {
            const int q = q0 + b;
            if (q < MAXQ && q < cnt) {
              double zd[8];
#pragma unroll
              for (int v = 0; v < VPL; ++v) to_double(z[b][v], zd + v * EPV);
              double s0 = 0.0, s1 = 0.0;
#pragma unroll
              for (int e = 0; e < 8; e += 2) { s0 = fma(xd[e], zd[e], s0); s1 = fma(xd[e + 1], zd[e + 1], s1); }
              accv[q] += s0 + s1;
            }
          }
        }
      }
    }
  } else {
    // reduction share of this lane: row rt of a tile <- element e_src of lane l_src, source warps
    // [8·(lane>>4), +8); lanes 0..15 write the outputs of rows 16·warp + lane
    const int rt_red = 16 * warp + (lane & 15);
    const int e_src = (rt_red / (32 * EPV)) * EPV + rt_red % EPV;
    const int l_src = (rt_red % (32 * EPV)) / EPV;
    const T* bg_col = ring + (p.f_bg % p.NS) * p.ld;
    int rd_slot = 0;                                 // slot / phase of the next tile to reduce
    unsigned rd_par = 0;
    auto bg_reduce = [&](long long jt, T xv_t) {       // reduce CTA-local tile jt (in order)
      const int slot = rd_slot;
      k1_mbar_wait(&fullb[slot], rd_par);
      if (++rd_slot == NSLOT) { rd_slot = 0; rd_par ^= 1u; }
      const BT2* rb = red + slot * (K1_WARPS * BgLayout<T>::W);
      double sx = 0.0, sy = 0.0;
      const int w0 = 8 * (lane >> 4);
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const BT2 v = rb[(w0 + w) * BgLayout<T>::W + e_src * BgLayout<T>::L + l_src];
        sx += (double)v.x;
        sy += (double)v.y;
      }
      sx += __shfl_xor_sync(0xffffffffu, sx, 16);
      sy += __shfl_xor_sync(0xffffffffu, sy, 16);
      const long long row = (blockIdx.x + jt * (long long)gridDim.x) * kSuperTile + rt_red;
      if (lane < 16 && row < p.n) {
        const double l = sqrt(sx * sx + sy * sy);                   // |l| (Q8)
        const double sp = (double)xv_t - l;                         // s = x - |l|
        ((T*)p.lowrank)[row] = (T)l;
        ((T*)p.sparse)[row] = (T)sp;
        p.mask[row] = (sp > (double)p.thr) ? 1 : 0;                 // strict '>'
      }
      __syncwarp();
      if (lane == 0) k1_mbar_arrive(&emptyb[slot]);
    };
    T xq[LAGR + 1];                                  // prefetched x_{f_bg} rows of pending tiles
#pragma unroll
    for (int q = 0; q <= LAGR; ++q) xq[q] = (T)0;
    int p_slot = 0, p_round = 0;            // partial slot of this tile, tiles / NSLOT
    // end of tile `it`: publish this warp's per-row partials, reduce tile it - LAGR
    auto tile_end = [&](const BgAcc<T>& bacc) {
      const int slot = p_slot;
      if (p_round > 0) k1_mbar_wait(&emptyb[slot], (unsigned)((p_round - 1) & 1));
      if (++p_slot == NSLOT) { p_slot = 0; ++p_round; }
      BT2* rb = red + slot * (K1_WARPS * BgLayout<T>::W) + warp * BgLayout<T>::W;
#pragma unroll
      for (int e = 0; e < 8; ++e) rb[e * BgLayout<T>::L + lane] = bacc.get(e);
      __syncwarp();
      if (lane == 0) k1_mbar_arrive(&fullb[slot]);
      if (it >= LAGR) bg_reduce(it - LAGR, xq[LAGR]);
    };
    auto tile_begin = [&](long long row0) {  // x_{f_bg} of this tile's reduction rows
#pragma unroll
      for (int q = LAGR; q > 0; --q) xq[q] = xq[q - 1];
      xq[0] = (lane < 16) ? __ldcs(bg_col + row0 + rt_red) : (T)0;
    };
    // ---- background, register streaming: CB columns (VPL LDG.128 each) in flight per lane
    for (long long tile = blockIdx.x; tile < NT; tile += gridDim.x, ++it) {
      const long long row0 = tile * kSuperTile;
      double xd[8];
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        VT xv = __ldg(reinterpret_cast<const VT*>(xslot + row0 + v * 32 * EPV) + lane);
        to_double(xv, xd + v * EPV);
      }
      tile_begin(row0);
      BgAcc<T> bacc;
      bacc.zero();
      const T* base = ring + row0;
#pragma unroll
      for (int q0 = 0; q0 < MAXQ; q0 += CB) {
        if (q0 < cnt) {
          VT z[CB][VPL];
#pragma unroll
          for (int b = 0; b < CB; ++b) {
            const int q = q0 + b;
            if (q < MAXQ && q < cnt) {
              const VT* zp = reinterpret_cast<const VT*>(base + col_off[warp][q]);
#pragma unroll
              for (int v = 0; v < VPL; ++v) z[b][v] = __ldcs(zp + v * 32 + lane);
            }
          }
#pragma unroll
          for (int b = 0; b < CB; ++b) {
            const int q = q0 + b;
            if (q < MAXQ && q < cnt) {
              double zd[8];
#pragma unroll
              for (int v = 0; v < VPL; ++v) to_double(z[b][v], zd + v * EPV);
              double s0 = 0.0, s1 = 0.0;
#pragma unroll
              for (int e = 0; e < 8; e += 2) { s0 = fma(xd[e], zd[e], s0); s1 = fma(xd[e + 1], zd[e + 1], s1); }
              accv[q] += s0 + s1;
              bacc.add(cw_s[warp][q], reinterpret_cast<const T*>(&z[b][0]));
            }
          }
        }
      }
      tile_end(bacc);
    }
    // drain the last LAGR tiles
    if (!(p.dbg & 1)) {
#pragma unroll
      for (int q = LAGR - 1; q >= 0; --q)
        if (it - 1 - q >= 0) bg_reduce(it - 1 - q, xq[q]);
    }
  }

  // per-column warp reduction of the lane partials (fixed order) -> this CTA's partials
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) {
    if (q < cnt) {
      const int kd = col_kd[warp][q];
      const double s = warp_sum(accv[q]);
      if (lane == 0 && kd >= 0) p.partials[(long long)kd * p.pgrid + blockIdx.x] = s;
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
  // warp per Gram column, lanes stride over the CTA partials, fixed-order butterfly: deterministic
  for (int k = warp; k < p.nd; k += K1_WARPS) {
    const double* pk = p.partials + (long long)k * p.pgrid;
    double s = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(pk + b);
    s = warp_sum(s);
    if (lane == 0) p.gout[k] = s;
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

// ---------------------------------------------------------------------------------------------
// K1 v2: the same pass with one 16-byte vector per lane per column (a 32·EPV-row tile: 128 fp32 /
// 64 fp64 rows), column batches double-buffered in registers (the next batch — or the next tile's
// first batch — is in flight while the current one is reduced), and a branch-free column loop:
// every warp walks exactly NQ columns, the ones past the union U pointing at the (L1-resident)
// x_t tile with a zero background coefficient and a discarded dot.  Column offsets are 32-bit, in
// 16-byte units.
// RC: the background coefficients are real (c.y == 0 for every column: a real λ_idx, the usual
// case for the slowest mode) — only the real part of l = X'c is accumulated.
template <typename T, bool RC = false> struct BgAcc2;
template <bool RC> struct BgAcc2<float, RC> {   // rows (0,1) and (2,3) of the lane, packed FFMA2
  using C2 = float2;
  using CW = float4;                           // (c.x, c.x, c.y, c.y)
  float2 re[2], im[2];
  static __device__ __forceinline__ CW make(double2 c) {
    return make_float4((float)c.x, (float)c.x, (float)c.y, (float)c.y);
  }
  __device__ __forceinline__ void zero() { re[0] = re[1] = im[0] = im[1] = make_float2(0.f, 0.f); }
  __device__ __forceinline__ void add(const CW c, const float4 z) {
    const float2 cr = make_float2(c.x, c.y), ci = make_float2(c.z, c.w);
    const float2 z01 = make_float2(z.x, z.y), z23 = make_float2(z.z, z.w);
    re[0] = __ffma2_rn(cr, z01, re[0]);
    re[1] = __ffma2_rn(cr, z23, re[1]);
    if (!RC) {
      im[0] = __ffma2_rn(ci, z01, im[0]);
      im[1] = __ffma2_rn(ci, z23, im[1]);
    }
  }
  __device__ __forceinline__ C2 get(int e) const {
    return (e & 1) ? make_float2(re[e >> 1].y, im[e >> 1].y) : make_float2(re[e >> 1].x, im[e >> 1].x);
  }
};
template <bool RC> struct BgAcc2<double, RC> {
  using C2 = double2;
  using CW = double2;
  double2 v[2];
  static __device__ __forceinline__ CW make(double2 c) { return c; }
  __device__ __forceinline__ void zero() { v[0] = v[1] = make_double2(0.0, 0.0); }
  __device__ __forceinline__ void add(const CW c, const double2 z) {
    v[0].x = fma(c.x, z.x, v[0].x);
    v[1].x = fma(c.x, z.y, v[1].x);
    if (!RC) { v[0].y = fma(c.y, z.x, v[0].y); v[1].y = fma(c.y, z.y, v[1].y); }
  }
  __device__ __forceinline__ C2 get(int e) const { return v[e]; }
};

template <int NQ> struct K1v2Shape {
  static constexpr int NB = NQ <= 8 ? 1 : 2 * ((NQ + K1V2_NBDIV - 1) / K1V2_NBDIV);     // batches per tile (even if > 1)
  static constexpr int CB = (NQ + NB - 1) / NB;                     // columns per batch
};

template <typename T, bool BG, int NQ>
__global__ void __launch_bounds__(K1_THREADS, 1) k1v2_kernel(const K1Params p) {
  using VT = typename VecOf<T>::type;
  using Acc = BgAcc2<T>;
  using BT2 = typename Acc::C2;
  using CW = typename Acc::CW;
  constexpr int EPV = VecOf<T>::E;             // rows per lane per tile
  constexpr int TILE = 32 * EPV;               // rows per tile
  constexpr int NB = K1v2Shape<NQ>::NB, CB = K1v2Shape<NQ>::CB;
  constexpr int LAGR = K1V2_LAGR;             // tiles between publishing and reducing
  constexpr int NSLOT = LAGR + K1V2_SLACK;     // reduction slots
  constexpr int RL = 33;                       // padded lane stride of the reduction slots
  constexpr int SLOTW = K1_WARPS * EPV * RL;   // BT2 elements per slot
  __shared__ unsigned col_off[K1_WARPS][NQ];   // ring offset of each warp column (16-byte units)
  __shared__ int col_kd[K1_WARPS][NQ];         // Gram-column index, or -1
  __shared__ __align__(16) CW cw_s[BG ? K1_WARPS : 1][BG ? NQ : 1];
  extern __shared__ __align__(16) unsigned char k1v2_dyn[];
  BT2* red = reinterpret_cast<BT2*>(k1v2_dyn);     // [NSLOT][K1_WARPS][EPV][RL]
  __shared__ unsigned long long fullb[NSLOT], emptyb[NSLOT];
  __shared__ int am_last;

  if (*(volatile int*)&p.st->status != 0) return;   // stream poisoned: discard (header contract)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long f_dot0 = p.f_new - p.nd + 1;
  const long long f_bg0 = p.f_bg - p.m + 1;
  const long long F0 = BG ? (f_dot0 < f_bg0 ? f_dot0 : f_bg0) : f_dot0;
  const int U = (int)(p.f_new - F0 + 1);
  const unsigned xoff = (unsigned)((p.f_new % p.NS) * p.ld / EPV);
  for (int e = tid; e < K1_WARPS * NQ; e += K1_THREADS) {
    const int w = e / NQ, q = e % NQ, j = w + K1_WARPS * q;
    const long long f = F0 + j;
    col_off[w][q] = (j < U) ? (unsigned)((f % p.NS) * p.ld / EPV) : xoff;
    col_kd[w][q] = (j < U && f >= f_dot0) ? (int)(f - f_dot0) : -1;
    if (BG) {
      const bool inb = j < U && f >= f_bg0 && f - f_bg0 < p.m;
      cw_s[w][q] = Acc::make(inb ? p.cbg[f - f_bg0] : make_double2(0.0, 0.0));
    }
  }
  if (BG && tid == 0) {
    for (int s = 0; s < NSLOT; ++s) { k1_mbar_init(&fullb[s], K1_WARPS); k1_mbar_init(&emptyb[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // real coefficients (every c.y == 0) select the real-only background accumulation
  bool creal = true;
  if (BG)
    for (int k = tid; k < p.m; k += K1_THREADS) creal = creal && (p.cbg[k].y == 0.0);
  const bool realc = __syncthreads_and(creal ? 1 : 0) != 0 && BG && !K1V2_NORC;
  auto body = [&](auto rc_tag) {
  constexpr bool RC = decltype(rc_tag)::value;
  using AccR = BgAcc2<T, RC>;

  const VT* __restrict__ ringv = (const VT*)p.ring;
  const long long NT = p.ld / TILE;
  const unsigned* my_off = col_off[warp];
  // real columns of this warp (j = warp + 16q < U); slots q >= cnt are dummies, which by default
  // stream the L1-resident x_t tile with a zero coefficient (branch-free; K1V2_SKIP=1 skips them).
  const int cnt = K1V2_SKIP ? (U > warp ? (U - warp + K1_WARPS - 1) / K1_WARPS : 0) : NQ;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;

  // background: every warp publishes its per-row (re, im) partials of each tile into slot
  // tile % NSLOT; the sums over the 16 warps are formed by ONE designated warp per tile
  // (tile & 15), LAGR tiles later, so the reductions are spread over the warps instead of all
  // warps reducing every tile in lockstep.  Fixed summation order: bitwise reproducible.
  const T* bg_col = (const T*)p.ring + (p.f_bg % p.NS) * p.ld;
  VT xbg;                                      // x_{f_bg} rows of the tile this warp reduces next
  auto bg_load_x = [&](long long jt) {
    const long long row0 = (blockIdx.x + jt * (long long)gridDim.x) * TILE;
    xbg = __ldcs(reinterpret_cast<const VT*>(bg_col + row0) + lane);
  };
  auto bg_reduce = [&](long long jt) {
    const int rs = (int)(jt % NSLOT);
    k1_mbar_wait(&fullb[rs], (unsigned)((jt / NSLOT) & 1));
    const BT2* rr = red + rs * SLOTW + lane;
    double sx[EPV], sy[EPV];
#pragma unroll
    for (int e = 0; e < EPV; ++e) { sx[e] = 0.0; sy[e] = 0.0; }
#pragma unroll
    for (int w = 0; w < K1_WARPS; ++w) {
#pragma unroll
      for (int e = 0; e < EPV; ++e) {
        const BT2 v = rr[w * (EPV * RL) + e * RL];
        sx[e] += (double)v.x;
        sy[e] += (double)v.y;
      }
    }
    __syncwarp();
    if (lane == 0) k1_mbar_arrive(&emptyb[rs]);          // slot may be refilled
    const long long row0 = (blockIdx.x + jt * (long long)gridDim.x) * TILE + lane * EPV;
    T xs[EPV], lo[EPV], sp[EPV];
    *reinterpret_cast<VT*>(xs) = xbg;
    unsigned char mk[EPV];
#pragma unroll
    for (int e = 0; e < EPV; ++e) {
      const double l = sqrt(sx[e] * sx[e] + sy[e] * sy[e]);   // |l| (Q8)
      const double sv = (double)xs[e] - l;                    // s = x - |l|
      lo[e] = (T)l;
      sp[e] = (T)sv;
      mk[e] = (sv > (double)p.thr) ? 1 : 0;                   // strict '>'
    }
    // outputs hold ld rows (padding rows come out as l = s = 0): whole vectors, no row guards
    *reinterpret_cast<VT*>((T*)p.lowrank + row0) = *reinterpret_cast<const VT*>(lo);
    *reinterpret_cast<VT*>((T*)p.sparse + row0) = *reinterpret_cast<const VT*>(sp);
    if constexpr (EPV == 4) {
      *reinterpret_cast<uchar4*>(p.mask + row0) = make_uchar4(mk[0], mk[1], mk[2], mk[3]);
    } else {
      *reinterpret_cast<uchar2*>(p.mask + row0) = make_uchar2(mk[0], mk[1]);
    }
  };

  auto load_batch = [&](VT (&z)[CB], int b, long long tile) {
    const VT* base = ringv + tile * 32 + lane;
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      const int q = b * CB + c;
      if (q < NQ && q < cnt) z[c] = __ldcs(base + my_off[q]);
    }
  };
  VT za[CB], zb[CB];
  long long tile = blockIdx.x;
  long long it = 0;
  if (tile < NT) load_batch(za, 0, tile);
  for (; tile < NT; tile += gridDim.x, ++it) {
    if (K1V2_PF > 0) {
      // L2 prefetch of this warp's column chunks K1V2_PF tiles ahead (one bulk prefetch of the
      // 16 x 32 B chunk per column, issued by lane q for column q): the loads of that tile then
      // hit L2, so fewer registers' worth of bytes in flight sustain the same bandwidth
      const long long pt = tile + (long long)K1V2_PF * gridDim.x;
      if (pt < NT && lane < NQ) {
        const VT* a = ringv + pt * 32 + my_off[lane];
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "n"(32 * (int)sizeof(VT)) : "memory");
      }
    }
    double xd[EPV];
    {
      const VT xv = __ldg(ringv + xoff + tile * 32 + lane);
      to_double(xv, xd);
    }
    if (BG && !(K1V2_DBG & 1) && it >= LAGR && (((it - LAGR) & (K1_WARPS - 1)) == warp)) bg_load_x(it - LAGR);
    AccR bacc;
    if (BG) bacc.zero();
    const long long next = tile + gridDim.x;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      VT (&cur)[CB] = (b & 1) ? zb : za;
      VT (&nxt)[CB] = (b & 1) ? za : zb;
      if (b + 1 < NB) load_batch(nxt, b + 1, tile);
      else if (NB > 1 && next < NT) load_batch(nxt, 0, next);     // next tile's first batch
#pragma unroll
      for (int c = 0; c < CB; ++c) {
        const int q = b * CB + c;
        if (q < NQ && q < cnt) {
          double zd[EPV];
          to_double(cur[c], zd);
#pragma unroll
          for (int e = 0; e < EPV; ++e) acc[q] = fma(xd[e], zd[e], acc[q]);
          if (BG && !(K1V2_DBG & 2)) bacc.add(cw_s[warp][q], cur[c]);
        }
      }
    }
    if (NB == 1 && next < NT) load_batch(za, 0, next);
    if (BG && (K1V2_DBG & 1)) {
      if (bacc.get(0).x == 12345.0) p.mask[0] = 7;      // keep the accumulators live
    } else if (BG) {
      // publish this warp's per-row (re, im) partials of the tile; the designated warp of tile
      // it - LAGR reduces it
      const int slot = (int)(it % NSLOT);
      if (it >= NSLOT) k1_mbar_wait(&emptyb[slot], (unsigned)(((it / NSLOT) - 1) & 1));
      BT2* rb = red + slot * SLOTW + warp * (EPV * RL);
#pragma unroll
      for (int e = 0; e < EPV; ++e) rb[e * RL + lane] = bacc.get(e);
      __syncwarp();
      if (lane == 0) k1_mbar_arrive(&fullb[slot]);
      if (it >= LAGR && (((it - LAGR) & (K1_WARPS - 1)) == warp)) bg_reduce(it - LAGR);
    }
  }
  if (BG && !(K1V2_DBG & 1)) {                 // drain the last LAGR tiles
    for (long long jt = it - LAGR > 0 ? it - LAGR : 0; jt < it; ++jt)
      if ((jt & (K1_WARPS - 1)) == warp) { bg_load_x(jt); bg_reduce(jt); }
  }

  // per-column warp reduction of the lane partials (fixed order) -> this CTA's partials
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int kd = col_kd[warp][q];
    const double s = warp_sum(acc[q]);
    if (lane == 0 && kd >= 0) p.partials[(long long)kd * p.pgrid + blockIdx.x] = s;
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
  for (int k = warp; k < p.nd; k += K1_WARPS) {
    const double* pk = p.partials + (long long)k * p.pgrid;
    double s = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(pk + b);
    s = warp_sum(s);
    if (lane == 0) p.gout[k] = s;
  }
  if (tid == 0) {
    p.st->k1_done = 0;
    if (BG) p.st->bg_frame = p.f_bg;
  }
  if (p.do_commit) {
    __syncthreads();
    commit_block(p.gout, p.nd, p.m, p.f_new, p.ghist, p.NH, p.st);
  }
  };  // body
  if (realc) body(std::true_type{});
  else body(std::false_type{});
}

__global__ void commit_kernel(const K1Params p) {
  if (*(volatile int*)&p.st->status != 0) return;
  for (int i = threadIdx.x; i < p.cfold_n; i += blockDim.x) p.cfold_dst[i] = p.cfold_src[i];
  commit_block(p.gout, p.nd, p.m, p.f_new, p.ghist, p.NH, p.st);
}

template <typename T, bool BG, int NQ>
static cudaError_t launch_k1_inst(const K1Params& p, int grid, int smem, cudaStream_t s) {
  cudaError_t e = set_max_dyn_smem((const void*)k1_gram_kernel<T, BG, NQ>, smem);
  static const int carve = [] { const char* c = std::getenv("SDMD_K1_CARVEOUT"); return c ? std::atoi(c) : -1; }();
  if (e == cudaSuccess && carve >= 0)      // experiment knob: shared-memory carveout (percent)
    e = cudaFuncSetAttribute(k1_gram_kernel<T, BG, NQ>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
  if (e == cudaSuccess) k1_gram_kernel<T, BG, NQ><<<grid, K1_THREADS, smem, s>>>(p);
  return e;
}

template <typename T, bool BG>
static cudaError_t launch_k1_nq(const K1Params& p, int grid, int smem, int U, cudaStream_t s) {
  // columns per warp: 14 covers m + lag <= 224 (e.g. m = 200, lag <= 24) with 6 fewer live registers
  return U <= K1_WARPS * 14 ? launch_k1_inst<T, BG, 14>(p, grid, smem, s)
                            : launch_k1_inst<T, BG, K1_NQMAX>(p, grid, smem, s);
}

template <typename T, bool BG, int NQ>
static cudaError_t launch_k1v2_inst(const K1Params& p, int grid, cudaStream_t s) {
  constexpr int EPV = VecOf<T>::E;
  const int smem = BG ? (K1V2_LAGR + K1V2_SLACK) * K1_WARPS * EPV * 33 * (int)(2 * sizeof(T)) : 0;
  if (smem > 48 * 1024) {
    const cudaError_t e = set_max_dyn_smem((const void*)k1v2_kernel<T, BG, NQ>, smem);
    if (e != cudaSuccess) return e;
  }
  k1v2_kernel<T, BG, NQ><<<grid, K1_THREADS, smem, s>>>(p);
  return cudaSuccess;
}

template <typename T, bool BG>
static cudaError_t launch_k1v2_nq(const K1Params& p, int grid, int U, cudaStream_t s) {
  const int need = (U + K1_WARPS - 1) / K1_WARPS;
  if (need <= 2) return launch_k1v2_inst<T, BG, 2>(p, grid, s);
  if (need <= 4) return launch_k1v2_inst<T, BG, 4>(p, grid, s);
  if (need <= 8) return launch_k1v2_inst<T, BG, 8>(p, grid, s);
  if (need <= 10) return launch_k1v2_inst<T, BG, 10>(p, grid, s);   // fewer dummy slots per warp
  if (need <= 12) return launch_k1v2_inst<T, BG, 12>(p, grid, s);
  if (need <= 13) return launch_k1v2_inst<T, BG, 13>(p, grid, s);
  if (need <= 14) return launch_k1v2_inst<T, BG, 14>(p, grid, s);
  if (need <= 16) return launch_k1v2_inst<T, BG, 16>(p, grid, s);
  return launch_k1v2_inst<T, BG, K1_NQMAX>(p, grid, s);
}

cudaError_t launch_k1(const K1Params& p, int dtype, int grid, cudaStream_t s) {
  const int es = dtype == 0 ? 4 : 8;
  if (!p.v1 && (unsigned long long)p.NS * (unsigned long long)p.ld * es / 16 < (1ull << 32)) {
    const int U = p.bg ? (p.nd > (int)(p.f_new - p.f_bg) + p.m ? p.nd : (int)(p.f_new - p.f_bg) + p.m) : p.nd;
    if (U > K1_MAXU) return cudaErrorInvalidValue;
    cudaError_t e;
    if (dtype == 0) e = p.bg ? launch_k1v2_nq<float, true>(p, grid, U, s) : launch_k1v2_nq<float, false>(p, grid, U, s);
    else e = p.bg ? launch_k1v2_nq<double, true>(p, grid, U, s) : launch_k1v2_nq<double, false>(p, grid, U, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  int smem = 0;
  if (p.bg) smem += K1_NSLOT * K1_WARPS * 8 * (dtype == 0 ? 40 : 36) * (dtype == 0 ? (int)sizeof(float2) : (int)sizeof(double2));
  // union of the Gram window and X' of the background frame
  const int U = p.bg ? (p.nd > (int)(p.f_new - p.f_bg) + p.m ? p.nd : (int)(p.f_new - p.f_bg) + p.m) : p.nd;
  if (U > K1_MAXU) return cudaErrorInvalidValue;
  cudaError_t e;
  if (dtype == 0) e = p.bg ? launch_k1_nq<float, true>(p, grid, smem, U, s) : launch_k1_nq<float, false>(p, grid, smem, U, s);
  else e = p.bg ? launch_k1_nq<double, true>(p, grid, smem, U, s) : launch_k1_nq<double, false>(p, grid, smem, U, s);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// Load every K1 instance at context creation: with lazy module loading the first launch of a
// kernel otherwise loads it mid-stream (measured: a 26 ms stall on the first background pass).
void preload_k1_kernels() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k1_gram_kernel<float, false, 14>);
  cudaFuncGetAttributes(&a, k1_gram_kernel<float, true, 14>);
  cudaFuncGetAttributes(&a, k1_gram_kernel<double, false, 14>);
  cudaFuncGetAttributes(&a, k1_gram_kernel<double, true, 14>);
  cudaFuncGetAttributes(&a, k1_gram_kernel<float, false, K1_NQMAX>);
  cudaFuncGetAttributes(&a, k1_gram_kernel<float, true, K1_NQMAX>);
  cudaFuncGetAttributes(&a, k1_gram_kernel<double, false, K1_NQMAX>);
  cudaFuncGetAttributes(&a, k1_gram_kernel<double, true, K1_NQMAX>);
  cudaFuncGetAttributes(&a, commit_kernel);
#define K1V2_PRELOAD(NQ)                                          \
  cudaFuncGetAttributes(&a, k1v2_kernel<float, false, NQ>);      \
  cudaFuncGetAttributes(&a, k1v2_kernel<float, true, NQ>);       \
  cudaFuncGetAttributes(&a, k1v2_kernel<double, false, NQ>);     \
  cudaFuncGetAttributes(&a, k1v2_kernel<double, true, NQ>);
  K1V2_PRELOAD(2) K1V2_PRELOAD(4) K1V2_PRELOAD(8) K1V2_PRELOAD(10) K1V2_PRELOAD(12) K1V2_PRELOAD(13)
  K1V2_PRELOAD(14) K1V2_PRELOAD(16)
  K1V2_PRELOAD(K1_NQMAX)
#undef K1V2_PRELOAD
}

cudaError_t launch_commit(const K1Params& p, cudaStream_t s) {
  commit_kernel<<<1, 256, 0, s>>>(p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Gram-history helpers (init_window path and get_gram)
// ---------------------------------------------------------------------------------------------

// Scatter a k x k window Gram (columns = frames first_frame .. first_frame+k-1) into ghist rows.
__global__ void ghist_from_gram_kernel(const double* G, int k, double* ghist, int NH, int m,
                                       long long first_frame) {
  const int j = blockIdx.x;                       // frame first_frame + j
  const long long f = first_frame + j;
  double* row = ghist + (f % NH) * (m + 1);
  for (int kk = threadIdx.x; kk < m + 1; kk += blockDim.x) {
    const int i = kk - m + j;                     // column index of x_{f-m+kk} in the window
    row[kk] = (i >= 0 && i <= j) ? G[(long long)j * k + i] : 0.0;
  }
}

cudaError_t launch_ghist_from_gram(const double* G, int k, double* ghist, int NH, int m,
                                   long long first_frame, cudaStream_t s) {
  ghist_from_gram_kernel<<<k, 128, 0, s>>>(G, k, ghist, NH, m, first_frame);
  return cudaGetLastError();
}

// Gather the logical-order k x k Gram of the window ending at frame f_last.
__global__ void gather_gram_kernel(const double* ghist, int NH, int m, long long f_last, int k,
                                   double* Gout) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= k * k) return;
  const int i = idx % k, j = idx / k;
  const int a = i < j ? i : j, b = i < j ? j : i;
  const long long fb = f_last - (k - 1) + b;      // frame of column b
  const int kk = a - b + m;                       // <x_{fb-m+kk}, x_fb> with fb-m+kk = frame of a
  Gout[idx] = ghist[(fb % NH) * (m + 1) + kk];
}

cudaError_t launch_gather_gram(const double* ghist, int NH, int m, long long f_last, int k,
                               double* Gout, cudaStream_t s) {
  const int n = k * k;
  gather_gram_kernel<<<(n + 255) / 256, 256, 0, s>>>(ghist, NH, m, f_last, k, Gout);
  return cudaGetLastError();
}

}  // namespace sdmd
