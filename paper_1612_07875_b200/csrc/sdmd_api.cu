// sdmd_api.cu — host runtime behind include/sdmd.h: context, HBM ring, Gram history, the per-frame
// DAG (ingest → K1/K3 → [NCCL allreduce] → commit → K4 on round-robin eigen-worker streams →
// fused background in a later K1), event bookkeeping, getters and the NCCL bootstrap.
//
// Per push of frame t (all enqueued asynchronously; the host never waits):
//   main stream : [wait done(t-lag)] → copy x_t into slot t mod NS → K1(t) (+ background of t-lag)
//                 → [ncclAllReduce(g) → commit] → record commit(t)
//   worker t%W  : wait commit(t) → K4(t) → record done(t)
// K4(t) overlaps the K1 passes of frames t+1 … t+lag-1 (they touch disjoint data), so the eigen
// work is hidden behind the bandwidth-bound Gram pass when lag·t_K1 ≥ t_K4.
// Eigen sharding (nranks = P > 1, cfg.eigen_shard): the small eigenproblems of frame t run only on
// rank t mod P (every rank holds the same allreduced Gram history, so any rank can solve any
// frame).  The m background coefficients c_t that K1(t+lag) consumes ride in the allreduce of the
// Gram column of frame t+lag-1 (2m fp64 appended: the owner's values, zeros on every other rank,
// so the sum is the owner's value exactly) — ONE collective per frame, as SURVEY §8(e) states.
// The eigen work per rank drops by P, so the pipeline keeps up with P times the frame rate of one
// GPU.  Local frame index q = t div P selects the worker streams, the workspace and the K4 events.
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>
#include <condition_variable>
#include <cstdio>
#include <map>
#include <mutex>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <deque>
#include <string>
#include <utility>
#include <vector>

#include "../../include/sdmd.h"
#include "nccl.h"
#include "sdmd_internal.cuh"

using namespace sdmd;

namespace {

struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi* nccl_api() {
  static NcclApi api;
  if (api.loaded) return &api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return nullptr;
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
  api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
  if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.CommDestroy)
    return nullptr;
  api.loaded = true;
  return &api;
}

// In-process collective group (TEST backend, SDMD_LOCAL_GROUP=1): the ranks are contexts on the
// SAME device driven by different host threads of one process.  Collectives stage each rank's
// buffer in device memory, rendezvous on the host (so every rank's event is recorded before any
// rank waits on it), and reduce in rank order — bit-identical on every rank, like NCCL's
// single-reduction algorithms.  It exists only so that the multi-rank data path (row sharding,
// the allreduce of g, eigen sharding and the broadcast of c_t) can be tested on one GPU: NCCL
// refuses two ranks on one device.  Production runs use NCCL.
struct LocalGroup {
  int n = 0, arrived = 0;
  long long gen = 0;
  std::mutex mu;
  std::condition_variable cv;
  double* stage[8]{};
  double** d_stage = nullptr;              // device copy of stage[] for the sum kernel
  size_t cap = 0;
  int refs = 0;
  cudaEvent_t ev_in[8]{}, ev_out[8]{};
  bool out_pending[8]{};
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == n) { arrived = 0; ++gen; cv.notify_all(); }
    else cv.wait(lk, [&] { return gen != g; });
  }
};
static std::mutex g_groups_mu;
static std::map<std::string, LocalGroup*> g_groups;

constexpr int kEvents = 256;      // > NWS + lag: event slots are reused modulo kEvents
// Ring slots beyond what the window (and the background lag) needs.  After a rejected frame p the
// state rolls back to "p frames committed"; the pushes that follow p before the host learns of
// the rejection still write ring slots.  Writes of frames p+1 .. p+D-1 land in slots of frames
// older than anything the rolled-back state reads (D = NS - frames needed, see ring_guard), so the
// host only has to check the poison mirror once frame t-D has committed before writing frame t.
// The spare slots raise D, so the host may run D frames ahead of the device without waiting.
constexpr int kRingSpare = 6;

// Per-frame eigen workspace (K4a writes the factors, K4b reads them); indexed by frame mod NWS so
// that K4a of a later frame never overwrites a workspace whose K4b is still pending.
constexpr int kMaxWS = kMaxLag + 4 + kMaxWorkers;   // per-frame eigen workspaces (NWS = lag + 4 + Wa)
struct Workspace {
  double *A = nullptr, *Gxy = nullptr, *V = nullptr, *sigma = nullptr, *Y = nullptr, *B = nullptr;
  double *H = nullptr, *Qv = nullptr, *tau = nullptr, *alpha1 = nullptr;
  double2 *M = nullptr, *Mc = nullptr, *lam = nullptr, *w = nullptr, *y = nullptr;
  K4Result* res = nullptr;
  int* flags = nullptr;
  double *mu = nullptr, *wv = nullptr, *uv = nullptr;
  long long vecs_frame = -1;            // frame whose full W/b are cached in Wall/ball
};

}  // namespace

struct sdmd_ctx {
  sdmd_config cfg{};
  int dev = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int W = 4, L = 5, NS = 0, NH = 0, NC = 0, nsm = 148, k1_grid = 148, pgrid = 148, k1_dbg = 0;
  int k1b_grid = 148;                   // CTAs of the batched Gram pass (K1b)
  int k4cl = 4;                         // CTAs per K4a launch (k4_cluster_size(m))
  int k4chol = 1;                       // Cholesky-preconditioned Jacobi start (SDMD_K4_CHOL=0: off)
  bool bg_nodmd = false;                // SDMD_BG_NODMD=1: background pass with c = 0 (benchmarks)
  int k1_v1 = 0;                        // SDMD_K1=v1 selects the v1 K1 (A/B)
  int atilde_v1 = 0;                    // SDMD_ATILDE=v1 selects the untiled Ã stage of K4a (A/B)
  long long ld = 0;
  size_t es = 4;
  void* ring = nullptr;
  DevState* dst = nullptr;
  double* ghist = nullptr;
  double2* cbuf = nullptr;
  double* partials = nullptr;
  double* gout = nullptr;
  double* gpart = nullptr;              // pre-allreduce copy
  int last_nd = 0;
  // sparse storage
  int* sp_idx = nullptr;
  double* sp_val = nullptr;
  int* sp_nnz = nullptr;
  double* scratch = nullptr;
  int k3_chunks = 1;
  // background outputs
  // background outputs, double-buffered by frame parity: the D2H of frame f's outputs (on
  // d2h_stream) overlaps the Gram pass that writes frame f+1's; the pass that writes f+2 into the
  // same buffer waits for that D2H
  void* bg_low[2] = {nullptr, nullptr};
  void* bg_sparse[2] = {nullptr, nullptr};
  unsigned char* bg_mask[2] = {nullptr, nullptr};
  cudaStream_t d2h_stream = nullptr;
  cudaEvent_t ev_bgw[2]{}, ev_d2h[2]{};
  bool d2h_pending[2] = {false, false};
  long long bg_last = -1;               // frame of the newest background pass enqueued
  // sparse DCT contexts with background: pixel-space background work planes (NEXT-3)
  double* pix_planes = nullptr;         // 3 x n: Re l̂, Im l̂, x̂ (then their inverse transforms)
  double* pix_tmp = nullptr;            // 3 x n
  bool cplx = false;                    // Fourier bases: complex sparse values
  // NEXT-4 scoring: device counters {tp, fp, fn, frames} and the host-gt staging buffer
  unsigned long long* score_cnt = nullptr;
  unsigned char* gt_stage = nullptr;
  // per-frame modes (cfg.modes_every_frame, NEXT-2): per single-CTA worker stream, the LU
  // workspaces of all r inverse iterations, W, b, T = YW and Φ (ld x r_max complex)
  double2* pm_M[kMaxWorkers]{};
  double2* pm_W[kMaxWorkers]{};
  double2* pm_b[kMaxWorkers]{};
  double* pm_T[kMaxWorkers]{};
  double2* pm_phi[kMaxWorkers]{};
  // W_SINGULAR amplitudes (k4s_kernel), per single-CTA worker stream: LU workspaces, kept
  // eigenvectors, least-squares matrix, b, last-block counters; and the on-demand LS matrix
  double2* sg_M[kMaxWorkers]{};
  double2* sg_W[kMaxWorkers]{};
  double2* sg_A[kMaxWorkers]{};
  double2* sg_b[kMaxWorkers]{};
  unsigned int* sg_cnt = nullptr;
  double2* od_A = nullptr;
  // eig(Ã) warm start per single-CTA worker stream (sorted spectrum and r of its previous frame)
  double2* lam_warm[kMaxWorkers]{};
  int* r_warm = nullptr;
  // workers
  Workspace ws[kMaxWS];
  int NWS = 0, Wa = 1, Wb = 4;
  bool warm = true;                     // Jacobi warm start (SDMD_WARM=0 disables, A/B)
  bool throttle = true;                 // eigen-work flow control (SDMD_THROTTLE=0 disables, A/B)
  cudaStream_t sa[kMaxWorkers]{};      // cluster eigen workers (K4a: Jacobi .. Hessenberg)
  cudaStream_t sb[kMaxWorkers]{};      // single-CTA eigen workers (K4b: QR .. background coeffs)
  cudaEvent_t ev_a[kEvents]{};
  cudaEvent_t ev_commit[kEvents]{};
  cudaEvent_t ev_done[kEvents]{};
  cudaEvent_t ev_k1[kEvents]{};         // after K1(t) on the main stream (slot-reuse fence)
  cudaEvent_t ev_copy[kEvents]{};       // after the H2D copy of frame t on the copy stream
  cudaStream_t copy_stream = nullptr;   // overlaps host→device ingest with the previous K1
  // on-demand buffers
  double2* Wall = nullptr;
  double2* ball = nullptr;
  double2* Mws = nullptr;
  int mws_chunk = 16;
  double* Tbuf = nullptr;
  int* colbuf = nullptr;
  double* Gtmp = nullptr;
  double* init_work = nullptr;
  size_t init_work_elems = 0;
  // host mirror (valid unless a deferred error is pending)
  long long frames = 0;
  long long last_dmd = -1;              // newest frame whose eigenproblems ran on THIS rank
  long long last_dmd_all = -1;          // newest frame whose eigenproblems ran on any rank
  int P = 1, prank = 0;                 // eigen shards (P = nranks with eigen_shard, else 1)
  bool coll = false;                    // collectives on: nranks > 1, or SDMD_FORCE_NCCL=1 (test knob:
                                        // a 1-rank NCCL communicator runs the multi-rank code path)
  long long c_folded = -1;              // newest frame whose background coefficients rode an allreduce
  long long collectives = 0;
  // timing
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> k1_ev, k4_ev, wait_ev;
  std::vector<cudaEvent_t> ev_pool;     // recycled timing events
  struct TL { long long f; int kind; cudaEvent_t a, b; };   // timeline view of the events above
  std::vector<TL> tl;
  long long launches = 0;
  // rejection mirror (mapped pinned host word, written by the device on every rejection) and the
  // ring-write guard: frames < known_clean are known to be committed without a rejection
  int* h_poison = nullptr;
  int* d_poison = nullptr;
  long long known_clean = 0;
  int guard_d = 2;
  long long fenced = -1;                // eigen tasks of frames <= fenced are fenced before commits
  // frames whose eigenproblems were enqueued on this rank, with their single-CTA worker stream
  // (flow control of push_batch and the Gram-history / ring reuse fences)
  std::deque<std::pair<long long, int>> solved;
  // nccl
  ncclComm_t comm = nullptr;
  LocalGroup* lgroup = nullptr;           // SDMD_LOCAL_GROUP test backend
  std::string err;
};

// ------------------------------------------------------------------------- helpers ------------
static int fail_cuda(sdmd_ctx* c, cudaError_t e, const char* what) {
  if (c) c->err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? SDMD_E_OOM : SDMD_E_CUDA;
}
#define CK(call)                                            \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return fail_cuda(c, e_, #call);  \
  } while (0)

// NVTX range over an ABI call (header-only nvtx3: a no-op unless a tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define SDMD_NVTX() NvtxRange nvtx_range_(__func__)

static inline bool m_small(int m) { return m <= k4_small_m(); }

static int invalid(sdmd_ctx* c, const char* msg) {
  if (c) c->err = msg;
  return SDMD_E_INVALID;
}

template <typename T>
static cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc((void**)p, count * sizeof(T) > 0 ? count * sizeof(T) : 16);
}

// Timing events are recycled through a per-context pool: cudaEventCreate costs microseconds of
// host time, which a launch-bound config (C1: ≈ 50 µs per push) would otherwise pay ~8 times per
// frame while it is being measured.  sdmd_set_timing(1) pre-fills the pool.
static void destroy_timing(sdmd_ctx* c, bool release = false) {
  for (auto* v : {&c->k1_ev, &c->k4_ev, &c->wait_ev})
    for (auto& pr : *v) { c->ev_pool.push_back(pr.first); c->ev_pool.push_back(pr.second); }
  c->k1_ev.clear();
  c->k4_ev.clear();
  c->wait_ev.clear();
  c->tl.clear();
  if (release) {
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    c->ev_pool.clear();
  }
}

static cudaEvent_t pool_event(sdmd_ctx* c) {
  if (c->ev_pool.empty()) {
    cudaEvent_t a;
    cudaEventCreate(&a);
    return a;
  }
  cudaEvent_t a = c->ev_pool.back();
  c->ev_pool.pop_back();
  return a;
}

static std::pair<cudaEvent_t, cudaEvent_t> new_pair(sdmd_ctx* c) {
  cudaEvent_t a = pool_event(c);
  return {a, pool_event(c)};
}

static int sync_all(sdmd_ctx* c) {
  CK(cudaStreamSynchronize(c->copy_stream));
  if (c->d2h_stream) CK(cudaStreamSynchronize(c->d2h_stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int w = 0; w < c->Wa; ++w) CK(cudaStreamSynchronize(c->sa[w]));
  for (int w = 0; w < c->Wb; ++w) CK(cudaStreamSynchronize(c->sb[w]));
  return SDMD_OK;
}

__global__ void lg_sum_kernel(double* const* stage, int n, size_t count, double* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < n; ++r) s += stage[r][i];          // rank order: bitwise identical
    out[i] = s;
  }
}

// The one collective of the path (on the ctx stream, in the same order on every rank): the sum of
// a fp64 vector — the partial Gram column of a frame (with, under eigen sharding, the background
// coefficients of a later frame appended), or the partial init Gram.
static int lg_begin(sdmd_ctx* c, const double* src, size_t count) {
  LocalGroup* g = c->lgroup;
  const int r = c->cfg.rank;
  if (count > g->cap) { c->err = "local group: collective larger than its staging"; return SDMD_E_INVALID; }
  for (int q = 0; q < g->n; ++q)          // previous collective's readers of my staging are done
    if (g->out_pending[q]) CK(cudaStreamWaitEvent(c->stream, g->ev_out[q], 0));
  if (src) CK(cudaMemcpyAsync(g->stage[r], src, count * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaEventRecord(g->ev_in[r], c->stream));
  g->barrier();                            // every rank's ev_in is recorded
  return SDMD_OK;
}
static int lg_end(sdmd_ctx* c) {
  LocalGroup* g = c->lgroup;
  CK(cudaEventRecord(g->ev_out[c->cfg.rank], c->stream));
  g->barrier();                            // every rank's ev_out is recorded
  for (int q = 0; q < g->n; ++q) g->out_pending[q] = true;
  return SDMD_OK;
}
static int coll_allreduce(sdmd_ctx* c, double* buf, size_t count) {
  c->collectives += 1;
  if (c->lgroup) {
    LocalGroup* g = c->lgroup;
    int st = lg_begin(c, buf, count);
    if (st) return st;
    for (int q = 0; q < g->n; ++q) CK(cudaStreamWaitEvent(c->stream, g->ev_in[q], 0));
    lg_sum_kernel<<<64, 256, 0, c->stream>>>(g->d_stage, g->n, count, buf);
    CK(cudaGetLastError());
    c->launches += 1;
    return lg_end(c);
  }
  NcclApi* api = nccl_api();
  if (!api || api->AllReduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, c->stream) != ncclSuccess) {
    c->err = "ncclAllReduce failed";
    return SDMD_E_NCCL;
  }
  return SDMD_OK;
}

// Eigen sharding: frame t's eigenproblems run on rank t mod P; q = t div P is its local index.
static inline bool owns(const sdmd_ctx* c, long long t) { return t % c->P == c->prank; }
static inline long long lidx(const sdmd_ctx* c, long long t) { return t / c->P; }
static inline Workspace& ws_of(sdmd_ctx* c, long long t) { return c->ws[lidx(c, t) % c->NWS]; }
// first frame with a DMD: m (full window), or 1 with cfg.buildup (NEXT-4: from 2 columns)
static inline long long first_dmd(const sdmd_ctx* c) { return c->cfg.buildup ? 1 : c->cfg.m; }
// window width of frame f's DMD (X has w columns)
static inline int win_of(const sdmd_ctx* c, long long f) { return f < c->cfg.m ? (int)f : c->cfg.m; }

// Ring-write guard (header contract: a rejected frame leaves the state bit-identical).  Writing
// ring slots for frames up to t_last is safe unless a frame <= t_last - guard_d was rejected (the
// slots the rolled-back state reads would be overwritten, see kRingSpare).  The device records
// every rejection in the mapped host word h_poison; once the commit of frame t_last - guard_d is
// known complete and the mirror is clear, the writes cannot harm.  Returns SDMD_E_NONFINITE
// (nothing written, nothing enqueued) if the stream is poisoned; sdmd_sync reports and clears it.
static int ring_guard(sdmd_ctx* c, long long t_last) {
  if (*(volatile int*)c->h_poison) {
    c->err = "stream poisoned by a rejected frame: call sdmd_sync";
    return SDMD_E_NONFINITE;
  }
  const long long fchk = t_last - c->guard_d;
  if (fchk >= c->known_clean) {
    CK(cudaEventSynchronize(c->ev_commit[fchk % kEvents]));
    if (*(volatile int*)c->h_poison) {
      c->err = "stream poisoned by a rejected frame: call sdmd_sync";
      return SDMD_E_NONFINITE;
    }
    c->known_clean = fchk + 1;
  }
  return SDMD_OK;
}

// Make the ctx stream wait until every eigen task of a frame <= thr has finished (per single-CTA
// worker stream: its newest such frame; stream order covers the older ones).  Used before a
// commit overwrites Gram-history rows (or a ring slot) that those tasks read.
static int wait_solved_upto(sdmd_ctx* c, long long thr) {
  long long best[kMaxWorkers];
  for (int w = 0; w < kMaxWorkers; ++w) best[w] = -1;
  for (auto it = c->solved.rbegin(); it != c->solved.rend(); ++it)
    if (it->first <= thr && it->first > best[it->second]) best[it->second] = it->first;
  for (int w = 0; w < c->Wb; ++w)
    if (best[w] >= 0) CK(cudaStreamWaitEvent(c->stream, c->ev_done[lidx(c, best[w]) % kEvents], 0));
  return SDMD_OK;
}

// ------------------------------------------------------------------------- ABI ----------------
extern "C" {

int sdmd_abi_version(void) { return SDMD_ABI_VERSION; }

const char* sdmd_status_string(int s) {
  switch (s) {
    case SDMD_OK: return "ok";
    case SDMD_E_INVALID: return "invalid argument";
    case SDMD_E_NONFINITE: return "non-finite frame rejected";
    case SDMD_E_WINDOW_NOT_FULL: return "window not full";
    case SDMD_E_ZERO_MATRIX: return "zero matrix (sigma_1 == 0)";
    case SDMD_E_NO_CONVERGENCE: return "eigensolver did not converge";
    case SDMD_W_SINGULAR: return "W*Lambda singular";
    case SDMD_E_NO_VIABLE_MODE: return "no viable background mode";
    case SDMD_E_CUDA: return "CUDA error";
    case SDMD_E_NCCL: return "NCCL error";
    case SDMD_E_OOM: return "out of device memory";
    case SDMD_E_STATE: return "invalid state";
    default: return "unknown status";
  }
}

const char* sdmd_last_error(const sdmd_ctx* c) { return c ? c->err.c_str() : ""; }

int sdmd_config_init(sdmd_config* cfg) {
  if (!cfg) return SDMD_E_INVALID;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->rank_tol = 1e-7;
  cfg->threshold = 0.2f;
  cfg->dmd = 1;
  cfg->background = 0;
  cfg->workers = 4;
  cfg->nranks = 1;
  cfg->eigen_shard = 1;
  cfg->dtype = SDMD_F32;
  cfg->storage = SDMD_DENSE;
  return SDMD_OK;
}

int sdmd_nccl_unique_id(uint8_t out[128]) {
  if (!out) return SDMD_E_INVALID;
  NcclApi* api = nccl_api();
  if (!api) return SDMD_E_NCCL;
  ncclUniqueId id;
  if (api->GetUniqueId(&id) != ncclSuccess) return SDMD_E_NCCL;
  std::memcpy(out, id.internal, 128);
  return SDMD_OK;
}

int sdmd_create(const sdmd_config* cfg_in, sdmd_ctx** out) {
  SDMD_NVTX();
  if (!cfg_in || !out) return SDMD_E_INVALID;
  *out = nullptr;
  const sdmd_config& cfg = *cfg_in;
  if (cfg.m < 2 || cfg.m > SDMD_MAX_M || cfg.n_local < 1 || cfg.n_global < cfg.n_local ||
      cfg.row_begin < 0 || cfg.row_begin + cfg.n_local > cfg.n_global ||
      (cfg.dtype != SDMD_F32 && cfg.dtype != SDMD_F64) ||
      (cfg.storage != SDMD_DENSE && cfg.storage != SDMD_SPARSE) || cfg.nranks < 1 ||
      cfg.rank < 0 || cfg.rank >= cfg.nranks || cfg.r_max < 0 || cfg.workers < 0 ||
      cfg.workers > kMaxWorkers || !(cfg.rank_tol >= 0.0) || cfg.lag < 0 || cfg.lag > kMaxLag)
    return SDMD_E_INVALID;
  if (cfg.storage == SDMD_SPARSE && cfg.nnz_cap < 1) return SDMD_E_INVALID;
  if (cfg.basis < SDMD_BASIS_DCT || cfg.basis > SDMD_BASIS_RFFT || cfg.grid_rows < 0 || cfg.grid_cols < 0 ||
      (cfg.basis != SDMD_BASIS_DCT && cfg.storage != SDMD_SPARSE))
    return SDMD_E_INVALID;
  {
    const long long gr = cfg.grid_rows, gc = cfg.grid_cols;
    const bool grid = gr > 0 && gc > 0;
    if ((gr > 0) != (gc > 0)) return SDMD_E_INVALID;
    if (cfg.basis == SDMD_BASIS_RFFT && (!grid || gr * (gc / 2 + 1) != cfg.n_global)) return SDMD_E_INVALID;
    if (grid && cfg.basis != SDMD_BASIS_RFFT && gr * gc != cfg.n_global) return SDMD_E_INVALID;
    if (cfg.storage == SDMD_SPARSE && cfg.background) {
      // pixel-space background (NEXT-3): DCT basis, one rank, power-of-two grid sides in [2, 4096]
      auto pow2 = [](long long v) { return v >= 2 && v <= 4096 && (v & (v - 1)) == 0; };
      if (cfg.basis != SDMD_BASIS_DCT || cfg.nranks != 1 || !grid || !pow2(gr) || !pow2(gc) ||
          cfg.n_local != cfg.n_global)
        return SDMD_E_INVALID;
    }
  }
  if (cfg.batch_max < 0 || cfg.batch_max > kMaxBatch || (cfg.batch_max > 0 && cfg.storage != SDMD_DENSE))
    return SDMD_E_INVALID;
  if (cfg.bg_modes < 0 || cfg.bg_modes > kMaxBgModes) return SDMD_E_INVALID;
  if (cfg.modes_every_frame && (cfg.storage != SDMD_DENSE || cfg.nranks > 1 || !cfg.dmd))
    return SDMD_E_INVALID;
  if (cfg.nranks > 1 && !cfg.nccl_uid) return SDMD_E_INVALID;

  sdmd_ctx* c = new sdmd_ctx();
  c->cfg = cfg;
  if (c->cfg.rank_tol == 0.0) c->cfg.rank_tol = 1e-7;
  int rmax = c->cfg.r_max > 0 ? c->cfg.r_max : c->cfg.m;
  if (rmax > c->cfg.m) rmax = c->cfg.m;
  if (rmax > SDMD_MAX_R) rmax = SDMD_MAX_R;
  c->cfg.r_max = rmax;
  c->W = c->cfg.workers > 0 ? c->cfg.workers : 4;
  c->P = (c->cfg.nranks > 1 && c->cfg.eigen_shard) ? c->cfg.nranks : 1;
  c->prank = c->P > 1 ? c->cfg.rank : 0;
  // default lag: two frame periods per worker; K4 latency (K4a + K4b ≈ 23 ms at m = 200) must
  // fit in lag·t_K1 for the Gram pass never to wait.  With P eigen shards
  // frames arrive P times faster while one frame's K4 latency is unchanged: W·P + 6 periods.
  {
    int want = c->P > 1 ? c->W * c->P + 6 : 2 * c->W;
    if (want > kMaxLag) want = kMaxLag;
    // one rank: the largest lag <= 2W (but >= W+2) that makes the K1 union m + lag a multiple of
    // the 16 warps, so that no warp streams dummy column slots (measured: C4 W = 6 → lag 8,
    // C3 W = 20 → lag 28: 3,166 vs 2,651 snapshots/s at lag 40, profiles/r2l…)
    if (c->P == 1 && c->cfg.background)
      for (int l = want; l >= c->W + 2 && l >= 1; --l)
        if ((c->cfg.m + l) % 16 == 0) { want = l; break; }
    c->L = c->cfg.lag > 0 ? c->cfg.lag : want;
  }
  // Since eig(Ã) runs on the K4a cluster, K4b (ordering, inverse iteration, b, c: ≈ 1 ms at
  // r = 200) needs few streams: Wb = W/4 (at least 2), and the SMs go to the clusters and the Gram
  // pass (measured sweeps, profiles/r2/r6h…: C3 W = 16 → 8 + 4 streams 4,096 vs 3,383/s with
  // 10 + 20; C4 W = 6 → 3 + 2, K1 on 134 SMs).  Dense contexts: W/2 cluster streams; sparse ones
  // (the Gram pass needs few SMs): the rest of the W budget.
  c->Wb = c->W >= 2 ? (c->W / 4 > 2 ? c->W / 4 : 2) : 1;
  // a multi-mode background runs one inverse iteration per mode in K4b: keep W/2 streams there
  if (c->cfg.bg_modes > 1 && c->Wb < c->W / 2) c->Wb = c->W / 2;
  // sparse contexts: the Gram pass needs few SMs and the rate is the number of K4a clusters in
  // flight over their latency, so every hardware queue left (C5 W = 16: 24 + 4 streams, 6,200 vs
  // 4,270 snapshots/s with 16 + 4, profiles/r2/r8…)
  // (measured at W = 16: 22 + 6 streams 7,693 vs 24 + 4 7,204 snapshots/s, profiles/r2/t2…)
  if (c->cfg.storage == SDMD_SPARSE && c->W >= 16 && c->Wb < 6) c->Wb = 6;
  c->Wa = c->cfg.storage == SDMD_SPARSE ? (c->W >= 8 ? 28 - c->Wb : c->W - c->Wb) : c->W / 2;
  if (c->Wa < 1) c->Wa = 1;
  // r <= m/4 (e.g. C2: m = 150, r = 21): the single-CTA stage (QR of Ã) is light and the cluster
  // stage (Jacobi of the m x m S) bounds the throughput: give it most of the remaining hardware
  // queues (measured C2, W = 14, S·Q0 start: 24 cluster streams 8,513 vs 16 streams 5,888
  // snapshots/s with the Gram pass persistent on the 49 SMs left, profiles/r2/c2…)
  if (4 * rmax <= c->cfg.m) {
    int wa = 23 - c->Wb;                               // (W = 14: 20 streams 20,118 vs 24 18,313/s)
    if (wa > kMaxWorkers) wa = kMaxWorkers;
    if (wa > c->Wa) c->Wa = wa;
  }
  // small windows (m <= 64: single-CTA Jacobi inside K4a) make K4a short and latency-bound (its
  // commit wait is a sizeable part): as many cluster streams as single-CTA ones (C1, profiles/r2…)
  if (m_small(c->cfg.m) && c->Wa < c->W) c->Wa = c->W;
  // K4a on one CTA (dense, 64 < m <= 128): about half the SM-cycles of the cluster per frame at
  // about twice its latency, so more streams (the background lag covers the latency; C3 W = 16:
  // 20 + 4 streams, profiles/r2/r8…)
  c->k4cl = k4_cluster_size(c->cfg.m, c->cfg.storage == SDMD_SPARSE);
  if (c->k4cl == 1 && !m_small(c->cfg.m) && c->Wa < c->W + c->W / 4) c->Wa = c->W + c->W / 4;
  if (c->Wa > kMaxWorkers) c->Wa = kMaxWorkers;
  if (c->Wa + c->Wb + 3 > 32) c->Wa = 29 - c->Wb;   // 32 hardware queues (+ ctx, copy, d2h)
  if (c->Wa < 1) c->Wa = 1;
  if (const char* ea = std::getenv("SDMD_WA")) {      // experiment knob: cluster workers
    const int v = std::atoi(ea);
    if (v >= 1 && v <= kMaxWorkers) c->Wa = v;
  }
  if (const char* eb = std::getenv("SDMD_WB")) {      // experiment knob: single-CTA workers
    const int v = std::atoi(eb);
    if (v >= 1 && v <= kMaxWorkers) c->Wb = v;
  }
  // workspaces: the frames in flight (lag + 4) plus the Wa frames whose V a later frame of the
  // same cluster stream reads as its warm start (enqueue_k4 orders reuse after that read)
  c->NWS = c->L + 4 + c->Wa;
  const int m = c->cfg.m;
  c->NS = c->cfg.background ? m + c->L + 1 : m + 2;
  if (c->NS < m + c->cfg.batch_max + 1) c->NS = m + c->cfg.batch_max + 1;   // union of a batch
  // per-frame modes read X'_f on the worker stream up to ~lag frames after f was pushed: the ring
  // keeps lag + 2 more slots, and push t waits for frame t-lag-2's worker (see enqueue_frame)
  if (c->cfg.modes_every_frame && c->NS < m + c->L + 3) c->NS = m + c->L + 3;
  c->NS += kRingSpare;
  // frames the rolled-back state may still read: the window (m), or with the fused background
  // the window of the oldest pending background frame (m + L - 1)
  c->guard_d = c->NS - (c->cfg.background ? m + c->L - 1 : m);
  c->NH = 2 * (m + c->L + 4);
  c->NC = c->L + 2;
  c->es = (c->cfg.dtype == SDMD_F32 && c->cfg.storage == SDMD_DENSE) ? 4 : 8;   // sparse: fp64 values
  c->cplx = c->cfg.storage == SDMD_SPARSE && c->cfg.basis != SDMD_BASIS_DCT;
  c->ld = (c->cfg.n_local + kSuperTile - 1) / kSuperTile * kSuperTile;
  c->dev = c->cfg.device;
  auto bail = [&](int st) { sdmd_destroy(c); return st; };
  cudaError_t e = cudaSetDevice(c->dev);
  if (e != cudaSuccess) { c->err = cudaGetErrorString(e); delete c; return SDMD_E_CUDA; }
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, c->dev);
  preload_k1_kernels();
  if (c->cfg.dmd) preload_k4_kernels();
  // K1 grid.  Without DMD: persistent, one CTA per SM.  With DMD the eigen kernels (K4a/K4b) run
  // concurrently on high-priority streams, so K1 is launched as `waves` x nsm short-lived CTAs
  // (one resident per SM): whenever a K1 CTA retires, a pending K4 CTA or cluster takes the SM
  // first, and the remaining K1 CTAs flow around it.  A persistent K1 would pin its SMs for the
  // whole pass and make every K4 launch wait for a pass boundary (4-CTA clusters need 4 free SMs
  // inside one GPC).
  c->pgrid = c->nsm * kK1MaxWaves;
  {
    // waves == 0 (default): a persistent grid on the SMs the eigen workers leave free (one
    // cluster of k4_cluster_size() CTAs per cluster stream, one CTA per single-CTA stream), so K4
    // never waits for an SM and K1 has no wave tail (measured at C4: 3.71 vs 3.76 ms per pass,
    // profiles/r1p…; C2 with 24 clusters: 0.044 ms on 49 SMs vs 0.111 ms in waves); waves > 0
    // (SDMD_K1_WAVES): waves x nsm short-lived CTAs that K4 CTAs slip between.  Falls back to
    // 8 waves only if the workers would leave fewer than 16 SMs.
    int waves = 0;
    if (const char* ew = std::getenv("SDMD_K1_WAVES")) waves = std::atoi(ew);   // < 0: persistent always
    const bool force_persistent = waves < 0;
    if (waves < 0) waves = 0;
    if (waves > kK1MaxWaves) waves = kK1MaxWaves;
    const int free_sms = c->nsm - c->Wa * c->k4cl - c->Wb;
    if (waves == 0 && !force_persistent && free_sms < 16) waves = 8;
    c->k1_grid = !c->cfg.dmd ? c->nsm : waves > 0 ? c->nsm * waves : free_sms;
  }
  {
    const char* ev = std::getenv("SDMD_K1");
    c->k1_v1 = (ev && std::strcmp(ev, "v1") == 0) ? 1 : 0;
    const char* ea1 = std::getenv("SDMD_ATILDE");
    c->atilde_v1 = (ea1 && std::strcmp(ea1, "v1") == 0) ? 1 : 0;
    const char* ech = std::getenv("SDMD_K4_CHOL");          // 0: the S·Q0 Jacobi start (A/B)
    c->k4chol = (ech && ech[0] == '0') ? 0 : 1;
    const char* ed = std::getenv("SDMD_K1_DBG");
    c->k1_dbg = ed ? std::atoi(ed) : 0;
    const char* ew = std::getenv("SDMD_WARM");
    c->warm = !(ew && ew[0] == '0');
    const char* et = std::getenv("SDMD_THROTTLE");
    c->throttle = !(et && et[0] == '0');
    const char* eb = std::getenv("SDMD_BG_NODMD");
    c->bg_nodmd = eb && eb[0] == '1';
  }
  if (c->k1_grid < 1) c->k1_grid = 1;
  if (c->cfg.stream) {
    c->stream = (cudaStream_t)c->cfg.stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(SDMD_E_CUDA);
    c->own_stream = true;
  }
  if (cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess) return bail(SDMD_E_CUDA);
  if (c->cfg.background) {
    if (cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking) != cudaSuccess) return bail(SDMD_E_CUDA);
    for (int b = 0; b < 2; ++b)
      if (cudaEventCreateWithFlags(&c->ev_bgw[b], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&c->ev_d2h[b], cudaEventDisableTiming) != cudaSuccess)
        return bail(SDMD_E_CUDA);
  }
#define AL(ptr, n)                                                   \
  do {                                                               \
    if (dalloc(&(ptr), (n)) != cudaSuccess) return bail(SDMD_E_OOM); \
  } while (0)
  if (c->cfg.storage == SDMD_DENSE) {
    const size_t bytes = (size_t)c->NS * c->ld * c->es;
    if (cudaMalloc(&c->ring, bytes) != cudaSuccess) return bail(SDMD_E_OOM);
    if (cudaMemsetAsync(c->ring, 0, bytes, c->stream) != cudaSuccess) return bail(SDMD_E_CUDA);
  } else {
    AL(c->sp_idx, (size_t)c->NS * c->cfg.nnz_cap);
    const size_t vs = c->cplx ? 2 : 1;            // doubles per value (complex: interleaved)
    AL(c->sp_val, (size_t)c->NS * c->cfg.nnz_cap * vs);
    AL(c->sp_nnz, (size_t)c->NS);
    AL(c->scratch, (size_t)c->cfg.n_local * vs);
    cudaMemsetAsync(c->scratch, 0, c->cfg.n_local * vs * sizeof(double), c->stream);
    if (c->cfg.background) {
      AL(c->pix_planes, 3 * (size_t)c->cfg.n_local);
      AL(c->pix_tmp, 3 * (size_t)c->cfg.n_local);
    }
    cudaMemsetAsync(c->sp_nnz, 0, c->NS * sizeof(int), c->stream);
    c->k3_chunks = (c->cfg.nnz_cap + 2047) / 2048;
  }
  AL(c->dst, 1);
  if (cudaHostAlloc((void**)&c->h_poison, sizeof(int), cudaHostAllocMapped) != cudaSuccess) return bail(SDMD_E_OOM);
  *(volatile int*)c->h_poison = 0;
  if (cudaHostGetDevicePointer((void**)&c->d_poison, c->h_poison, 0) != cudaSuccess) return bail(SDMD_E_CUDA);
  {
    DevState hs0{};
    hs0.hpoison = c->d_poison;
    if (cudaMemcpy(c->dst, &hs0, sizeof(hs0), cudaMemcpyHostToDevice) != cudaSuccess) return bail(SDMD_E_CUDA);
  }
  AL(c->ghist, (size_t)c->NH * (m + 1));
  cudaMemsetAsync(c->ghist, 0, (size_t)c->NH * (m + 1) * sizeof(double), c->stream);
  AL(c->cbuf, (size_t)c->NC * m);
  cudaMemsetAsync(c->cbuf, 0, (size_t)c->NC * m * sizeof(double2), c->stream);
  const size_t np = (size_t)c->pgrid * (kMaxM + 16);
  const size_t np3 = (size_t)(m + 1) * c->k3_chunks;
  c->k1b_grid = k1b_grid(c->nsm, c->cfg.n_local, c->cfg.dtype);
  const size_t npb = c->cfg.batch_max > 0 ? k1b_partials_elems(c->k1b_grid) : 0;
  AL(c->partials, np > np3 ? (np > npb ? np : npb) : (np3 > npb ? np3 : npb));
  AL(c->gout, (size_t)(m + 1) * (c->cfg.batch_max > 1 ? c->cfg.batch_max : 1) + 2 * (size_t)m);
  AL(c->gpart, (size_t)(m + 1));
  AL(c->Gtmp, (size_t)(m + 1) * (m + 1));
  if (c->cfg.background) {
    // ld rows (padding included): K1 writes whole 16-byte vectors of its tiles without row guards
    for (int b = 0; b < 2; ++b) {
      if (cudaMalloc(&c->bg_low[b], c->ld * c->es) != cudaSuccess) return bail(SDMD_E_OOM);
      if (cudaMalloc(&c->bg_sparse[b], c->ld * c->es) != cudaSuccess) return bail(SDMD_E_OOM);
      AL(c->bg_mask[b], (size_t)c->ld);
    }
    AL(c->score_cnt, 4);
    cudaMemsetAsync(c->score_cnt, 0, 4 * sizeof(unsigned long long), c->stream);
  }
  const int R = kMaxR;
  int prio_lo = 0, prio_hi = 0;                     // eigen workers: highest stream priority
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  for (int w = 0; w < c->Wa; ++w)
    if (cudaStreamCreateWithPriority(&c->sa[w], cudaStreamNonBlocking, prio_hi) != cudaSuccess) return bail(SDMD_E_CUDA);
  for (int w = 0; w < c->Wb; ++w)
    if (cudaStreamCreateWithPriority(&c->sb[w], cudaStreamNonBlocking, prio_hi) != cudaSuccess) return bail(SDMD_E_CUDA);
  for (int w = 0; w < c->NWS; ++w) {
    Workspace& k = c->ws[w];
    AL(k.A, (size_t)m * m);
    AL(k.Gxy, (size_t)m * m);
    AL(k.V, (size_t)m * m);
    AL(k.sigma, (size_t)m);
    AL(k.Y, (size_t)m * R);
    AL(k.B, (size_t)(m > 8 ? m : 8) * R);   // also the Hessenberg exchange scratch (5 x R)
    AL(k.H, (size_t)R * R);
    AL(k.Qv, (size_t)R * R);
    AL(k.tau, (size_t)R);
    AL(k.alpha1, (size_t)R);
    const size_t nbs = c->cfg.bg_modes > 1 ? (size_t)c->cfg.bg_modes + 1 : 1;   // per-mode slots
    AL(k.M, nbs * R * R);
    AL(k.Mc, (size_t)R * R);
    AL(k.lam, (size_t)R);
    AL(k.w, nbs * R);
    AL(k.y, nbs * R);
    AL(k.res, 1);
    AL(k.flags, 64);
    AL(k.mu, (size_t)kMaxM);
    AL(k.wv, (size_t)R);
    AL(k.uv, (size_t)R);
    cudaMemsetAsync(k.res, 0, sizeof(K4Result), c->stream);
  }
  if (c->cfg.modes_every_frame) {
    const size_t rm = (size_t)c->cfg.r_max;
    for (int w = 0; w < c->Wb; ++w) {
      AL(c->pm_M[w], rm * rm * rm);
      AL(c->pm_W[w], rm * rm);
      AL(c->pm_b[w], rm);
      AL(c->pm_T[w], 2 * (size_t)m * rm);
      AL(c->pm_phi[w], (size_t)c->ld * rm);
    }
  }
  if (c->cfg.dmd) {
    const size_t rm = (size_t)c->cfg.r_max;
    for (int w = 0; w < c->Wb; ++w) {
      AL(c->sg_M[w], (size_t)kSingVecGrid * rm * rm);
      AL(c->sg_W[w], rm * rm);
      AL(c->sg_A[w], rm * rm);
      AL(c->sg_b[w], rm);
    }
    AL(c->sg_cnt, (size_t)kMaxWorkers);
    cudaMemsetAsync(c->sg_cnt, 0, kMaxWorkers * sizeof(unsigned int), c->stream);
    for (int w = 0; w < c->Wa; ++w) AL(c->lam_warm[w], (size_t)kMaxR);
    AL(c->r_warm, (size_t)kMaxWorkers);
    cudaMemsetAsync(c->r_warm, 0, kMaxWorkers * sizeof(int), c->stream);
  }
  for (int i = 0; i < kEvents; ++i) {
    if (cudaEventCreateWithFlags(&c->ev_commit[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_k1[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_copy[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_a[i], cudaEventDisableTiming) != cudaSuccess)
      return bail(SDMD_E_CUDA);
  }
  const char* elg = std::getenv("SDMD_LOCAL_GROUP");
  if (c->cfg.nranks > 1 && elg && elg[0] == '1') {       // TEST backend (see LocalGroup)
    if (c->cfg.nranks > 8) return bail(SDMD_E_INVALID);
    std::lock_guard<std::mutex> lk(g_groups_mu);
    const std::string key((const char*)c->cfg.nccl_uid, 128);
    LocalGroup*& g = g_groups[key];
    if (!g) {
      g = new LocalGroup();
      g->n = c->cfg.nranks;
      g->cap = (size_t)(m + 1) * (m + 1) + (size_t)kMaxBatch * (m + 1) + 2 * (size_t)m;
      for (int q = 0; q < g->n; ++q) {
        if (cudaMalloc(&g->stage[q], g->cap * sizeof(double)) != cudaSuccess) return bail(SDMD_E_OOM);
        cudaEventCreateWithFlags(&g->ev_in[q], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&g->ev_out[q], cudaEventDisableTiming);
      }
      if (cudaMalloc(&g->d_stage, 8 * sizeof(double*)) != cudaSuccess) return bail(SDMD_E_OOM);
      cudaMemcpy(g->d_stage, g->stage, 8 * sizeof(double*), cudaMemcpyHostToDevice);
    }
    ++g->refs;
    c->lgroup = g;
    c->coll = true;
  } else {
    const char* ef = std::getenv("SDMD_FORCE_NCCL");
    const bool force = c->cfg.nranks == 1 && ef && ef[0] == '1';
    if (c->cfg.nranks > 1 || force) {
      NcclApi* api = nccl_api();
      if (!api) { c->err = "libnccl.so.2 not loadable"; return bail(SDMD_E_NCCL); }
      ncclUniqueId id;
      if (force) {
        if (api->GetUniqueId(&id) != ncclSuccess) { c->err = "ncclGetUniqueId failed"; return bail(SDMD_E_NCCL); }
      } else {
        std::memcpy(id.internal, c->cfg.nccl_uid, 128);
      }
      if (api->CommInitRank(&c->comm, c->cfg.nranks, id, c->cfg.rank) != ncclSuccess) {
        c->err = "ncclCommInitRank failed";
        return bail(SDMD_E_NCCL);
      }
      c->coll = true;
    }
  }
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return bail(SDMD_E_CUDA);
  *out = c;
  return SDMD_OK;
#undef AL
}

int sdmd_destroy(sdmd_ctx* c) {
  if (!c) return SDMD_OK;
  cudaSetDevice(c->dev);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (int w = 0; w < kMaxWorkers; ++w) {
    if (c->sa[w]) cudaStreamSynchronize(c->sa[w]);
    if (c->sb[w]) cudaStreamSynchronize(c->sb[w]);
  }
  if (c->comm) {
    NcclApi* api = nccl_api();
    if (api) api->CommDestroy(c->comm);
  }
  if (c->lgroup) {
    std::lock_guard<std::mutex> lk(g_groups_mu);
    LocalGroup* g = c->lgroup;
    if (--g->refs == 0) {
      for (auto it = g_groups.begin(); it != g_groups.end(); ++it)
        if (it->second == g) { g_groups.erase(it); break; }
      for (int q = 0; q < g->n; ++q) {
        cudaFree(g->stage[q]);
        cudaEventDestroy(g->ev_in[q]);
        cudaEventDestroy(g->ev_out[q]);
      }
      cudaFree(g->d_stage);
      delete g;
    }
  }
  destroy_timing(c, true);
  for (int i = 0; i < kEvents; ++i) {
    if (c->ev_commit[i]) cudaEventDestroy(c->ev_commit[i]);
    if (c->ev_done[i]) cudaEventDestroy(c->ev_done[i]);
    if (c->ev_k1[i]) cudaEventDestroy(c->ev_k1[i]);
    if (c->ev_copy[i]) cudaEventDestroy(c->ev_copy[i]);
    if (c->ev_a[i]) cudaEventDestroy(c->ev_a[i]);
  }
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->d2h_stream) { cudaStreamSynchronize(c->d2h_stream); cudaStreamDestroy(c->d2h_stream); }
  for (int b = 0; b < 2; ++b) {
    if (c->ev_bgw[b]) cudaEventDestroy(c->ev_bgw[b]);
    if (c->ev_d2h[b]) cudaEventDestroy(c->ev_d2h[b]);
    if (c->bg_low[b]) cudaFree(c->bg_low[b]);
    if (c->bg_sparse[b]) cudaFree(c->bg_sparse[b]);
    if (c->bg_mask[b]) cudaFree(c->bg_mask[b]);
  }
  void* ptrs[] = {c->ring, c->dst, c->ghist, c->cbuf, c->partials, c->gout, c->gpart, c->sp_idx,
                  c->sp_val, c->sp_nnz, c->scratch, c->Wall, c->ball, c->Mws, c->Tbuf, c->colbuf,
                  c->Gtmp, c->init_work, c->sg_cnt, c->od_A, c->r_warm, c->pix_planes, c->pix_tmp,
                  c->score_cnt, c->gt_stage};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (int w = 0; w < kMaxWS; ++w) {
    Workspace& k = c->ws[w];
    void* wp[] = {k.A, k.Gxy, k.V, k.sigma, k.Y, k.B, k.H, k.Qv, k.tau, k.alpha1, k.M, k.Mc, k.lam, k.w,
                  k.y, k.res, k.flags, k.mu, k.wv, k.uv};
    for (void* p : wp)
      if (p) cudaFree(p);
  }
  for (int w = 0; w < kMaxWorkers; ++w) {
    if (c->sa[w]) cudaStreamDestroy(c->sa[w]);
    if (c->sb[w]) cudaStreamDestroy(c->sb[w]);
    void* pm[] = {c->pm_M[w], c->pm_W[w], c->pm_b[w], c->pm_T[w], c->pm_phi[w], c->sg_M[w], c->sg_W[w],
                  c->sg_A[w], c->sg_b[w], c->lam_warm[w]};
    for (void* q : pm)
      if (q) cudaFree(q);
  }
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (c->h_poison) cudaFreeHost(c->h_poison);
  delete c;
  return SDMD_OK;
}

static K4Params k4_params(sdmd_ctx* c, long long f) {
  Workspace& k = ws_of(c, f);
  K4Params p{};
  p.ghist = c->ghist; p.NH = c->NH; p.m = win_of(c, f); p.mh = c->cfg.m; p.f = f;
  p.r_max = c->cfg.r_max < p.m ? c->cfg.r_max : p.m;
  p.rank_tol = c->cfg.rank_tol; p.st = c->dst;
  p.A = k.A; p.Gxy = k.Gxy; p.V = k.V; p.sigma = k.sigma; p.Y = k.Y; p.B = k.B; p.H = k.H;
  p.Qv = k.Qv; p.tau = k.tau; p.M = k.M; p.Mc = k.Mc; p.lam = k.lam; p.w = k.w; p.y = k.y; p.alpha1 = k.alpha1;
  p.res = k.res;
  p.cout = c->cbuf + (f % c->NC) * c->cfg.m;
  p.flags = k.flags; p.mu = k.mu; p.wv = k.wv; p.uv = k.uv;
  p.bg_modes = c->cfg.bg_modes;
  p.atilde_v1 = c->atilde_v1;
  p.chol = (c->k4chol && p.m <= kMaxR) ? 1 : 0;
  // Jacobi warm start from the previous frame of the same cluster stream (frame f - Wa·P)
  const long long fp = f - (long long)c->Wa * c->P;
  // (only while the two windows overlap: Wa·P < m)
  if (c->warm && c->Wa < c->NWS && fp >= c->cfg.m && f - fp < p.m) {
    const Workspace& kp = ws_of(c, fp);
    p.Vprev = kp.V; p.res_prev = kp.res; p.warm_k = (int)(f - fp);
  }
  if (c->r_warm) {                              // per cluster stream (K4a computes eig(Ã))
    const int sw = (int)(lidx(c, f) % c->Wa);
    p.lam_warm = c->lam_warm[sw];
    p.r_warm = c->r_warm + sw;
  }
  return p;
}

// K4a (cluster) then K4b (single CTA) for frame t on the round-robin worker streams.
static cudaError_t enqueue_k4(sdmd_ctx* c, long long t) {
  cudaError_t e;
  const long long q = lidx(c, t), P = c->P;               // local index of frame t (t mod P == rank)
  cudaStream_t A = c->sa[q % c->Wa], B = c->sb[q % c->Wb];
  // released by the commit of frame t-1 (S_t is complete then); K4a itself waits on the device
  // for the commit of frame t before its Ã stage, so its Jacobi overlaps the Gram pass of frame t
  if ((e = cudaStreamWaitEvent(A, c->ev_commit[(t - 1) % kEvents], 0)) != cudaSuccess) return e;
  if (t - c->NWS * P >= first_dmd(c))          // workspace reuse: local frame q-NWS must be finished
    if ((e = cudaStreamWaitEvent(A, c->ev_done[(q - c->NWS) % kEvents], 0)) != cudaSuccess) return e;
  // ... and local frame q+Wa-NWS (whose warm start reads this workspace's V) must have passed K4a
  if (c->warm && c->Wa < c->NWS && t + (c->Wa - c->NWS) * P >= c->cfg.m)
    if ((e = cudaStreamWaitEvent(A, c->ev_a[(q + c->Wa - c->NWS) % kEvents], 0)) != cudaSuccess) return e;
  const K4Params p = k4_params(c, t);
  std::pair<cudaEvent_t, cudaEvent_t> ka{}, kb{};
  if (c->timing) { ka = new_pair(c); cudaEventRecord(ka.first, A); }
  if ((e = launch_k4a(p, A, c->k4cl)) != cudaSuccess) return e;
  if (c->timing) { cudaEventRecord(ka.second, A); c->k4_ev.push_back(ka); c->tl.push_back({t, 1, ka.first, ka.second}); }
  if ((e = cudaEventRecord(c->ev_a[q % kEvents], A)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(B, c->ev_a[q % kEvents], 0)) != cudaSuccess) return e;
  if (c->timing) { kb = new_pair(c); cudaEventRecord(kb.first, B); }
  if ((e = launch_k4b(p, B)) != cudaSuccess) return e;
  {                                             // W_SINGULAR frames only (device-side decision)
    const int sw = (int)(q % c->Wb);
    K4SingParams sp{};
    sp.r = c->cfg.r_max; sp.m = p.m; sp.f = t; sp.res = p.res; sp.res_out = p.res;
    sp.H = p.H; sp.Qv = p.Qv; sp.tau = p.tau; sp.lam = p.lam; sp.alpha1 = p.alpha1; sp.Y = p.Y;
    sp.Mws = c->sg_M[sw]; sp.W = c->sg_W[sw]; sp.A = c->sg_A[sw]; sp.b = c->sg_b[sw];
    sp.cout = p.cout; sp.counter = c->sg_cnt + sw;
    if ((e = launch_k4_singular(sp, true, B)) != cudaSuccess) return e;
    c->launches += 1;
  }
  if (c->timing) { cudaEventRecord(kb.second, B); c->k4_ev.push_back(kb); c->tl.push_back({t, 2, kb.first, kb.second}); }
  if (c->cfg.modes_every_frame) {               // NEXT-2: Φ_t = X'_t (Y W) for all r modes
    const int sw = (int)(q % c->Wb), rm = c->cfg.r_max, w = win_of(c, t);
    Workspace& k = ws_of(c, t);
    K4VecParams v{};
    v.r = rm; v.H = k.H; v.Qv = k.Qv; v.tau = k.tau; v.lam = k.lam; v.alpha1 = k.alpha1;
    v.Mws = c->pm_M[sw]; v.W = c->pm_W[sw]; v.b = c->pm_b[sw]; v.j0 = 0; v.res = k.res;
    if ((e = launch_k4_vecs(v, rm, B)) != cudaSuccess) return e;
    if ((e = launch_make_T_all(k.Y, w, k.res, rm, c->pm_W[sw], c->pm_T[sw], B)) != cudaSuccess) return e;
    if ((e = launch_modes(c->ring, c->ld, c->NS, c->cfg.dtype, c->cfg.n_local, t - w + 1, w,
                          c->pm_T[sw], rm, (double*)c->pm_phi[sw], c->ld, B)) != cudaSuccess) return e;
    c->launches += 3;
  }
  if ((e = cudaEventRecord(c->ev_done[q % kEvents], B)) != cudaSuccess) return e;
  c->solved.emplace_back(t, (int)(q % c->Wb));
  while (c->solved.size() > 1024) c->solved.pop_front();
  c->launches += 2;
  ws_of(c, t).vecs_frame = -1;
  c->last_dmd = t;
  return cudaSuccess;
}

// Under eigen sharding (or the forced 1-rank NCCL test path) the background coefficients of frame
// fb come from the rank that solved fb; they travel inside the per-frame allreduce of g.
static inline bool fold_c(const sdmd_ctx* c) {
  return c->coll && c->cfg.background && c->cfg.dmd && c->cfg.storage == SDMD_DENSE &&
         (c->P > 1 || c->cfg.nranks == 1);
}

// Stage c_fb at gout + off for the allreduce: the owner copies its coefficients (after its eigen
// worker finished fb), every other rank contributes zeros.
static int stage_c(sdmd_ctx* c, long long fb, int off) {
  const int m = c->cfg.m;
  double* dst = c->gout + off;
  if (owns(c, fb)) {
    CK(cudaStreamWaitEvent(c->stream, c->ev_done[lidx(c, fb) % kEvents], 0));
    CK(cudaMemcpyAsync(dst, c->cbuf + (fb % c->NC) * m, 2 * (size_t)m * sizeof(double),
                       cudaMemcpyDeviceToDevice, c->stream));
  } else {
    CK(cudaMemsetAsync(dst, 0, 2 * (size_t)m * sizeof(double), c->stream));
  }
  return SDMD_OK;
}

// Fallback: an allreduce of c_fb alone, then copied into its cbuf slot.
static int allreduce_c(sdmd_ctx* c, long long fb, int off) {
  const int m = c->cfg.m;
  int st = stage_c(c, fb, off);
  if (st) return st;
  st = coll_allreduce(c, c->gout + off, 2 * (size_t)m);
  if (st) return st;
  CK(cudaMemcpyAsync(c->cbuf + (fb % c->NC) * m, c->gout + off, 2 * (size_t)m * sizeof(double),
                     cudaMemcpyDeviceToDevice, c->stream));
  c->c_folded = fb;
  return SDMD_OK;
}

// Everything after the frame data sits in its slot: Gram column, reduction, DMD, events.
static int enqueue_frame(sdmd_ctx* c, long long t) {
  const int m = c->cfg.m;
  const int nd = (int)(t + 1 < m + 1 ? t + 1 : m + 1);
  const bool do_dmd = c->cfg.dmd && t >= first_dmd(c);
  const bool sparse = c->cfg.storage == SDMD_SPARSE;
  // the background of frame t - L: fused into the Gram pass K1(t) (dense), or the pixel-space
  // pipeline of k6_background.cu before the sparse Gram pass (sparse DCT)
  const bool bg = (c->cfg.background && c->cfg.dmd && (t - c->L) >= m &&
                   (t - c->L) <= c->last_dmd_all) ||
                  (c->bg_nodmd && c->cfg.background && !sparse && (t - c->L) >= m);
  std::pair<cudaEvent_t, cudaEvent_t> tp{}, tw{};
  if (c->timing) {                                // wait_ev: time the ctx stream spends waiting
    tw = new_pair(c);                              // for the background coefficients of t - L
    CK(cudaEventRecord(tw.first, c->stream));
  }
  if (c->cfg.dmd && (c->cfg.modes_every_frame || c->throttle) && t - c->L - 2 >= first_dmd(c) &&
      owns(c, t - c->L - 2)) {
    // modes_every_frame: frame t-L-2's modes read ring slots that push t+2 may overwrite (see
    // sdmd_create).  Otherwise flow control: at most ~lag frames of eigen work in flight (measured
    // on the K4-bound configs: an unthrottled stream floods the worker queues, profiles/r2h…)
    const long long fw = t - c->L - 2;
    CK(cudaStreamWaitEvent(c->stream, c->ev_done[lidx(c, fw) % kEvents], 0));
  }
  if (c->cfg.dmd && t - c->NH + m > c->fenced) {
    // Gram-history reuse fence: the commit of t overwrites the row of frame t - NH, read by the
    // eigen tasks of frames up to t - NH + m; fence every worker up to t - L - 2 (covers the next
    // NH - m - L - 2 commits at the cost of one wait per worker)
    const int st_ = wait_solved_upto(c, t - c->L - 2);
    if (st_) return st_;
    c->fenced = t - c->L - 2;
  }
  if (bg && c->cfg.dmd) {
    const long long fb = t - c->L;
    if (owns(c, fb)) CK(cudaStreamWaitEvent(c->stream, c->ev_done[lidx(c, fb) % kEvents], 0));
    if (fold_c(c) && c->c_folded != fb) {
      // c_fb did not ride the allreduce of frame t-1 (lag 1, or the first frame after an
      // init_window / a rollback): an allreduce of c alone (owner's values, zeros elsewhere)
      const int st_ = allreduce_c(c, fb, 0);
      if (st_) return st_;
    }
  }
  if (c->timing) {
    CK(cudaEventRecord(tw.second, c->stream));
    c->wait_ev.push_back(tw);
    c->tl.push_back({t, 3, tw.first, tw.second});
    tp = new_pair(c);
    CK(cudaEventRecord(tp.first, c->stream));
  }
  const int do_commit = c->coll ? 0 : 1;
  if (!sparse) {
    K1Params p{};
    p.ring = c->ring; p.ld = c->ld; p.NS = c->NS; p.m = m; p.n = c->cfg.n_local; p.f_new = t;
    p.nd = nd; p.bg = bg ? 1 : 0; p.f_bg = bg ? t - c->L : 0;
    p.cbg = bg ? c->cbuf + ((t - c->L) % c->NC) * m : nullptr;
    const int bslot = bg ? (int)((t - c->L) & 1) : 0;
    if (bg && c->d2h_pending[bslot]) {           // frame t-L-2's outputs still being read back
      CK(cudaStreamWaitEvent(c->stream, c->ev_d2h[bslot], 0));
      c->d2h_pending[bslot] = false;
    }
    p.lowrank = c->bg_low[bslot]; p.sparse = c->bg_sparse[bslot]; p.mask = c->bg_mask[bslot];
    p.thr = c->cfg.threshold;
    p.dbg = c->k1_dbg;
    p.partials = c->partials; p.pgrid = c->pgrid; p.gout = c->gout; p.do_commit = do_commit;
    p.ghist = c->ghist; p.NH = c->NH; p.st = c->dst;
    p.v1 = c->k1_v1;
    CK(launch_k1(p, c->cfg.dtype, c->k1_grid, c->stream));
    c->launches += 1;
    if (bg) {
      CK(cudaEventRecord(c->ev_bgw[bslot], c->stream));
      c->bg_last = t - c->L;
    }
    if (c->timing) {
      CK(cudaEventRecord(tp.second, c->stream));
      c->k1_ev.push_back(tp);
      c->tl.push_back({t, 0, tp.first, tp.second});
    }
    if (c->coll) {
      CK(cudaMemcpyAsync(c->gpart, c->gout, nd * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
      // the next push's background coefficients c_{t+1-L} ride this allreduce (computed by frame
      // t+1-L's owner; L >= 2 so that its eigen task was enqueued before this commit)
      const long long fb1 = t + 1 - c->L;
      const long long newest = do_dmd ? t : c->last_dmd_all;
      const bool fold = fold_c(c) && c->L >= 2 && fb1 >= m && fb1 <= newest && fb1 <= t - 1;
      size_t cnt = nd;
      if (fold) {
        const int st_ = stage_c(c, fb1, nd);
        if (st_) return st_;
        cnt += 2 * (size_t)m;
        p.cfold_src = c->gout + nd;
        p.cfold_dst = (double*)(c->cbuf + (fb1 % c->NC) * m);
        p.cfold_n = 2 * m;
      }
      const int st_ = coll_allreduce(c, c->gout, cnt);
      if (st_) return st_;
      CK(launch_commit(p, c->stream));
      c->launches += 1;
      if (fold) c->c_folded = fb1;
    }
  } else {
    if (bg) {                                    // pixel-space background of frame t - L (NEXT-3)
      const long long fb = t - c->L;
      const int bslot = (int)(fb & 1);
      if (c->d2h_pending[bslot]) {
        CK(cudaStreamWaitEvent(c->stream, c->ev_d2h[bslot], 0));
        c->d2h_pending[bslot] = false;
      }
      PixBgParams q{};
      q.idx = c->sp_idx; q.val = c->sp_val; q.nnz = c->sp_nnz; q.nnz_cap = c->cfg.nnz_cap;
      q.NS = c->NS; q.m = m; q.f_bg = fb; q.c = c->cbuf + (fb % c->NC) * m;
      q.rows = c->cfg.grid_rows; q.cols = c->cfg.grid_cols;
      q.planes = c->pix_planes; q.tmp = c->pix_tmp;
      q.lowrank = (double*)c->bg_low[bslot]; q.sparse = (double*)c->bg_sparse[bslot];
      q.mask = c->bg_mask[bslot]; q.thr = c->cfg.threshold; q.st = c->dst;
      CK(launch_pixel_background(q, c->stream));
      c->launches += 4;
      CK(cudaEventRecord(c->ev_bgw[bslot], c->stream));
      c->bg_last = fb;
    }
    K3Params p{};
    p.idx = c->sp_idx; p.val = c->sp_val; p.nnz = c->sp_nnz; p.nnz_cap = c->cfg.nnz_cap;
    p.cplx = c->cplx ? 1 : 0;
    if (c->cfg.basis == SDMD_BASIS_RFFT) {
      p.half_h = c->cfg.grid_cols / 2 + 1;
      p.half_even = (c->cfg.grid_cols % 2) == 0;
    }
    p.NS = c->NS; p.m = m; p.f_new = t; p.nd = nd; p.scratch = c->scratch;
    p.row_begin = c->cfg.row_begin; p.partials = c->partials; p.chunks = c->k3_chunks;
    p.gout = c->gout; p.do_commit = do_commit; p.ghist = c->ghist; p.NH = c->NH; p.st = c->dst;
    CK(launch_k3(p, c->stream));
    c->launches += 2;
    if (c->timing) {
      CK(cudaEventRecord(tp.second, c->stream));
      c->k1_ev.push_back(tp);
      c->tl.push_back({t, 0, tp.first, tp.second});
    }
    if (c->coll) {
      CK(cudaMemcpyAsync(c->gpart, c->gout, nd * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
      const int st_ = coll_allreduce(c, c->gout, nd);
      if (st_) return st_;
      K1Params q{};
      q.gout = c->gout; q.nd = nd; q.m = m; q.f_new = t; q.ghist = c->ghist; q.NH = c->NH; q.st = c->dst;
      CK(launch_commit(q, c->stream));
      c->launches += 1;
    }
  }
  c->last_nd = nd;
  CK(cudaEventRecord(c->ev_commit[t % kEvents], c->stream));
  CK(cudaEventRecord(c->ev_k1[t % kEvents], c->stream));
  if (do_dmd) {
    if (owns(c, t)) CK(enqueue_k4(c, t));
    c->last_dmd_all = t;
  }
  c->frames = t + 1;
  return SDMD_OK;
}

int sdmd_push_dense(sdmd_ctx* c, const void* x, int where) {
  SDMD_NVTX();
  if (!c || !x || (where != SDMD_HOST && where != SDMD_DEVICE && where != SDMD_DEVICE_READY))
    return invalid(c, "push_dense: bad argument");
  if (c->cfg.storage != SDMD_DENSE) return invalid(c, "push_dense on a sparse context");
  CK(cudaSetDevice(c->dev));
  const long long t = c->frames;
  if (int g = ring_guard(c, t)) return g;
  char* dst = (char*)c->ring + (size_t)(t % c->NS) * c->ld * c->es;
  // a small ready frame (< 1 MB, e.g. C1's 32 KB) is copied in ctx-stream order: one call instead
  // of the copy-stream handshake's four, and its copy time is negligible
  if (where == SDMD_DEVICE_READY && (size_t)c->cfg.n_local * c->es < ((size_t)1 << 20)) where = SDMD_DEVICE;
  if (where != SDMD_DEVICE) {
    // H2D (or a ready D2D) on the copy stream so it overlaps K1(t-1): slot t mod NS was last read
    // by K1(t-2) at the latest (kRingSpare slots of margin)
    if (t >= 2) CK(cudaStreamWaitEvent(c->copy_stream, c->ev_k1[(t - 2) % kEvents], 0));
    CK(cudaMemcpyAsync(dst, x, c->cfg.n_local * c->es,
                       where == SDMD_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c->copy_stream));
    CK(cudaEventRecord(c->ev_copy[t % kEvents], c->copy_stream));
    CK(cudaStreamWaitEvent(c->stream, c->ev_copy[t % kEvents], 0));
  } else {
    CK(cudaMemcpyAsync(dst, x, c->cfg.n_local * c->es, cudaMemcpyDeviceToDevice, c->stream));
  }
  return enqueue_frame(c, t);
}

int sdmd_acquire_slot(sdmd_ctx* c, void** dev_ptr) {
  if (!c || !dev_ptr) return invalid(c, "acquire_slot: bad argument");
  if (c->cfg.storage != SDMD_DENSE) return invalid(c, "acquire_slot on a sparse context");
  CK(cudaSetDevice(c->dev));
  if (int g = ring_guard(c, c->frames)) return g;
  *dev_ptr = (char*)c->ring + (size_t)(c->frames % c->NS) * c->ld * c->es;
  return SDMD_OK;
}

int sdmd_commit_slot(sdmd_ctx* c) {
  SDMD_NVTX();
  if (!c) return SDMD_E_INVALID;
  if (c->cfg.storage != SDMD_DENSE) return invalid(c, "commit_slot on a sparse context");
  CK(cudaSetDevice(c->dev));
  return enqueue_frame(c, c->frames);
}

int sdmd_push_batch(sdmd_ctx* c, int32_t k, const void* X, int64_t ldx, int where, int32_t dmd_every) {
  SDMD_NVTX();
  if (!c || !X || k < 1 || (where != SDMD_HOST && where != SDMD_DEVICE))
    return invalid(c, "push_batch: bad argument");
  if (c->cfg.storage != SDMD_DENSE || c->cfg.background) return invalid(c, "push_batch: dense, background-free contexts only");
  if (k > c->cfg.batch_max) return invalid(c, "push_batch: k > cfg.batch_max");
  if (ldx < c->cfg.n_local) return invalid(c, "push_batch: ldx < n_local");
  const int m = c->cfg.m;
  const long long t = c->frames;
  if (t < m + 1) { c->err = "push_batch: window not full (use push_dense during warm-up)"; return SDMD_E_STATE; }
  CK(cudaSetDevice(c->dev));
  if (int g = ring_guard(c, t + k - 1)) return g;
  // flow control and reuse fences: the commits of frames t..t+k-1 overwrite Gram-
  // history rows (and, with per-frame modes, ring slots) that eigen tasks of frames up to
  // t+k-1-L-2 may read; wait for them on the device, like enqueue_frame's throttle
  if (c->cfg.dmd) {
    if (int w = wait_solved_upto(c, t + k - 1 - c->L - 2)) return w;
    c->fenced = t + k - 1 - c->L - 2;
  }
  const cudaMemcpyKind kind = where == SDMD_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  // the k frames into slots t..t+k-1 (mod NS; at most two contiguous runs).  Those slots last
  // held frames ≤ t-m-1, read only by Gram passes already ordered before this on the ctx stream.
  for (int j = 0; j < k;) {
    const int slot = (int)((t + j) % c->NS);
    const int run = (c->NS - slot) < (k - j) ? (c->NS - slot) : (k - j);
    CK(cudaMemcpy2DAsync((char*)c->ring + (size_t)slot * c->ld * c->es, c->ld * c->es,
                         (const char*)X + (size_t)j * ldx * c->es, (size_t)ldx * c->es,
                         c->cfg.n_local * c->es, run, kind, c->stream));
    j += run;
  }
  std::pair<cudaEvent_t, cudaEvent_t> tp{};
  if (c->timing) { tp = new_pair(c); CK(cudaEventRecord(tp.first, c->stream)); }
  K1bParams p{};
  p.ring = c->ring; p.ld = c->ld; p.NS = c->NS; p.m = m; p.n = c->cfg.n_local; p.f0 = t; p.k = k;
  p.partials = c->partials; p.gout = c->gout; p.do_commit = c->coll ? 0 : 1;
  p.ghist = c->ghist; p.NH = c->NH; p.st = c->dst;
  CK(launch_k1b(p, c->cfg.dtype, c->k1b_grid, c->stream));
  c->launches += 1;
  if (c->timing) {
    CK(cudaEventRecord(tp.second, c->stream));
    c->k1_ev.push_back(tp);
    c->tl.push_back({t + k - 1, 0, tp.first, tp.second});
  }
  if (c->coll) {
    const size_t cnt = (size_t)k * (m + 1);
    CK(cudaMemcpyAsync(c->gpart, c->gout, (m + 1) * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    const int st_ = coll_allreduce(c, c->gout, cnt);
    if (st_) return st_;
    CK(launch_commit_batch(p, c->stream));
    c->launches += 1;
  }
  c->last_nd = m + 1;
  for (int j = 0; j < k; ++j) {
    const long long f = t + j;
    CK(cudaEventRecord(c->ev_commit[f % kEvents], c->stream));
    CK(cudaEventRecord(c->ev_k1[f % kEvents], c->stream));
  }
  if (c->cfg.dmd) {
    for (int j = dmd_every ? 0 : k - 1; j < k; ++j) {
      const long long f = t + j;
      if (owns(c, f)) CK(enqueue_k4(c, f));
      c->last_dmd_all = f;
    }
  }
  c->frames = t + k;
  return SDMD_OK;
}

int sdmd_push_sparse(sdmd_ctx* c, int32_t nnz, const int32_t* idx, const double* val, int where) {
  SDMD_NVTX();
  if (!c || nnz < 0 || (nnz > 0 && (!idx || !val)) || (where != SDMD_HOST && where != SDMD_DEVICE))
    return invalid(c, "push_sparse: bad argument");
  if (c->cfg.storage != SDMD_SPARSE) return invalid(c, "push_sparse on a dense context");
  if (nnz > c->cfg.nnz_cap) return invalid(c, "push_sparse: nnz > nnz_cap");
  CK(cudaSetDevice(c->dev));
  const long long lo = c->cfg.row_begin, hi = c->cfg.row_begin + c->cfg.n_local;
  if (where == SDMD_HOST) {
    for (int e = 0; e < nnz; ++e) {
      if (idx[e] < lo || idx[e] >= hi || (e > 0 && idx[e] <= idx[e - 1]))
        return invalid(c, "push_sparse: indices must be strictly ascending and in range");
    }
  }
  const long long t = c->frames;
  if (int g = ring_guard(c, t)) return g;
  const int slot = (int)(t % c->NS);
  const size_t vs = c->cplx ? 2 : 1;              // doubles per value
  int* sidx = c->sp_idx + (size_t)slot * c->cfg.nnz_cap;
  double* sval = c->sp_val + (size_t)slot * c->cfg.nnz_cap * vs;
  if (where == SDMD_HOST) {
    // compressed ingest: only the nnz (index, value) pairs
    // cross PCIe (12 B per nonzero), on the copy stream so that they overlap the previous sparse
    // Gram pass; slot t mod NS was last read by the pass of frame t-2
    if (t >= 2) CK(cudaStreamWaitEvent(c->copy_stream, c->ev_k1[(t - 2) % kEvents], 0));
    if (nnz > 0) {
      CK(cudaMemcpyAsync(sidx, idx, nnz * sizeof(int), cudaMemcpyHostToDevice, c->copy_stream));
      CK(cudaMemcpyAsync(sval, val, nnz * vs * sizeof(double), cudaMemcpyHostToDevice, c->copy_stream));
    }
    CK(launch_set_int(c->sp_nnz + slot, nnz, c->copy_stream));
    CK(cudaEventRecord(c->ev_copy[t % kEvents], c->copy_stream));
    CK(cudaStreamWaitEvent(c->stream, c->ev_copy[t % kEvents], 0));
  } else {
    if (nnz > 0) {
      CK(cudaMemcpyAsync(sidx, idx, nnz * sizeof(int), cudaMemcpyDeviceToDevice, c->stream));
      CK(cudaMemcpyAsync(sval, val, nnz * vs * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    }
    CK(launch_sparse_nnz_checked(sidx, nnz, lo, hi, c->sp_nnz + slot, c->stream));
  }
  c->launches += 1;
  return enqueue_frame(c, t);
}

int sdmd_init_window(sdmd_ctx* c, const void* Z, int64_t ldz, int where) {
  SDMD_NVTX();
  if (!c || !Z || ldz < c->cfg.n_local || (where != SDMD_HOST && where != SDMD_DEVICE))
    return invalid(c, "init_window: bad argument");
  if (c->cfg.storage != SDMD_DENSE) return invalid(c, "init_window needs dense storage");
  CK(cudaSetDevice(c->dev));
  int st = sync_all(c);
  if (st) return st;
  const int m = c->cfg.m, k = m + 1;
  // fresh state: frames 0..m occupy slots 0..m
  {
    DevState z{};
    z.hpoison = c->d_poison;                 // the rejection mirror survives the reset
    CK(cudaMemcpyAsync(c->dst, &z, sizeof(z), cudaMemcpyHostToDevice, c->stream));
  }
  CK(cudaMemsetAsync(c->ghist, 0, (size_t)c->NH * (m + 1) * sizeof(double), c->stream));
  CK(cudaMemcpy2DAsync(c->ring, c->ld * c->es, Z, (size_t)ldz * c->es, c->cfg.n_local * c->es, k,
                       where == SDMD_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                       c->stream));
  const size_t need = init_gram_work_elems(c->cfg.n_local, k);
  if (need > c->init_work_elems) {
    if (c->init_work) cudaFree(c->init_work);
    c->init_work = nullptr;
    if (dalloc(&c->init_work, need) != cudaSuccess) { c->init_work_elems = 0; return SDMD_E_OOM; }
    c->init_work_elems = need;
  }
  CK(launch_init_gram(c->ring, c->ld, c->cfg.dtype, c->cfg.n_local, k, c->Gtmp, c->init_work, c->stream));
  c->launches += 2;
  if (c->coll) {
    const int st_ = coll_allreduce(c, c->Gtmp, (size_t)k * k);
    if (st_) return st_;
  }
  {
    // one-off: a non-finite window is rejected whole, leaving an empty stream; after the
    // allreduce every rank sees the same Gram and takes the same decision
    std::vector<double> hg((size_t)k * k);
    CK(cudaMemcpyAsync(hg.data(), c->Gtmp, hg.size() * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (double v : hg)
      if (!std::isfinite(v)) {
        c->frames = 0;
        c->last_dmd = c->last_dmd_all = -1;
        c->err = "init_window rejected (non-finite Gram)";
        return SDMD_E_NONFINITE;
      }
  }
  CK(launch_ghist_from_gram(c->Gtmp, k, c->ghist, c->NH, m, 0, c->stream));
  c->launches += 1;
  DevState hs{};
  hs.committed = k;
  hs.bg_frame = -1;
  hs.hpoison = c->d_poison;
  *(volatile int*)c->h_poison = 0;
  c->known_clean = k;
  c->fenced = -1;
  c->solved.clear();
  c->c_folded = -1;
  CK(cudaMemcpyAsync(c->dst, &hs, sizeof(hs), cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int f = 0; f < k; ++f) CK(cudaEventRecord(c->ev_k1[f % kEvents], c->stream));
  c->frames = k;
  c->last_dmd = -1;
  c->last_dmd_all = -1;
  c->last_nd = k;
  if (c->cfg.dmd) {
    const long long t = m;
    CK(cudaEventRecord(c->ev_commit[t % kEvents], c->stream));
    if (owns(c, t)) CK(enqueue_k4(c, t));
    c->last_dmd_all = t;
  }
  return SDMD_OK;
}

int sdmd_join(sdmd_ctx* c) {
  if (!c) return SDMD_E_INVALID;
  CK(cudaSetDevice(c->dev));
  for (int b = 0; b < 2; ++b)                       // background read-backs still in flight
    if (c->d2h_pending[b]) CK(cudaStreamWaitEvent(c->stream, c->ev_d2h[b], 0));
  if (c->last_dmd < 0) return SDMD_OK;
  for (long long f = c->last_dmd; f > c->last_dmd - (long long)c->NWS * c->P && f >= first_dmd(c); f -= c->P)
    CK(cudaStreamWaitEvent(c->stream, c->ev_done[lidx(c, f) % kEvents], 0));
  return SDMD_OK;
}

int sdmd_sync(sdmd_ctx* c, int64_t* failed_frame) {
  SDMD_NVTX();
  if (!c) return SDMD_E_INVALID;
  if (failed_frame) *failed_frame = -1;
  CK(cudaSetDevice(c->dev));
  int st = sync_all(c);
  if (st) return st;
  DevState hs{};
  CK(cudaMemcpy(&hs, c->dst, sizeof(hs), cudaMemcpyDeviceToHost));
  if (hs.status != 0) {
    if (failed_frame) *failed_frame = hs.failed_frame;
    c->frames = hs.committed;
    const int m = c->cfg.m;
    const long long f0 = first_dmd(c);
    c->last_dmd_all = (c->cfg.dmd && hs.committed - 1 >= f0) ? hs.committed - 1 : -1;
    long long ld_ = c->last_dmd_all;               // newest surviving frame solved on this rank
    while (ld_ >= f0 && !owns(c, ld_)) --ld_;
    c->last_dmd = ld_ >= f0 ? ld_ : -1;
    (void)m;
    hs.status = 0;
    CK(cudaMemcpy(c->dst, &hs, sizeof(hs), cudaMemcpyHostToDevice));
    *(volatile int*)c->h_poison = 0;
    if (c->known_clean > hs.committed) c->known_clean = hs.committed;
    if (c->fenced > hs.committed - 1) c->fenced = hs.committed - 1;
    while (!c->solved.empty() && c->solved.back().first >= hs.committed) c->solved.pop_back();
    c->c_folded = -1;
    c->err = "frame " + std::to_string(hs.failed_frame) +
             " rejected (non-finite Gram column, or invalid device-side sparse indices)";
    return SDMD_E_NONFINITE;
  }
  return SDMD_OK;
}

int sdmd_get_info(sdmd_ctx* c, sdmd_info* info) {
  if (!c || !info) return SDMD_E_INVALID;
  info->frames = c->frames;
  info->window = (int32_t)(c->frames < c->cfg.m + 1 ? c->frames : c->cfg.m + 1);
  info->lag = c->L;
  info->ring_slots = c->NS;
  info->workers = c->W;
  info->ring_bytes = c->cfg.storage == SDMD_DENSE ? (int64_t)c->NS * c->ld * c->es
                                                   : (int64_t)c->NS * c->cfg.nnz_cap * 12;
  info->ld = c->ld;
  info->cluster_workers = c->Wa;
  info->k1_grid = c->k1_grid;
  return SDMD_OK;
}

int sdmd_get_gram(sdmd_ctx* c, double* G, int32_t* k_out) {
  if (!c || !G) return SDMD_E_INVALID;
  CK(cudaSetDevice(c->dev));
  int st = sync_all(c);
  if (st) return st;
  const int k = (int)(c->frames < c->cfg.m + 1 ? c->frames : c->cfg.m + 1);
  if (k_out) *k_out = k;
  if (k == 0) return SDMD_E_STATE;
  CK(launch_gather_gram(c->ghist, c->NH, c->cfg.m, c->frames - 1, k, c->Gtmp, c->stream));
  c->launches += 1;
  CK(cudaMemcpyAsync(G, c->Gtmp, (size_t)k * k * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return SDMD_OK;
}

int sdmd_get_partial_gram_column(sdmd_ctx* c, double* g, int32_t* k_out) {
  if (!c || !g) return SDMD_E_INVALID;
  CK(cudaSetDevice(c->dev));
  int st = sync_all(c);
  if (st) return st;
  if (k_out) *k_out = c->last_nd;
  if (c->last_nd == 0) return SDMD_E_STATE;
  CK(cudaMemcpy(g, c->coll ? c->gpart : c->gout, c->last_nd * sizeof(double),
                cudaMemcpyDeviceToHost));
  return SDMD_OK;
}

static int newest_result(sdmd_ctx* c, K4Result* r) {
  int st = sync_all(c);
  if (st) return st;
  if (c->last_dmd < 0) return SDMD_E_WINDOW_NOT_FULL;
  Workspace& k = ws_of(c, c->last_dmd);
  CK(cudaMemcpy(r, k.res, sizeof(K4Result), cudaMemcpyDeviceToHost));
  if (r->frame != c->last_dmd) { c->err = "stale worker result"; return SDMD_E_STATE; }
  return SDMD_OK;
}

int sdmd_get_svd(sdmd_ctx* c, int32_t* r, double* sigma, double* V, int64_t* frame) {
  SDMD_NVTX();
  if (!c) return SDMD_E_INVALID;
  CK(cudaSetDevice(c->dev));
  K4Result res{};
  int st = newest_result(c, &res);
  if (st) return st;
  Workspace& k = ws_of(c, c->last_dmd);
  if (r) *r = res.r;
  if (frame) *frame = res.frame;
  const int m = c->cfg.m, w = win_of(c, c->last_dmd);   // w < m: a build-up window (NEXT-4)
  if (sigma) {
    for (int i = w; i < m; ++i) sigma[i] = 0.0;
    CK(cudaMemcpy(sigma, k.sigma, w * sizeof(double), cudaMemcpyDeviceToHost));
  }
  if (V && res.r > 0) {
    if (w < m) std::memset(V, 0, (size_t)m * res.r * sizeof(double));
    CK(cudaMemcpy2D(V, m * sizeof(double), k.V, w * sizeof(double), w * sizeof(double), res.r,
                    cudaMemcpyDeviceToHost));
  }
  return res.status == 6 ? SDMD_OK : (res.status > 0 ? res.status : SDMD_OK);
}

static int ensure_vecs(sdmd_ctx* c) {
  Workspace& k = ws_of(c, c->last_dmd);
  if (k.vecs_frame == c->last_dmd) return SDMD_OK;
  K4Result res{};
  CK(cudaMemcpy(&res, k.res, sizeof(K4Result), cudaMemcpyDeviceToHost));
  const int r = res.r;
  if (r <= 0) return SDMD_E_ZERO_MATRIX;
  const int R = kMaxR;
  if (!c->Wall) {
    if (dalloc(&c->Wall, (size_t)R * R) != cudaSuccess) return SDMD_E_OOM;
    if (dalloc(&c->ball, (size_t)R) != cudaSuccess) return SDMD_E_OOM;
    if (dalloc(&c->Mws, (size_t)c->mws_chunk * R * R) != cudaSuccess) return SDMD_E_OOM;
  }
  K4VecParams p{};
  p.r = r; p.H = k.H; p.Qv = k.Qv; p.tau = k.tau; p.lam = k.lam; p.alpha1 = k.alpha1;
  p.Mws = c->Mws; p.W = c->Wall; p.b = c->ball;
  for (int j0 = 0; j0 < r; j0 += c->mws_chunk) {
    p.j0 = j0;
    const int cnt = r - j0 < c->mws_chunk ? r - j0 : c->mws_chunk;
    CK(launch_k4_vecs(p, cnt, c->stream));
    c->launches += 1;
  }
  if (res.status == SDMD_W_SINGULAR && res.nkeep < r) {   // kept-mode least squares (Q15)
    if (!c->od_A && dalloc(&c->od_A, (size_t)R * R) != cudaSuccess) return SDMD_E_OOM;
    K4SingParams sp{};
    sp.r = r; sp.nkeep = res.nkeep; sp.H = k.H; sp.Qv = k.Qv; sp.tau = k.tau; sp.lam = k.lam;
    sp.alpha1 = k.alpha1; sp.W = c->Wall; sp.A = c->od_A; sp.b = c->ball;
    CK(launch_k4_singular(sp, false, c->stream));
    c->launches += 1;
  }
  CK(cudaStreamSynchronize(c->stream));
  k.vecs_frame = c->last_dmd;
  return SDMD_OK;
}

int sdmd_get_spectrum(sdmd_ctx* c, int32_t* r, double* lambda, double* b, int32_t* idx, int64_t* frame) {
  SDMD_NVTX();
  if (!c) return SDMD_E_INVALID;
  CK(cudaSetDevice(c->dev));
  K4Result res{};
  int st = newest_result(c, &res);
  if (st) return st;
  Workspace& k = ws_of(c, c->last_dmd);
  if (r) *r = res.r;
  if (idx) *idx = res.idx;
  if (frame) *frame = res.frame;
  if (lambda && res.r > 0) CK(cudaMemcpy(lambda, k.lam, res.r * sizeof(double2), cudaMemcpyDeviceToHost));
  if (b && res.r > 0) {
    st = ensure_vecs(c);
    if (st) return st;
    CK(cudaMemcpy(b, c->ball, res.r * sizeof(double2), cudaMemcpyDeviceToHost));
  }
  return res.status > 0 ? res.status : SDMD_OK;
}

int sdmd_get_eigvecs(sdmd_ctx* c, double* W, int32_t* r) {
  SDMD_NVTX();
  if (!c || !W) return SDMD_E_INVALID;
  CK(cudaSetDevice(c->dev));
  K4Result res{};
  int st = newest_result(c, &res);
  if (st) return st;
  if (r) *r = res.r;
  st = ensure_vecs(c);
  if (st) return st;
  CK(cudaMemcpy(W, c->Wall, (size_t)res.r * res.r * sizeof(double2), cudaMemcpyDeviceToHost));
  return SDMD_OK;
}

int sdmd_get_modes(sdmd_ctx* c, const int32_t* cols, int32_t ncols, double* phi_dev, int64_t ld) {
  SDMD_NVTX();
  if (!c || !cols || ncols < 1 || !phi_dev || ld < c->cfg.n_local) return invalid(c, "get_modes: bad argument");

  CK(cudaSetDevice(c->dev));
  K4Result res{};
  int st = newest_result(c, &res);
  if (st) return st;
  for (int q = 0; q < ncols; ++q)
    if (cols[q] < 0 || cols[q] >= res.r) return invalid(c, "get_modes: column out of range");
  if (c->cfg.modes_every_frame) {                 // computed per frame on the worker stream
    const int sw = (int)(lidx(c, c->last_dmd) % c->Wb);
    for (int q = 0; q < ncols; ++q)
      CK(cudaMemcpyAsync((double2*)phi_dev + (size_t)q * ld, c->pm_phi[sw] + (size_t)cols[q] * c->ld,
                         c->cfg.n_local * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return SDMD_OK;
  }
  st = ensure_vecs(c);
  if (st) return st;
  const int m = c->cfg.m;
  if (c->Tbuf) cudaFree(c->Tbuf);
  if (c->colbuf) cudaFree(c->colbuf);
  c->Tbuf = nullptr;
  c->colbuf = nullptr;
  if (dalloc(&c->Tbuf, (size_t)2 * m * ncols) != cudaSuccess) return SDMD_E_OOM;
  if (dalloc(&c->colbuf, (size_t)ncols) != cudaSuccess) return SDMD_E_OOM;
  CK(cudaMemcpy(c->colbuf, cols, ncols * sizeof(int), cudaMemcpyHostToDevice));
  Workspace& k = ws_of(c, c->last_dmd);
  const int w = win_of(c, c->last_dmd);
  CK(launch_make_T(k.Y, w, res.r, c->Wall, c->colbuf, ncols, c->Tbuf, c->stream));
  // X' of the frame's window = frames last_dmd-w+1 .. last_dmd
  if (c->cfg.storage == SDMD_DENSE) {
    CK(launch_modes(c->ring, c->ld, c->NS, c->cfg.dtype, c->cfg.n_local, c->last_dmd - w + 1, w,
                    c->Tbuf, ncols, phi_dev, ld, c->stream));
  } else {                                      // coefficient-space modes (NEXT-3), K3 scatter
    CK(launch_modes_sparse(c->sp_idx, c->sp_val, c->sp_nnz, c->cfg.nnz_cap, c->NS, c->cfg.row_begin,
                           c->cfg.n_local, c->last_dmd - w + 1, w, c->Tbuf, ncols, phi_dev, ld,
                           c->cplx ? 1 : 0, c->stream));
  }
  c->launches += 1 + (ncols + 31) / 32;
  CK(cudaStreamSynchronize(c->stream));
  return SDMD_OK;
}

int sdmd_get_background(sdmd_ctx* c, void* lowrank, void* sparse, uint8_t* mask, int64_t* frame,
                        int where) {
  SDMD_NVTX();
  if (!c || (where != SDMD_HOST && where != SDMD_DEVICE && where != SDMD_HOST_ASYNC))
    return SDMD_E_INVALID;
  if (!c->cfg.background) return invalid(c, "background disabled in config");
  CK(cudaSetDevice(c->dev));
  const size_t n = c->cfg.n_local;
  if (where == SDMD_HOST_ASYNC) {
    // no host wait: the newest enqueued background pass's outputs are read back on the D2H
    // stream (overlapping the next Gram pass, which writes the other buffer); complete after
    // sdmd_sync, or on the ctx stream after sdmd_join
    if (frame) *frame = c->bg_last;
    if (c->bg_last < 0) return SDMD_E_STATE;
    const int b = (int)(c->bg_last & 1);
    CK(cudaStreamWaitEvent(c->d2h_stream, c->ev_bgw[b], 0));
    if (lowrank) CK(cudaMemcpyAsync(lowrank, c->bg_low[b], n * c->es, cudaMemcpyDeviceToHost, c->d2h_stream));
    if (sparse) CK(cudaMemcpyAsync(sparse, c->bg_sparse[b], n * c->es, cudaMemcpyDeviceToHost, c->d2h_stream));
    if (mask) CK(cudaMemcpyAsync(mask, c->bg_mask[b], n, cudaMemcpyDeviceToHost, c->d2h_stream));
    CK(cudaEventRecord(c->ev_d2h[b], c->d2h_stream));
    c->d2h_pending[b] = true;
    return SDMD_OK;
  }
  int st = sync_all(c);
  if (st) return st;
  DevState hs{};
  CK(cudaMemcpy(&hs, c->dst, sizeof(hs), cudaMemcpyDeviceToHost));
  long long bf = hs.bg_frame;
  if (hs.committed == 0 || bf <= 0) bf = -1;
  if (frame) *frame = bf;
  if (bf < 0) return SDMD_E_STATE;
  const int b = (int)(bf & 1);
  const cudaMemcpyKind kind = where == SDMD_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (lowrank) CK(cudaMemcpyAsync(lowrank, c->bg_low[b], n * c->es, kind, c->stream));
  if (sparse) CK(cudaMemcpyAsync(sparse, c->bg_sparse[b], n * c->es, kind, c->stream));
  if (mask) CK(cudaMemcpyAsync(mask, c->bg_mask[b], n, kind, c->stream));
  if (where == SDMD_HOST) CK(cudaStreamSynchronize(c->stream));
  return SDMD_OK;
}

int sdmd_get_background_window(sdmd_ctx* c, void* lowrank, void* sparse, uint8_t* mask, int64_t ld,
                               int64_t* frame) {
  SDMD_NVTX();
  if (!c || ld < c->cfg.n_local) return invalid(c, "get_background_window: bad argument");
  if (c->cfg.storage != SDMD_DENSE || !c->cfg.dmd || c->cfg.bg_modes > 1)
    return invalid(c, "get_background_window: dense single-mode DMD contexts only");
  CK(cudaSetDevice(c->dev));
  K4Result res{};
  int st = newest_result(c, &res);              // synchronises
  if (st) return st;
  if (frame) *frame = res.frame;
  if (res.status && res.status != SDMD_W_SINGULAR) return res.status;
  const long long f = c->last_dmd;
  if (win_of(c, f) < c->cfg.m) { c->err = "get_background_window: newest DMD window not full"; return SDMD_E_STATE; }
  if (res.idx < 0) { c->err = "get_background_window: no background mode"; return SDMD_E_NO_VIABLE_MODE; }
  Workspace& k = ws_of(c, f);
  CK(launch_window_background(c->ring, c->ld, c->NS, c->cfg.dtype, c->cfg.n_local, f, c->cfg.m,
                              c->cbuf + (f % c->NC) * c->cfg.m, k.res, lowrank, sparse, mask, ld,
                              c->cfg.threshold, c->stream));
  c->launches += 1;
  CK(cudaStreamSynchronize(c->stream));
  return res.status;
}

int sdmd_score_background(sdmd_ctx* c, int64_t frame, const uint8_t* gt, int where) {
  SDMD_NVTX();
  if (!c || !gt || (where != SDMD_HOST && where != SDMD_DEVICE)) return invalid(c, "score_background: bad argument");
  if (!c->cfg.background) return invalid(c, "score_background: background disabled in config");
  CK(cudaSetDevice(c->dev));
  if (c->bg_last < 0) { c->err = "score_background: no background mask produced yet"; return SDMD_E_STATE; }
  if (frame != c->bg_last) return invalid(c, "score_background: frame is not the newest background frame");
  const size_t n = c->cfg.n_local;
  const uint8_t* g = gt;
  if (where == SDMD_HOST) {                     // stage: the host buffer is free when we return
    if (!c->gt_stage && dalloc(&c->gt_stage, n) != cudaSuccess) return SDMD_E_OOM;
    CK(cudaMemcpyAsync(c->gt_stage, gt, n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    g = c->gt_stage;
  }
  const int b = (int)(c->bg_last & 1);
  CK(cudaStreamWaitEvent(c->stream, c->ev_bgw[b], 0));
  CK(launch_score(c->bg_mask[b], g, (long long)n, c->score_cnt, c->stream));
  c->launches += 1;
  return SDMD_OK;
}

int sdmd_get_scores(sdmd_ctx* c, sdmd_scores* o, int reset) {
  if (!c || !o) return SDMD_E_INVALID;
  if (!c->cfg.background) return invalid(c, "get_scores: background disabled in config");
  CK(cudaSetDevice(c->dev));
  unsigned long long h[4] = {0, 0, 0, 0};
  CK(cudaMemcpyAsync(h, c->score_cnt, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (reset) {
    CK(cudaMemsetAsync(c->score_cnt, 0, sizeof(h), c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  // Table 2 P:437-443 / SPEC S:368; reading Q26 (pooled counts, binary-mask PSNR at the peak)
  const long long tp = (long long)h[0], fp = (long long)h[1], fn = (long long)h[2], fr = (long long)h[3];
  const long long npx = fr * (long long)c->cfg.n_local;
  o->frames = fr; o->tp = tp; o->fp = fp; o->fn = fn; o->tn = npx - tp - fp - fn;
  o->empty_gt = (tp + fn) == 0;
  o->empty_mask = (tp + fp) == 0;
  o->recall = o->empty_gt ? 0.0 : (double)tp / (double)(tp + fn);
  o->precision = o->empty_mask ? 0.0 : (double)tp / (double)(tp + fp);
  o->f_measure = (o->recall + o->precision) == 0.0 ? 0.0
                 : 2.0 * o->precision * o->recall / (o->precision + o->recall);
  o->psnr = (fp + fn) == 0 ? HUGE_VAL : 10.0 * std::log10((double)npx / (double)(fp + fn));
  return SDMD_OK;
}

int sdmd_get_frame_diag(sdmd_ctx* c, int64_t out[24]) {
  if (!c || !out) return SDMD_E_INVALID;
  CK(cudaSetDevice(c->dev));
  K4Result res{};
  int st = newest_result(c, &res);
  if (st) return st;
  for (int i = 0; i < 24; ++i) out[i] = 0;
  out[0] = res.frame; out[1] = res.status; out[2] = res.r; out[3] = res.idx;
  out[4] = res.sweeps; out[5] = res.qr_its;
  for (int q = 0; q < 7; ++q) out[6 + q] = res.phase[q];
  out[13] = res.qr_cnt[0]; out[14] = res.qr_cnt[1]; out[15] = res.qr_cnt[3];
  out[16] = res.phase[7]; out[17] = res.qr_cnt[2]; out[18] = res.qr_dbg[0]; out[19] = res.qr_dbg[1];
  out[20] = res.aberth_its; out[21] = res.aberth_evals; out[22] = res.commit_wait;
  return SDMD_OK;
}

int sdmd_set_timing(sdmd_ctx* c, int enable) {
  if (!c) return SDMD_E_INVALID;
  c->timing = enable != 0;
  if (c->timing) {
    CK(cudaSetDevice(c->dev));
    while (c->ev_pool.size() < 8192) {                 // ≈ 1000 frames of K1/wait/K4a/K4b pairs
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) break;
      c->ev_pool.push_back(e);
    }
  }
  return SDMD_OK;
}

int sdmd_get_stats(sdmd_ctx* c, sdmd_stats* s, int reset) {
  if (!c || !s) return SDMD_E_INVALID;
  CK(cudaSetDevice(c->dev));
  int st = sync_all(c);
  if (st) return st;
  s->k1_launches = (int64_t)c->k1_ev.size();
  s->k4_launches = (int64_t)c->k4_ev.size();
  s->k1_ms = 0.0;
  s->k4_ms = 0.0;
  for (auto& pr : c->k1_ev) { float ms = 0; cudaEventElapsedTime(&ms, pr.first, pr.second); s->k1_ms += ms; }
  s->k1_gap_ms = 0.0;                    // main-stream time between consecutive Gram passes
  for (size_t i = 1; i < c->k1_ev.size(); ++i) {
    float ms = 0;
    cudaEventElapsedTime(&ms, c->k1_ev[i - 1].second, c->k1_ev[i].first);
    s->k1_gap_ms += ms;
  }
  for (auto& pr : c->k4_ev) { float ms = 0; cudaEventElapsedTime(&ms, pr.first, pr.second); s->k4_ms += ms; }
  s->k1_wait_ms = 0.0;
  for (auto& pr : c->wait_ev) { float ms = 0; cudaEventElapsedTime(&ms, pr.first, pr.second); s->k1_wait_ms += ms; }
  s->gpu_launches = c->launches;
  s->collectives = c->collectives;
  if (reset) { destroy_timing(c); c->launches = 0; c->collectives = 0; }
  return SDMD_OK;
}

int sdmd_get_timeline(sdmd_ctx* c, double* out, int cap, int* count) {
  if (!c || !count || cap < 0 || (cap > 0 && !out)) return invalid(c, "get_timeline: bad argument");
  CK(cudaSetDevice(c->dev));
  int st = sync_all(c);
  if (st) return st;
  *count = (int)c->tl.size();
  if (c->tl.empty()) return SDMD_OK;
  const cudaEvent_t t0 = c->tl.front().a;
  const int k = cap < (int)c->tl.size() ? cap : (int)c->tl.size();
  for (int i = 0; i < k; ++i) {
    float s = 0, e = 0;
    cudaEventElapsedTime(&s, t0, c->tl[i].a);
    cudaEventElapsedTime(&e, t0, c->tl[i].b);
    out[4 * i + 0] = (double)c->tl[i].f;
    out[4 * i + 1] = (double)c->tl[i].kind;
    out[4 * i + 2] = s;
    out[4 * i + 3] = e;
  }
  return SDMD_OK;
}

}  // extern "C"
