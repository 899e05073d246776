/*
 * sdmd.h — C ABI of the B200-native streaming method-of-snapshots SVD / DMD library
 *          (hot path of arXiv 1612.07875, "streaming DMD"; PAPER.md cited as P:<line>).
 *
 * One context (sdmd_ctx) owns a sliding window of tall-skinny snapshots x_t (n rows each) in an
 * HBM ring buffer, the window's Gram matrix G = Zᵀ Z (Z = [x_{t-m} … x_t], n x (m+1)), and the
 * small on-device eigenproblems that turn G into the DMD of the window:
 *
 *   push x_t  →  g_k = <x_{t-m+k}, x_t>, k = 0..m           (§3.1; Alg 1)
 *             →  [allreduce of g over row shards]             (row sharding; no paper analogue)
 *             →  commit: G ← slide(G) with g as last row/col  (Alg 1)
 *             →  S = XᵀX = G[0:m,0:m]:   S V = V Λ,  Σ = sqrt|Λ| sorted desc   (§2.1; Alg 1)
 *             →  Ã = (VΣ⁻¹)ᵀ XᵀX' (VΣ⁻¹),  XᵀX' = G[0:m,1:m+1]                 (Eq. Atilde; Alg 2)
 *             →  Ã W = W Λ                                                     (Alg 2)
 *             →  α₁ = Σ V[0,:]ᵀ,  b = (WΛ)⁻¹ α₁  (only b_idx per frame)          (§3.3; Alg 3)
 *             →  idx = argmin |log λ_i|                                         (Alg 3)
 *             →  l = b_idx φ_idx λ_idx^m,  s = x − |l|,  mask = s > threshold   (Alg 3)
 *
 * Everything after sdmd_create runs on the GPU (sm_100a).  There is no CPU fallback: every
 * entry point returns SDMD_E_CUDA if the device work cannot be launched.
 *
 * Conventions
 *  - Every function returns an int status (enum below); 0 = SDMD_OK.  No exceptions, no abort,
 *    no exit cross the ABI.  Argument/shape errors are returned before anything is enqueued.
 *  - Matrices are column-major unless stated.  Complex numbers are interleaved (re, im) doubles.
 *  - `where` says where a caller buffer lives: SDMD_HOST (pageable or pinned host memory) or
 *    SDMD_DEVICE (device pointer on the ctx's device).
 *  - Stream semantics: all device work of a ctx is ordered on the ctx stream (cfg.stream, or a
 *    stream the ctx creates) plus internal eigen-worker streams joined back to it.  DEVICE
 *    inputs must stay valid and unmodified until the ctx stream passes the push (e.g. until
 *    sdmd_sync).  HOST inputs are read in stream order as well (pinned memory: asynchronously;
 *    pageable memory: copied before the call returns).  Calls that return HOST outputs
 *    synchronise the ctx first.
 *  - Device-detected errors (non-finite frame) are recorded in a device status word; the frame
 *    is rejected ON THE DEVICE (state bit-identical) and every frame pushed after it is
 *    discarded until the next sdmd_sync(), which returns the error and the rejected frame index.
 *    The device also sets a host-visible mirror of the status; a push (or sdmd_acquire_slot)
 *    whose ring slot could hold data the rolled-back state still needs first waits for the
 *    commit of the frame `D` pushes earlier (D = ring slots − frames the state reads, >= 8 thanks
 *    to spare slots) and, if the stream is poisoned, returns SDMD_E_NONFINITE WITHOUT writing or
 *    enqueuing anything; call sdmd_sync to learn the rejected frame and resume.  The host thus
 *    never runs more than D frames ahead of the device's commits.
 *  - One writer per ctx.  With nranks > 1, sdmd_init_window and sdmd_push_* are collective:
 *    every rank calls them in the same order (NCCL semantics).
 *
 * Environment (read at sdmd_create; experiment and test knobs, defaults are the measured best):
 *    SDMD_K1_WAVES=w     Gram pass as w x SMs short CTAs instead of the persistent grid
 *    SDMD_K1=v1          the earlier 8-rows-per-lane Gram kernel (A/B; checked by the tests)
 *    SDMD_WARM=0         no Jacobi warm start;   SDMD_THROTTLE=0  no eigen-work flow control
 *    SDMD_WA=n           n cluster eigen streams; SDMD_BG_NODMD=1 background pass with c = 0
 *    SDMD_LOCAL_GROUP=1  TEST ONLY: nranks > 1 contexts of one process on one device exchange
 *                        through an in-process group instead of NCCL (keyed by nccl_uid bytes;
 *                        each rank driven by its own host thread)
 */
#ifndef SDMD_H
#define SDMD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDMD_ABI_VERSION 4
#define SDMD_MAX_M 256   /* largest window width m supported                              */
#define SDMD_MAX_LAG 64  /* largest background lag (frames)                                     */
#define SDMD_MAX_BATCH 8 /* largest k of sdmd_push_batch                                          */
#define SDMD_MAX_BG_MODES 8 /* largest background mode set (plus a conjugate partner)             */
#define SDMD_MAX_R 224   /* largest rank r (shared-memory Hessenberg QR)    */

enum sdmd_status {
  SDMD_OK = 0,
  SDMD_E_INVALID = 1,          /* bad argument, shape or config          */
  SDMD_E_NONFINITE = 2,        /* a pushed frame had a non-finite self inner product  */
  SDMD_E_WINDOW_NOT_FULL = 3,  /* fewer than m+1 frames pushed yet (warm-up, Q14)             */
  SDMD_E_ZERO_MATRIX = 4,      /* σ₁ == 0 (all-zero window) or r == 0                 */
  SDMD_E_NO_CONVERGENCE = 5,   /* an on-device eigensolver exceeded its sweep budget   */
  SDMD_W_SINGULAR = 6,         /* WΛ numerically singular; amplitudes of zero modes set to 0 */
  SDMD_E_NO_VIABLE_MODE = 7,   /* every DMD eigenvalue is zero: no background mode    */
  SDMD_E_CUDA = 8,             /* CUDA runtime error (details in sdmd_last_error)             */
  SDMD_E_NCCL = 9,             /* NCCL error or NCCL unavailable for nranks > 1               */
  SDMD_E_OOM = 10,             /* device allocation failed                                    */
  SDMD_E_STATE = 11            /* call not valid in the current state (e.g. no DMD computed)  */
};

enum sdmd_dtype { SDMD_F32 = 0, SDMD_F64 = 1 };
enum sdmd_storage { SDMD_DENSE = 0, SDMD_SPARSE = 1 };
/* Basis of sparse snapshots (§3.5 P:355-363 "Fourier" compression; readings Q10, Q11, Q27):
 *  SDMD_BASIS_DCT   real orthonormal 2-D DCT-II coefficients; val = nnz doubles
 *  SDMD_BASIS_FFT   unitary 2-D DFT of a real field, FULL spectrum stored (every bin's conjugate
 *                   partner present); val = nnz interleaved complex (re, im); g = Σ Re(conj(ẑ) x̂)
 *  SDMD_BASIS_RFFT  the stored HALF spectrum of a real grid_rows x grid_cols field (rfft2 layout:
 *                   index ky*(grid_cols/2+1) + kx); val = nnz interleaved complex; every bin off
 *                   the self-conjugate columns kx = 0 and kx = grid_cols/2 (even grid_cols)
 *                   counts twice (its omitted conjugate partner), g = Σ w Re(conj(ẑ) x̂)        */
enum sdmd_basis { SDMD_BASIS_DCT = 0, SDMD_BASIS_FFT = 1, SDMD_BASIS_RFFT = 2 };
enum sdmd_where { SDMD_HOST = 0, SDMD_DEVICE = 1, SDMD_HOST_ASYNC = 2 /* pinned host, stream-ordered */,
                  SDMD_DEVICE_READY = 3 /* device buffer already complete: sdmd_push_dense only */ };

typedef struct sdmd_ctx sdmd_ctx; /* opaque; owns ALL device state (ring, G history, factors) */

typedef struct sdmd_config {
  /* rows: this rank holds rows [row_begin, row_begin + n_local) of n_global (dense), or the
   * coefficient indices in that range (sparse).  Single GPU: row_begin = 0, n_local = n_global. */
  int64_t n_global;
  int64_t row_begin;
  int64_t n_local;
  int32_t m;          /* width of X; the window holds m+1 snapshots. 2 <= m <= SDMD_MAX_M */
  int32_t dtype;      /* dense storage dtype SDMD_F32 | SDMD_F64 (sparse values are always f64) */
  int32_t storage;    /* SDMD_DENSE | SDMD_SPARSE (orthonormal-DCT coefficient snapshots, §3.5) */
  int32_t nnz_cap;    /* sparse: max nonzeros per snapshot held by this rank                   */
  int32_t r_max;      /* rank cap; 0 → min(m, SDMD_MAX_R)                                      */
  double rank_tol;    /* r = min(r_max, #{σ_i > rank_tol·σ₁}); 0 → 1e-7 (reading Q7)         */
  float threshold;    /* foreground threshold on s = x − |l| (".2"), strict '>'          */
  int32_t background; /* 1: compute the newest background column every push (fused into the Gram
                       * pass, emitted with a lag of `lag` frames, see sdmd_info); 0: off       */
  int32_t dmd;        /* 1: run the DMD (a5..a10) on every push once the window is full       */
  int32_t workers;    /* eigen-worker budget W, 1..24 (0 → 4): the context runs max(2, W/4) single-
                       * CTA streams (K4b; W/2 with bg_modes > 1) and W/2 four-CTA cluster streams (K4a; W − W/4 for sparse
                       * storage; min(2W, 30 − W, 20) when r_max <= m/4; W when m <= 64).  About
                       * W + 2 streams in all: set CUDA_DEVICE_MAX_CONNECTIONS >= that (e.g. 32)
                       * before CUDA initialises, else streams share hardware queues and the
                       * eigen stages serialise behind unrelated waits                          */
  int32_t device;     /* CUDA device ordinal                                                   */
  void* stream;       /* cudaStream_t to order work on, or NULL (the ctx creates one)          */
  int32_t rank;       /* this rank, 0..nranks-1                                                 */
  int32_t nranks;     /* row shards; > 1 needs NCCL (uid from sdmd_nccl_unique_id on rank 0)   */
  const uint8_t* nccl_uid; /* 128 bytes, identical on all ranks; ignored when nranks == 1       */
  int32_t lag;        /* background lag in frames, 1..64; 0 → 2·workers (one rank) or workers·nranks + 6
                       * (eigen-sharded ranks), at most 64.  K1(t+lag)
                       * consumes the background coefficients of frame t, so K4 may take up to
                       * lag frame periods before the Gram pass waits                          */
  int32_t eigen_shard; /* nranks > 1: 1 → the eigenproblems of frame t run only on rank t mod
                       * nranks; its m background coefficients ride the allreduce of a later
                       * frame's Gram column (owner's values, zeros elsewhere: one collective per
                       * push) before the Gram pass that consumes them; the getters of a rank
                       * then report the newest frame it solved.  0 → replicated on every rank */
  int32_t batch_max;  /* largest k accepted by sdmd_push_batch, 0..SDMD_MAX_BATCH (0: batching
                       * off); the ring holds m + batch_max + 1 slots                          */
  int32_t bg_modes;   /* background modes: 0 or 1 → the single
                       * slowest mode of Alg 3; nb = 2..SDMD_MAX_BG_MODES → l = Σ_{p∈B} b_p φ_p λ_p^m
                       * over B = the nb smallest |log λ| (Q5's order), closed under conjugation
                       * (reading Q25); one inverse iteration per mode in K4     */
  int32_t buildup;    /* 1: DMD during the build-up ("start the
                       * algorithm with only 2 columns"): every push from the 2nd frame on runs
                       * the DMD of the growing window (X = the t columns x_0..x_{t-1}); the
                       * getters then report windows narrower than m (sigma zero-padded, V
                       * with leading dimension m).  No background before the window is full */
  int32_t modes_every_frame; /* 1 (dense, one rank): the DMD modes Φ = X'(YW) of every frame are
                       * computed on its eigen-worker stream (all r eigenvectors, then K2 on
                       * DMMA; SURVEY §8(f) NEXT-2 "full Φ every frame") and sdmd_get_modes
                       * returns the newest frame's columns without recomputing.  Meant for
                       * small r (C2: r = 21); at C4 (r = 200) it would cost ~0.1 s per frame */
  int32_t basis;      /* sparse storage: enum sdmd_basis (0 = DCT)                              */
  int32_t grid_rows;  /* 2-D grid of the sparse transform (0: unknown).  DCT / FFT: n_global =   */
  int32_t grid_cols;  /* grid_rows*grid_cols; RFFT: n_global = grid_rows*(grid_cols/2+1) and the
                       * grid is required (the weights depend on grid_cols).  A sparse DCT context
                       * with background = 1 returns its background in PIXEL space (SURVEY §8(f)
                       * NEXT-3 "inverse-DCT kernel for pixel-space background"): one rank, grid
                       * sides powers of two in [2, 4096], pixels row-major, fp64 outputs        */
} sdmd_config;

typedef struct sdmd_info {
  int64_t frames;       /* frames accepted so far (exact after sdmd_sync)                        */
  int32_t window;       /* columns currently held (<= m+1)                                       */
  int32_t lag;          /* background of frame t is produced by the push of frame t + lag        */
  int32_t ring_slots;   /* HBM ring slots                                                        */
  int32_t workers;      /* single-CTA eigen-stage streams (K4b)                                  */
  int64_t ring_bytes;   /* device bytes of the ring                                              */
  int64_t ld;           /* ring slot stride in elements                                          */
  int32_t cluster_workers; /* streams of the 4-CTA cluster eigen stage (K4a)                     */
  int32_t k1_grid;      /* CTAs per Gram pass                                                    */
} sdmd_info;

typedef struct sdmd_stats {
  int64_t k1_launches;  /* Gram-update (K1/K3) launches timed since the last reset               */
  double k1_ms;         /* their summed device time (CUDA events on the ctx stream)             */
  int64_t k4_launches;  /* per-frame eigen (K4) launches                                         */
  double k4_ms;         /* summed device time of K4 (events on the worker streams)               */
  int64_t gpu_launches; /* all kernels this ctx launched since the last reset                   */
  double k1_gap_ms;     /* summed ctx-stream time between consecutive Gram passes (ingest, waits) */
  double k1_wait_ms;    /* part of k1_gap_ms spent waiting for background coefficients (K4)     */
  int64_t collectives;  /* collectives (allreduce/broadcast) issued since the last reset: one per
                         * push at nranks > 1 (the Gram column and, under eigen sharding, the
                         * background coefficients of a later frame share it)                  */
} sdmd_stats;

/* BMC-style scores of the background masks (Table 2 P:437-443 "Recall,
 * Precision, F-measure, Psnr"; reading Q26): counts pooled over every mask scored
 * since the last reset, this rank's rows. */
typedef struct sdmd_scores {
  int64_t frames;       /* masks scored                                                          */
  int64_t tp, fp, fn, tn; /* pixel counts: mask & gt, mask & !gt, !mask & gt, !mask & !gt         */
  double recall;        /* tp / (tp + fn); 0 with empty_gt                                        */
  double precision;     /* tp / (tp + fp); 0 with empty_mask                                      */
  double f_measure;     /* 2PR / (P + R); 0 when P + R = 0                                        */
  double psnr;          /* binary mask images at the range's peak: 10 log10(N / (fp + fn)) dB over
                         * the N pixels scored; +inf when no pixel differs                         */
  int32_t empty_gt;     /* tp + fn == 0 (recall undefined)                                 */
  int32_t empty_mask;   /* tp + fp == 0 (precision undefined)                              */
} sdmd_scores;

/* Fill *cfg with defaults (rank_tol 1e-7, threshold 0.2, dmd 1, background 0, workers 4, …).
 * n_global/n_local/m must still be set by the caller. */
int sdmd_config_init(sdmd_config* cfg);

/* Create a context: allocates the ring (ring_slots x ld elements of dtype), the Gram history, the
 * eigen-worker workspaces and, for nranks > 1, the NCCL communicator.  *out owned by the caller,
 * released with sdmd_destroy.  Errors: E_INVALID (shape), E_OOM, E_CUDA, E_NCCL. */
int sdmd_create(const sdmd_config* cfg, sdmd_ctx** out);
int sdmd_destroy(sdmd_ctx* ctx);

/* First window in one call (Alg 1 first branch "xtx = X.T * X"): Z is n_local x (m+1),
 * column-major with leading dimension ldz >= n_local, oldest column first, dtype = cfg.dtype.
 * The batch Gram runs on the fp64 tensor pipe (DMMA, kernel K2); the DMD of the window is then
 * computed if cfg.dmd.  Replaces any previous state.  Dense storage only.  A window whose Gram
 * has a non-finite entry is rejected whole: SDMD_E_NONFINITE, the stream is left empty (0 frames). */
int sdmd_init_window(sdmd_ctx* ctx, const void* Z, int64_t ldz, int where);

/* Push one dense snapshot (n_local values of cfg.dtype).  While fewer than m+1 frames are held
 * the column is appended (warm-up, Q14); afterwards the oldest column is dropped (§3.1).  Work is
 * enqueued asynchronously; see the header notes for the NONFINITE contract.
 * where = SDMD_HOST (copied on the context's copy stream, overlapping the previous Gram pass),
 * SDMD_DEVICE (copied into the ring in ctx-stream order, after the work already queued there —
 * including the previous Gram pass), or SDMD_DEVICE_READY: a device buffer whose contents are
 * complete when the call is made (a host-synchronised producer, a static pool); it is copied on
 * the copy stream like a host frame, so the copy overlaps the previous Gram pass instead of
 * sitting between two passes (frames under 1 MB are copied in ctx-stream order as for
 * SDMD_DEVICE: one call, negligible copy time).  In every case x must stay unmodified until the
 * ctx stream passes the push. */
int sdmd_push_dense(sdmd_ctx* ctx, const void* x, int where);

/* Push one sparse snapshot in an orthonormal coefficient basis (§3.5): nnz pairs,
 * idx strictly ascending in [row_begin, row_begin + n_local) (int32), val fp64 — nnz doubles for
 * cfg.basis = SDMD_BASIS_DCT, nnz interleaved complex (2·nnz doubles) for the Fourier bases.
 * nnz <= nnz_cap.  The Gram column uses sparse–sparse inner products (weighted real parts for the
 * Fourier bases, see enum sdmd_basis); nothing is densified in HBM.
 * Errors: nnz > nnz_cap, or (where = SDMD_HOST) indices not strictly ascending / out of range ->
 * SDMD_E_INVALID, nothing queued.  Device-resident indices are checked on the device: a violation
 * rejects the frame like a non-finite one (nothing scattered; the next sdmd_sync returns
 * SDMD_E_NONFINITE with failed_frame = this frame, consistently on every rank). */
int sdmd_push_sparse(sdmd_ctx* ctx, int32_t nnz, const int32_t* idx, const double* val,
                     int where);

/* Push k = 1..cfg.batch_max dense snapshots at once (the paper's future work
 * "dynamic updating with more than one column at a time … to catch up").  X holds k
 * columns of n_local values (cfg.dtype), column-major with leading dimension ldx >= n_local,
 * oldest first.  One pass (kernel K1b, fp64 DMMA) computes the k new Gram columns
 * <x_{t+j-m+i}, x_{t+j}> from the union window of m + k columns — each window element is read
 * once per batch instead of once per frame — and commits them; the results equal k successive
 * sdmd_push_dense calls up to the fixed summation order.  dmd_every = 1: the DMD (a5..a10) runs
 * for every one of the k windows; 0: only for the newest (catch-up mode: the intermediate
 * windows' eigenproblems are skipped).  Requires a full window (>= m+1 frames held) and
 * cfg.background == 0 (else E_STATE / E_INVALID, nothing enqueued).  A batch containing a
 * non-finite value is rejected as a whole (the deferred NONFINITE of sdmd_sync names its first
 * bad frame).  With nranks > 1 the k(m+1) partial values are allreduced in one NCCL call. */
int sdmd_push_batch(sdmd_ctx* ctx, int32_t k, const void* X, int64_t ldx, int where,
                    int32_t dmd_every);

/* Zero-copy ingest: *dev_ptr receives the device address of the slot the next dense frame will
 * occupy (n_local values); fill it (on the ctx stream or before), then sdmd_commit_slot. */
int sdmd_acquire_slot(sdmd_ctx* ctx, void** dev_ptr);
int sdmd_commit_slot(sdmd_ctx* ctx);

/* Order the ctx stream after every eigen-worker launch enqueued so far (device-side join; the
 * host does not wait).  Work enqueued on the ctx stream afterwards — e.g. a CUDA event that ends a
 * timed region — follows the DMD of every pushed frame. */
int sdmd_join(sdmd_ctx* ctx);

/* Wait for all queued work.  Returns the first deferred device error (SDMD_E_NONFINITE) since the
 * previous sync and, if failed_frame != NULL, the index of the rejected frame (-1 if none). */
int sdmd_sync(sdmd_ctx* ctx, int64_t* failed_frame);

int sdmd_get_info(sdmd_ctx* ctx, sdmd_info* info);

/* Gram of the current window in logical (oldest-first) order: k x k doubles where k = columns
 * held (<= m+1), written to host memory G (column-major, ld k).  *k_out receives k. */
int sdmd_get_gram(sdmd_ctx* ctx, double* G, int32_t* k_out);

/* This rank's pre-allreduce Gram column of the last push (k doubles, oldest first). */
int sdmd_get_partial_gram_column(sdmd_ctx* ctx, double* g, int32_t* k_out);

/* Method-of-snapshots SVD of X = window[:, 0:m] of the newest DMD frame (Alg 1): sigma gets m
 * values (descending, sqrt|eig|), V gets m x r (column-major, ld m) or is NULL.  *frame gets the
 * frame index.  Returns E_WINDOW_NOT_FULL during warm-up, or the frame's own status. */
int sdmd_get_svd(sdmd_ctx* ctx, int32_t* r, double* sigma, double* V, int64_t* frame);

/* DMD spectrum of the newest DMD frame: r eigenvalues of Ã (interleaved complex, ordered by |λ|
 * desc, Re desc, Im desc), background index idx (into that order), and, if b != NULL, all r
 * amplitudes b = (WΛ)⁻¹α₁ (computed on demand from left/right eigenvectors).  lambda needs 2r
 * doubles (pass SDMD_MAX_R-sized buffers). */
int sdmd_get_spectrum(sdmd_ctx* ctx, int32_t* r, double* lambda, double* b, int32_t* idx,
                      int64_t* frame);

/* Right eigenvectors W of Ã for the newest DMD frame (r x r complex, column-major, unit-norm,
 * largest entry real positive), host memory. */
int sdmd_get_eigvecs(sdmd_ctx* ctx, double* W, int32_t* r);

/* DMD modes of the newest DMD frame, this rank's rows: Φ[:, cols] = X' V Σ⁻¹ W[:, cols]
 * (Eq. Phi), computed on demand on the fp64 tensor pipe (K2).  phi_dev: device buffer,
 * n_local x ncols complex (interleaved), column-major with leading dimension ld >= n_local.
 * Sparse contexts return the modes in the coefficient space of the pushed snapshots (NEXT-3:
 * Φ̂ = X̂'(YW), accumulated over the sparse window columns in fixed order). */
int sdmd_get_modes(sdmd_ctx* ctx, const int32_t* cols, int32_t ncols, double* phi_dev, int64_t ld);

/* Newest background column produced (frame index in *frame, -1 if none yet): lowrank = |l|,
 * sparse = x − |l| (cfg.dtype, n_local values each; either may be NULL) and mask (uint8, 1 where
 * sparse > threshold; may be NULL).  A sparse DCT context returns them in pixel space: n_local =
 * grid_rows·grid_cols fp64 values, row-major (l = IDCT2(X̂'c), x = IDCT2(x̂), NEXT-3).  where = SDMD_HOST (synchronises) or SDMD_DEVICE (copies on
 * the ctx stream) or SDMD_HOST_ASYNC (pinned host buffers; no host wait: the outputs of the
 * newest enqueued background pass — its frame in *frame — are read back on the context's D2H
 * stream, overlapping the next Gram pass (the outputs are double-buffered by frame parity); the
 * host buffers are valid after sdmd_sync, or on the ctx stream after sdmd_join). */
int sdmd_get_background(sdmd_ctx* ctx, void* lowrank, void* sparse, uint8_t* mask, int64_t* frame,
                        int where);

/* Alg 3's first-window branch (reading Q24) on the window of the newest DMD frame f:
 * for every window column e = 0..m (frames f-m..f), l_e = b_idx φ_idx λ_idx^e, lowrank = |l_e|,
 * sparse = z_e − |l_e|, mask = sparse > threshold.  Outputs are DEVICE buffers (any may be NULL),
 * n_local x (m+1) column-major with leading dimension ld >= n_local (cfg.dtype; mask uint8);
 * *frame = f.  Dense single-mode contexts with dmd = 1 and a full window.  Synchronises.
 * Returns the frame's status (OK or W_SINGULAR), E_STATE / E_NO_VIABLE_MODE when there is no
 * full-window DMD with a background mode. */
int sdmd_get_background_window(sdmd_ctx* ctx, void* lowrank, void* sparse, uint8_t* mask,
                               int64_t ld, int64_t* frame);

/* Score the newest background mask produced (frame `frame`, which must be the frame
 * sdmd_get_background reports, else SDMD_E_INVALID) against the ground-truth foreground mask gt
 * (n_local bytes, nonzero = foreground; SDMD_HOST: copied before the call returns, SDMD_DEVICE:
 * stream-ordered).  Counts accumulate on the device (kernel on the ctx stream, no host wait).
 * Errors: E_INVALID (background off, bad where, frame mismatch), E_STATE (no mask yet). */
int sdmd_score_background(sdmd_ctx* ctx, int64_t frame, const uint8_t* gt, int where);

/* Read (synchronises) and optionally reset the accumulated scores. */
int sdmd_get_scores(sdmd_ctx* ctx, sdmd_scores* out, int reset);

/* Diagnostics of the newest DMD frame: out[0]=frame, [1]=status, [2]=r, [3]=idx, [4]=Jacobi
 * sweeps, [5]=QR iterations, [6..12]=SM cycles spent in the K4 phases (build S, Jacobi, sort/V,
 * Ã, Hessenberg, QR, eigenvectors+c), [13]=single-bulge chase steps, [14]=multishift global
 * steps, [15]=multishift sweeps, [16]=SM cycles spent computing multishift shifts, [17]=single-
 * bulge iterations, [18..19]=SM cycles of the multishift chase phases, [20]=Ehrlich–Aberth
 * iterations of eig(Ã) (0: QR used, −1: Aberth did not certify → QR), [21]=Hyman evaluations.
 * Synchronises. */
int sdmd_get_frame_diag(sdmd_ctx* ctx, int64_t out[24]);

/* Kernel timing (CUDA events around every K1/K3 and K4 launch) and launch counts. */
int sdmd_set_timing(sdmd_ctx* ctx, int enable);
int sdmd_get_stats(sdmd_ctx* ctx, sdmd_stats* stats, int reset);
/* Device timeline of the timed launches since the last stats reset (tracing aid).  Writes
 * min(cap, count) records of 4 doubles {frame, kind, start_ms, end_ms} to host `out`; kind 0 = Gram
 * pass (K1/K3), 1 = K4a, 2 = K4b, 3 = ctx-stream wait for background coefficients; times are
 * relative to the first record's start.  *count = records available.  Synchronises the context.
 * Errors: SDMD_E_INVALID (null ctx/count, cap < 0, out null with cap > 0). */
int sdmd_get_timeline(sdmd_ctx* ctx, double* out, int cap, int* count);

/* NCCL bootstrap: rank 0 calls this and broadcasts the 128 bytes (e.g. torch.distributed). */
int sdmd_nccl_unique_id(uint8_t out[128]);

const char* sdmd_status_string(int status);
const char* sdmd_last_error(const sdmd_ctx* ctx);
int sdmd_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SDMD_H */
