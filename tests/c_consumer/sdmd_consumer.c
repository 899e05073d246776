/* A plain C consumer of the C ABI (include/sdmd.h), compiled with gcc and linked against
 * libsdmd.so — no Python, no torch.  Mode "cpu": argument/shape validation and status strings
 * only (works without a GPU: every call must fail cleanly, never crash).  Mode "gpu": a streamed
 * DMD of a planted rank-2 signal x_t = Re(φ λ^t) + ... with a known eigenvalue pair e^{±iθ}
 * ("same eigenvalues as A"), pushed from host memory; prints the recovered spectrum and
 * exits 0 iff both eigenvalues match to 1e-9. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "sdmd.h"

static int cpu_mode(void) {
  sdmd_config cfg;
  sdmd_ctx* ctx = NULL;
  if (sdmd_abi_version() != SDMD_ABI_VERSION) { printf("abi mismatch\n"); return 1; }
  if (sdmd_config_init(&cfg) != SDMD_OK) return 2;
  if (strcmp(sdmd_status_string(SDMD_E_NONFINITE), "non-finite frame rejected") != 0) return 3;
  cfg.n_local = cfg.n_global = 1000;
  cfg.m = 1;                                           /* m < 2: rejected before any device work */
  if (sdmd_create(&cfg, &ctx) != SDMD_E_INVALID || ctx != NULL) return 4;
  cfg.m = 8;
  cfg.storage = SDMD_SPARSE;                           /* sparse without nnz_cap */
  if (sdmd_create(&cfg, &ctx) != SDMD_E_INVALID) return 5;
  if (sdmd_push_dense(NULL, NULL, SDMD_HOST) != SDMD_E_INVALID) return 6;
  if (sdmd_sync(NULL, NULL) != SDMD_E_INVALID) return 7;
  if (sdmd_get_scores(NULL, NULL, 0) != SDMD_E_INVALID) return 8;
  printf("cpu ok (abi %d)\n", sdmd_abi_version());
  return 0;
}

static int gpu_mode(void) {
  const int n = 2048, m = 8, T = 24;
  const double th = 0.3, rho = 0.98;
  sdmd_config cfg;
  sdmd_config_init(&cfg);
  cfg.n_local = cfg.n_global = n;
  cfg.m = m;
  cfg.dtype = SDMD_F64;
  cfg.workers = 1;
  sdmd_ctx* ctx = NULL;
  int st = sdmd_create(&cfg, &ctx);
  if (st) { printf("create: %s\n", sdmd_status_string(st)); return 10; }
  double* x = (double*)malloc(sizeof(double) * n);
  for (int t = 0; t < T; ++t) {
    /* x_t = ρ^t (a cos(tθ) − b sin(tθ)): eigenvalues ρ e^{±iθ} of the rank-2 propagator */
    const double c = pow(rho, t) * cos(t * th), s = pow(rho, t) * sin(t * th);
    for (int i = 0; i < n; ++i) {
      const double a = sin(0.01 * i + 0.3), b = cos(0.023 * i * i / n + 1.1);
      x[i] = a * c - b * s;
    }
    st = sdmd_push_dense(ctx, x, SDMD_HOST);
    if (st) { printf("push %d: %s\n", t, sdmd_status_string(st)); return 11; }
  }
  int64_t failed = -1;
  if ((st = sdmd_sync(ctx, &failed))) { printf("sync: %s\n", sdmd_status_string(st)); return 12; }
  int32_t r = 0, idx = -1;
  int64_t frame = -1;
  double lam[2 * SDMD_MAX_R];
  st = sdmd_get_spectrum(ctx, &r, lam, NULL, &idx, &frame);
  if (st) { printf("spectrum: %s\n", sdmd_status_string(st)); return 13; }
  const double er = rho * cos(th), ei = rho * sin(th);
  double e0 = hypot(lam[0] - er, fabs(lam[1]) - ei), e1 = hypot(lam[2] - er, fabs(lam[3]) - ei);
  printf("gpu: frame %lld r %d lambda (%.15f, %.15f) (%.15f, %.15f) err %.2e %.2e\n", (long long)frame, r,
         lam[0], lam[1], lam[2], lam[3], e0, e1);
  sdmd_destroy(ctx);
  free(x);
  return (r == 2 && e0 < 1e-9 && e1 < 1e-9 && lam[1] * lam[3] < 0) ? 0 : 14;
}

int main(int argc, char** argv) {
  if (argc > 1 && strcmp(argv[1], "gpu") == 0) return gpu_mode();
  return cpu_mode();
}
