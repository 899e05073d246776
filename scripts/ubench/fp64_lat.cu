// Latency of dependent fp64 operations on this GPU (clock64 cycles per op), single thread.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x0, int n) {
  double x = x0;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 1.0000001, 1e-9);
  t1 = clock64(); cyc[0] = t1 - t0; out[0] = x;
  x = x0; t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64(); cyc[1] = t1 - t0; out[1] = x;
  x = x0; t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  t1 = clock64(); cyc[2] = t1 - t0; out[2] = x;
  x = x0; t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x + 1.0);
  t1 = clock64(); cyc[3] = t1 - t0; out[3] = x;
  x = x0; t0 = clock64();
  for (int i = 0; i < n; ++i) x = __drcp_rn(x + 1.0);
  t1 = clock64(); cyc[4] = t1 - t0; out[4] = x;
  float y = (float)x0; t0 = clock64();
  for (int i = 0; i < n; ++i) y = 1.0f / (y + 1.0f);
  t1 = clock64(); cyc[5] = t1 - t0; out[5] = y;
  __shared__ double sh[64];
  sh[threadIdx.x] = x0; int j = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { j = (int)sh[j & 31]; }
  t1 = clock64(); cyc[6] = t1 - t0; out[6] = j;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 64); cudaMalloc(&c, 64);
  const int n = 10000;
  k<<<1, 1>>>(d, c, 0.5, n);
  long long h[8]; cudaMemcpy(h, c, 56, cudaMemcpyDeviceToHost);
  const char* nm[] = {"dfma", "ddiv", "dsqrt", "drsqrt", "drcp_rn", "fdiv", "lds_chain"};
  for (int i = 0; i < 7; ++i) printf("%-10s %.1f cycles/op\n", nm[i], (double)h[i] / n);
  return 0;
}
