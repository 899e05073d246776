// fp64 tensor-core (DMMA m8n8k4) peak microbenchmark for the K2 / K1b roofline denominators.
// MEASURED_PEAKS.json carries no fp64 entry, so this measures one: every warp issues long chains
// of independent mma.sync.m8n8k4.f64 (8 accumulators, no memory traffic), grid = SMs x CTAs/SM.
// flops per mma = 2*8*8*4 = 512.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// dmma_peak.cu -o dmma_peak ; run: ./dmma_peak  -> one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;   // never true; keeps the chain alive
}

__global__ void dfma_loop(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  const double a = 0.999999, b = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  double best_dmma = 0, best_dfma = 0;
  int best_w = 0;
  for (int warps = 2; warps <= 16; warps *= 2) {
    for (int rep = 0; rep < 3; ++rep) {
      dmma_loop<<<sms * 2, 32 * warps>>>(out, iters / 10);
      cudaEventRecord(e0);
      dmma_loop<<<sms * 2, 32 * warps>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 512.0 * 8 * iters * (double)(sms * 2) * warps;
      double tf = fl / (ms * 1e-3) / 1e12;
      if (tf > best_dmma) { best_dmma = tf; best_w = warps; }
      if (rep == 2) printf("{\"warps_per_sm\": %d, \"dmma_f64_tflops\": %.3f}\n", 2 * warps, tf);
    }
  }
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    dfma_loop<<<sms * 4, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)(sms * 4) * 256;
    double tf = fl / (ms * 1e-3) / 1e12;
    if (tf > best_dfma) best_dfma = tf;
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"dmma_f64_tflops\": %.3f, \"dmma_warps_per_cta\": %d, \"dfma_f64_tflops\": %.3f, "
         "\"sms\": %d, \"clock_khz_attr\": %d, \"err\": \"%s\"}\n",
         best_dmma, best_w, best_dfma, sms, clk, cudaGetErrorString(err));
  return 0;
}
