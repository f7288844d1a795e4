// FP64 peak microbenchmark for the roofline denominators of DESIGN.md §7:
//   (1) DFMA throughput (FP64 FMA pipe), (2) DMMA.8x8x4 throughput (mma.sync f64).
// Each thread runs many independent dependency chains so the pipe, not latency, bounds it.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void k_dmma(double* out, double a) {
  double c[8][2];
  double av = a * (threadIdx.x + 1), bv = a * 0.5;
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d;
  cudaMalloc(&d, 4096 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 512;
  float best_f = 1e30f, best_m = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(d, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best_f) best_f = ms;
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(d, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best_m) best_m = ms;
  }
  const double nthr = (double)blocks * threads;
  const double f_flops = nthr * ITERS * 16 * 2.0;
  const double m_flops = (nthr / 32.0) * ITERS * 8 * (8.0 * 8 * 4 * 2);
  printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, "
         "\"dfma_ms\": %.3f, \"dmma_ms\": %.3f, \"err\": \"%s\"}\n",
         sms, clk / 1e3, f_flops / best_f / 1e9, m_flops / best_m / 1e9, best_f, best_m,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
