// DMMA (mma.sync m8n8k4 f64) throughput against resident warps per SM and independent accumulator
// chains per warp -- the occupancy / ILP the FP64 tensor kernels (block-Jacobi round, wide-QR
// update, TSQR pass B) need to approach the 37 TFLOP/s of tools/fp64_peak.cu (64 warps x 8 chains).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_ilp tools/dmma_ilp.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int NCH>
__global__ void k_dmma(double* out, double a) {
  double c[NCH][2];
  double av = a * (threadIdx.x + 1), bv = a * 0.5;
#pragma unroll
  for (int i = 0; i < NCH; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int NCH>
static void run(int sms, int warps_per_sm, double* d) {
  const int threads = warps_per_sm <= 32 ? warps_per_sm * 32 : 1024;
  const int blocks = sms * (warps_per_sm * 32 / threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k_dmma<NCH><<<blocks, threads>>>(d, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  const double flops = 2.0 * 256.0 * NCH * ITERS * (double)blocks * threads / 32.0;
  printf("{\"warps_per_sm\": %d, \"chains\": %d, \"tflops\": %.2f}\n", warps_per_sm, NCH, flops / best / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 4096 * sizeof(double));
  for (int w : {4, 8, 16, 32, 64}) {
    run<4>(sms, w, d);
    run<8>(sms, w, d);
    run<16>(sms, w, d);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
