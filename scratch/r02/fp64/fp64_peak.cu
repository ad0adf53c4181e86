// FP64 DFMA peak of this B200: every thread runs 8 independent FMA chains
// (enough ILP to cover the pipe latency), grid = SMs x 8 CTAs x 256 threads.
// Prints one JSON line: TFLOP/s (2 flops per DFMA), clocks via cudaDeviceProp.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_dfma(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double *out;
  cudaMalloc(&out, sizeof(double));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  for (int w = 0; w < 3; ++w) k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * (double)blocks * threads * iters * 16 * 8;
  printf("{\"fp64_dfma_tflops\": %.3f, \"ms\": %.3f, \"sms\": %d, \"max_clock_mhz\": %d, "
         "\"per_sm_per_clk_dfma\": %.2f}\n",
         flops / (best * 1e-3) / 1e12, best, sms, clk / 1000,
         flops / 2.0 / (best * 1e-3) / (sms * (clk * 1e3)));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
