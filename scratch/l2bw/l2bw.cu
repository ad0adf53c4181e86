// L2 read-throughput microbenchmark (diagnostic, not part of the library):
// every thread streams 16-byte loads over an L2-resident buffer (ld.global.cg
// bypasses L1), repeatedly; bytes / time = the chip's LTS read throughput.
#include <cuda_runtime.h>
#include <stdint.h>
extern "C" __global__ void k_l2read(const double2 *buf, int64_t n2, int reps, double *out) {
  double ax = 0.0, ay = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
      const double2 v = __ldcg(buf + i);
      ax += v.x;
      ay += v.y;
    }
  }
  if (ax + ay == 12345.678) out[0] = ax;  // keep the loads
}
extern "C" int l2_read_bw(const void *buf, int64_t bytes, int reps, int blocks, int threads,
                          double *out, float *ms) {
  const int64_t n2 = bytes / 16;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_l2read<<<blocks, threads>>>((const double2 *)buf, n2, 1, out);  // warm L2
  cudaEventRecord(a);
  k_l2read<<<blocks, threads>>>((const double2 *)buf, n2, reps, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
