// Microbenchmark: 1D cp.async.bulk global->shared streaming bandwidth as a
// function of copy size and pipeline depth (persistent CTAs, one producer lane).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int COPIES>  // copies per stage (issued by lanes 0..COPIES-1)
__global__ void k_stream(const char *src, size_t total, int copy_bytes, int depth, double *sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bars[16];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const size_t stage_bytes = (size_t)copy_bytes * COPIES;
  const size_t nchunks = total / stage_bytes;
  if (threadIdx.x == 0) {
    for (int k = 0; k < depth; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bars[k])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](size_t chunk, int k) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bars[k])),
                   "r"((uint32_t)stage_bytes) : "memory");
    __syncwarp();
    if (lane < COPIES) {
      const char *g = src + chunk * stage_bytes + (size_t)lane * copy_bytes;
      char *d = sm + (size_t)k * stage_bytes + (size_t)lane * copy_bytes;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su(d)), "l"(g), "r"((uint32_t)copy_bytes), "r"(su(&bars[k])) : "memory");
    }
  };
  if (w == 0)
    for (int k = 0; k < depth; ++k) {
      size_t c = blockIdx.x + (size_t)k * gridDim.x;
      if (c < nchunks) issue(c, k);
    }
  double acc = 0;
  int it = 0;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
    const int k = it % depth;
    const uint32_t par = (it / depth) & 1;
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
                 ::"r"(su(&bars[k])), "r"(par) : "memory");
    acc += ((const double *)(sm + (size_t)k * stage_bytes))[threadIdx.x % (stage_bytes / 8)];
    __syncthreads();
    if (w == 0) {
      size_t nc = c + (size_t)depth * gridDim.x;
      if (nc < nchunks) issue(nc, k);
    }
  }
  if (acc == 12345.0) sink[0] = acc;
}

int main() {
  const size_t total = 2ull << 30;
  char *src; double *sink;
  cudaMalloc(&src, total); cudaMalloc(&sink, 8);
  cudaMemset(src, 0, total);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int sizes[] = {256, 1024, 2048, 4096, 8192, 16384, 32768};
  printf("copy_bytes copies/stage depth ctas/sm smem_KB GB/s\n");
  for (int cs : sizes)
    for (int copies : {1, 8, 16}) for (int depth : {2, 4, 8}) for (int per : {1, 2, 4}) {
      size_t smem = (size_t)cs * copies * depth;
      if (smem * per > 220 * 1024 || smem > 200 * 1024) continue;
      auto kern = copies == 1 ? k_stream<1> : (copies == 8 ? k_stream<8> : k_stream<16>);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int grid = sms * per;
      kern<<<grid, 128, smem>>>(src, total, cs, depth, sink);
      cudaEventRecord(a);
      for (int r = 0; r < 3; ++r) kern<<<grid, 128, smem>>>(src, total, cs, depth, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      printf("%6d %3d %2d %d %6.1f %7.0f\n", cs, copies, depth, per, smem / 1024.0, 3.0 * total / (ms * 1e-3) / 1e9);
    }
  return 0;
}
