// bdem_common.cuh -- launch helpers and deterministic reductions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bdem_sm100.h"

namespace bdem {

constexpr int kRedBlocks = BDEM_RED_BLOCKS;
constexpr int kClampCounter = 5;  // sys->counter slot: queued indefinite blocks
constexpr int kThreads = 256;

// SpMV coefficient layout in sys->scoef (see BDEM_CF_* in the header): the
// 14 coefficients of a 32-position block are one contiguous 3.5 KB record;
// inside it, coefficient k of lane l sits at 64 (k >> 1) + 2 l + (k & 1)
// (pairs of coefficients interleaved per lane), so a lane reads its 14
// values as 7 aligned 16-byte loads and a warp's load of one pair is a
// contiguous 512-byte segment.
// offset of coefficient k from the lane's base cf_idx(pos, 0)
__host__ __device__ __forceinline__ constexpr int cf_rel(int k) {
  return 64 * (k >> 1) + (k & 1);
}
__host__ __device__ __forceinline__ int64_t cf_idx(int64_t pos, int k) {
  return (pos & ~int64_t(31)) * BDEM_CF_COUNT + 2 * (pos & 31) + cf_rel(k);
}

// the 14 coupling coefficients of one position
struct Coef {
  double n[3], al, be, C[9];
};
template <bool kGlobal>
__device__ __forceinline__ Coef load_coef(const double *base) {
  Coef c;
  double v[BDEM_CF_COUNT];
  const double2 *b2 = reinterpret_cast<const double2 *>(base);
#pragma unroll
  for (int j = 0; j < BDEM_CF_COUNT / 2; ++j) {
    const double2 t = kGlobal ? __ldg(b2 + 32 * j) : b2[32 * j];
    v[2 * j] = t.x;
    v[2 * j + 1] = t.y;
  }
#pragma unroll
  for (int t = 0; t < 3; ++t) c.n[t] = v[BDEM_CF_N + t];
  c.al = v[BDEM_CF_ALPHA];
  c.be = v[BDEM_CF_BETA];
#pragma unroll
  for (int t = 0; t < 9; ++t) c.C[t] = v[BDEM_CF_C + t];
  return c;
}
// coefficients 2j and 2j + 1 of one position as one 16-byte store (a warp's
// store of a pair is one contiguous 512-byte segment)
__device__ __forceinline__ void store_coef_pair(double *base, int j, double a, double b) {
  *reinterpret_cast<double2 *>(base + cf_rel(2 * j)) = make_double2(a, b);
}
__device__ __forceinline__ void store_coef(double *base, const double v[BDEM_CF_COUNT]) {
#pragma unroll
  for (int j = 0; j < BDEM_CF_COUNT / 2; ++j) store_coef_pair(base, j, v[2 * j], v[2 * j + 1]);
}

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// kernels launched by this library (defined in topology_kernels.cu)
void count_launches(int64_t k);

inline int launch_status(int64_t kernels = 1) {
  count_launches(kernels);
  return cudaGetLastError() == cudaSuccess ? BDEM_OK : BDEM_ERR_CUDA;
}

inline unsigned int grid_for(int64_t n, int threads = kThreads, int cap = 1 << 20) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned int>(g);
}

// Deterministic block sum: fixed xor-butterfly inside warps, fixed order
// across warps.  Result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NT / 32; ++k) s += sh[k];
  }
  return s;
}

// Two / three block sums in one shared-memory round (2 barriers instead of
// 2 per value); each value is reduced exactly as block_sum does (same
// butterfly, same warp order), so the results are bit-identical to it.
// `sh` holds K * NT / 32 doubles.  Results valid in thread 0.
template <int NT, int K>
__device__ __forceinline__ void block_sum_k(double (&v)[K], double *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) sh[k * (NT / 32) + w] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < NT / 32; ++q) s += sh[k * (NT / 32) + q];
      v[k] = s;
    }
  }
}

template <int NT>
__device__ __forceinline__ double block_max(double v, double *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NT / 32; ++k) s = fmax(s, sh[k]);
  }
  return s;
}

// partial layout: red[col * kRedBlocks + block]
__device__ __forceinline__ double *red_slot(double *red, int col, int block) {
  return red + static_cast<int64_t>(col) * kRedBlocks + block;
}

// "last block finishes" pattern: every block has stored its partials; the
// block that increments `counter` last sums them in a fixed order.  Returns
// true in all threads of the last block.
__device__ __forceinline__ bool last_block(unsigned int *counter) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(counter, 1u);
    am_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (am_last) {
    __threadfence();
    if (threadIdx.x == 0) *counter = 0u;
  }
  return am_last;
}

// fixed-order sum of nb partials of one column, by one block
template <int NT>
__device__ __forceinline__ double sum_partials(const double *red, int col, int nb, double *sh) {
  double v = 0.0;
  const volatile double *col_ptr = red + static_cast<int64_t>(col) * kRedBlocks;
  for (int b = threadIdx.x; b < nb; b += NT) v += col_ptr[b];
  return block_sum<NT>(v, sh);
}

}  // namespace bdem
