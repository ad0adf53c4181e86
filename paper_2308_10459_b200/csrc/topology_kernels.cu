// topology_kernels.cu -- per-step topology work: hash-grid broad phase,
// connected components over intact bonds, ordered compaction of flags.
//
// Sorting / scans use CUB (header library shipped with the CUDA toolkit)
// inside this library; everything else is hand-written.
#include <atomic>

#include <cub/cub.cuh>

#include "bdem_common.cuh"

namespace bdem {

// ---------------------------------------------------------------------------
// broad phase (contact.py:140-173, solver.py:856-878)
// ---------------------------------------------------------------------------
struct GridHdr {
  long long lo[3];
  long long hi[3];
  unsigned long long rmax_bits;  // max inflated radius (non-negative double's bits)
  double cell;
};

// contact_candidates (solver.py:866-870): inflated radii r + dt |v| +
// dt^2 |g| with numpy's order of operations (|v| = sqrt((x x + y y) + z z);
// travel = dt |v|; travel += dt2g; r + travel), and their maximum (the bits
// of non-negative doubles order like the values)
__global__ void k_inflate(const double *v, const double *radius, int64_t n, double dt,
                          double dt2g, double *out, GridHdr *hdr) {
  __shared__ unsigned long long sh[kThreads / 32];
  unsigned long long m = 0ull;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double x = v[3 * e], y = v[3 * e + 1], z = v[3 * e + 2];
    double travel = dt * sqrt((x * x + y * y) + z * z);
    travel += dt2g;
    const double r = radius[e] + travel;
    out[e] = r;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(r);
    m = bits > m ? bits : m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long u = __shfl_xor_sync(0xffffffffu, m, o);
    m = u > m ? u : m;
  }
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < kThreads / 32; ++k) m = sh[k] > m ? sh[k] : m;
    atomicMax(&hdr->rmax_bits, m);
  }
}

// cell = 2 max(inflated) + 1e-12 (solver.py:871), on the device
__global__ void k_cell_from_rmax(GridHdr *hdr) {
  hdr->cell = 2.0 * __longlong_as_double((long long)hdr->rmax_bits) + 1e-12;
}

__global__ void k_cells(const double *p, int64_t n, const GridHdr *cellh, long long *cxyz,
                        GridHdr *hdr) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  const double cell = cellh->cell;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const long long v = (long long)floor(p[3 * e + c] / cell);
    cxyz[3 * e + c] = v;
    atomicMin(&hdr->lo[c], v);
    atomicMax(&hdr->hi[c], v);
  }
}

__device__ __forceinline__ long long cell_key(long long x, long long y, long long z,
                                              const long long lo[3], long long ny,
                                              long long nz) {
  // +1 margin so neighbour offsets -1..1 stay non-negative and unique
  return ((x - lo[0] + 1) * ny + (y - lo[1] + 1)) * nz + (z - lo[2] + 1);
}

__global__ void k_keys(const long long *cxyz, int64_t n, GridHdr hdr, long long ny, long long nz,
                       unsigned long long *keys, int32_t *ids) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  keys[e] = (unsigned long long)cell_key(cxyz[3 * e], cxyz[3 * e + 1], cxyz[3 * e + 2], hdr.lo,
                                         ny, nz);
  ids[e] = (int32_t)e;
}

__device__ __forceinline__ int64_t lower_bound(const unsigned long long *k, int64_t n,
                                               unsigned long long v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (k[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// pass 0: count pairs per element a (a < b); pass 1: write and sort them,
// interleaved (pairs) or as two planes (pi, pj) when pairs == NULL
__global__ void k_pairs(const double *p, const double *rad, int64_t n, const long long *cxyz,
                        GridHdr hdr, long long ny, long long nz, const unsigned long long *skeys,
                        const int32_t *sids, const int64_t *labels, int32_t *count,
                        const int64_t *offs, int32_t *pairs, int pass, int32_t *pi = nullptr,
                        int32_t *pj = nullptr) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  const long long cx = cxyz[3 * a], cy = cxyz[3 * a + 1], cz = cxyz[3 * a + 2];
  const double pa0 = p[3 * a], pa1 = p[3 * a + 1], pa2 = p[3 * a + 2], ra = rad[a];
  const int64_t la = labels ? labels[a] : 0;
  int cnt = 0;
  int64_t base = pass ? offs[a] : 0;
  for (int dx = -1; dx <= 1; ++dx)
    for (int dy = -1; dy <= 1; ++dy) {
      // the three dz cells are consecutive keys
      const long long k0 = cell_key(cx + dx, cy + dy, cz - 1, hdr.lo, ny, nz);
      int64_t s = lower_bound(skeys, n, (unsigned long long)k0);
      for (; s < n && skeys[s] <= (unsigned long long)(k0 + 2); ++s) {
        const int b = sids[s];
        if (b <= a) continue;
        if (labels && labels[b] == la) continue;
        const double d0 = p[3 * (int64_t)b] - pa0, d1 = p[3 * (int64_t)b + 1] - pa1,
                     d2 = p[3 * (int64_t)b + 2] - pa2;
        const double dist = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
        if (!(dist < ra + rad[b])) continue;
        if (pass && pairs) {
          // insertion into the sorted segment [base, base+cnt)
          int64_t w = base + cnt;
          while (w > base && pairs[2 * (w - 1) + 1] > b) {
            pairs[2 * w] = pairs[2 * (w - 1)];
            pairs[2 * w + 1] = pairs[2 * (w - 1) + 1];
            --w;
          }
          pairs[2 * w] = (int32_t)a;
          pairs[2 * w + 1] = b;
        } else if (pass) {
          int64_t w = base + cnt;
          while (w > base && pj[w - 1] > b) {
            pj[w] = pj[w - 1];
            --w;
          }
          pj[w] = b;
          pi[base + cnt] = (int32_t)a;
        }
        ++cnt;
      }
    }
  if (!pass) count[a] = cnt;
}

// ---------------------------------------------------------------------------
// connected components (geometry.py:264-310)
// ---------------------------------------------------------------------------
__global__ void k_cc_init(int32_t *parent, int64_t n) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) parent[e] = (int32_t)e;
}

__global__ void k_cc_hook(const int32_t *bi, const int32_t *bj, const int8_t *status, int64_t nb,
                          int32_t *parent, int32_t *changed) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= nb || status[b] == 2) return;
  const int32_t pi = parent[bi[b]], pj = parent[bj[b]];
  if (pi == pj) return;
  const int32_t lo = pi < pj ? pi : pj, hi = pi < pj ? pj : pi;
  const int32_t old = atomicMin(&parent[hi], lo);
  if (old > lo) *changed = 1;
}

__global__ void k_cc_jump(int32_t *parent, int64_t n) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int32_t pe = parent[e];
  const int32_t pp = parent[pe];
  if (pp != pe) parent[e] = pp;
}

__global__ void k_cc_roots(const int32_t *parent, int64_t n, int32_t *is_root) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) is_root[e] = parent[e] == (int32_t)e ? 1 : 0;
}

__global__ void k_cc_label(const int32_t *parent, const int32_t *rank, int64_t n, int64_t *labels) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) labels[e] = rank[parent[e]];
}

// ---------------------------------------------------------------------------
// element adjacency of the frozen contact pairs (sorted i<j): pairs with
// i == e are [pi_ptr[e], pi_ptr[e+1]); pairs with j == e are
// pj_idx[pj_ptr[e] .. pj_ptr[e+1]) in ascending pair order
// ---------------------------------------------------------------------------
__global__ void k_pair_counts(const int32_t *pi, const int32_t *pj, int64_t m, int32_t *ci,
                              int32_t *cj, int32_t *iota) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  atomicAdd(&ci[pi[k]], 1);
  atomicAdd(&cj[pj[k]], 1);
  iota[k] = (int32_t)k;
}

__global__ void k_split_pairs(const int32_t *pairs, int64_t m, int32_t *pi, int32_t *pj) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  pi[k] = pairs[2 * k];
  pj[k] = pairs[2 * k + 1];
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace bdem

namespace bdem {
static std::atomic<long long> g_launches{0};
void count_launches(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
}  // namespace bdem

using namespace bdem;

extern "C" {

int64_t bdem_launch_count(void) { return (int64_t)g_launches.load(); }

// workspace layout for the broad phase
static size_t bp_cub_bytes(int64_t n) {
  size_t sort_b = 0, scan_b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_b, (unsigned long long *)nullptr,
                                  (unsigned long long *)nullptr, (int32_t *)nullptr,
                                  (int32_t *)nullptr, (int)n);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_b, (int32_t *)nullptr, (int64_t *)nullptr, (int)n + 1);
  return sort_b > scan_b ? sort_b : scan_b;
}

int64_t bdem_broadphase_workspace(int64_t n) {
  if (n < 1) n = 1;
  size_t b = 0;
  b += align256(sizeof(GridHdr));
  b += align256(sizeof(long long) * 3 * n);             // cxyz
  b += 2 * align256(sizeof(unsigned long long) * n);    // keys, sorted keys
  b += 2 * align256(sizeof(int32_t) * n);               // ids, sorted ids
  b += align256(sizeof(int32_t) * (n + 1));             // counts
  b += align256(sizeof(int64_t) * (n + 1));             // offsets
  b += align256(bp_cub_bytes(n));
  return (int64_t)b;
}

// the broad phase proper; the cell size is hdr->cell on the device (set by
// the caller: a host value copied in, or k_cell_from_rmax).  Writes
// interleaved pairs, or two planes (pi, pj) when pairs == NULL and pi != NULL;
// with no output buffer only counts.
static int broadphase_impl(const double *p, const double *radii, int64_t n,
                           const int64_t *labels, char *w, GridHdr *hdr, int32_t *pairs,
                           int32_t *pi, int32_t *pj, int64_t cap, int64_t *n_out,
                           cudaStream_t st, int64_t launched) {
  long long *cxyz = reinterpret_cast<long long *>(w); w += align256(sizeof(long long) * 3 * n);
  unsigned long long *keys = reinterpret_cast<unsigned long long *>(w); w += align256(sizeof(unsigned long long) * n);
  unsigned long long *skeys = reinterpret_cast<unsigned long long *>(w); w += align256(sizeof(unsigned long long) * n);
  int32_t *ids = reinterpret_cast<int32_t *>(w); w += align256(sizeof(int32_t) * n);
  int32_t *sids = reinterpret_cast<int32_t *>(w); w += align256(sizeof(int32_t) * n);
  int32_t *cnt = reinterpret_cast<int32_t *>(w); w += align256(sizeof(int32_t) * (n + 1));
  int64_t *offs = reinterpret_cast<int64_t *>(w); w += align256(sizeof(int64_t) * (n + 1));
  void *cub_tmp = w;
  size_t cub_bytes = bp_cub_bytes(n);

  k_cells<<<grid_for(n), kThreads, 0, st>>>(p, n, hdr, cxyz, hdr);
  GridHdr h;
  cudaMemcpyAsync(&h, hdr, sizeof(GridHdr), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return BDEM_ERR_CUDA;
  const long long nx = h.hi[0] - h.lo[0] + 3, ny = h.hi[1] - h.lo[1] + 3, nz = h.hi[2] - h.lo[2] + 3;
  const long double span = (long double)nx * ny * nz;
  if (span > 9.0e18L) return BDEM_ERR_ARG;  // key space overflow
  k_keys<<<grid_for(n), kThreads, 0, st>>>(cxyz, n, h, ny, nz, keys, ids);
  int end_bit = 1;
  while (end_bit < 64 && ((unsigned long long)(nx * ny * nz) >> end_bit) != 0ull) ++end_bit;
  cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, keys, skeys, ids, sids, (int)n, 0, end_bit, st);
  k_pairs<<<grid_for(n), kThreads, 0, st>>>(p, radii, n, cxyz, h, ny, nz, skeys, sids, labels, cnt,
                                            nullptr, nullptr, 0);
  cudaMemsetAsync(cnt + n, 0, sizeof(int32_t), st);
  cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, cnt, offs, (int)n + 1, st);
  int64_t total = 0;
  cudaMemcpyAsync(&total, offs + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return BDEM_ERR_CUDA;
  *n_out = total;
  if ((pairs == nullptr && pi == nullptr) || total == 0) return launch_status(launched + 5);
  if (total > cap) return BDEM_ERR_CAPACITY;
  k_pairs<<<grid_for(n), kThreads, 0, st>>>(p, radii, n, cxyz, h, ny, nz, skeys, sids, labels, cnt,
                                            offs, pairs, 1, pi, pj);
  return launch_status(launched + 6);
}

int bdem_broadphase(const double *p, const double *radii, int64_t n, double cell,
                    const int64_t *labels, void *work, int32_t *pairs, int64_t cap,
                    int64_t *n_out, void *stream) {
  if (n < 0 || !(cell > 0.0) || !n_out) return BDEM_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  if (n < 2) {
    *n_out = 0;
    return BDEM_OK;
  }
  char *w = static_cast<char *>(work);
  GridHdr *hdr = reinterpret_cast<GridHdr *>(w); w += align256(sizeof(GridHdr));
  GridHdr h0;
  for (int c = 0; c < 3; ++c) { h0.lo[c] = LLONG_MAX; h0.hi[c] = LLONG_MIN; }
  h0.rmax_bits = 0ull;
  h0.cell = cell;
  cudaMemcpyAsync(hdr, &h0, sizeof(GridHdr), cudaMemcpyHostToDevice, st);
  return broadphase_impl(p, radii, n, labels, w, hdr, pairs, nullptr, nullptr, cap, n_out, st, 0);
}

int64_t bdem_pair_adjacency_workspace(int64_t n, int64_t cap) {
  if (n < 1) n = 1;
  if (cap < 1) cap = 1;
  size_t scan_b = 0, sort_b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_b, (int32_t *)nullptr, (int32_t *)nullptr,
                                (int)n + 1);
  cub::DeviceRadixSort::SortPairs(nullptr, sort_b, (int32_t *)nullptr, (int32_t *)nullptr,
                                  (int32_t *)nullptr, (int32_t *)nullptr, (int)cap);
  return (int64_t)(2 * align256(sizeof(int32_t) * (n + 1)) + 2 * align256(sizeof(int32_t) * cap) +
                   align256(scan_b > sort_b ? scan_b : sort_b));
}

// element adjacency of sys->pair_i/pair_j (n_pair pairs, sorted i<j)
static int pair_adjacency(const bdem_system_t *sys, void *work, cudaStream_t st) {
  const int64_t n = sys->n_elem, m = sys->n_pair;
  if (m == 0) return BDEM_OK;
  char *w = static_cast<char *>(work);
  int32_t *ci = reinterpret_cast<int32_t *>(w); w += align256(sizeof(int32_t) * (n + 1));
  int32_t *cj = reinterpret_cast<int32_t *>(w); w += align256(sizeof(int32_t) * (n + 1));
  int32_t *iota = reinterpret_cast<int32_t *>(w); w += align256(sizeof(int32_t) * sys->pair_cap);
  int32_t *kout = reinterpret_cast<int32_t *>(w); w += align256(sizeof(int32_t) * sys->pair_cap);
  void *cub_tmp = w;
  size_t scan_b = 0, sort_b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_b, ci, (int32_t *)nullptr, (int)n + 1);
  cub::DeviceRadixSort::SortPairs(nullptr, sort_b, (int32_t *)nullptr, (int32_t *)nullptr,
                                  (int32_t *)nullptr, (int32_t *)nullptr, (int)sys->pair_cap);
  size_t tmp_b = scan_b > sort_b ? scan_b : sort_b;
  cudaMemsetAsync(ci, 0, sizeof(int32_t) * (n + 1), st);
  cudaMemsetAsync(cj, 0, sizeof(int32_t) * (n + 1), st);
  k_pair_counts<<<grid_for(m), kThreads, 0, st>>>(sys->pair_i, sys->pair_j, m, ci, cj, iota);
  cub::DeviceScan::ExclusiveSum(cub_tmp, tmp_b, ci, const_cast<int32_t *>(sys->pi_ptr), (int)n + 1, st);
  cub::DeviceScan::ExclusiveSum(cub_tmp, tmp_b, cj, const_cast<int32_t *>(sys->pj_ptr), (int)n + 1, st);
  // stable radix sort by j: pair indices ascending within each j
  int end_bit = 1;
  while (end_bit < 31 && (n >> end_bit) != 0) ++end_bit;
  cub::DeviceRadixSort::SortPairs(cub_tmp, tmp_b, sys->pair_j, kout, iota,
                                  const_cast<int32_t *>(sys->pj_idx), (int)m, 0, end_bit, st);
  return launch_status(4);
}

int bdem_set_pairs(bdem_system_t *sys, const int32_t *pairs, int64_t m, void *work,
                   void *stream) {
  if (!sys || m < 0 || m > sys->pair_cap) return BDEM_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  sys->n_pair = m;
  if (m == 0) return BDEM_OK;
  k_split_pairs<<<grid_for(m), kThreads, 0, st>>>(pairs, m, const_cast<int32_t *>(sys->pair_i),
                                                   const_cast<int32_t *>(sys->pair_j));
  const int rc = launch_status();
  return rc != BDEM_OK ? rc : pair_adjacency(sys, work, st);
}

int bdem_contact_pairs(bdem_system_t *sys, const double *p, const double *v, double dt,
                       double dt2g, const int64_t *labels, void *bp_work, void *adj_work,
                       double *radii, int64_t *n_out, void *stream) {
  if (!sys || !n_out) return BDEM_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  const int64_t n = sys->n_elem;
  sys->n_pair = 0;
  *n_out = 0;
  if (n < 2) return BDEM_OK;
  char *w = static_cast<char *>(bp_work);
  GridHdr *hdr = reinterpret_cast<GridHdr *>(w); w += align256(sizeof(GridHdr));
  GridHdr h0;
  for (int c = 0; c < 3; ++c) { h0.lo[c] = LLONG_MAX; h0.hi[c] = LLONG_MIN; }
  h0.rmax_bits = 0ull;
  h0.cell = 0.0;
  cudaMemcpyAsync(hdr, &h0, sizeof(GridHdr), cudaMemcpyHostToDevice, st);
  k_inflate<<<kRedBlocks, kThreads, 0, st>>>(v, sys->radius, n, dt, dt2g, radii, hdr);
  k_cell_from_rmax<<<1, 1, 0, st>>>(hdr);
  const int rc = broadphase_impl(p, radii, n, labels, w, hdr, nullptr,
                                 const_cast<int32_t *>(sys->pair_i),
                                 const_cast<int32_t *>(sys->pair_j), sys->pair_cap, n_out, st, 2);
  if (rc != BDEM_OK) return rc;
  sys->n_pair = *n_out;
  return pair_adjacency(sys, adj_work, st);
}

static size_t cc_cub_bytes(int64_t n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int32_t *)nullptr, (int32_t *)nullptr, (int)n);
  return b;
}

int64_t bdem_components_workspace(int64_t n) {
  if (n < 1) n = 1;
  return (int64_t)(3 * align256(sizeof(int32_t) * (n + 1)) + align256(sizeof(int32_t)) +
                   align256(cc_cub_bytes(n + 1)));
}

int bdem_components(int64_t n, int64_t n_bond, const int32_t *bi, const int32_t *bj,
                    const int8_t *status, void *work, int64_t *labels, int64_t *n_comp,
                    void *stream) {
  if (n < 0 || n_bond < 0) return BDEM_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    if (n_comp) *n_comp = 0;
    return BDEM_OK;
  }
  char *w = static_cast<char *>(work);
  int32_t *parent = reinterpret_cast<int32_t *>(w); w += align256(sizeof(int32_t) * (n + 1));
  int32_t *isroot = reinterpret_cast<int32_t *>(w); w += align256(sizeof(int32_t) * (n + 1));
  int32_t *rank = reinterpret_cast<int32_t *>(w); w += align256(sizeof(int32_t) * (n + 1));
  int32_t *changed = reinterpret_cast<int32_t *>(w); w += align256(sizeof(int32_t));
  void *cub_tmp = w;
  size_t cub_bytes = cc_cub_bytes(n + 1);
  int jumps = 1;
  while ((int64_t(1) << jumps) < n) ++jumps;
  ++jumps;
  k_cc_init<<<grid_for(n), kThreads, 0, st>>>(parent, n);
  for (int round = 0; round < 10000; ++round) {
    int32_t h_changed = 0;
    cudaMemsetAsync(changed, 0, sizeof(int32_t), st);
    if (n_bond > 0)
      k_cc_hook<<<grid_for(n_bond), kThreads, 0, st>>>(bi, bj, status, n_bond, parent, changed);
    for (int j = 0; j < jumps; ++j) k_cc_jump<<<grid_for(n), kThreads, 0, st>>>(parent, n);
    cudaMemcpyAsync(&h_changed, changed, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return BDEM_ERR_CUDA;
    if (!h_changed) break;
  }
  k_cc_roots<<<grid_for(n), kThreads, 0, st>>>(parent, n, isroot);
  cudaMemsetAsync(isroot + n, 0, sizeof(int32_t), st);
  cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, isroot, rank, (int)n + 1, st);
  k_cc_label<<<grid_for(n), kThreads, 0, st>>>(parent, rank, n, labels);
  count_launches(4);
  if (n_comp) {
    int32_t nc = 0;
    cudaMemcpyAsync(&nc, rank + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return BDEM_ERR_CUDA;
    *n_comp = nc;
  }
  return launch_status();
}

// ascending indices of nonzero flags (event compaction, bonds.py:564-569)
int64_t bdem_select_workspace(int64_t n) {
  size_t b = 0;
  cub::DeviceSelect::Flagged(nullptr, b, cub::CountingInputIterator<int32_t>(0),
                             (const uint8_t *)nullptr, (int32_t *)nullptr, (int64_t *)nullptr,
                             (int)(n < 1 ? 1 : n));
  return (int64_t)align256(b) + 256;
}

int bdem_select_flagged(const uint8_t *flags, int64_t n, int32_t *out_idx, void *work,
                        int64_t *n_out, void *stream) {
  if (n < 0 || !n_out) return BDEM_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    *n_out = 0;
    return BDEM_OK;
  }
  size_t b = 0;
  cub::DeviceSelect::Flagged(nullptr, b, cub::CountingInputIterator<int32_t>(0), flags, out_idx,
                             (int64_t *)nullptr, (int)n);
  char *w = static_cast<char *>(work);
  int64_t *d_num = reinterpret_cast<int64_t *>(w);
  void *tmp = w + 256;
  cub::DeviceSelect::Flagged(tmp, b, cub::CountingInputIterator<int32_t>(0), flags, out_idx, d_num,
                             (int)n, st);
  cudaMemcpyAsync(n_out, d_num, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return BDEM_ERR_CUDA;
  return launch_status();
}

int bdem_abi_version(void) { return BDEM_ABI_VERSION; }

int64_t bdem_system_size(void) { return (int64_t)sizeof(bdem_system_t); }

int bdem_device_sm(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major * 10 + minor;
}

}  // extern "C"
