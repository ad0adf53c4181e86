// surface_kernels.cu -- per-frame surface reconstruction (reconstruct_surface,
// geometry.py:313-343) on the device.
//
// Every element owns the boundary faces of its tet plus, for each broken bond,
// the bond's face on its side.  The reference emits, per fragment in label
// order, per member element in ascending id, the element's faces in ascending
// local index, each face's three rest vertices (relative to the tet centroid)
// transported by the element pose: v = p + rotate(q, rest).  Here: face bit
// masks (boundary | broken, atomicOr), a stable radix sort of elements by
// fragment label, a scan of the per-element face counts, and one thread per
// element writing its faces at the scanned offset -- the same order.
#include <cub/cub.cuh>

#include "bdem_common.cuh"

namespace bdem {

__constant__ int kFaceVerts[4][3] = {{0, 2, 1}, {0, 1, 3}, {1, 2, 3}, {0, 3, 2}};

__global__ void k_surf_mask(bdem_system_t S, const int32_t *bmask, const int64_t *labels,
                            int32_t *mask, int32_t *key, int32_t *val) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= S.n_elem) return;
  mask[e] = bmask[e];
  key[e] = (int32_t)labels[e];
  val[e] = (int32_t)e;
}

// broken bonds add their face on each side (update_surface_on_break's faces)
__global__ void k_surf_broken(bdem_system_t S, const int8_t *face_i, const int8_t *face_j,
                              int32_t *mask) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= S.n_bond) return;
  if (S.status[b] != 2 || face_i[b] < 0) return;  // intact, or padding / no mesh face
  atomicOr(mask + S.bond_i[b], 1 << face_i[b]);
  atomicOr(mask + S.bond_j[b], 1 << face_j[b]);
}

__global__ void k_surf_count(int64_t n, const int32_t *mask, const int32_t *order,
                             int32_t *count) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  count[k] = __popc(mask[order[k]]);
}

// rotate_vec (quat.py:106-114): (s^2 - t.t) d + 2 (t.d) t + 2 s (t x d), every
// product and sum rounded on its own in numpy's order (no FMA contraction), so
// the surface vertices -- and the OBJ text -- are bit-identical to the reference
#define M_(a, b) __dmul_rn(a, b)
#define A_(a, b) __dadd_rn(a, b)
#define S_(a, b) __dsub_rn(a, b)
__device__ __forceinline__ void rotate(const double q[4], const double d[3], double out[3]) {
  const double s = q[3];
  const double td = A_(A_(M_(q[0], d[0]), M_(q[1], d[1])), M_(q[2], d[2]));
  const double tt = A_(A_(M_(q[0], q[0]), M_(q[1], q[1])), M_(q[2], q[2]));
  const double c[3] = {S_(M_(q[1], d[2]), M_(q[2], d[1])), S_(M_(q[2], d[0]), M_(q[0], d[2])),
                       S_(M_(q[0], d[1]), M_(q[1], d[0]))};
  const double a = S_(M_(s, s), tt), td2 = M_(2.0, td), s2 = M_(2.0, s);
#pragma unroll
  for (int k = 0; k < 3; ++k) out[k] = A_(A_(M_(a, d[k]), M_(td2, q[k])), M_(s2, c[k]));
}

__global__ void k_surf_write(int64_t n, const double *p, const double *q, const double *tet_rel,
                             const int32_t *mask, const int32_t *order, const int32_t *comp,
                             const int32_t *offset, int64_t cap, double *verts,
                             int32_t *face_comp) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t e = order[k];
  const int m = mask[e];
  if (!m) return;
  double pe[3], qe[4];
#pragma unroll
  for (int c = 0; c < 3; ++c) pe[c] = p[3 * e + c];
#pragma unroll
  for (int c = 0; c < 4; ++c) qe[c] = q[4 * e + c];
  int64_t f = offset[k];
  for (int local = 0; local < 4; ++local) {
    if (!(m & (1 << local))) continue;
    if (f < cap) {
      for (int v = 0; v < 3; ++v) {
        const double *rest = tet_rel + 12 * e + 3 * kFaceVerts[local][v];
        double r[3];
        rotate(qe, rest, r);
#pragma unroll
        for (int c = 0; c < 3; ++c) verts[9 * f + 3 * v + c] = A_(pe[c], r[c]);
      }
      face_comp[f] = comp[k];
    }
    ++f;
  }
}

}  // namespace bdem

using namespace bdem;

namespace {
inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
size_t cub_bytes(int64_t n) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (const int32_t *)nullptr, (int32_t *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, (int)n);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const int32_t *)nullptr, (int32_t *)nullptr,
                                (int)n + 1);
  return a > b ? a : b;
}
}  // namespace

extern "C" {

int64_t bdem_surface_workspace(int64_t n_elem) {
  const int64_t n = n_elem > 0 ? n_elem : 1;
  return (int64_t)(6 * align256(4 * (size_t)(n + 1)) + align256(cub_bytes(n)));
}

int bdem_surface(const bdem_system_t *sys, const double *p, const double *q,
                 const double *tet_rel, const int32_t *bmask, const int8_t *face_i,
                 const int8_t *face_j, const int64_t *labels, void *work, double *verts,
                 int32_t *face_comp, int64_t cap_faces, int64_t *n_faces, void *stream) {
  if (!sys || !p || !q || !tet_rel || !bmask || !labels || !work || !n_faces) return BDEM_ERR_ARG;
  const bdem_system_t S = *sys;
  const int64_t n = S.n_elem;
  *n_faces = 0;
  if (n == 0) return BDEM_OK;
  cudaStream_t st = as_stream(stream);
  char *w = static_cast<char *>(work);
  const size_t seg = align256(4 * (size_t)(n + 1));
  int32_t *mask = reinterpret_cast<int32_t *>(w);
  int32_t *key = reinterpret_cast<int32_t *>(w + seg);
  int32_t *val = reinterpret_cast<int32_t *>(w + 2 * seg);
  int32_t *key_s = reinterpret_cast<int32_t *>(w + 3 * seg);
  int32_t *val_s = reinterpret_cast<int32_t *>(w + 4 * seg);
  int32_t *cnt = reinterpret_cast<int32_t *>(w + 5 * seg);
  int32_t *off = key;  // unsorted keys are dead after the sort: face offsets
  void *tmp = w + 6 * seg;
  size_t tmp_bytes = cub_bytes(n);
  const int T = 256;
  const unsigned gn = (unsigned)((n + T - 1) / T);
  k_surf_mask<<<gn, T, 0, st>>>(S, bmask, labels, mask, key, val);
  if (S.n_bond > 0 && face_i && face_j)
    k_surf_broken<<<(unsigned)((S.n_bond + T - 1) / T), T, 0, st>>>(S, face_i, face_j, mask);
  int bits = 1;
  while (bits < 31 && (int64_t(1) << bits) < n) ++bits;
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, key_s, val, val_s, (int)n, 0, bits, st);
  k_surf_count<<<gn, T, 0, st>>>(n, mask, val_s, cnt);
  cudaMemsetAsync(cnt + n, 0, sizeof(int32_t), st);
  tmp_bytes = cub_bytes(n);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, off, (int)n + 1, st);
  int32_t total = 0;
  cudaMemcpyAsync(&total, off + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return BDEM_ERR_CUDA;
  *n_faces = total;
  if (total > cap_faces || !verts || !face_comp) return launch_status(4);  // caller re-sizes
  k_surf_write<<<gn, T, 0, st>>>(n, p, q, tet_rel, mask, val_s, key_s, off, cap_faces, verts,
                                 face_comp);
  return launch_status(5);
}

}  // extern "C"
