// friction_kernels.cu -- post-step Coulomb-type friction (contact.py:267-350,
// called by stable_step when mu_s > 0 or mu_r > 0, solver.py:923-925).
//
// The reference sweeps the contact pairs in ascending order, each pair
// correcting both sides with velocities already corrected by earlier pairs;
// then the collider contacts per collider in ascending element order.  Here
// the pairs are grouped into dependency waves by the host (wave of a pair =
// 1 + the latest wave of an earlier pair sharing an element), so pairs of one
// wave touch disjoint elements and every element sees its corrections in the
// reference order.  The collider part is independent per element.
#include <vector>

#include "bdem_common.cuh"
#include "bdem_math.cuh"
#include "colliders.cuh"

namespace bdem {

__device__ __forceinline__ void ld3(const double *a, int64_t e, double v[3]) {
  v[0] = a[3 * e]; v[1] = a[3 * e + 1]; v[2] = a[3 * e + 2];
}
__device__ __forceinline__ void st3(double *a, int64_t e, const double v[3]) {
  a[3 * e] = v[0]; a[3 * e + 1] = v[1]; a[3 * e + 2] = v[2];
}
__device__ __forceinline__ double norm3(const double v[3]) {
  return sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
}

// _friction_delta (contact.py:267-282)
__device__ __forceinline__ void friction_delta(const double rel[3], const double own[3], double fn,
                                               double coeff, double scale, double dt,
                                               double out[3]) {
  out[0] = out[1] = out[2] = 0.0;
  const double own_n = norm3(own), rel_n = norm3(rel);
  if (own_n == 0.0 || rel_n == 0.0 || fn == 0.0) return;
  const double factor = fmin(1.0, coeff * fn * dt / (scale * rel_n));
  double delta[3], dir[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    delta[c] = -factor * rel[c];
    dir[c] = own[c] / own_n;
  }
  double along = (delta[0] * dir[0] + delta[1] * dir[1]) + delta[2] * dir[2];
  along = fmin(0.0, fmax(along, -own_n));
#pragma unroll
  for (int c = 0; c < 3; ++c) out[c] = along * dir[c];
}

// friction_post_step + the in-place update of correct() (contact.py:285-330)
__device__ __forceinline__ void friction_correct(const bdem_system_t &S, int64_t k,
                                                 const double vrel[3], const double wrel[3],
                                                 const double nrm[3], double fn, double mu_s,
                                                 double mu_r, double dt, double *v, double *w,
                                                 uint8_t *touched) {
  if (S.slot[k] < 0) return;
  double vi[3], wi[3], dv[3], dw[3];
  ld3(v, k, vi);
  ld3(w, k, wi);
  const double vn = (vrel[0] * nrm[0] + vrel[1] * nrm[1]) + vrel[2] * nrm[2];
  double vt[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) vt[c] = vrel[c] - vn * nrm[c];
  const double m = S.mass[k], r = S.radius[k];
  const double inertia = 0.4 * m * (r * r);
  friction_delta(vt, vi, fn, mu_s, m, dt, dv);
  friction_delta(wrel, wi, fn, mu_r, inertia / (r * r * r), dt, dw);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    vi[c] += dv[c];
    wi[c] += dw[c];
  }
  st3(v, k, vi);
  st3(w, k, wi);
  touched[k] = 1;
}

// w = Im(2 tangent(qdot) * conj(q))  (angular_velocity, quat.py:116-134)
__global__ void k_friction_init(bdem_system_t S, const double *q, const double *qd, double *w,
                                uint8_t *touched) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= S.n_elem) return;
  double qe[4], de[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) { qe[c] = q[4 * e + c]; de[c] = qd[4 * e + c]; }
  const double rad = ((qe[0] * de[0] + qe[1] * de[1]) + qe[2] * de[2]) + qe[3] * de[3];
  double t[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) t[c] = de[c] - rad * qe[c];
  // t * conj(q): vec = ts*(-qv) + qs*tv + tv x (-qv), scalar dropped
  const double tv0 = t[0], tv1 = t[1], tv2 = t[2], ts = t[3];
  const double qv0 = -qe[0], qv1 = -qe[1], qv2 = -qe[2], qs = qe[3];
  const double c0 = tv1 * qv2 - tv2 * qv1, c1 = tv2 * qv0 - tv0 * qv2, c2 = tv0 * qv1 - tv1 * qv0;
  w[3 * e] = 2.0 * ((ts * qv0 + qs * tv0) + c0);
  w[3 * e + 1] = 2.0 * ((ts * qv1 + qs * tv1) + c1);
  w[3 * e + 2] = 2.0 * ((ts * qv2 + qs * tv2) + c2);
  touched[e] = 0;
}

// pair is in contact after the step: |p_a - p_b| < r_a + r_b (contact.py:334-336)
__global__ void k_friction_flags(bdem_system_t S, const double *p, uint8_t *flags) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= S.n_pair) return;
  const int64_t a = S.pair_i[k], b = S.pair_j[k];
  double pa[3], pb[3], d[3];
  ld3(p, a, pa);
  ld3(p, b, pb);
#pragma unroll
  for (int c = 0; c < 3; ++c) d[c] = pa[c] - pb[c];
  flags[k] = norm3(d) < S.radius[a] + S.radius[b] ? 1 : 0;
}

__global__ void k_friction_gather(bdem_system_t S, const int32_t *idx, int64_t m, int32_t *ends) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= m) return;
  const int32_t k = idx[t];
  ends[2 * t] = S.pair_i[k];
  ends[2 * t + 1] = S.pair_j[k];
}

__device__ __forceinline__ void friction_pair(const bdem_system_t &S, const double *p, int64_t k,
                                              double mu_s, double mu_r, double dt, double *v,
                                              double *w, uint8_t *touched) {
  const int64_t a = S.pair_i[k], b = S.pair_j[k];
  double pa[3], pb[3], d[3];
  ld3(p, a, pa);
  ld3(p, b, pb);
#pragma unroll
  for (int c = 0; c < 3; ++c) d[c] = pa[c] - pb[c];
  const double dist = norm3(d);
  if (dist >= S.radius[a] + S.radius[b]) return;
  double nrm[3];
  if (dist > 1e-12) {
#pragma unroll
    for (int c = 0; c < 3; ++c) nrm[c] = d[c] / dist;
  } else {
    nrm[0] = 1.0; nrm[1] = 0.0; nrm[2] = 0.0;
  }
  const double fn = S.k_element * dist;
  double va[3], vb[3], wa[3], wb[3], vr[3], wr[3], mn[3];
  ld3(v, a, va); ld3(v, b, vb); ld3(w, a, wa); ld3(w, b, wb);
#pragma unroll
  for (int c = 0; c < 3; ++c) { vr[c] = va[c] - vb[c]; wr[c] = wa[c] - wb[c]; }
  friction_correct(S, a, vr, wr, nrm, fn, mu_s, mu_r, dt, v, w, touched);
  ld3(v, a, va); ld3(w, a, wa);
#pragma unroll
  for (int c = 0; c < 3; ++c) { vr[c] = vb[c] - va[c]; wr[c] = wb[c] - wa[c]; mn[c] = -nrm[c]; }
  friction_correct(S, b, vr, wr, mn, fn, mu_s, mu_r, dt, v, w, touched);
}

__global__ void k_friction_wave(bdem_system_t S, const double *p, const int32_t *order,
                                int32_t t0, int32_t t1, double mu_s, double mu_r, double dt,
                                double *v, double *w, uint8_t *touched) {
  const int64_t t = t0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= t1) return;
  friction_pair(S, p, order[t], mu_s, mu_r, dt, v, w, touched);
}

// A run of consecutive small waves in ONE CTA: a __syncthreads between waves
// orders each wave's velocity writes before the next wave reads them.
__global__ void __launch_bounds__(1024) k_friction_waves(bdem_system_t S, const double *p,
                                                         const int32_t *order,
                                                         const int32_t *wave_ptr, int32_t wb,
                                                         int32_t we, double mu_s, double mu_r,
                                                         double dt, double *v, double *w,
                                                         uint8_t *touched) {
  for (int32_t l = wb; l < we; ++l) {
    const int32_t t1 = wave_ptr[l + 1];
    for (int32_t t = wave_ptr[l] + threadIdx.x; t < t1; t += blockDim.x)
      friction_pair(S, p, order[t], mu_s, mu_r, dt, v, w, touched);
    __syncthreads();
  }
}

// Collider contacts per element in collider order (contact.py:342-347), then
// qdot = quat_rate(q, w) = 0.5 (w,0) * q for touched elements (contact.py:348-350).
__global__ void k_friction_colliders(bdem_system_t S, const double *p, const double *q,
                                     double mu_s, double mu_r, double dt, double *v,
                                     const double *w_in, uint8_t *touched, double *qd) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= S.n_elem) return;
  double *w = const_cast<double *>(w_in);
  double pe[3];
  ld3(p, e, pe);
  for (int ci = 0; ci < S.n_colliders; ++ci) {
    double g, dg[3], H[6];
    collider_eval(S.colliders[ci], pe, g, dg, H);
    if (!(g < 0.0)) continue;
    const double fn = S.k_contact * fabs(g) * norm3(dg);
    double vi[3], wi[3];
    ld3(v, e, vi);
    ld3(w, e, wi);
    friction_correct(S, e, vi, wi, dg, fn, mu_s, mu_r, dt, v, w, touched);
  }
  if (!touched[e]) return;
  double wv[3], qe[4];
  ld3(w, e, wv);
#pragma unroll
  for (int c = 0; c < 4; ++c) qe[c] = q[4 * e + c];
  // (w,0) * q: vec = 0*qv + qs*w + w x qv ; scalar = -w.qv
  const double cx = wv[1] * qe[2] - wv[2] * qe[1];
  const double cy = wv[2] * qe[0] - wv[0] * qe[2];
  const double cz = wv[0] * qe[1] - wv[1] * qe[0];
  qd[4 * e] = 0.5 * (qe[3] * wv[0] + cx);
  qd[4 * e + 1] = 0.5 * (qe[3] * wv[1] + cy);
  qd[4 * e + 2] = 0.5 * (qe[3] * wv[2] + cz);
  qd[4 * e + 3] = 0.5 * (-((wv[0] * qe[0] + wv[1] * qe[1]) + wv[2] * qe[2]));
}

}  // namespace bdem

using namespace bdem;

namespace {
constexpr int kWaveBig = 8192;  // waves at least this large get a full-grid launch
inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
struct FrictionWork {
  double *w;
  uint8_t *touched, *flags;
  int32_t *idx, *ends, *order, *wave_ptr;
  void *sel;
};
FrictionWork carve(void *work, int64_t n, int64_t m) {
  char *c = static_cast<char *>(work);
  FrictionWork f;
  f.w = reinterpret_cast<double *>(c); c += align256(sizeof(double) * 3 * n);
  f.touched = reinterpret_cast<uint8_t *>(c); c += align256(n);
  f.flags = reinterpret_cast<uint8_t *>(c); c += align256(m);
  f.idx = reinterpret_cast<int32_t *>(c); c += align256(4 * m);
  f.ends = reinterpret_cast<int32_t *>(c); c += align256(8 * m);
  f.order = reinterpret_cast<int32_t *>(c); c += align256(4 * m);
  f.wave_ptr = reinterpret_cast<int32_t *>(c); c += align256(4 * (m + 1));
  f.sel = c;
  return f;
}
}  // namespace

extern "C" {

int64_t bdem_friction_workspace(int64_t n_elem, int64_t n_pair) {
  const int64_t n = n_elem, m = n_pair;
  return (int64_t)(align256(sizeof(double) * 3 * n) + align256(n) + align256(m) +
                   align256(4 * m) + align256(8 * m) + align256(4 * m) + align256(4 * (m + 1))) +
         bdem_select_workspace(m);
}

int64_t bdem_friction_schedule(const int32_t *ends, int64_t m, int64_t n_elem, int32_t *order,
                               int32_t *wave_ptr) {
  if (m < 0 || n_elem < 0 || (m > 0 && (!ends || !order || !wave_ptr))) return -BDEM_ERR_ARG;
  if (m == 0) {
    if (wave_ptr) wave_ptr[0] = 0;
    return 0;
  }
  static thread_local std::vector<int32_t> last;
  if ((int64_t)last.size() < n_elem) last.assign(n_elem, 0);
  std::vector<int32_t> level(m);
  int32_t depth = 0;
  for (int64_t k = 0; k < m; ++k) {
    const int32_t a = ends[2 * k], b = ends[2 * k + 1];
    if (a < 0 || b < 0 || a >= n_elem || b >= n_elem) {
      for (int64_t t = 0; t < k; ++t) last[ends[2 * t]] = last[ends[2 * t + 1]] = 0;
      return -BDEM_ERR_ARG;
    }
    const int32_t l = 1 + (last[a] > last[b] ? last[a] : last[b]);
    last[a] = last[b] = l;
    level[k] = l - 1;
    depth = l > depth ? l : depth;
  }
  for (int64_t k = 0; k < m; ++k) last[ends[2 * k]] = last[ends[2 * k + 1]] = 0;
  // counting sort by wave, stable in pair order
  for (int32_t l = 0; l <= depth; ++l) wave_ptr[l] = 0;
  for (int64_t k = 0; k < m; ++k) ++wave_ptr[level[k] + 1];
  for (int32_t l = 0; l < depth; ++l) wave_ptr[l + 1] += wave_ptr[l];
  std::vector<int32_t> fill(wave_ptr, wave_ptr + depth);
  for (int64_t k = 0; k < m; ++k) order[fill[level[k]]++] = (int32_t)k;
  return depth;
}

int bdem_friction(const bdem_system_t *sys, const double *p, const double *q, double *v,
                  double *qdot, double mu_s, double mu_r, double dt, void *work,
                  int64_t *n_waves, void *stream) {
  if (!sys || !p || !q || !v || !qdot || !work) return BDEM_ERR_ARG;
  if (n_waves) *n_waves = 0;
  if (mu_s == 0.0 && mu_r == 0.0) return BDEM_OK;
  const bdem_system_t S = *sys;
  cudaStream_t st = as_stream(stream);
  const int64_t n = S.n_elem, m = S.n_pair;
  if (n == 0) return BDEM_OK;
  FrictionWork f = carve(work, n, m);
  const int T = 256;
  k_friction_init<<<(unsigned)((n + T - 1) / T), T, 0, st>>>(S, q, qdot, f.w, f.touched);
  count_launches(1);
  if (m > 0) {
    k_friction_flags<<<(unsigned)((m + T - 1) / T), T, 0, st>>>(S, p, f.flags);
    count_launches(1);
    int64_t active = 0;
    int rc = bdem_select_flagged(f.flags, m, f.idx, f.sel, &active, stream);
    if (rc != BDEM_OK) return rc;
    if (active > 0) {
      k_friction_gather<<<(unsigned)((active + T - 1) / T), T, 0, st>>>(S, f.idx, active, f.ends);
      count_launches(1);
      std::vector<int32_t> ends(2 * active), order(active), wave(active + 1), pord(active);
      cudaMemcpyAsync(ends.data(), f.ends, sizeof(int32_t) * 2 * active, cudaMemcpyDeviceToHost,
                      st);
      std::vector<int32_t> idx(active);
      cudaMemcpyAsync(idx.data(), f.idx, sizeof(int32_t) * active, cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) return BDEM_ERR_CUDA;
      const int64_t depth = bdem_friction_schedule(ends.data(), active, n, order.data(),
                                                   wave.data());
      if (depth < 0) return (int)-depth;
      for (int64_t t = 0; t < active; ++t) pord[t] = idx[order[t]];  // original pair ids
      cudaMemcpyAsync(f.order, pord.data(), sizeof(int32_t) * active, cudaMemcpyHostToDevice, st);
      cudaMemcpyAsync(f.wave_ptr, wave.data(), sizeof(int32_t) * (depth + 1),
                      cudaMemcpyHostToDevice, st);
      int64_t l = 0;
      while (l < depth) {
        const int32_t sz = wave[l + 1] - wave[l];
        if (sz >= kWaveBig) {
          k_friction_wave<<<(unsigned)((sz + T - 1) / T), T, 0, st>>>(
              S, p, f.order, wave[l], wave[l + 1], mu_s, mu_r, dt, v, f.w, f.touched);
          count_launches(1);
          ++l;
          continue;
        }
        int64_t e = l;
        while (e < depth && wave[e + 1] - wave[e] < kWaveBig) ++e;
        k_friction_waves<<<1, 1024, 0, st>>>(S, p, f.order, f.wave_ptr, (int32_t)l, (int32_t)e,
                                             mu_s, mu_r, dt, v, f.w, f.touched);
        count_launches(1);
        l = e;
      }
      // host vectors must outlive the async H2D copies
      if (cudaStreamSynchronize(st) != cudaSuccess) return BDEM_ERR_CUDA;
      if (n_waves) *n_waves = depth;
    }
  }
  k_friction_colliders<<<(unsigned)((n + T - 1) / T), T, 0, st>>>(S, p, q, mu_s, mu_r, dt, v, f.w,
                                                                   f.touched, qdot);
  return launch_status(1);
}

}  // extern "C"
