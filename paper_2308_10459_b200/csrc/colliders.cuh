// colliders.cuh -- signed distance, gradient and Hessian of the analytic
// colliders (contact.py:38-125): half-space, sphere, axis-aligned box.
#pragma once
#include "bdem_common.cuh"

namespace bdem {

__device__ inline void collider_eval(const bdem_collider_t &C, const double p[3], double &g,
                              double dg[3], double H[6]) {
#pragma unroll
  for (int t = 0; t < 6; ++t) H[t] = 0.0;
  if (C.kind == BDEM_COLLIDER_HALFSPACE) {
    g = ((p[0] * C.a[0] + p[1] * C.a[1]) + p[2] * C.a[2]) - C.a[3];
    dg[0] = C.a[0]; dg[1] = C.a[1]; dg[2] = C.a[2];
  } else if (C.kind == BDEM_COLLIDER_SPHERE) {
    const double d[3] = {p[0] - C.a[0], p[1] - C.a[1], p[2] - C.a[2]};
    const double r = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    const double rs = fmax(r, 1e-12);
    g = r - C.a[3];
    double n[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) { n[c] = div_nz(d[c], rs); dg[c] = n[c]; }
    const int pr[6] = {0, 0, 0, 1, 1, 2}, pc[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int t = 0; t < 6; ++t) H[t] = div_nz((pr[t] == pc[t] ? 1.0 : 0.0) - n[pr[t]] * n[pc[t]], rs);
  } else {  // box
    double loc[3], d[3], pos[3], sign[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      loc[c] = p[c] - C.a[c];
      d[c] = fabs(loc[c]) - C.a[3 + c];
      pos[c] = fmax(d[c], 0.0);
      sign[c] = loc[c] >= 0.0 ? 1.0 : -1.0;
    }
    const double on = sqrt((pos[0] * pos[0] + pos[1] * pos[1]) + pos[2] * pos[2]);
    const double inside = fmin(fmax(fmax(d[0], d[1]), d[2]), 0.0);
    g = on + inside;
    if (on > 0.0) {
      const double ons = fmax(on, 1e-300);
      double n[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) { n[c] = div_nz(sign[c] * pos[c], ons); dg[c] = n[c]; }
      const int pr[6] = {0, 0, 0, 1, 1, 2}, pc[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        const double act = (pr[t] == pc[t] && pos[pr[t]] > 0.0) ? 1.0 : 0.0;
        H[t] = div_nz(act - n[pr[t]] * n[pc[t]], ons);
      }
    } else {
      // first axis of largest d (selects, not d[ax]: a run-time index would
      // put d in local memory)
      int ax = 0;
      double dmax = d[0];
      if (d[1] > dmax) { ax = 1; dmax = d[1]; }
      if (d[2] > dmax) ax = 2;
#pragma unroll
      for (int c = 0; c < 3; ++c) dg[c] = (c == ax ? 1.0 : 0.0) * sign[c];
    }
  }
}

}  // namespace bdem
