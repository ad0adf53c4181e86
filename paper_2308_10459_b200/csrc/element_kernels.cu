// element_kernels.cu -- per-element kernels: ordered gradient gather,
// reduced gradient, diagonal blocks + block-Jacobi inverses, objective
// reductions, line-search trial point, predictor and velocity update.
//
// The gather reproduces np.add.at's sequential order (integrator.py:98-103):
// for element e, first the bonds with i == e (ascending), then the bonds
// with j == e (ascending), then contact pairs the same way, then colliders,
// then gravity and inertia.  No atomics: results are deterministic and,
// up to the per-bond arithmetic, bit-identical in summation order.
#include "bdem_common.cuh"
#include "bdem_math.cuh"
#include "colliders.cuh"

// the staged pieces and row sums (1) and the j-end coefficient pairs (2) are
// read once here: evict-first loads keep the bond pass's not-yet-read outputs
// in L2 longer (bond + element 498.7 -> 496.7 us, then 490.2 -> 485.6 us)
#ifndef BDEM_ELEM_CS
#define BDEM_ELEM_CS 2
#endif
#if BDEM_ELEM_CS
#define LDS1(a) __ldcs(a)
#else
#define LDS1(a) (*(a))
#endif


namespace bdem {

__device__ __forceinline__ void load_p(const double *p, int64_t e, double pe[3]) {
  pe[0] = p[3 * e + 0];
  pe[1] = p[3 * e + 1];
  pe[2] = p[3 * e + 2];
}
__device__ __forceinline__ void load_q(const double *q, int64_t e, double qe[4]) {
  const double2 *q2 = reinterpret_cast<const double2 *>(q) + 2 * e;
  const double2 a = q2[0], c = q2[1];
  qe[0] = a.x; qe[1] = a.y; qe[2] = c.x; qe[3] = c.y;
}
__device__ __forceinline__ void store_q(double *q, int64_t e, const double qe[4]) {
  double2 *q2 = reinterpret_cast<double2 *>(q) + 2 * e;
  q2[0] = make_double2(qe[0], qe[1]);
  q2[1] = make_double2(qe[2], qe[3]);
}

// staged stretch piece of bond position b: returns k c, fills n and the
// clamped block a+ = alpha n n^T + beta I (sym6)
__device__ __forceinline__ double stage_stretch(const double *st, const double *cf, int64_t nb,
                                                int64_t b, double n[3], double a[6]) {
  // pairs (n0 n1) (n2 alpha) (beta C00): three 16-byte loads
  const double2 *cb = reinterpret_cast<const double2 *>(cf + cf_idx(b, 0));
#if BDEM_ELEM_CS >= 2
  const double2 c01 = __ldcs(cb), c23 = __ldcs(cb + 32), c45 = __ldcs(cb + 64);
#else
  const double2 c01 = cb[0], c23 = cb[32], c45 = cb[64];
#endif
  n[0] = c01.x; n[1] = c01.y; n[2] = c23.x;
  stretch_apos(c23.y, c45.x, n, a);
  return LDS1(st + BDEM_ST_KC * nb + b);
}

// ---------------------------------------------------------------------------
// element assembly
// ---------------------------------------------------------------------------
#ifndef BDEM_ELEM_MINB
#define BDEM_ELEM_MINB 2
#endif
__global__ void __launch_bounds__(kThreads, BDEM_ELEM_MINB) k_element_assemble(bdem_system_t S, const double *p,
                                                               const double *q, double *z) {
  __shared__ double sh[kThreads / 32];
  double acc_f = 0.0, acc_g2 = 0.0, acc_c2 = 0.0, acc_dev = 0.0, acc_sing = 0.0;
  const int64_t nb = S.n_bond, pc = S.pair_cap;
  const int64_t nrow = ((S.n_elem + 31) >> 5) << 5;
  const double *st = S.stage;
  bool any_col_hess = false;
  for (int i = 0; i < S.n_colliders; ++i) any_col_hess |= S.colliders[i].kind != BDEM_COLLIDER_HALFSPACE;

  // one thread per SELL row (lane = row & 31 keeps the staged reads coalesced)
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < S.n_elem;
       row += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = S.row_elem[row];
    double pe[3], qe[4];
    load_p(p, e, pe);
    load_q(q, e, qe);
    double gp[3] = {0.0, 0.0, 0.0}, gq[4] = {0.0, 0.0, 0.0, 0.0};
    double P[6] = {0, 0, 0, 0, 0, 0}, R[6] = {0, 0, 0, 0, 0, 0};
    double ebond = 0.0;
    const int sl = (int)(row >> 5), lane = (int)(row & 31);
    // bonds with i == e: their pieces were summed in order by the bond pass
    // (ipart); slots from ikpre on staged their (i,i) rotation quadrant
    if (nb > 0) {
      const double *ip = S.ipart;
#pragma unroll
      for (int c = 0; c < 3; ++c) gp[c] = LDS1(ip + (BDEM_IP_GP + c) * nrow + row);
#pragma unroll
      for (int c = 0; c < 4; ++c) gq[c] = LDS1(ip + (BDEM_IP_GQ + c) * nrow + row);
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        P[t] = LDS1(ip + (BDEM_IP_P + t) * nrow + row);
        R[t] = LDS1(ip + (BDEM_IP_R + t) * nrow + row);
      }
      ebond = LDS1(ip + BDEM_IP_E * nrow + row);
      const int kpre = S.ikpre[row];
      if (kpre >= 0) {
        for (int64_t b = S.slice_base[sl] + lane + 32 * (int64_t)kpre; b < S.slice_base[sl + 1];
             b += 32) {
#pragma unroll
          for (int t = 0; t < 6; ++t) R[t] += st[(BDEM_ST_A + t) * nb + b];
        }
      }
    }
    // bonds with j == e (ascending bond id)
    // not unrolled: 1 / 2 / 3 / 4 iterations in flight ran 160.8 / 163.5 / 164.5 / 167.7 us
#pragma unroll 1
    for (int64_t k = S.jslice_base[sl] + lane; k < S.jslice_base[sl + 1]; k += 32) {
      const int64_t b = S.jpos[k];
      if (b < 0) continue;
      double n[3], apos[6];
      const double kc = stage_stretch(st, S.scoef, nb, b, n, apos);
#pragma unroll
      for (int c = 0; c < 3; ++c) gp[c] += kc * n[c];
#pragma unroll
      for (int c = 0; c < 4; ++c) gq[c] += LDS1(st + (BDEM_ST_GQJ + c) * nb + b);
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        P[t] += apos[t];
        R[t] += LDS1(st + (BDEM_ST_D + t) * nb + b);
      }
    }
    // contacts: pairs then colliders into a separate accumulator (integrator.py:56-85,104-105)
    double gc[3] = {0.0, 0.0, 0.0};
    double epair = 0.0, ecol = 0.0;
    if (S.n_pair > 0) {
      const double *ps = S.pstage;
      for (int k = S.pi_ptr[e]; k < S.pi_ptr[e + 1]; ++k) {
#pragma unroll
        for (int c = 0; c < 3; ++c) gc[c] += ps[(BDEM_PS_GI + c) * pc + k];
#pragma unroll
        for (int t = 0; t < 6; ++t) P[t] += ps[(BDEM_PS_A + t) * pc + k];
        epair += ps[BDEM_PS_E * pc + k];
      }
      for (int kk = S.pj_ptr[e]; kk < S.pj_ptr[e + 1]; ++kk) {
        const int64_t k = S.pj_idx[kk];
#pragma unroll
        for (int c = 0; c < 3; ++c) gc[c] += -ps[(BDEM_PS_GI + c) * pc + k];
#pragma unroll
        for (int t = 0; t < 6; ++t) P[t] += ps[(BDEM_PS_A + t) * pc + k];
      }
    }
    double Hc[6] = {0, 0, 0, 0, 0, 0};
    bool hc_nonzero = false;
    for (int ci = 0; ci < S.n_colliders; ++ci) {
      double g, dg[3], Hs[6];
      collider_eval(S.colliders[ci], pe, g, dg, Hs);
      if (g < 0.0) {
        const double k = S.k_contact;
        ecol += 0.5 * k * (g * g);
#pragma unroll
        for (int c = 0; c < 3; ++c) gc[c] += (k * g) * dg[c];
        const int pr[6] = {0, 0, 0, 1, 1, 2}, pcc[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
        for (int t = 0; t < 6; ++t) Hc[t] += k * (dg[pr[t]] * dg[pcc[t]] + g * Hs[t]);
        hc_nonzero = true;
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) gp[c] += gc[c];
    const double m = S.mass[e];
#pragma unroll
    for (int c = 0; c < 3; ++c) gp[c] -= m * S.gravity[c];
    const double pg = (pe[0] * S.gravity[0] + pe[1] * S.gravity[1]) + pe[2] * S.gravity[2];
    double fe = ((ebond + epair) + ecol) - m * pg;

    const int s = S.slot[e];
    if (s >= 0) {
      const double mp = S.mp_dt2[e], mq = S.mq_dt2[e];
      double dpv[3], dqv[4];
#pragma unroll
      for (int c = 0; c < 3; ++c) dpv[c] = pe[c] - S.p_hat[3 * e + c];
      double qh[4];
      load_q(S.q_hat, e, qh);
#pragma unroll
      for (int c = 0; c < 4; ++c) dqv[c] = qe[c] - qh[c];
#pragma unroll
      for (int c = 0; c < 3; ++c) gp[c] = gp[c] + mp * dpv[c];
#pragma unroll
      for (int c = 0; c < 4; ++c) gq[c] = gq[c] + mq * dqv[c];
      fe += 0.5 * (mp * ((dpv[0] * dpv[0] + dpv[1] * dpv[1]) + dpv[2] * dpv[2])) +
            0.5 * (mq * (((dqv[0] * dqv[0] + dqv[1] * dqv[1]) + dqv[2] * dqv[2]) + dqv[3] * dqv[3]));
      // reduced gradient (solver.py:116-123)
      double zr[3];
      gl_apply(qe, gq, zr);
      const int64_t nf6 = S.vstride;
      z[0 * nf6 + s] = gp[0]; z[1 * nf6 + s] = gp[1]; z[2 * nf6 + s] = gp[2];
      z[3 * nf6 + s] = zr[0]; z[4 * nf6 + s] = zr[1]; z[5 * nf6 + s] = zr[2];
      acc_g2 += (((gp[0] * gp[0] + gp[1] * gp[1]) + gp[2] * gp[2]) +
                 ((zr[0] * zr[0] + zr[1] * zr[1]) + zr[2] * zr[2]));
      const double qq = ((qe[0] * qe[0] + qe[1] * qe[1]) + qe[2] * qe[2]) + qe[3] * qe[3];
      const double cons = 0.5 * (qq - 1.0);
      acc_c2 += cons * cons;
      acc_dev = fmax(acc_dev, fabs(sqrt(qq) - 1.0));
      // element terms (solver.py:164-173) and diagonal blocks (solver.py:231-237)
      double Ep[6] = {mp, 0.0, 0.0, mp, 0.0, mp};
      if (hc_nonzero) {
#pragma unroll
        for (int t = 0; t < 6; ++t) Ep[t] = Hc[t] + Ep[t];
        if (any_col_hess) psd_clamp<3>(Ep);
      }
      const double curv = -(((qe[0] * gq[0] + qe[1] * gq[1]) + qe[2] * gq[2]) + qe[3] * gq[3]);
      const double erot = fmax(mq + curv, 0.0);
#pragma unroll
      for (int t = 0; t < 6; ++t) P[t] += Ep[t];
      R[0] += erot; R[3] += erot; R[5] += erot;
      const int64_t nf = S.vstride;
      double *dg = S.diag + s;
      double *mi = S.minv + s;
#pragma unroll
      for (int t = 0; t < 6; ++t) { dg[t * nf] = P[t]; dg[(6 + t) * nf] = R[t]; }
      // block-Jacobi (linalg.py:100-121): singular -> identity.  The
      // eigenvalue test lambda_min <= 1e-12 max|lambda| is decided by a cheap
      // certificate when it can be (pd_certify3: both blocks positive
      // definite with lambda_min >= det / |S|_F^2 far above the threshold),
      // else by the eigenvalues themselves; same decision either way
      bool singular;
      double fp_, lbp, fr_, lbr;
      const bool okp = pd_certify3(P, fp_, lbp), okr = pd_certify3(R, fr_, lbr);
      if (okp && okr && fmin(lbp, lbr) > 2e-12 * sqrt(fmax(fp_, fr_))) {
        singular = false;
      } else {
        double lp, ap_, lr, ar;
        eig3_minmax(P, lp, ap_);
        eig3_minmax(R, lr, ar);
        const double scale = fmax(fmax(ap_, ar), 1e-300);
        singular = fmin(lp, lr) <= 1e-12 * scale;
      }
      if (singular) {
        const double I6[6] = {1, 0, 0, 1, 0, 1};
#pragma unroll
        for (int t = 0; t < 6; ++t) { mi[t * nf] = I6[t]; mi[(6 + t) * nf] = I6[t]; }
        acc_sing += 1.0;
      } else {
        double Pi[6], Ri[6];
        inv3_sym(P, Pi);
        inv3_sym(R, Ri);
#pragma unroll
        for (int t = 0; t < 6; ++t) { mi[t * nf] = Pi[t]; mi[(6 + t) * nf] = Ri[t]; }
      }
    }
    if (S.grad_p != nullptr) {   // ImplicitProblem.value_and_gradient (integrator.py:195-200)
#pragma unroll
      for (int c = 0; c < 3; ++c) S.grad_p[3 * e + c] = gp[c];
      store_q(S.grad_q, e, gq);
    }
    acc_f += fe;
  }
  double v;
  v = block_sum<kThreads>(acc_f, sh);
  if (threadIdx.x == 0) *red_slot(S.red, BDEM_SC_F, blockIdx.x) = v;
  v = block_sum<kThreads>(acc_g2, sh);
  if (threadIdx.x == 0) *red_slot(S.red, BDEM_SC_GNORM2, blockIdx.x) = v;
  v = block_sum<kThreads>(acc_c2, sh);
  if (threadIdx.x == 0) *red_slot(S.red, BDEM_SC_CNORM2, blockIdx.x) = v;
  v = block_max<kThreads>(acc_dev, sh);
  if (threadIdx.x == 0) *red_slot(S.red, BDEM_SC_MAXDEV, blockIdx.x) = v;
  v = block_sum<kThreads>(acc_sing, sh);
  if (threadIdx.x == 0) *red_slot(S.red, BDEM_SC_NSING, blockIdx.x) = v;
}

// fixed-order finish of per-block partials -> scalars
// one block per column (grid = ncol): each column is reduced exactly as
// before (same per-thread strided partial sums, same block_sum order)
__global__ void __launch_bounds__(kThreads) k_reduce_finish(bdem_system_t S, int col0, int ncol,
                                                            int nblocks) {
  __shared__ double sh[kThreads / 32];
  for (int c = col0 + blockIdx.x; c < col0 + ncol; c += gridDim.x) {
    double v;
    if (c == BDEM_SC_MAXDEV) {
      double m = 0.0;
      for (int b = threadIdx.x; b < nblocks; b += kThreads) m = fmax(m, *red_slot(S.red, c, b));
      v = block_max<kThreads>(m, sh);
    } else {
      v = sum_partials<kThreads>(S.red, c, nblocks, sh);
    }
    if (threadIdx.x == 0) S.scalars[c] = v;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// element part of the objective at an (optionally moved) point
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_element_energy(bdem_system_t S, const double *p,
                                                             const double *q, const double *dp,
                                                             const double *dq, double alpha,
                                                             double *pt, double *qt,
                                                             int with_inertia) {
  __shared__ double sh[kThreads / 32];
  double acc_in = 0.0, acc_col = 0.0, acc_g = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < S.n_elem;
       e += (int64_t)gridDim.x * blockDim.x) {
    double pe[3], qe[4];
    load_p(p, e, pe);
    load_q(q, e, qe);
    const bool fr = S.slot[e] >= 0;
    if (dp != nullptr) {
      // p_t = p + alpha dp ; q_t = normalize(geodesic(q, alpha dq)) on free rows
      double dpe[3];
      load_p(dp, e, dpe);
#pragma unroll
      for (int c = 0; c < 3; ++c) pe[c] = pe[c] + alpha * dpe[c];
      if (fr) {
        double dqe[4], ad[4], out[4];
        load_q(dq, e, dqe);
#pragma unroll
        for (int c = 0; c < 4; ++c) ad[c] = alpha * dqe[c];
        retract_normalize(qe, ad, out);
#pragma unroll
        for (int c = 0; c < 4; ++c) qe[c] = out[c];
      }
      pt[3 * e + 0] = pe[0]; pt[3 * e + 1] = pe[1]; pt[3 * e + 2] = pe[2];
      store_q(qt, e, qe);
    }
    for (int ci = 0; ci < S.n_colliders; ++ci) {
      double g, dg[3], Hs[6];
      collider_eval(S.colliders[ci], pe, g, dg, Hs);
      if (g < 0.0) acc_col += 0.5 * S.k_contact * (g * g);
    }
    acc_g += -(S.mass[e] * ((pe[0] * S.gravity[0] + pe[1] * S.gravity[1]) + pe[2] * S.gravity[2]));
    if (with_inertia && fr) {
      double dpv[3], dqv[4], qh[4];
      load_q(S.q_hat, e, qh);
#pragma unroll
      for (int c = 0; c < 3; ++c) dpv[c] = pe[c] - S.p_hat[3 * e + c];
#pragma unroll
      for (int c = 0; c < 4; ++c) dqv[c] = qe[c] - qh[c];
      acc_in += 0.5 * (S.mp_dt2[e] * ((dpv[0] * dpv[0] + dpv[1] * dpv[1]) + dpv[2] * dpv[2])) +
                0.5 * (S.mq_dt2[e] *
                       (((dqv[0] * dqv[0] + dqv[1] * dqv[1]) + dqv[2] * dqv[2]) + dqv[3] * dqv[3]));
    }
  }
  double v;
  v = block_sum<kThreads>(acc_in, sh);
  if (threadIdx.x == 0) *red_slot(S.red, BDEM_SC_FT, blockIdx.x) = v;
  v = block_sum<kThreads>(acc_col, sh);
  if (threadIdx.x == 0) *red_slot(S.red, BDEM_SC_ECOL, blockIdx.x) = v;
  v = block_sum<kThreads>(acc_g, sh);
  if (threadIdx.x == 0) *red_slot(S.red, BDEM_SC_EGRAV, blockIdx.x) = v;
}

// kinetic energy (elements.py:114-117) -> partial column EKIN
__global__ void __launch_bounds__(kThreads) k_kinetic(bdem_system_t S, const double *v,
                                                      const double *qd) {
  __shared__ double sh[kThreads / 32];
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < S.n_elem;
       e += (int64_t)gridDim.x * blockDim.x) {
    double ve[3], we[4];
    load_p(v, e, ve);
    load_q(qd, e, we);
    const double m = S.mass[e], r = S.radius[e];
    acc += 0.5 * (m * ((ve[0] * ve[0] + ve[1] * ve[1]) + ve[2] * ve[2])) +
           0.5 * (((1.6 * m) * (r * r)) * (((we[0] * we[0] + we[1] * we[1]) + we[2] * we[2]) + we[3] * we[3]));
  }
  const double s = block_sum<kThreads>(acc, sh);
  if (threadIdx.x == 0) *red_slot(S.red, BDEM_SC_EKIN, blockIdx.x) = s;
}

// ---------------------------------------------------------------------------
// direction, predictor, velocity update, normalisation
// ---------------------------------------------------------------------------
__global__ void k_direction(bdem_system_t S, const double *q, const double *y, double sign,
                            double *dp, double *dq) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= S.n_free) return;
  const int64_t e = S.free_elem[s];
  const int64_t nf = S.vstride;
  double qe[4], yr[3], w[4];
  load_q(q, e, qe);
#pragma unroll
  for (int c = 0; c < 3; ++c) dp[3 * e + c] = sign * y[c * nf + s];
#pragma unroll
  for (int c = 0; c < 3; ++c) yr[c] = sign * y[(3 + c) * nf + s];
  glt_apply(qe, yr, w);
  store_q(dq, e, w);
}

__global__ void k_predict(bdem_system_t S, const double *p, const double *q, const double *v,
                          const double *qd, const double *pp, const double *qp, double dt,
                          double *ph, double *qh, double *mp, double *mq, double *p0,
                          double *q0) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= S.n_elem) return;
  double pe[3], qe[4], ppe[3], qpe[4];
  load_p(p, e, pe);
  load_q(q, e, qe);
  load_p(pp, e, ppe);
  load_q(qp, e, qpe);
  double hq[4];
#pragma unroll
  for (int c = 0; c < 3; ++c) ph[3 * e + c] = 2.0 * pe[c] - ppe[c];
#pragma unroll
  for (int c = 0; c < 4; ++c) hq[c] = 2.0 * qe[c] - qpe[c];
  store_q(qh, e, hq);
  const bool fr = S.slot[e] >= 0;
  const double dt2 = dt * dt;
  const double m = S.mass[e], r = S.radius[e];
  mp[e] = fr ? m / dt2 : 0.0;
  mq[e] = fr ? ((1.6 * m) * (r * r)) / dt2 : 0.0;
  double out[4];
  if (fr) {
    double ve[3], we[4], st[4];
    load_p(v, e, ve);
    load_q(qd, e, we);
#pragma unroll
    for (int c = 0; c < 3; ++c) p0[3 * e + c] = pe[c] + dt * ve[c];
#pragma unroll
    for (int c = 0; c < 4; ++c) st[c] = dt * we[c];
#ifdef BDEM_MUTATE_RETRACT  // mutation check of the parity tests only (never shipped)
#pragma unroll
    for (int c = 0; c < 4; ++c) st[c] *= 1.0 + BDEM_MUTATE_RETRACT;
#endif
    retract_normalize(qe, st, out);  // geodesic then quat_normalize(q0)
  } else {
#pragma unroll
    for (int c = 0; c < 3; ++c) p0[3 * e + c] = pe[c];
    normalize4(qe, out);
  }
  store_q(q0, e, out);
}

__global__ void k_normalize_free(bdem_system_t S, double *q) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= S.n_free) return;
  const int64_t e = S.free_elem[s];
  double qe[4], out[4];
  load_q(q, e, qe);
  normalize4(qe, out);
  store_q(q, e, out);
}

__global__ void k_finish_step(bdem_system_t S, const double *p, const double *q,
                              const double *pc, const double *qc, double dt, double *v,
                              double *qd) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= S.n_free) return;
  const int64_t e = S.free_elem[s];
  double pe[3], qe[4], pce[3], qce[4], w[4], out[4];
  load_p(p, e, pe);
  load_q(q, e, qe);
  load_p(pc, e, pce);
  load_q(qc, e, qce);
#pragma unroll
  for (int c = 0; c < 3; ++c) v[3 * e + c] = div_nz(pe[c] - pce[c], dt);
#pragma unroll
  for (int c = 0; c < 4; ++c) w[c] = div_nz(qe[c] - qce[c], dt);
  const double qw = ((qe[0] * w[0] + qe[1] * w[1]) + qe[2] * w[2]) + qe[3] * w[3];
#pragma unroll
  for (int c = 0; c < 4; ++c) out[c] = w[c] - qw * qe[c];
  store_q(qd, e, out);
}

// dot product with last-block finish into scalars[col]
__global__ void __launch_bounds__(kThreads) k_dot(bdem_system_t S, const double *a,
                                                  const double *b, int64_t n, int col) {
  __shared__ double sh[kThreads / 32];
  double acc = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    acc += a[k] * b[k];
  const double s = block_sum<kThreads>(acc, sh);
  if (threadIdx.x == 0) *red_slot(S.red, col, blockIdx.x) = s;
  if (last_block(S.counter + 1)) {
    const double tot = sum_partials<kThreads>(S.red, col, gridDim.x, sh);
    if (threadIdx.x == 0) S.scalars[col] = tot;
  }
}

// element rows <-> a packed buffer of 14 doubles per listed element (p 3,
// q 4, v 3, qdot 4): the pinned-state backup / restore of stable_step
// (solver.py:894-896, 910-916) and the driver rows at t + dt (:898-900)
__global__ void k_rows_copy(const int32_t *ids, int64_t m, double *p, double *q, double *v,
                            double *qdot, double *buf, int to_buf) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int64_t e = ids[k];
  double *r = buf + 14 * k;
  if (to_buf) {
#pragma unroll
    for (int c = 0; c < 3; ++c) { r[c] = p[3 * e + c]; r[7 + c] = v[3 * e + c]; }
#pragma unroll
    for (int c = 0; c < 4; ++c) { r[3 + c] = q[4 * e + c]; r[10 + c] = qdot[4 * e + c]; }
  } else {
#pragma unroll
    for (int c = 0; c < 3; ++c) { p[3 * e + c] = r[c]; v[3 * e + c] = r[7 + c]; }
#pragma unroll
    for (int c = 0; c < 4; ++c) { q[4 * e + c] = r[3 + c]; qdot[4 * e + c] = r[10 + c]; }
  }
}

__global__ void k_reset_errors(int32_t *err) {
  const int t = threadIdx.x;
  if (t < BDEM_ERRSLOT_COUNT)
    err[t] = (t == BDEM_ERRSLOT_DEGENERATE_FIRST || t == BDEM_ERRSLOT_ANTIPODAL_FIRST)
                 ? 0x7fffffff : 0;
}

// ambient contact Hessian blocks (PotentialModel.hessian_blocks): pairs
// [[a,-a],[-a,a]] (contact.py:209-223) and summed collider blocks
// (contact.py:243-247, integrator.py:76-83), row-major
__global__ void __launch_bounds__(kThreads) k_contact_blocks(bdem_system_t S, const double *p,
                                                             double *pair_pp, double *elem_pp) {
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (pair_pp != nullptr) {
    for (int64_t k = t0; k < S.n_pair; k += stride) {
      const int64_t i = S.pair_i[k], j = S.pair_j[k];
      double d[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) d[c] = p[3 * j + c] - p[3 * i + c];
      const double len = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
      const double depth = fmax(0.0, (S.radius[i] + S.radius[j]) - len);
      double n[3];
      if (len < 1e-12) {
        n[0] = 1.0; n[1] = 0.0; n[2] = 0.0;
      } else {
        const double l = fmax(len, 1e-300);
#pragma unroll
        for (int c = 0; c < 3; ++c) n[c] = div_nz(d[c], l);
      }
      const bool touch = depth > 0.0;
      const double f = depth / fmax(len, 1e-300);
      double *H = pair_pp + 36 * k;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double nn = n[r] * n[c];
          const double a = touch ? S.k_element * (nn - f * ((r == c ? 1.0 : 0.0) - nn)) : 0.0;
          H[6 * r + c] = a;
          H[6 * (r + 3) + c + 3] = a;
          H[6 * r + c + 3] = -a;
          H[6 * (r + 3) + c] = -a;
        }
    }
  }
  if (elem_pp != nullptr) {
    for (int64_t e = t0; e < S.n_elem; e += stride) {
      double pe[3];
      load_p(p, e, pe);
      double Hc[6] = {0, 0, 0, 0, 0, 0};
      for (int ci = 0; ci < S.n_colliders; ++ci) {
        double g, dg[3], Hs[6];
        collider_eval(S.colliders[ci], pe, g, dg, Hs);
        const int pr[6] = {0, 0, 0, 1, 1, 2}, pcc[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
        for (int t = 0; t < 6; ++t)
          Hc[t] += g < 0.0 ? S.k_contact * (dg[pr[t]] * dg[pcc[t]] + g * Hs[t]) : 0.0;
      }
      double *H = elem_pp + 9 * e;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) H[3 * r + c] = Hc[sidx<3>(r, c)];
    }
  }
}

}  // namespace bdem

using namespace bdem;

extern "C" {

int bdem_element_assemble(const bdem_system_t *sys, const double *p, const double *q,
                          double *z, void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  k_element_assemble<<<kRedBlocks, kThreads, 0, as_stream(stream)>>>(*sys, p, q, z);
  return launch_status();
}

int bdem_reduce_finish(const bdem_system_t *sys, int col0, int ncol, int nblocks,
                       void *stream) {
  if (!sys || col0 < 0 || col0 + ncol > BDEM_SC_COUNT || nblocks > kRedBlocks) return BDEM_ERR_ARG;
  k_reduce_finish<<<ncol > 0 ? ncol : 1, kThreads, 0, as_stream(stream)>>>(*sys, col0, ncol,
                                                                           nblocks);
  return launch_status();
}

int bdem_trial_point(const bdem_system_t *sys, const double *p, const double *q,
                     const double *dp, const double *dq, double alpha, double *p_t,
                     double *q_t, void *stream) {
  if (!sys || !dp || !dq || !p_t || !q_t) return BDEM_ERR_ARG;
  k_element_energy<<<kRedBlocks, kThreads, 0, as_stream(stream)>>>(*sys, p, q, dp, dq, alpha,
                                                                    p_t, q_t, 1);
  return launch_status();
}

int bdem_contact_blocks(const bdem_system_t *sys, const double *p, double *pair_pp,
                        double *elem_pp, void *stream) {
  if (!sys || !p) return BDEM_ERR_ARG;
  const int64_t m = sys->n_pair > sys->n_elem ? sys->n_pair : sys->n_elem;
  if (m == 0 || (!pair_pp && !elem_pp)) return BDEM_OK;
  k_contact_blocks<<<grid_for(m), kThreads, 0, as_stream(stream)>>>(*sys, p, pair_pp, elem_pp);
  return launch_status();
}

int bdem_element_energy(const bdem_system_t *sys, const double *p, const double *q,
                        int with_inertia, void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  k_element_energy<<<kRedBlocks, kThreads, 0, as_stream(stream)>>>(
      *sys, p, q, nullptr, nullptr, 0.0, nullptr, nullptr, with_inertia);
  return launch_status();
}

int bdem_kinetic(const bdem_system_t *sys, const double *v, const double *qdot, void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  k_kinetic<<<kRedBlocks, kThreads, 0, as_stream(stream)>>>(*sys, v, qdot);
  return launch_status();
}

int bdem_direction(const bdem_system_t *sys, const double *q, const double *y, double sign,
                   double *dp, double *dq, void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  if (sys->n_free == 0) return BDEM_OK;
  k_direction<<<grid_for(sys->n_free), kThreads, 0, as_stream(stream)>>>(*sys, q, y, sign, dp, dq);
  return launch_status();
}

int bdem_dot(const bdem_system_t *sys, const double *a, const double *b, int64_t n, int sc_col,
             void *stream) {
  if (!sys || sc_col < 0 || sc_col >= BDEM_SC_COUNT) return BDEM_ERR_ARG;
  k_dot<<<kRedBlocks, kThreads, 0, as_stream(stream)>>>(*sys, a, b, n, sc_col);
  return launch_status();
}

int bdem_predict(const bdem_system_t *sys, const double *p, const double *q, const double *v,
                 const double *qdot, const double *p_prev, const double *q_prev, double dt,
                 double *p_hat, double *q_hat, double *mp_dt2, double *mq_dt2, double *p0,
                 double *q0, void *stream) {
  if (!sys || dt <= 0.0) return BDEM_ERR_ARG;
  k_predict<<<grid_for(sys->n_elem), kThreads, 0, as_stream(stream)>>>(
      *sys, p, q, v, qdot, p_prev, q_prev, dt, p_hat, q_hat, mp_dt2, mq_dt2, p0, q0);
  return launch_status();
}

int bdem_normalize_free(const bdem_system_t *sys, double *q, void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  if (sys->n_free == 0) return BDEM_OK;
  k_normalize_free<<<grid_for(sys->n_free), kThreads, 0, as_stream(stream)>>>(*sys, q);
  return launch_status();
}

int bdem_finish_step(const bdem_system_t *sys, const double *p, const double *q,
                     const double *p_c, const double *q_c, double dt, double *v, double *qdot,
                     void *stream) {
  if (!sys || dt <= 0.0) return BDEM_ERR_ARG;
  if (sys->n_free == 0) return BDEM_OK;
  k_finish_step<<<grid_for(sys->n_free), kThreads, 0, as_stream(stream)>>>(*sys, p, q, p_c, q_c,
                                                                           dt, v, qdot);
  return launch_status();
}

int bdem_rows_copy(const int32_t *ids, int64_t m, double *p, double *q, double *v,
                   double *qdot, double *buf, int to_buf, void *stream) {
  if (m < 0) return BDEM_ERR_ARG;
  if (m == 0) return BDEM_OK;
  k_rows_copy<<<grid_for(m), kThreads, 0, as_stream(stream)>>>(ids, m, p, q, v, qdot, buf, to_buf);
  return launch_status();
}

int bdem_reset_errors(const bdem_system_t *sys, void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  k_reset_errors<<<1, 32, 0, as_stream(stream)>>>(sys->err);
  return launch_status();
}

}  // extern "C"
