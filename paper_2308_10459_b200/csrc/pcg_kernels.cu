// pcg_kernels.cu -- reduced-system SpMV, block-Jacobi and the PCG state
// machine (linalg.py:40-97) with all control scalars kept on the device.
//
// Matrix storage: the reduced Newton matrix (assemble_reduced_system,
// solver.py:198-258) is never formed as CSR.  Its pieces stay where the
// assembly kernels wrote them:
//   * per bond:  a+ (sym 3x3, position coupling is -a+) and C (3x3 rotation
//                coupling, used as C for row i and C^T for row j),
//   * per pair:  a+ (position coupling -a+),
//   * per free element: the 6x6 diagonal as two sym 3x3 blocks P, R.
// Each stored coefficient is read once per row that uses it (twice per bond,
// the second read mostly from L2), i.e. half the bytes of a BSR copy.
//
// PCG control flow: every kernel reads sys->pcg[STATE] first and returns if
// the solve has stopped, so the host can enqueue several iterations ahead
// and synchronise only once per chunk.
#include "bdem_common.cuh"
#include "bdem_math.cuh"

namespace bdem {

enum { PCG_RUNNING = 0, PCG_CONVERGED = 1, PCG_BREAKDOWN = 2, PCG_MAXIT = 3 };
enum { CNT_SPMV = 2, CNT_UPDATE = 3, CNT_INIT = 4 };
// partial-sum columns of sys->red owned by PCG (disjoint from BDEM_SC_*)
enum { RC_PAP = 20, RC_AP2 = 21, RC_PP2 = 22, RC_RR = 23, RC_RZ = 24, RC_IRR = 25, RC_IRZ = 26 };

__device__ __forceinline__ void load6(const double *x, int64_t s, double v[6]) {
  const double2 *x2 = reinterpret_cast<const double2 *>(x + 6 * s);
  const double2 a = x2[0], b = x2[1], c = x2[2];
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; v[4] = c.x; v[5] = c.y;
}
__device__ __forceinline__ void store6(double *x, int64_t s, const double v[6]) {
  double2 *x2 = reinterpret_cast<double2 *>(x + 6 * s);
  x2[0] = make_double2(v[0], v[1]);
  x2[1] = make_double2(v[2], v[3]);
  x2[2] = make_double2(v[4], v[5]);
}

// y_s = (A x)_s for one free slot s
__device__ __forceinline__ void spmv_row(const bdem_system_t &S, const double *x, int64_t s,
                                         const double xs[6], double y[6]) {
  const int64_t nb = S.n_bond;
  const double *st = S.stage;
  const double *dg = S.diag + 12 * s;
  symv3(dg, xs, y);
  symv3(dg + 6, xs + 3, y + 3);
  const int64_t e = S.free_elem[s];
  const int a0 = S.adj_ptr[e], am = S.adj_mid[e], a1 = S.adj_ptr[e + 1];
  for (int k = a0; k < a1; ++k) {
    const int o = S.adj_oslot[k];
    if (o < 0) continue;
    const int64_t b = S.adj_bond[k];
    double xo[6];
    load6(x, o, xo);
    double a[6];
#pragma unroll
    for (int t = 0; t < 6; ++t) a[t] = st[(BDEM_ST_APOS + t) * nb + b];
    double ap[3];
    symv3(a, xo, ap);
    y[0] -= ap[0]; y[1] -= ap[1]; y[2] -= ap[2];
    double C[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) C[t] = st[(BDEM_ST_C + t) * nb + b];
    if (k < am) {  // row i: C x_j
#pragma unroll
      for (int r = 0; r < 3; ++r)
        y[3 + r] += (C[3 * r] * xo[3] + C[3 * r + 1] * xo[4]) + C[3 * r + 2] * xo[5];
    } else {       // row j: C^T x_i
#pragma unroll
      for (int r = 0; r < 3; ++r)
        y[3 + r] += (C[r] * xo[3] + C[3 + r] * xo[4]) + C[6 + r] * xo[5];
    }
  }
  if (S.n_pair > 0) {
    const int64_t pc = S.pair_cap;
    const double *ps = S.pstage;
    for (int k = S.pi_ptr[e]; k < S.pi_ptr[e + 1]; ++k) {
      const int o = S.slot[S.pair_j[k]];
      if (o < 0) continue;
      double xo[6], a[6], ap[3];
      load6(x, o, xo);
#pragma unroll
      for (int t = 0; t < 6; ++t) a[t] = ps[(BDEM_PS_A + t) * pc + k];
      symv3(a, xo, ap);
      y[0] -= ap[0]; y[1] -= ap[1]; y[2] -= ap[2];
    }
    for (int kk = S.pj_ptr[e]; kk < S.pj_ptr[e + 1]; ++kk) {
      const int64_t k = S.pj_idx[kk];
      const int o = S.slot[S.pair_i[k]];
      if (o < 0) continue;
      double xo[6], a[6], ap[3];
      load6(x, o, xo);
#pragma unroll
      for (int t = 0; t < 6; ++t) a[t] = ps[(BDEM_PS_A + t) * pc + k];
      symv3(a, xo, ap);
      y[0] -= ap[0]; y[1] -= ap[1]; y[2] -= ap[2];
    }
  }
}

__device__ __forceinline__ void precond_row(const bdem_system_t &S, int64_t s, const double r[6],
                                            double z[6]) {
  const double *mi = S.minv + 12 * s;
  symv3(mi, r, z);
  symv3(mi + 6, r + 3, z + 3);
}

// mode 0: plain y = A x; mode 1: PCG step (y = A p + boost p, p.Ap, |Ap|^2, |p|^2)
__global__ void __launch_bounds__(kThreads) k_spmv(bdem_system_t S, const double *x, double *y,
                                                   int mode) {
  __shared__ double sh[kThreads / 32];
  double *pcg = S.pcg;
  if (mode == 1 && pcg[BDEM_PCG_STATE] != PCG_RUNNING) return;
  const double boost = mode == 1 ? pcg[BDEM_PCG_BOOST] : 0.0;
  double acc_xy = 0.0, acc_yy = 0.0, acc_xx = 0.0;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S.n_free;
       s += (int64_t)gridDim.x * blockDim.x) {
    double xs[6], ys[6];
    load6(x, s, xs);
    spmv_row(S, x, s, xs, ys);
    if (boost != 0.0) {
#pragma unroll
      for (int c = 0; c < 6; ++c) ys[c] = ys[c] + boost * xs[c];
    }
    store6(y, s, ys);
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      acc_xy += xs[c] * ys[c];
      acc_yy += ys[c] * ys[c];
      acc_xx += xs[c] * xs[c];
    }
  }
  if (mode == 0) return;
  double v = block_sum<kThreads>(acc_xy, sh);
  if (threadIdx.x == 0) *red_slot(S.red, RC_PAP, blockIdx.x) = v;
  v = block_sum<kThreads>(acc_yy, sh);
  if (threadIdx.x == 0) *red_slot(S.red, RC_AP2, blockIdx.x) = v;
  v = block_sum<kThreads>(acc_xx, sh);
  if (threadIdx.x == 0) *red_slot(S.red, RC_PP2, blockIdx.x) = v;
  if (!last_block(S.counter + CNT_SPMV)) return;
  const double pap = sum_partials<kThreads>(S.red, RC_PAP, gridDim.x, sh);
  const double ap2 = sum_partials<kThreads>(S.red, RC_AP2, gridDim.x, sh);
  const double pp2 = sum_partials<kThreads>(S.red, RC_PP2, gridDim.x, sh);
  if (threadIdx.x == 0) {
    pcg[BDEM_PCG_PAP] = pap;
    pcg[BDEM_PCG_APNORM2] = ap2;
    pcg[BDEM_PCG_PNORM2] = pp2;
    if (pap <= 0.0) {  // breakdown: boost for the restart (linalg.py:74-77)
      const double sc = sqrt(ap2) / fmax(sqrt(pp2), 1e-300);
      pcg[BDEM_PCG_BOOST] = fmax(boost * 100.0, 1e-10 * fmax(sc, 1.0));
      pcg[BDEM_PCG_STATE] = PCG_BREAKDOWN;
    } else {
      pcg[BDEM_PCG_ALPHA] = pcg[BDEM_PCG_RZ] / pap;
    }
  }
}

// x += alpha p; r -= alpha Ap; z = M^-1 r; r.r, r.z (linalg.py:79-89)
__global__ void __launch_bounds__(kThreads) k_pcg_update(bdem_system_t S, double *x, double *r,
                                                         double *zv, const double *p,
                                                         const double *ap) {
  __shared__ double sh[kThreads / 32];
  double *pcg = S.pcg;
  if (pcg[BDEM_PCG_STATE] != PCG_RUNNING) return;
  const double alpha = pcg[BDEM_PCG_ALPHA];
  double acc_rr = 0.0, acc_rz = 0.0;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S.n_free;
       s += (int64_t)gridDim.x * blockDim.x) {
    double xs[6], rs[6], ps[6], aps[6], zs[6];
    load6(x, s, xs);
    load6(r, s, rs);
    load6(p, s, ps);
    load6(ap, s, aps);
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      xs[c] = xs[c] + alpha * ps[c];
      rs[c] = rs[c] - alpha * aps[c];
      acc_rr += rs[c] * rs[c];
    }
    store6(x, s, xs);
    store6(r, s, rs);
    precond_row(S, s, rs, zs);
    store6(zv, s, zs);
#pragma unroll
    for (int c = 0; c < 6; ++c) acc_rz += rs[c] * zs[c];
  }
  double v = block_sum<kThreads>(acc_rr, sh);
  if (threadIdx.x == 0) *red_slot(S.red, RC_RR, blockIdx.x) = v;
  v = block_sum<kThreads>(acc_rz, sh);
  if (threadIdx.x == 0) *red_slot(S.red, RC_RZ, blockIdx.x) = v;
  if (!last_block(S.counter + CNT_UPDATE)) return;
  const double rr = sum_partials<kThreads>(S.red, RC_RR, gridDim.x, sh);
  const double rz_new = sum_partials<kThreads>(S.red, RC_RZ, gridDim.x, sh);
  if (threadIdx.x == 0) {
    const double k = pcg[BDEM_PCG_K] + 1.0;
    pcg[BDEM_PCG_K] = k;
    pcg[BDEM_PCG_RR] = rr;
    const double rel = sqrt(rr) / pcg[BDEM_PCG_BNORM];
    pcg[BDEM_PCG_REL] = rel;
    if (rel <= pcg[BDEM_PCG_TOL]) {
      pcg[BDEM_PCG_STATE] = PCG_CONVERGED;
    } else {
      pcg[BDEM_PCG_BETA] = rz_new / pcg[BDEM_PCG_RZ];
      pcg[BDEM_PCG_RZ] = rz_new;
      if (k >= pcg[BDEM_PCG_MAXIT]) pcg[BDEM_PCG_STATE] = PCG_MAXIT;
    }
  }
}

// p = z + beta p (linalg.py:91)
__global__ void __launch_bounds__(kThreads) k_pcg_pupdate(bdem_system_t S, double *p,
                                                          const double *zv) {
  const double *pcg = S.pcg;
  if (pcg[BDEM_PCG_STATE] != PCG_RUNNING) return;
  const double beta = pcg[BDEM_PCG_BETA];
  const int64_t n6 = 6 * S.n_free;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n6;
       k += (int64_t)gridDim.x * blockDim.x)
    p[k] = zv[k] + beta * p[k];
}

// x = 0, r = sign b, z = M^-1 r, p = z, r.z, |b| (linalg.py:52-68)
__global__ void __launch_bounds__(kThreads) k_pcg_init(bdem_system_t S, const double *b,
                                                       double sign, double *x, double *r,
                                                       double *zv, double *p, double tol,
                                                       double maxit, double boost) {
  __shared__ double sh[kThreads / 32];
  double acc_rr = 0.0, acc_rz = 0.0;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S.n_free;
       s += (int64_t)gridDim.x * blockDim.x) {
    double bs[6], zs[6];
    const double zero[6] = {0, 0, 0, 0, 0, 0};
    load6(b, s, bs);
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      bs[c] = sign * bs[c];
      acc_rr += bs[c] * bs[c];
    }
    store6(x, s, zero);
    store6(r, s, bs);
    precond_row(S, s, bs, zs);
    store6(zv, s, zs);
    store6(p, s, zs);
#pragma unroll
    for (int c = 0; c < 6; ++c) acc_rz += bs[c] * zs[c];
  }
  double v = block_sum<kThreads>(acc_rr, sh);
  if (threadIdx.x == 0) *red_slot(S.red, RC_IRR, blockIdx.x) = v;
  v = block_sum<kThreads>(acc_rz, sh);
  if (threadIdx.x == 0) *red_slot(S.red, RC_IRZ, blockIdx.x) = v;
  if (!last_block(S.counter + CNT_INIT)) return;
  const double rr = sum_partials<kThreads>(S.red, RC_IRR, gridDim.x, sh);
  const double rz = sum_partials<kThreads>(S.red, RC_IRZ, gridDim.x, sh);
  if (threadIdx.x == 0) {
    double *pcg = S.pcg;
    pcg[BDEM_PCG_RZ] = rz;
    pcg[BDEM_PCG_BNORM] = sqrt(rr);
    pcg[BDEM_PCG_RR] = rr;
    pcg[BDEM_PCG_REL] = 1.0;
    pcg[BDEM_PCG_TOL] = tol;
    pcg[BDEM_PCG_MAXIT] = maxit;
    pcg[BDEM_PCG_BOOST] = boost;
    pcg[BDEM_PCG_K] = 0.0;
    pcg[BDEM_PCG_STATE] = (rr == 0.0 || maxit <= 0.0) ? (rr == 0.0 ? PCG_CONVERGED : PCG_MAXIT)
                                                      : PCG_RUNNING;
  }
}

__global__ void k_precond(bdem_system_t S, const double *r, double *zv) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= S.n_free) return;
  double rs[6], zs[6];
  load6(r, s, rs);
  precond_row(S, s, rs, zs);
  store6(zv, s, zs);
}

// self_repulsion_terms + clamp of the pair block (contact.py:180-224, solver.py:162)
__global__ void __launch_bounds__(kThreads) k_pair(bdem_system_t S, const double *p,
                                                   int energy_only) {
  __shared__ double sh[kThreads / 32];
  const int64_t pc = S.pair_cap;
  double acc = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < S.n_pair;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = S.pair_i[k], j = S.pair_j[k];
    double d[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) d[c] = p[3 * j + c] - p[3 * i + c];
    const double len = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    const double depth = fmax(0.0, (S.radius[i] + S.radius[j]) - len);
    const double ke = S.k_element;
    const double E = 0.5 * ke * (depth * depth);
    acc += E;
    if (energy_only) continue;
    double n[3];
    if (len < 1e-12) {
      n[0] = 1.0; n[1] = 0.0; n[2] = 0.0;
    } else {
      const double l = fmax(len, 1e-300);
#pragma unroll
      for (int c = 0; c < 3; ++c) n[c] = d[c] / l;
    }
    const bool touch = depth > 0.0;
    double *ps = S.pstage;
    ps[BDEM_PS_E * pc + k] = E;
#pragma unroll
    for (int c = 0; c < 3; ++c) ps[(BDEM_PS_GI + c) * pc + k] = touch ? (ke * depth) * n[c] : 0.0;
    const int pr[6] = {0, 0, 0, 1, 1, 2}, pcc[6] = {0, 1, 2, 1, 2, 2};
    // a = k (nn - (depth/l)(I - nn)): eigenvalues k (along n) and -k depth/l,
    // so the clamp of [[a,-a],[-a,a]] keeps k nn.
#pragma unroll
    for (int t = 0; t < 6; ++t) ps[(BDEM_PS_A + t) * pc + k] = touch ? ke * (n[pr[t]] * n[pcc[t]]) : 0.0;
  }
  if (!energy_only) return;
  const double s = block_sum<kThreads>(acc, sh);
  if (threadIdx.x == 0) *red_slot(S.red, BDEM_SC_EPAIR, blockIdx.x) = s;
}

}  // namespace bdem

using namespace bdem;

extern "C" {

int bdem_spmv(const bdem_system_t *sys, const double *x, double *y, void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  k_spmv<<<kRedBlocks, kThreads, 0, as_stream(stream)>>>(*sys, x, y, 0);
  return launch_status();
}

int bdem_precond_apply(const bdem_system_t *sys, const double *r, double *zv, void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  if (sys->n_free == 0) return BDEM_OK;
  k_precond<<<grid_for(sys->n_free), kThreads, 0, as_stream(stream)>>>(*sys, r, zv);
  return launch_status();
}

int bdem_pcg_init(const bdem_system_t *sys, const double *b, double sign, double *x, double *r,
                  double *zv, double *pv, double tol, int max_iter, double boost,
                  void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  k_pcg_init<<<kRedBlocks, kThreads, 0, as_stream(stream)>>>(*sys, b, sign, x, r, zv, pv, tol,
                                                              (double)max_iter, boost);
  return launch_status();
}

int bdem_pcg_iterate(const bdem_system_t *sys, double *x, double *r, double *zv, double *pv,
                     double *ap, int n_iter, void *stream) {
  if (!sys || n_iter < 0) return BDEM_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  for (int it = 0; it < n_iter; ++it) {
    k_spmv<<<kRedBlocks, kThreads, 0, st>>>(*sys, pv, ap, 1);
    k_pcg_update<<<kRedBlocks, kThreads, 0, st>>>(*sys, x, r, zv, pv, ap);
    k_pcg_pupdate<<<kRedBlocks, kThreads, 0, st>>>(*sys, pv, zv);
  }
  return launch_status(3 * (int64_t)n_iter);
}

int bdem_pcg_spmv(const bdem_system_t *sys, const double *pv, double *ap, void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  k_spmv<<<kRedBlocks, kThreads, 0, as_stream(stream)>>>(*sys, pv, ap, 1);
  return launch_status();
}

int bdem_pcg_update(const bdem_system_t *sys, double *x, double *r, double *zv, double *pv,
                    const double *ap, void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  k_pcg_update<<<kRedBlocks, kThreads, 0, st>>>(*sys, x, r, zv, pv, ap);
  k_pcg_pupdate<<<kRedBlocks, kThreads, 0, st>>>(*sys, pv, zv);
  return launch_status(2);
}

int bdem_pair_assemble(const bdem_system_t *sys, const double *p, int energy_only,
                       void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  if (sys->n_pair == 0 && !energy_only) return BDEM_OK;
  k_pair<<<kRedBlocks, kThreads, 0, as_stream(stream)>>>(*sys, p, energy_only);
  return launch_status();
}

}  // extern "C"
