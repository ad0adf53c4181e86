// bond_kernels.cu -- per-bond kernels: ambient debug evaluation, the fused
// production assembly (energy + gradient + SPD-clamped reduced blocks),
// the line-search energy pass and the fracture/plasticity update.
//
// One thread per bond; bond data are structure-of-arrays planes so every
// load and store of a warp is a coalesced 256-byte transaction.  Endpoint
// states (p: 24 B, q: 32 B rows) are gathered through L1/L2.
#include "bdem_common.cuh"
#include "bdem_math.cuh"

namespace bdem {

struct BondIn {
  int i, j;
  int8_t status;
  double l0, d0[3], F[3][3], kn, kt, kd[3], scale;
};

__device__ __forceinline__ void load_bond(const bdem_system_t &S, int64_t b, BondIn &B) {
  const int64_t nb = S.n_bond;
  const double *g = S.geom;
  B.i = S.bond_i[b];
  B.j = S.bond_j[b];
  B.status = S.status[b];
  B.l0 = g[BDEM_BG_L0 * nb + b];
#pragma unroll
  for (int c = 0; c < 3; ++c) B.d0[c] = g[(BDEM_BG_D0 + c) * nb + b];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) B.F[r][c] = g[(BDEM_BG_FRAME + 3 * r + c) * nb + b];
  B.kn = g[BDEM_BG_KN * nb + b];
  B.kt = g[BDEM_BG_KT * nb + b];
#pragma unroll
  for (int c = 0; c < 3; ++c) B.kd[c] = g[(BDEM_BG_KDIAG + c) * nb + b];
  B.scale = S.bstate[BDEM_BS_SCALE * nb + b];
}

__device__ __forceinline__ void load_pq(const double *p, const double *q, int e, double pe[3],
                                        double qe[4]) {
  pe[0] = p[3 * (int64_t)e + 0];
  pe[1] = p[3 * (int64_t)e + 1];
  pe[2] = p[3 * (int64_t)e + 2];
  const double2 *q2 = reinterpret_cast<const double2 *>(q) + 2 * (int64_t)e;
  const double2 a = q2[0], c = q2[1];
  qe[0] = a.x; qe[1] = a.y; qe[2] = c.x; qe[3] = c.y;
}

__device__ __forceinline__ void flag_error(int32_t *err, int kind, int64_t b) {
  const int cnt = kind == BDEM_ERR_DEGENERATE_BOND ? BDEM_ERRSLOT_DEGENERATE_COUNT
                                                    : BDEM_ERRSLOT_ANTIPODAL_COUNT;
  atomicAdd(&err[cnt], 1);
  atomicMin(&err[cnt + 1], static_cast<int32_t>(b));
}

// ---------------------------------------------------------------------------
// ambient debug kernel: BondSet.energy_terms (bonds.py:473-504)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_bond_ambient(bdem_system_t S, const double *p,
                                                      const double *q, int64_t n_idx,
                                                      const int32_t *idx, double *E,
                                                      double *gpi, double *gpj, double *gqi,
                                                      double *gqj, double *hpp, double *hqq,
                                                      int want_hess) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_idx) return;
  const int64_t b = idx[t];
  BondIn B;
  load_bond(S, b, B);
  double pi[3], pj[3], qi[4], qj[4];
  load_pq(p, q, B.i, pi, qi);
  load_pq(p, q, B.j, pj, qj);
  const double ks = B.scale * B.kn, kts = B.scale * B.kt;
  double kds[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) kds[c] = B.scale * B.kd[c];
  const Stretch st = stretch_eval(pi, pj, B.l0, ks);
  const Shear sh = shear_eval(qi, qj, B.d0, kts);
  const BendTwist bt = bendtwist_eval(qi, qj, B.F, kds);
  if (st.degenerate) flag_error(S.err, BDEM_ERR_DEGENERATE_BOND, b);
  if (sh.antipodal) flag_error(S.err, BDEM_ERR_ANTIPODAL, b);
  E[t] = (st.E + sh.E) + bt.E;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    gpi[3 * t + c] = -st.gj[c];
    gpj[3 * t + c] = st.gj[c];
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    gqi[4 * t + c] = sh.g[c] + bt.gi[c];
    gqj[4 * t + c] = sh.g[c] + bt.gj[c];
  }
  if (!want_hess) return;
  double a[6];
  stretch_block(st, st.c_over_l, a);
  double *H = hpp + 36 * t;
  const int sym3[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double v = a[sym3[r][c]];
      H[6 * r + c] = v;
      H[6 * (r + 3) + c + 3] = v;
      H[6 * r + c + 3] = -v;
      H[6 * (r + 3) + c] = -v;
    }
  double hu[4][4], Hb[4][4];
  shear_hu(sh, B.d0, hu);
  double *Q = hqq + 64 * t;
  for (int which = 0; which < 3; ++which) {
    bendtwist_block(bt, B.F, which, Hb);
    const int r0 = (which == 1) ? 4 : 0, c0 = (which == 0) ? 0 : 4;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double v = hu[r][c] + Hb[r][c];
        Q[8 * (r0 + r) + c0 + c] = v;
        if (which == 2) Q[8 * (c0 + c) + r0 + r] = hu[c][r] + Hb[r][c];
      }
  }
}

// ---------------------------------------------------------------------------
// fused production bond pass: energy, gradient contributions and the clamped
// reduced blocks (energy_terms + build_clamped_pieces, solver.py:141-162)
// ---------------------------------------------------------------------------
// One thread per SELL row: it walks the row's i-role slots (the bonds with
// i == e in ascending id; lane = row & 31, so slot k of a warp's 32 rows is
// one contiguous 256-byte segment per plane) and
//   * writes the bond's SpMV coupling coefficients (scoef) and the pieces the
//     element pass gathers for the j end (stage: kc, dE/dq_j, (j,j) quadrant);
//   * adds the i-end pieces (-kc n, dE/dq_i, a+, (i,i) quadrant, energy) to
//     the row's partial sums in exactly the order the element pass used to
//     (np.add.at, integrator.py:100-103), so the gathered gradient and
//     diagonal blocks are unchanged bit for bit while the i-role pieces
//     never travel through HBM.  The partial sums live in shared memory
//     (one column per thread) so they do not compete with the bond
//     arithmetic for registers.
// A rotation block that fails the register PSD certificate is queued for
// the eigen-clamp pass (k_bond_clamp), which rewrites it after this kernel;
// from that slot on the row stages its (i,i) quadrants (ikpre) and the
// element pass continues the sum from there.
// 64-thread CTAs, 6 per SM (168 registers, 52 B of spills; at 8 per SM the
// 128-register cap spilled ~320 B per bond through L1, 441 vs 461 us on the
// plate, scratch/r02/ab_rows.sh).
#ifndef BDEM_ASM_MINB
#define BDEM_ASM_MINB 6
#endif
#ifndef BDEM_ASM_THREADS
#define BDEM_ASM_THREADS 64
#endif
#define ACC_T volatile double
// 1: the next slot's operand lines are prefetched into L2 while the current
// slot computes (387 -> 368 us on the plate).  Two slots ahead, only the
// early operands, one lane per line, and prefetches paired with the loads
// were all measured slower or equal (profiles/r02/README.md, session 4).
#ifndef BDEM_ASM_PF
#define BDEM_ASM_PF 1
#endif
// row blocks in descending order: the rows the element pass (ascending)
// starts with are the ones this pass wrote last, still in L2 (bond + element
// 505.8 -> 500.0 us)
// the 18 geometry planes are read once per assembly: evict-first loads keep
// them from displacing the outputs the element pass is about to read (bond
// pass 340.0 -> 333.8 us, bond + element 496.6 -> 490.5 us; the same hint on
// status / j index / scale, or evict-first stores of the C coefficients, did
// not help)
#ifndef BDEM_ASM_GEO_CS
#define BDEM_ASM_GEO_CS 1
#endif
#ifndef BDEM_ASM_REVERSE
#define BDEM_ASM_REVERSE 1
#endif
__device__ __forceinline__ void prefetch_l2(const void *a) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}

// row partial sums in shared memory: acc[first + c][t] += v[c] for c < N,
// all loads issued before the adds and all stores after them (volatile
// accesses keep program order, so an interleaved load/add/store sequence
// would serialise on the shared-memory latency)
template <int N>
__device__ __forceinline__ void acc_add(ACC_T (*acc)[BDEM_ASM_THREADS], int first, int t,
                                        const double v[N]) {
  double cur[N];
#pragma unroll
  for (int c = 0; c < N; ++c) cur[c] = acc[first + c][t];
#pragma unroll
  for (int c = 0; c < N; ++c) cur[c] += v[c];
#pragma unroll
  for (int c = 0; c < N; ++c) acc[first + c][t] = cur[c];
}

__global__ void __launch_bounds__(BDEM_ASM_THREADS, BDEM_ASM_MINB) k_bond_rows(bdem_system_t S, const double *p,
                                                       const double *q) {
  __shared__ double acc_sh[BDEM_IP_COUNT][BDEM_ASM_THREADS];
  // volatile: every partial-sum update is a shared-memory read-modify-write
  // (the compiler would otherwise keep the 20 sums in registers and spill)
  ACC_T(*acc)[BDEM_ASM_THREADS] = acc_sh;
  const int t = threadIdx.x;
  const int64_t nrow = ((S.n_elem + 31) >> 5) << 5;
#if BDEM_ASM_REVERSE
  const unsigned int blk = gridDim.x - 1 - blockIdx.x;
#else
  const unsigned int blk = blockIdx.x;
#endif
  const int64_t row = blk * (int64_t)BDEM_ASM_THREADS + t;
  if (row >= nrow) return;
#pragma unroll
  for (int k = 0; k < BDEM_IP_COUNT; ++k) acc[k][t] = 0.0;
  const int sl = (int)(row >> 5), lane = (int)(row & 31);
  const int e = S.row_elem[row];
  const int64_t nb = S.n_bond;
  double *st_out = S.stage;
  int kpre = (S.asm_flags & BDEM_ASM_STAGE_ALL_A) ? 0 : -1;
  const int64_t b_end = S.slice_base[sl + 1];
  const int64_t b_beg = S.slice_base[sl] + lane;
  const double *g = S.geom;
  int k = 0;
#pragma unroll 1
  for (int64_t b = b_beg; b < b_end; b += 32, ++k) {
    double *cf = S.scoef + cf_idx(b, 0);
    const int8_t stat = S.status[b];
#if BDEM_ASM_PF
    // the next slot's operands are pulled into L2 while this slot computes
    // (no registers held): its loads then pay the L2 latency, not DRAM's
    if (b + 32 < b_end) {
      const int64_t bn = b + 32;
      prefetch_l2(S.status + bn);
      prefetch_l2(S.bond_j + bn);
      prefetch_l2(S.bstate + BDEM_BS_SCALE * nb + bn);
#pragma unroll
      for (int f = 0; f < BDEM_BG_KDIAG + 3; ++f) prefetch_l2(g + f * nb + bn);
    }
#endif
#if BDEM_ASM_GEO_CS
#define GEO(f) __ldcs(g + (f) * nb + b)
#else
#define GEO(f) g[(f) * nb + b]
#endif
    if (stat == 2) {  // broken or padding: no energy, no coupling
#pragma unroll
      for (int c = 0; c < BDEM_ST_COUNT; ++c) st_out[c * nb + b] = 0.0;
      const double zero[BDEM_CF_COUNT] = {};
      store_coef(cf, zero);
      continue;
    }
    // pieces are stored (and summed) as soon as they are final so the
    // stretch state is dead before the rotation block is formed
    double pi[3], qi[4], pj[3], qj[4];
    load_pq(p, q, e, pi, qi);
    const double scale = S.bstate[BDEM_BS_SCALE * nb + b];
    load_pq(p, q, S.bond_j[b], pj, qj);

    // stretch: energy, gradient (kc n) and the closed-form clamp of
    // [[a,-a],[-a,a]]: a+ = k (nn + max(c/l,0) (I - nn)) = alpha nn + beta I
    double e_s, beta_cf;
    {
      const double ks = scale * GEO(BDEM_BG_KN);
      const Stretch st = stretch_eval(pi, pj, GEO(BDEM_BG_L0), ks);
      if (st.degenerate) flag_error(S.err, BDEM_ERR_DEGENERATE_BOND, b);
      const double f = st.c_over_l > 0.0 ? st.c_over_l : 0.0;
      const double beta = ks * f;
      const double alpha = ks - beta;
      e_s = st.E;
      st_out[BDEM_ST_KC * nb + b] = st.kc;
      static_assert(BDEM_CF_N == 0 && BDEM_CF_ALPHA == 3 && BDEM_CF_BETA == 4 && BDEM_CF_C == 5,
                    "coefficient pairs: (n0 n1) (n2 alpha) (beta C00) (C01 C02) ...");
      store_coef_pair(cf, 0, st.n[0], st.n[1]);
      store_coef_pair(cf, 1, st.n[2], alpha);
      beta_cf = beta;   // shares its pair with C00
      double apos[6], gpc[3];
      stretch_apos(alpha, beta, st.n, apos);
#pragma unroll
      for (int c = 0; c < 3; ++c) gpc[c] = acc[BDEM_IP_GP + c][t];
      // same expression as the element pass's j-role sum (same contraction)
#pragma unroll
      for (int c = 0; c < 3; ++c) gpc[c] += -(st.kc * st.n[c]);
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[BDEM_IP_GP + c][t] = gpc[c];
      acc_add<6>(acc, BDEM_IP_P, t, apos);
    }

    double S6[21];
    {
      double d0[3], F[3][3], kds[3];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) F[r][c] = GEO(BDEM_BG_FRAME + 3 * r + c);
#pragma unroll
      for (int c = 0; c < 3; ++c) kds[c] = scale * GEO(BDEM_BG_KDIAG + c);
#pragma unroll
      for (int c = 0; c < 3; ++c) d0[c] = GEO(BDEM_BG_D0 + c);
      const Shear sh = shear_eval(qi, qj, d0, scale * GEO(BDEM_BG_KT));
      if (sh.antipodal) flag_error(S.err, BDEM_ERR_ANTIPODAL, b);
      const RotGrad ro = rot_grad(qi, qj, F, kds);
      double eg[5];
      eg[0] = (e_s + sh.E) + ro.E_b;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        eg[1 + c] = sh.g[c] + ro.gbi[c];
        st_out[(BDEM_ST_GQJ + c) * nb + b] = sh.g[c] + ro.gbj[c];
      }
      acc_add<1>(acc, BDEM_IP_E, t, eg);
      acc_add<4>(acc, BDEM_IP_GQ, t, eg + 1);
      rot_block(qi, qj, d0, F, kds, sh, ro.rs, ro.rv, ro.w, S6);
    }
#undef GEO
    store_coef_pair(cf, 2, beta_cf, S6[sidx<6>(0, 3)]);
    store_coef_pair(cf, 3, S6[sidx<6>(0, 4)], S6[sidx<6>(0, 5)]);
    store_coef_pair(cf, 4, S6[sidx<6>(1, 3)], S6[sidx<6>(1, 4)]);
    store_coef_pair(cf, 5, S6[sidx<6>(1, 5)], S6[sidx<6>(2, 3)]);
    store_coef_pair(cf, 6, S6[sidx<6>(2, 4)], S6[sidx<6>(2, 5)]);
    const int pr[6] = {0, 0, 0, 1, 1, 2}, pc[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int u = 0; u < 6; ++u) st_out[(BDEM_ST_D + u) * nb + b] = S6[sidx<6>(pr[u] + 3, pc[u] + 3)];

    // PSD blocks (all of them at identity orientations) are final; an
    // indefinite one is queued for the register-resident eigen-clamp pass
    // (k_bond_clamp), which overwrites its staged quadrants and coefficients
    const double mx = max_abs21(S6);
    if (mx != 0.0 && !psd6_regs(S6, 4e-14 * mx)) {
      const unsigned int slot = atomicAdd(S.counter + kClampCounter, 1u);
      S.clamp_list[slot] = (int32_t)b;
      if (kpre < 0) kpre = k;
    }
    if (kpre < 0) {
      double a6[6];
#pragma unroll
      for (int u = 0; u < 6; ++u) a6[u] = S6[sidx<6>(pr[u], pc[u])];
      acc_add<6>(acc, BDEM_IP_R, t, a6);
    } else {
#pragma unroll
      for (int u = 0; u < 6; ++u) st_out[(BDEM_ST_A + u) * nb + b] = S6[sidx<6>(pr[u], pc[u])];
    }
  }
#pragma unroll
  for (int c = 0; c < BDEM_IP_COUNT; ++c) S.ipart[c * nrow + row] = acc[c][t];
  S.ikpre[row] = kpre;
}

// ---------------------------------------------------------------------------
// eigen-clamp pass for the queued indefinite rotation blocks (spd_project,
// solver.py:89-113): one thread per queued bond, Jacobi in registers
// ---------------------------------------------------------------------------
// occupancy: unbounded, the Jacobi pass takes 182 registers (2 CTAs = 8
// warps per SM); capped at 168 (3 CTAs, 36 B of spills) it runs 12% faster
// (C5-like random-q blocks, profiles/r01/README.md); 32- or 64-thread CTAs
// at 182 registers do not help
#ifndef BDEM_CLAMP_THREADS
#define BDEM_CLAMP_THREADS 128
#endif
#ifndef BDEM_CLAMP_MINB
#define BDEM_CLAMP_MINB 3
#endif
__global__ void __launch_bounds__(BDEM_CLAMP_THREADS, BDEM_CLAMP_MINB) k_bond_clamp(bdem_system_t S) {
  const unsigned int n = S.counter[kClampCounter];
  const int64_t nb = S.n_bond;
  double *st = S.stage;
  for (unsigned int t = blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += gridDim.x * blockDim.x) {
    const int64_t b = S.clamp_list[t];
    double A[21];
    const int pr[6] = {0, 0, 0, 1, 1, 2}, pc[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      A[sidx<6>(pr[q], pc[q])] = st[(BDEM_ST_A + q) * nb + b];
      A[sidx<6>(pr[q] + 3, pc[q] + 3)] = st[(BDEM_ST_D + q) * nb + b];
    }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) A[sidx<6>(r, c + 3)] = S.scoef[cf_idx(b, BDEM_CF_C + 3 * r + c)];
    jacobi_clamp_regs<6>(A);
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      st[(BDEM_ST_A + q) * nb + b] = A[sidx<6>(pr[q], pc[q])];
      st[(BDEM_ST_D + q) * nb + b] = A[sidx<6>(pr[q] + 3, pc[q] + 3)];
    }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) S.scoef[cf_idx(b, BDEM_CF_C + 3 * r + c)] = A[sidx<6>(r, c + 3)];
  }
}

// ---------------------------------------------------------------------------
// energy-only pass (PotentialModel.value, integrator.py:87-89)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_bond_energy(bdem_system_t S, const double *p,
                                                          const double *q, int col) {
  __shared__ double sh_red[kThreads / 32];
  double acc = 0.0;
  const int64_t nb = S.n_bond;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    if (S.status[b] == 2) continue;
    const int i = S.bond_i[b], j = S.bond_j[b];
    const double *g = S.geom;
    const double sc = S.bstate[BDEM_BS_SCALE * nb + b];
    double pi[3], pj[3], qi[4], qj[4];
    load_pq(p, q, i, pi, qi);
    load_pq(p, q, j, pj, qj);
    // stretch
    const double l0 = g[BDEM_BG_L0 * nb + b];
    const double d0_ = pj[0] - pi[0], d1_ = pj[1] - pi[1], d2_ = pj[2] - pi[2];
    const double len = sqrt((d0_ * d0_ + d1_ * d1_) + d2_ * d2_);
    if (len < kDegenerateRel * l0) flag_error(S.err, BDEM_ERR_DEGENERATE_BOND, b);
    const double c = len - l0;
    const double e_s = 0.5 * (sc * g[BDEM_BG_KN * nb + b]) * (c * c);
    // shear
    double d0[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) d0[k] = g[(BDEM_BG_D0 + k) * nb + b];
    double u[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) u[k] = qi[k] + qj[k];
    const double un2 = ((u[0] * u[0] + u[1] * u[1]) + u[2] * u[2]) + u[3] * u[3];
    if (un2 < kAntipodalTol * kAntipodalTol) flag_error(S.err, BDEM_ERR_ANTIPODAL, b);
    const double proj = (d0[0] * u[0] + d0[1] * u[1]) + d0[2] * u[2];
    const double utut = (u[0] * u[0] + u[1] * u[1]) + u[2] * u[2];
    double rho = ((2.0 * (proj * proj)) - utut + u[3] * u[3]) / un2;
    rho = rho < -1.0 + 1e-12 ? -1.0 + 1e-12 : rho;
    rho = rho > 1.0 ? 1.0 : rho;
    const double th = acos(rho);
    const double e_h = 0.5 * (sc * g[BDEM_BG_KT * nb + b]) * (th * th);
    // bend/twist: t = F G_l(q_j) q_i
    double v[3];
    gl_apply(qj, qi, v);
    double e_b = 0.0;
    {
      double t[3], kt[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        t[r] = (g[(BDEM_BG_FRAME + 3 * r) * nb + b] * v[0] +
                g[(BDEM_BG_FRAME + 3 * r + 1) * nb + b] * v[1]) +
               g[(BDEM_BG_FRAME + 3 * r + 2) * nb + b] * v[2];
        kt[r] = (sc * g[(BDEM_BG_KDIAG + r) * nb + b]) * t[r];
      }
      e_b = 0.5 * ((t[0] * kt[0] + t[1] * kt[1]) + t[2] * kt[2]);
    }
    acc += (e_s + e_h) + e_b;
  }
  const double s = block_sum<kThreads>(acc, sh_red);
  if (threadIdx.x == 0) *red_slot(S.red, col, blockIdx.x) = s;
}

// ---------------------------------------------------------------------------
// fracture / plasticity update (bonds.py:506-570)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double pow_np(double x, double a) {
  // numpy's float power fast paths for the scalar exponents it special-cases
  if (a == 2.0) return x * x;
  if (a == 1.0) return x;
  if (a == 0.5) return sqrt(x);
  return pow(x, a);
}

__global__ void __launch_bounds__(kThreads) k_bond_update(bdem_system_t S, const double *p,
                                                          const double *q, double youngs,
                                                          int plastic_on, double eps_c,
                                                          double eps_y, double weak,
                                                          double dexp, uint8_t *flags) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nb = S.n_bond;
  if (b >= nb) return;
  const int8_t status = S.status[b];
  if (status == 2) {
    flags[b] = 0;
    return;
  }
  const double *g = S.geom;
  double *bs = S.bstate;
  const int i = S.bond_i[b], j = S.bond_j[b];
  double pi[3], pj[3], qi[4], qj[4];
  load_pq(p, q, i, pi, qi);
  load_pq(p, q, j, pj, qj);
  double scale = bs[BDEM_BS_SCALE * nb + b];
  const double l0 = g[BDEM_BG_L0 * nb + b];
  const double d0_ = pj[0] - pi[0], d1_ = pj[1] - pi[1], d2_ = pj[2] - pi[2];
  const double len = sqrt((d0_ * d0_ + d1_ * d1_) + d2_ * d2_);
  const double fn = (scale * g[BDEM_BG_KN * nb + b]) * fabs(len - l0);
  double v[3], t[3], kt[3];
  gl_apply(qj, qi, v);
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    t[r] = (g[(BDEM_BG_FRAME + 3 * r) * nb + b] * v[0] +
            g[(BDEM_BG_FRAME + 3 * r + 1) * nb + b] * v[1]) +
           g[(BDEM_BG_FRAME + 3 * r + 2) * nb + b] * v[2];
    kt[r] = (scale * g[(BDEM_BG_KDIAG + r) * nb + b]) * t[r];
  }
  const double mt = fabs(kt[0]);
  const double mb = hypot(kt[1], kt[2]);
  const double r0 = g[BDEM_BG_RADIUS * nb + b];
  const double section = bs[BDEM_BS_DAMAGE * nb + b] * g[BDEM_BG_SECTION * nb + b];
  const double sigma = div_nz(fn, section) + div_nz(mb * r0, g[BDEM_BG_SECOND * nb + b]);
  const double tau = div_nz(mt * r0, g[BDEM_BG_POLAR * nb + b]);
  bs[BDEM_BS_SIGMA * nb + b] = sigma;
  bs[BDEM_BS_TAU * nb + b] = tau;
  bool broke = false;
  int8_t new_status = status;
  if (plastic_on) {
    const double strain = div_nz(len - l0, l0);
    const double sy = youngs * eps_y;
    const double vm = sqrt(sigma * sigma + 3.0 * (tau * tau));
    if (vm > sy) {
      const double k_new = 1.0 - weak * (1.0 - sy / vm);
      scale = fmin(scale, k_new);
      bs[BDEM_BS_SCALE * nb + b] = scale;
      const double ep = fmax(0.0, strain - eps_y);
      bs[BDEM_BS_PLASTIC * nb + b] = fmax(bs[BDEM_BS_PLASTIC * nb + b], ep);
      bs[BDEM_BS_DAMAGE * nb + b] = fmin(bs[BDEM_BS_DAMAGE * nb + b], exp(-pow_np(ep, dexp)));
      if (new_status < 1) new_status = 1;
    }
    broke |= strain > eps_c;
  }
  broke |= (sigma > g[BDEM_BG_TENSILE * nb + b]) || (tau > g[BDEM_BG_SHEAR * nb + b]);
  if (broke) new_status = 2;
  if (new_status != status) S.status[b] = new_status;
  flags[b] = broke ? 1 : 0;
}

// (sigma, tau) of the flagged positions, for the ordered event list
// [(bond, sigma, tau)] of update_bond_states (bonds.py:564-570)
__global__ void k_event_records(bdem_system_t S, const int32_t *pos, int64_t m, double *out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int64_t b = pos[k];
  out[2 * k] = S.bstate[BDEM_BS_SIGMA * S.n_bond + b];
  out[2 * k + 1] = S.bstate[BDEM_BS_TAU * S.n_bond + b];
}

}  // namespace bdem

using namespace bdem;

extern "C" {

int bdem_bond_eval_ambient(const bdem_system_t *sys, const double *p, const double *q,
                           int64_t n_idx, const int32_t *idx, double *E, double *gpi,
                           double *gpj, double *gqi, double *gqj, double *hpp, double *hqq,
                           int want_hess, void *stream) {
  if (!sys || n_idx < 0) return BDEM_ERR_ARG;
  if (n_idx == 0) return BDEM_OK;
  k_bond_ambient<<<grid_for(n_idx, 128), 128, 0, as_stream(stream)>>>(
      *sys, p, q, n_idx, idx, E, gpi, gpj, gqi, gqj, hpp, hqq, want_hess);
  return launch_status();
}

int bdem_bond_assemble(const bdem_system_t *sys, const double *p, const double *q,
                       void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  if (sys->n_bond == 0) return BDEM_OK;
  cudaStream_t st = as_stream(stream);
  cudaMemsetAsync(sys->counter + kClampCounter, 0, sizeof(unsigned int), st);
  const int64_t nrow = ((sys->n_elem + 31) >> 5) << 5;
  if (nrow > (int64_t)grid_for(nrow, BDEM_ASM_THREADS) * BDEM_ASM_THREADS) return BDEM_ERR_ARG;
  k_bond_rows<<<grid_for(nrow, BDEM_ASM_THREADS), BDEM_ASM_THREADS, 0, st>>>(*sys, p, q);
  // the clamp pass reads the queue length on the device; idle threads exit
  k_bond_clamp<<<kRedBlocks * (128 / BDEM_CLAMP_THREADS), BDEM_CLAMP_THREADS, 0, st>>>(*sys);
  return launch_status(2);
}

int bdem_bond_energy(const bdem_system_t *sys, const double *p, const double *q, int col,
                     void *stream) {
  if (!sys || col < 0 || col >= BDEM_SC_COUNT) return BDEM_ERR_ARG;
  k_bond_energy<<<kRedBlocks, kThreads, 0, as_stream(stream)>>>(*sys, p, q, col);
  return launch_status();
}

int bdem_event_records(const bdem_system_t *sys, const int32_t *pos, int64_t m, double *out,
                       void *stream) {
  if (!sys || m < 0) return BDEM_ERR_ARG;
  if (m == 0) return BDEM_OK;
  k_event_records<<<grid_for(m), kThreads, 0, as_stream(stream)>>>(*sys, pos, m, out);
  return launch_status();
}

int bdem_bond_update(const bdem_system_t *sys, const double *p, const double *q,
                     double youngs, const double *plastic, uint8_t *flags, void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  if (sys->n_bond == 0) return BDEM_OK;
  const int on = plastic != nullptr;
  k_bond_update<<<grid_for(sys->n_bond), kThreads, 0, as_stream(stream)>>>(
      *sys, p, q, youngs, on, on ? plastic[0] : 0.0, on ? plastic[1] : 0.0,
      on ? plastic[2] : 0.0, on ? plastic[3] : 1.0, flags);
  return launch_status();
}

}  // extern "C"
