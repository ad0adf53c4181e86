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
#include <cstdlib>

#include "bdem_common.cuh"
#include "bdem_math.cuh"

namespace bdem {

enum { PCG_RUNNING = 0, PCG_CONVERGED = 1, PCG_BREAKDOWN = 2, PCG_MAXIT = 3 };

// Diagnostic builds only (-DBDEM_TIMELINE=1, not the shipped library): every
// PCG kernel stamps %globaltimer at its first CTA's arrival, its first CTA's
// release from griddepcontrol.wait and its last CTA's exit, per iteration,
// so the gaps at the kernel boundaries of the PDL chain can be read back
// (bdem_timeline_read).  Slot = (kernel, pcg K & 1023).
#ifndef BDEM_TIMELINE
#define BDEM_TIMELINE 0
#endif
#if BDEM_TIMELINE
__device__ unsigned long long g_tl[3 * 1024 * 3];
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TL_ARRIVE(kid, it) \
  if (threadIdx.x == 0) atomicMin(&g_tl[((kid) * 1024 + ((it) & 1023)) * 3 + 0], tl_now());
#define TL_RELEASE(kid, it) \
  if (threadIdx.x == 0) atomicMin(&g_tl[((kid) * 1024 + ((it) & 1023)) * 3 + 1], tl_now());
#define TL_EXIT(kid, it)  \
  __syncthreads();        \
  if (threadIdx.x == 0) atomicMax(&g_tl[((kid) * 1024 + ((it) & 1023)) * 3 + 2], tl_now());
#else
#define TL_ARRIVE(kid, it)
#define TL_RELEASE(kid, it)
#define TL_EXIT(kid, it)
#endif

// Programmatic dependent launch: the PCG kernels are launched with
// programmatic stream serialisation, so a kernel's CTAs are scheduled as the
// previous kernel's CTAs retire; each waits here until the previous grid has
// completed and its writes are visible (a no-op for ordinary launches).
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
enum { CNT_SPMV = 2, CNT_UPDATE = 3, CNT_INIT = 4 };
// partial-sum columns of sys->red owned by PCG (disjoint from BDEM_SC_*)
enum { RC_PAP = 20, RC_AP2 = 21, RC_PP2 = 22, RC_RR = 23, RC_RZ = 24, RC_IRR = 25, RC_IRZ = 26,
       RC_IRN = 27 };

// The SpMV's gathers of x (each row's block is gathered by
// ~12 bonds) carry an L2 evict-last cache policy, so the streamed
// coefficients evict them last (1% per PCG iteration; the same hint on the
// slot indices and diagonal blocks measured 1% slower)
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double ld_keep(const double *a) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(l2_evict_last_policy()));
  return v;
}

// 1: the slice's diagonal rows (read after the slice barrier) are prefetched
// into L2 at the top of the slice: 123.2 -> 122.0 us, PCG iteration 176.9 ->
// 175.8 us.  Prefetching the CTA's next slice (records, index lines: 152-162
// us, a grid-wide wave ahead overflows what L2 retains) or the warp's next
// in-slice records (no gain) was measured and dropped (profiles/r02/README.md).
#ifndef BDEM_SPMV_PF
#define BDEM_SPMV_PF 1
#endif
__device__ __forceinline__ void prefetch_l2(const void *a) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}

// reduced vectors are 6 planes of stride vstride: component c of slot s at
// x[c * vstride + s], so a warp touching 32 consecutive slots reads 256 contiguous
// bytes per component
__device__ __forceinline__ void load6(const double *x, int64_t s, int64_t nf, double v[6]) {
#pragma unroll
  for (int c = 0; c < 6; ++c) v[c] = x[c * nf + s];
}
__device__ __forceinline__ void load6_ro(const double *x, int64_t s, int64_t nf, double v[6]) {
#pragma unroll
  for (int c = 0; c < 6; ++c) v[c] = ld_keep(x + c * nf + s);
}
__device__ __forceinline__ void store6(double *x, int64_t s, int64_t nf, const double v[6]) {
#pragma unroll
  for (int c = 0; c < 6; ++c) x[c * nf + s] = v[c];
}

__device__ __forceinline__ void load_sym(const double *planes, int64_t s, int64_t nf, double v[6]) {
#pragma unroll
  for (int t = 0; t < 6; ++t) v[t] = planes[t * nf + s];
}

__device__ __forceinline__ void precond_row(const bdem_system_t &S, int64_t s, const double r[6],
                                            double z[6]) {
  const int64_t nf = S.vstride;
  double mp[6], mr[6];
  load_sym(S.minv, s, nf, mp);
  load_sym(S.minv + 6 * nf, s, nf, mr);
  symv3(mp, r, z);
  symv3(mr, r + 3, z + 3);
}

// component c (= w, w + W, ...) of y for the 32 rows of slice sl:
// y = D x + sum of the staged slot partials (fixed order) - pair couplings
template <int W, bool kRot = true>
__device__ __forceinline__ void spmv_tail(const bdem_system_t &S, const double *x, double *y,
                                          int sl, int w, int lane, const double (*part)[6][32],
                                          double boost, double &acc_xy, double &acc_yy,
                                          double &acc_xx, int s) {
  const int64_t nf = S.vstride;
  // s = the row's free slot (row_slot = slot[row_elem], loaded by the caller
  // at the start of the slice); the element id only for the contact pairs
  if (s < 0) return;
  const int64_t e = S.n_pair > 0 ? __ldg(S.row_elem + (int64_t)sl * 32 + lane) : -1;
  // kRot false: the rotation half of x is identically zero (see
  // pcg_rot_active), so y's rotation half is zero and not formed
  for (int c = w; c < (kRot ? 6 : 3); c += W) {
    const int base = c < 3 ? 0 : 3, rr = c - base;
    const double *dg = S.diag + (c < 3 ? 0 : 6 * nf);
    double xs[3], dgr[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      xs[t] = __ldg(x + (base + t) * nf + s);
      dgr[t] = __ldg(dg + sidx<3>(rr, t) * nf + s);
    }
    double yc = (dgr[0] * xs[0] + dgr[1] * xs[1]) + dgr[2] * xs[2];
#pragma unroll
    for (int ww = 0; ww < W; ++ww) yc += part[ww][c][lane];
    if (c < 3 && S.n_pair > 0) {
      const int64_t pc = S.pair_cap;
      const double *ps = S.pstage;
      for (int k = S.pi_ptr[e]; k < S.pi_ptr[e + 1]; ++k) {
        const int o = S.slot[S.pair_j[k]];
        if (o < 0) continue;
        yc -= (ps[(BDEM_PS_A + sidx<3>(c, 0)) * pc + k] * x[0 * nf + o] +
               ps[(BDEM_PS_A + sidx<3>(c, 1)) * pc + k] * x[1 * nf + o]) +
              ps[(BDEM_PS_A + sidx<3>(c, 2)) * pc + k] * x[2 * nf + o];
      }
      for (int kk = S.pj_ptr[e]; kk < S.pj_ptr[e + 1]; ++kk) {
        const int64_t k = S.pj_idx[kk];
        const int o = S.slot[S.pair_i[k]];
        if (o < 0) continue;
        yc -= (ps[(BDEM_PS_A + sidx<3>(c, 0)) * pc + k] * x[0 * nf + o] +
               ps[(BDEM_PS_A + sidx<3>(c, 1)) * pc + k] * x[1 * nf + o]) +
              ps[(BDEM_PS_A + sidx<3>(c, 2)) * pc + k] * x[2 * nf + o];
      }
    }
    // (a select, not xs[rr]: a run-time index would put xs in local memory)
    const double xc = rr == 0 ? xs[0] : (rr == 1 ? xs[1] : xs[2]);
    if (boost != 0.0) yc = yc + boost * xc;
    y[c * nf + s] = yc;
    acc_xy += xc * yc;
    acc_yy += yc * yc;
    acc_xx += xc * xc;
  }
}

// PCG-mode epilogue shared by the SpMV kernels: per-block partials of p.Ap,
// |Ap|^2, |p|^2 (one shared-memory round); the last block sets alpha, or
// flags breakdown and only then sums |Ap|^2 and |p|^2 for the restart boost
// (linalg.py:69-77).  Same partials and fixed-order sums as before.
template <int NT>
__device__ __forceinline__ void spmv_pcg_epilogue(const bdem_system_t &S, double boost,
                                                  double acc_xy, double acc_yy, double acc_xx,
                                                  double *sh) {
  double *pcg = S.pcg;
  __shared__ double sh3[3 * (NT / 32)];
  __shared__ double pap_sh;
  double v3[3] = {acc_xy, acc_yy, acc_xx};
  block_sum_k<NT, 3>(v3, sh3);
  if (threadIdx.x == 0) {
    *red_slot(S.red, RC_PAP, blockIdx.x) = v3[0];
    *red_slot(S.red, RC_AP2, blockIdx.x) = v3[1];
    *red_slot(S.red, RC_PP2, blockIdx.x) = v3[2];
  }
  if (!last_block(S.counter + CNT_SPMV)) return;
  const double pap = sum_partials<NT>(S.red, RC_PAP, gridDim.x, sh);
  if (threadIdx.x == 0) {
    pap_sh = pap;
    pcg[BDEM_PCG_PAP] = pap;
    if (pap > 0.0) pcg[BDEM_PCG_ALPHA] = pcg[BDEM_PCG_RZ] / pap;
  }
  __syncthreads();
  if (pap_sh > 0.0) return;
  // breakdown: boost for the restart (linalg.py:74-77)
  const double ap2 = sum_partials<NT>(S.red, RC_AP2, gridDim.x, sh);
  const double pp2 = sum_partials<NT>(S.red, RC_PP2, gridDim.x, sh);
  if (threadIdx.x == 0) {
    pcg[BDEM_PCG_APNORM2] = ap2;
    pcg[BDEM_PCG_PNORM2] = pp2;
    const double sc = sqrt(ap2) / fmax(sqrt(pp2), 1e-300);
    pcg[BDEM_PCG_BOOST] = fmax(boost * 100.0, 1e-10 * fmax(sc, 1.0));
    pcg[BDEM_PCG_STATE] = PCG_BREAKDOWN;
  }
}

// ---------------------------------------------------------------------------
// SpMV, slot-parallel form.  One CTA works on one 32-element slice at a time:
// warp w takes slots w, w+8, ... of the slice's i-role and j-role lists
// (lane = element), so every thread issues one independent set of loads
// (index -> 15 coefficient planes + the neighbour's x block) and the
// coefficient loads of a warp are contiguous 256-byte segments.  Partial
// products go to shared memory; warps 0..5 then form component c of
// y = D x + sum_slots in a fixed order (deterministic).
// mode 0: plain y = A x;  mode 1: PCG step (y = A p + boost p, p.Ap, |Ap|^2,
// |p|^2 and the breakdown test, linalg.py:69-77).
// ---------------------------------------------------------------------------
#ifndef BDEM_SPMV_WARPS
#define BDEM_SPMV_WARPS 4
#endif
#ifndef BDEM_SPMV_MINB
#define BDEM_SPMV_MINB 8
#endif
constexpr int kSpmvWarps = BDEM_SPMV_WARPS;
constexpr int kSpmvThreads = 32 * kSpmvWarps;

// where slot k of a slice lives: i-role (coefficients at b, neighbour slot o,
// C applied as is) or j-role (C^T); o < 0 = nothing to do
struct SlotRef {
  int64_t b;
  int o;
  bool tr;
};

__device__ __forceinline__ SlotRef slot_ref(const bdem_system_t &S, int64_t i0, int ki,
                                            int64_t j0, int kj, int lane, int k) {
  SlotRef r{0, -1, false};
  if (k < ki) {
    r.b = i0 + 32 * k + lane;
    r.o = __ldg(S.pos_oslot + r.b);
  } else if (k < ki + kj) {
    const int64_t jk = j0 + 32 * (k - ki) + lane;
    r.o = __ldg(S.jslot + jk);
    r.b = __ldg(S.jpos + jk);
    r.tr = true;
  }
  return r;
}

template <bool kRot = true>
__device__ __forceinline__ void slot_apply(const bdem_system_t &S, const double *x,
                                           const SlotRef &r, double acc[6]) {
  if (r.o < 0) return;
  if (!kRot) {
    // position half only: 5 of the 14 coefficients, 3 of the 6 x components
    const double *base = S.scoef + cf_idx(r.b, 0);
    double xo[3], n[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) xo[t] = __ldg(x + t * S.vstride + r.o);
    // n0 n1 | n2 alpha | beta (C0): three 16-byte loads
    const double2 *b2 = reinterpret_cast<const double2 *>(base);
    const double2 c01 = __ldg(b2), c23 = __ldg(b2 + 32), c45 = __ldg(b2 + 64);
    n[0] = c01.x; n[1] = c01.y; n[2] = c23.x;
    const double al = c23.y, be = c45.x;
    static_assert(BDEM_CF_N == 0 && BDEM_CF_ALPHA == 3 && BDEM_CF_BETA == 4, "pair layout");
    const double nx = al * ((n[0] * xo[0] + n[1] * xo[1]) + n[2] * xo[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c] -= nx * n[c] + be * xo[c];
    return;
  }
  const int64_t nb = S.n_bond;
  const double *st = S.stage;
  double xo[6], n[3], C[9];
  load6_ro(x, r.o, S.vstride, xo);
  const Coef cv = load_coef<true>(S.scoef + cf_idx(r.b, 0));
#pragma unroll
  for (int t = 0; t < 3; ++t) n[t] = cv.n[t];
  const double al = cv.al, be = cv.be;
#pragma unroll
  for (int t = 0; t < 9; ++t) C[t] = cv.C[t];
  // a+ x = alpha (n.x) n + beta x ; coupling -a+
  const double nx = al * ((n[0] * xo[0] + n[1] * xo[1]) + n[2] * xo[2]);
#pragma unroll
  for (int c = 0; c < 3; ++c) acc[c] -= nx * n[c] + be * xo[c];
  if (!r.tr) {
#pragma unroll
    for (int q = 0; q < 3; ++q)
      acc[3 + q] += (C[3 * q] * xo[3] + C[3 * q + 1] * xo[4]) + C[3 * q + 2] * xo[5];
  } else {
#pragma unroll
    for (int q = 0; q < 3; ++q)
      acc[3 + q] += (C[q] * xo[3] + C[3 + q] * xo[4]) + C[6 + q] * xo[5];
  }
}

struct SliceBounds {
  int64_t i0, j0;
  int ki, kj;
};

__device__ __forceinline__ SliceBounds slice_bounds(const bdem_system_t &S, int sl, int ns) {
  SliceBounds sb{0, 0, 0, 0};
  if (sl < ns) {
    const int a0 = __ldg(S.slice_base + sl), a1 = __ldg(S.slice_base + sl + 1);
    const int c0 = __ldg(S.jslice_base + sl), c1 = __ldg(S.jslice_base + sl + 1);
    sb.i0 = a0; sb.ki = (a1 - a0) >> 5;
    sb.j0 = c0; sb.kj = (c1 - c0) >> 5;
  }
  return sb;
}

// ---------------------------------------------------------------------------
// SpMV, slot-parallel form.  One CTA of 4 warps walks 32-element slices
// (strided over the grid); in each slice warp w handles slots w, w+4, ... of
// the slice's i-role then j-role lists (lane = element), so each thread
// issues one independent set of loads per slot: 14 coefficient planes
// (contiguous 256-byte warp segments, AoSoA-32) and the neighbour's x block
// (evict-last L2 policy: each block is gathered ~12 times).  The next slot's
// indices are loaded while the current slot's data is in flight; the row's
// free slot comes from row_slot in one load.  Partial products meet in a
// double-buffered shared-memory array (one barrier per slice); warp c forms
// component c (and c + 4) of y = D x + sum of the warp partials in a fixed
// order (deterministic).  The kernel is memory-latency bound at the
// 64-register / 8-CTA point; every variant that keeps more loads in flight
// spilled (profiles/r01/README.md).
// mode 0: plain y = A x;  mode 1: PCG step (y = A p + boost p, p.Ap, |Ap|^2,
// |p|^2 and the breakdown test, linalg.py:69-77).
// ---------------------------------------------------------------------------
template <bool kRot>
__device__ __forceinline__ void spmv_slices(const bdem_system_t &S, const double *x, double *y,
                                            double boost, double (*part2)[kSpmvWarps][6][32],
                                            double &acc_xy, double &acc_yy, double &acc_xx) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ns = (int)((S.n_elem + 31) >> 5);
  const int s_begin = blockIdx.x, s_end = ns, step = gridDim.x;
  int buf = 0;
#pragma unroll 1
  for (int sl = s_begin; sl < s_end; sl += step, buf ^= 1) {
    // partial products alternate between two buffers, so one barrier per
    // slice suffices: a warp may start the next slice while others still
    // read this slice's partials in the tail
    double (*part)[6][32] = part2[buf];
    const SliceBounds cb = slice_bounds(S, sl, ns);
    const int s_row = __ldg(S.row_slot + (int64_t)sl * 32 + lane);
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#if BDEM_SPMV_PF
    // this slice's diagonal rows (read after the barrier) into L2 now
    if (s_row >= 0) {
#pragma unroll
      for (int t = 0; t < 12 / kSpmvWarps; ++t)
        if (kRot || w + kSpmvWarps * t < 6)   // rotation-free: only the position block P
          prefetch_l2(S.diag + (int64_t)(w + kSpmvWarps * t) * S.vstride + s_row);
    }
#endif
    // software pipeline on the (cheap, integer) slot indices: the next slot's
    // index loads are in flight while this slot's coefficients arrive
    const int kt = cb.ki + cb.kj;
    SlotRef cur = slot_ref(S, cb.i0, cb.ki, cb.j0, cb.kj, lane, w);
#pragma unroll 1
    for (int k = w; k < kt; k += kSpmvWarps) {
      const SlotRef nxt = slot_ref(S, cb.i0, cb.ki, cb.j0, cb.kj, lane, k + kSpmvWarps);
      slot_apply<kRot>(S, x, cur, acc);
      cur = nxt;
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) part[w][q][lane] = acc[q];
    __syncthreads();
    spmv_tail<kSpmvWarps, kRot>(S, x, y, sl, w, lane, part, boost, acc_xy, acc_yy, acc_xx,
                                s_row);
  }
}

// Rotation-free PCG (bdem_pcg_set_rot_skip): when the rotation half of the
// right-hand side is identically zero (pcg_init found no non-zero entry,
// e.g. identity orientations with no rotational load: every shear and
// bend/twist gradient vanishes exactly), the rotation halves of r, z, p, x
// and Ap stay exactly zero through the whole solve (the reduced matrix has
// no position/rotation coupling), so every PCG kernel skips them.  Each
// skipped term is an exact zero, so iterates and scalars are bit-identical
// to the full solve (up to the sign of zeros).
__device__ __forceinline__ bool pcg_rot_active(const double *pcg) {
  return pcg[BDEM_PCG_ROTZERO] == 0.0;
}

__global__ void __launch_bounds__(kSpmvThreads, BDEM_SPMV_MINB) k_spmv(bdem_system_t S, const double *x, double *y,
                                                       int mode) {
  __shared__ double part[2][kSpmvWarps][6][32];
  __shared__ double sh[kSpmvThreads / 32];
#if BDEM_TIMELINE
  const unsigned long long t_arrive = tl_now();
#endif
  griddep_wait();
  double *pcg = S.pcg;
  if (mode == 1 && pcg[BDEM_PCG_STATE] != PCG_RUNNING) return;
#if BDEM_TIMELINE
  const int tl_it = (int)pcg[BDEM_PCG_K];
  if (mode == 1 && threadIdx.x == 0) {
    atomicMin(&g_tl[(0 * 1024 + (tl_it & 1023)) * 3 + 0], t_arrive);
    TL_RELEASE(0, tl_it)
  }
#endif
  const double boost = mode == 1 ? pcg[BDEM_PCG_BOOST] : 0.0;
  double acc_xy = 0.0, acc_yy = 0.0, acc_xx = 0.0;
  if (mode == 0 || pcg_rot_active(pcg))
    spmv_slices<true>(S, x, y, boost, part, acc_xy, acc_yy, acc_xx);
  else
    spmv_slices<false>(S, x, y, boost, part, acc_xy, acc_yy, acc_xx);
  if (mode == 0) return;
  spmv_pcg_epilogue<kSpmvThreads>(S, boost, acc_xy, acc_yy, acc_xx, sh);
  TL_EXIT(0, tl_it)
}

// x += alpha p; r -= alpha Ap; z = M^-1 r; r.r, r.z (linalg.py:79-89)
#ifndef BDEM_UPD_MINB
#define BDEM_UPD_MINB 4
#endif
__global__ void __launch_bounds__(kThreads, BDEM_UPD_MINB) k_pcg_update(bdem_system_t S, double *x, double *r,
                                                         double *zv, const double *p,
                                                         const double *ap) {
  __shared__ double sh[kThreads / 32];
#if BDEM_TIMELINE
  const unsigned long long t_arrive = tl_now();
#endif
  griddep_wait();
  double *pcg = S.pcg;
  if (pcg[BDEM_PCG_STATE] != PCG_RUNNING) return;
#if BDEM_TIMELINE
  const int tl_it = (int)pcg[BDEM_PCG_K];
  if (threadIdx.x == 0) {
    atomicMin(&g_tl[(1 * 1024 + (tl_it & 1023)) * 3 + 0], t_arrive);
    TL_RELEASE(1, tl_it)
  }
#endif
  const double alpha = pcg[BDEM_PCG_ALPHA];
  const int halves = pcg_rot_active(pcg) ? 2 : 1;
  double acc_rr = 0.0, acc_rz = 0.0;
  // two consecutive slots per thread with 16-byte loads (planes are 256-B
  // aligned, stride vstride); padding slots carry zeros and stay zero
  const int64_t nf = S.vstride;
  const double2 *p2 = reinterpret_cast<const double2 *>(p);
  const double2 *ap2 = reinterpret_cast<const double2 *>(ap);
  double2 *x2 = reinterpret_cast<double2 *>(x);
  double2 *r2 = reinterpret_cast<double2 *>(r);
  double2 *z2 = reinterpret_cast<double2 *>(zv);
  const double2 *mi2 = reinterpret_cast<const double2 *>(S.minv);
  const int64_t h2 = nf >> 1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < h2;
       t += (int64_t)gridDim.x * blockDim.x) {
    // position half (components 0..2, P^-1) then rotation half (3..5, R^-1)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h >= halves) break;
      double ra[3], rb[3], ma[6], mb[6], za[3], zb[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int64_t k = (3 * h + c) * h2 + t;
        // x, r, Ap and M^-1 are next touched an SpMV later (0.5 GB of
        // coefficients streamed in between): evict-first loads / stores keep
        // them from displacing the SpMV's L2 working set
        const double2 xv = __ldcs(x2 + k), rv = __ldcs(r2 + k), pv = p2[k], av = __ldcs(ap2 + k);
        __stcs(x2 + k, make_double2(xv.x + alpha * pv.x, xv.y + alpha * pv.y));
        ra[c] = rv.x - alpha * av.x;
        rb[c] = rv.y - alpha * av.y;
        __stcs(r2 + k, make_double2(ra[c], rb[c]));
      }
#pragma unroll
      for (int tt = 0; tt < 6; ++tt) {
        const double2 m = __ldcs(mi2 + (6 * h + tt) * h2 + t);
        ma[tt] = m.x;
        mb[tt] = m.y;
      }
      symv3(ma, ra, za);
      symv3(mb, rb, zb);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        z2[(3 * h + c) * h2 + t] = make_double2(za[c], zb[c]);
        acc_rr += ra[c] * ra[c];
        acc_rz += ra[c] * za[c];
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        acc_rr += rb[c] * rb[c];
        acc_rz += rb[c] * zb[c];
      }
    }
  }
  __shared__ double sh2[2 * (kThreads / 32)];
  double v2[2] = {acc_rr, acc_rz};
  block_sum_k<kThreads, 2>(v2, sh2);
  if (threadIdx.x == 0) {
    *red_slot(S.red, RC_RR, blockIdx.x) = v2[0];
    *red_slot(S.red, RC_RZ, blockIdx.x) = v2[1];
  }
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
  TL_EXIT(1, tl_it)
}

// p = z + beta p (linalg.py:91)
__global__ void __launch_bounds__(kThreads) k_pcg_pupdate(bdem_system_t S, double *p,
                                                          const double *zv) {
#if BDEM_TIMELINE
  const unsigned long long t_arrive = tl_now();
#endif
  griddep_wait();
  const double *pcg = S.pcg;
  if (pcg[BDEM_PCG_STATE] != PCG_RUNNING) return;
#if BDEM_TIMELINE
  const int tl_it = (int)pcg[BDEM_PCG_K];
  if (threadIdx.x == 0) {
    atomicMin(&g_tl[(2 * 1024 + (tl_it & 1023)) * 3 + 0], t_arrive);
    TL_RELEASE(2, tl_it)
  }
#endif
  const double beta = pcg[BDEM_PCG_BETA];
  // double2 units over 6 planes (3 with the rotation half inactive)
  const int64_t n6 = pcg_rot_active(pcg) ? 3 * S.vstride : (3 * S.vstride) / 2;
  double2 *p2 = reinterpret_cast<double2 *>(p);
  const double2 *z2 = reinterpret_cast<const double2 *>(zv);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n6;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double2 zz = __ldcs(z2 + k), pp = p2[k];   // last use of z this iteration
    p2[k] = make_double2(zz.x + beta * pp.x, zz.y + beta * pp.y);
  }
  TL_EXIT(2, tl_it)
}

// x = 0, r = sign b, z = M^-1 r, p = z, r.z, |b| (linalg.py:52-68)
__global__ void __launch_bounds__(kThreads) k_pcg_init(bdem_system_t S, const double *b,
                                                       double sign, double *x, double *r,
                                                       double *zv, double *p, double tol,
                                                       double maxit, double boost,
                                                       int rot_skip) {
  __shared__ double sh[kThreads / 32];
  double acc_rr = 0.0, acc_rz = 0.0, acc_nz = 0.0;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S.n_free;
       s += (int64_t)gridDim.x * blockDim.x) {
    double bs[6], zs[6];
    const double zero[6] = {0, 0, 0, 0, 0, 0};
    load6(b, s, S.vstride, bs);
    if (bs[3] != 0.0 || bs[4] != 0.0 || bs[5] != 0.0) acc_nz = 1.0;
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      bs[c] = sign * bs[c];
      acc_rr += bs[c] * bs[c];
    }
    store6(x, s, S.vstride, zero);
    store6(r, s, S.vstride, bs);
    precond_row(S, s, bs, zs);
    store6(zv, s, S.vstride, zs);
    store6(p, s, S.vstride, zs);
#pragma unroll
    for (int c = 0; c < 6; ++c) acc_rz += bs[c] * zs[c];
  }
  double v = block_sum<kThreads>(acc_rr, sh);
  if (threadIdx.x == 0) *red_slot(S.red, RC_IRR, blockIdx.x) = v;
  v = block_sum<kThreads>(acc_rz, sh);
  if (threadIdx.x == 0) *red_slot(S.red, RC_IRZ, blockIdx.x) = v;
  v = block_sum<kThreads>(acc_nz, sh);
  if (threadIdx.x == 0) *red_slot(S.red, RC_IRN, blockIdx.x) = v;
  if (!last_block(S.counter + CNT_INIT)) return;
  const double rr = sum_partials<kThreads>(S.red, RC_IRR, gridDim.x, sh);
  const double rz = sum_partials<kThreads>(S.red, RC_IRZ, gridDim.x, sh);
  const double nz = sum_partials<kThreads>(S.red, RC_IRN, gridDim.x, sh);
  if (threadIdx.x == 0) {
    double *pcg = S.pcg;
    // rotation half active unless the skip is enabled and b's rotation
    // half is identically zero (see pcg_rot_active)
    pcg[BDEM_PCG_ROTZERO] = (rot_skip && nz == 0.0) ? 1.0 : 0.0;
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
  load6(r, s, S.vstride, rs);
  precond_row(S, s, rs, zs);
  store6(zv, s, S.vstride, zs);
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
      atomicAdd(&S.err[BDEM_ERRSLOT_COINCIDENT_CONTACT], 1);   // host logs contact.py:202's warning
    } else {
      const double l = fmax(len, 1e-300);
#pragma unroll
      for (int c = 0; c < 3; ++c) n[c] = div_nz(d[c], l);
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

// launch with programmatic stream serialisation (see griddep_wait)
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
static bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char *env = getenv("BDEM_PDL");
    on = env ? atoi(env) != 0 : 1;
  }
  return on != 0;
}

// resident-grid size of k_spmv (one wave), capped by the partial-sum slots
static unsigned int spmv_grid() {
  static unsigned int g = 0;
  if (g == 0) {
    int dev = 0, sms = 148, per_sm = 4;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv, kSpmvThreads, 0);
    long long want = (long long)sms * (per_sm > 0 ? per_sm : 1);
    g = (unsigned int)(want < kRedBlocks ? want : kRedBlocks);
  }
  return g;
}

static int g_rot_skip = -1;
static int rot_skip_on() {
  if (g_rot_skip < 0) {
    const char *env = getenv("BDEM_ROT_SKIP");
    g_rot_skip = env ? (atoi(env) != 0) : 0;
  }
  return g_rot_skip;
}

// Problem-sized grids.  Every PCG kernel strides its grid over work items
// (slices, slot pairs, rows) and sums per-block partials over gridDim.x.
// When a system has fewer items than the full grid has threads (slices) --
// small and mid-size systems -- each busy thread (CTA) already handles a
// single item, and the surplus blocks only add +0.0 partials; launching
// just the busy blocks gives the same partials in the same order
// (bit-identical scalars) without the idle CTAs' launch, barrier and
// last-block costs.
static unsigned int fit_grid(int64_t items, int64_t per_block, unsigned int cap) {
  const int64_t g = (items + per_block - 1) / per_block;
  return g < 1 ? 1u : (g < (int64_t)cap ? (unsigned int)g : cap);
}
static unsigned int spmv_fit(const bdem_system_t &S) {
  return fit_grid((S.n_elem + 31) >> 5, 1, spmv_grid());
}
static unsigned int update_fit(const bdem_system_t &S) {
  return fit_grid(S.vstride >> 1, kThreads, kRedBlocks);    // slot pairs
}
static unsigned int pupdate_fit(const bdem_system_t &S) {
  return fit_grid(3 * S.vstride, kThreads, kRedBlocks);     // double2 units, 6 planes
}

// one SpMV launch (plain or PCG mode)
static void launch_spmv(const bdem_system_t &S, const double *x, double *y, int mode,
                        cudaStream_t st) {
  k_spmv<<<spmv_fit(S), kSpmvThreads, 0, st>>>(S, x, y, mode);
}

}  // namespace bdem

using namespace bdem;

extern "C" {

#if BDEM_TIMELINE
// diagnostic builds: reset / read the PCG kernel timeline (3 x 1024 x 3 u64)
int bdem_timeline_reset(void) {
  static unsigned long long init[3 * 1024 * 3];
  for (int k = 0; k < 3 * 1024; ++k) {
    init[3 * k] = ~0ull;
    init[3 * k + 1] = ~0ull;
    init[3 * k + 2] = 0ull;
  }
  return cudaMemcpyToSymbol(g_tl, init, sizeof(init)) == cudaSuccess ? 0 : 1;
}
int bdem_timeline_read(unsigned long long *out) {
  return cudaMemcpyFromSymbol(out, g_tl, sizeof(unsigned long long) * 3 * 1024 * 3) ==
                 cudaSuccess ? 0 : 1;
}
#endif
int bdem_pcg_set_rot_skip(int on) {
  const int prev = rot_skip_on();
  if (on == 0 || on == 1) g_rot_skip = on;
  return prev;
}

int bdem_spmv(const bdem_system_t *sys, const double *x, double *y, void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  launch_spmv(*sys, x, y, 0, as_stream(stream));
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
  k_pcg_init<<<fit_grid(sys->n_free, kThreads, kRedBlocks), kThreads, 0, as_stream(stream)>>>(
      *sys, b, sign, x, r, zv, pv, tol, (double)max_iter, boost, rot_skip_on());
  return launch_status();
}

int bdem_pcg_iterate(const bdem_system_t *sys, double *x, double *r, double *zv, double *pv,
                     double *ap, int n_iter, void *stream) {
  if (!sys || n_iter < 0) return BDEM_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  // programmatic dependent launch chain SpMV -> update -> p update
  auto spmv_k = k_spmv;
  const bool pdl = pdl_enabled();
  for (int it = 0; it < n_iter; ++it) {
    if (pdl) {
      launch_pdl(spmv_k, spmv_fit(*sys), kSpmvThreads, st, *sys, (const double *)pv, ap, 1);
      launch_pdl(k_pcg_update, update_fit(*sys), kThreads, st, *sys, x, r, zv,
                 (const double *)pv, (const double *)ap);
      launch_pdl(k_pcg_pupdate, pupdate_fit(*sys), kThreads, st, *sys, pv, (const double *)zv);
    } else {
      launch_spmv(*sys, pv, ap, 1, st);
      k_pcg_update<<<update_fit(*sys), kThreads, 0, st>>>(*sys, x, r, zv, pv, ap);
      k_pcg_pupdate<<<pupdate_fit(*sys), kThreads, 0, st>>>(*sys, pv, zv);
    }
  }
  return launch_status(3 * (int64_t)n_iter);
}

int bdem_pcg_spmv(const bdem_system_t *sys, const double *pv, double *ap, void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  launch_spmv(*sys, pv, ap, 1, as_stream(stream));
  return launch_status();
}

int bdem_pcg_update(const bdem_system_t *sys, double *x, double *r, double *zv, double *pv,
                    const double *ap, void *stream) {
  if (!sys) return BDEM_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  k_pcg_update<<<update_fit(*sys), kThreads, 0, st>>>(*sys, x, r, zv, pv, ap);
  k_pcg_pupdate<<<pupdate_fit(*sys), kThreads, 0, st>>>(*sys, pv, zv);
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
