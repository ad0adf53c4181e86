/*
 * bdem_sm100.h -- C ABI of the B200-native Newton hot path of the bonded
 * discrete element method with quaternion manifold optimisation
 * (arXiv 2308.10459).  Library: paper_2308_10459_b200/lib/libbdem_sm100.so
 * (sm_100a, FP64, hand-written CUDA; no torch types cross this boundary).
 *
 * The reference (pure Python package `bdem`, /root/reference/pkg/src/bdem)
 * has no FFI; its seams are duck-typed Python callables.  Each entry point
 * below names the reference function it replaces (file:line).  The Python
 * host (paper_2308_10459_b200/_lib.py) binds these with ctypes.
 *
 * Conventions
 *  - All pointers inside bdem_system_t and all pointer arguments are DEVICE
 *    pointers owned by the caller; the library never allocates on hot calls.
 *  - `stream` is a cudaStream_t passed as void*.  Calls are asynchronous.
 *  - Return value: BDEM_OK or BDEM_ERR_* (launch/argument errors).  Data
 *    errors (degenerate bonds, antipodal pairs) are reported through the
 *    device int array `sys->err` (see BDEM_ERRSLOT_*), read back by the host
 *    together with the scalar results it synchronises on anyway.
 *  - Layouts: p (n,3), q (n,4) scalar-last row-major like the reference;
 *    per-bond data in structure-of-arrays planes of length n_bond, indexed
 *    by SELL-32 position (see bdem_system_t); per-free-element blocks in
 *    planes of stride vstride.  Reduced vectors (z, y, PCG x/r/z/p/Ap) are
 *    6 planes [pos x,y,z, rot x,y,z] of stride vstride: component c of free
 *    slot s is v[c * vstride + s].
 */
#ifndef BDEM_SM100_H
#define BDEM_SM100_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BDEM_ABI_VERSION 7

enum {
  BDEM_OK = 0,
  BDEM_ERR_DEGENERATE_BOND = 1, /* bonds.py:165-168 DegenerateBondError   */
  BDEM_ERR_ANTIPODAL = 2,       /* bonds.py:223-227 DegenerateShearError  */
  BDEM_ERR_NONFINITE = 3,
  BDEM_ERR_ARG = 4,
  BDEM_ERR_CUDA = 5,
  BDEM_ERR_CAPACITY = 6         /* output larger than the given capacity */
};

/* device error words (int32) in sys->err */
enum {
  BDEM_ERRSLOT_DEGENERATE_COUNT = 0,
  BDEM_ERRSLOT_DEGENERATE_FIRST = 1, /* smallest offending bond index */
  BDEM_ERRSLOT_ANTIPODAL_COUNT = 2,
  BDEM_ERRSLOT_ANTIPODAL_FIRST = 3,
  BDEM_ERRSLOT_COINCIDENT_CONTACT = 4, /* not an error: contact pairs with coincident
                                          centres took the +x fallback normal
                                          (contact.py:200-203); the host logs the
                                          reference's warning */
  BDEM_ERRSLOT_COUNT = 8
};

/* bond geometry planes (each n_bond doubles) -- BondSet fields bonds.py:418-447 */
enum {
  BDEM_BG_L0 = 0,     /* rest_length                              */
  BDEM_BG_D0 = 1,     /* d0[3]                                    */
  BDEM_BG_FRAME = 4,  /* frame[3][3] row-major (world->local)     */
  BDEM_BG_KN = 13,    /* kn                                       */
  BDEM_BG_KT = 14,    /* kt                                       */
  BDEM_BG_KDIAG = 15, /* k_diag[3] (twist, bend, bend)            */
  BDEM_BG_RADIUS = 18,
  BDEM_BG_SECTION = 19,
  BDEM_BG_SECOND = 20,
  BDEM_BG_POLAR = 21,
  BDEM_BG_TENSILE = 22,
  BDEM_BG_SHEAR = 23,
  BDEM_BG_COUNT = 24
};

/* mutable bond state planes (each n_bond doubles) -- bonds.py:443-448 */
enum {
  BDEM_BS_SCALE = 0, /* stiffness_scale */
  BDEM_BS_DAMAGE = 1,
  BDEM_BS_PLASTIC = 2, /* plastic_strain */
  BDEM_BS_SIGMA = 3,
  BDEM_BS_TAU = 4,
  BDEM_BS_COUNT = 5
};

/* per-bond staging written by bdem_bond_assemble (each n_bond doubles): the
 * j-role pieces the element pass gathers for the bond's j end, and the
 * clamped (i,i) rotation quadrant of the positions whose row could not fold
 * it into its i-role partial sum (see BDEM_IP_* / ikpre) */
enum {
  BDEM_ST_KC = 0,    /* k c: dE/dp_j = kc n, dE/dp_i = -kc n          */
  BDEM_ST_GQJ = 1,   /* d E / d q_j [4]                               */
  BDEM_ST_D = 5,     /* clamped (j,j) rotation quadrant (sym 6)        */
  BDEM_ST_A = 11,    /* clamped (i,i) rotation quadrant (sym 6), only
                        for slots >= ikpre[row] of its row            */
  BDEM_ST_COUNT = 17
};

/* i-role partial sums of one SELL row, written by bdem_bond_assemble (each
 * plane n_rows = 32 * n_slices doubles, indexed by row): the row thread of
 * the bond pass walks its i-role slots in ascending bond id and adds each
 * bond's pieces in np.add.at order (integrator.py:100-103); the element pass
 * continues these sums with the j-role pieces.  The rotation quadrant of a
 * slot is folded into BDEM_IP_R only while every earlier slot of the row had
 * a PSD-certified block: ikpre[row] is the first slot whose (possibly
 * eigen-clamped) quadrant is staged in BDEM_ST_A instead (-1: none). */
enum {
  BDEM_IP_GP = 0,    /* sum of -kc n (position gradient) [3]          */
  BDEM_IP_GQ = 3,    /* sum of dE/dq_i [4]                            */
  BDEM_IP_P = 7,     /* sum of clamped stretch blocks a+ (sym 6)      */
  BDEM_IP_R = 13,    /* sum of (i,i) rotation quadrants (sym 6)       */
  BDEM_IP_E = 19,    /* sum of bond energies                          */
  BDEM_IP_COUNT = 20
};

/* sys->asm_flags */
enum {
  BDEM_ASM_STAGE_ALL_A = 1 /* stage every (i,i) quadrant (ikpre = 0): tests */
};

/* Off-diagonal coupling coefficients of a bond, read by the SpMV: stored
 * AoSoA-32 in sys->scoef -- the 14 coefficients of the 32 positions of a
 * slot form one contiguous 3.5 KB record at (pos & ~31) * BDEM_CF_COUNT;
 * inside it coefficient k of lane l = pos & 31 sits at 64 (k >> 1) + 2 l +
 * (k & 1), i.e. coefficient pairs interleaved per lane: a lane reads its 14
 * values as 7 aligned 16-byte loads and a warp's load of one pair is a
 * contiguous 512-byte segment. */
enum {
  BDEM_CF_N = 0,     /* unit bond direction n [3]                     */
  BDEM_CF_ALPHA = 3, /* clamped stretch block a+ = alpha n n^T + beta I */
  BDEM_CF_BETA = 4,  /*   (off-diagonal coupling -a+)                 */
  BDEM_CF_C = 5,     /* clamped reduced rotation block (i,j) quadrant, 3x3 row-major */
  BDEM_CF_COUNT = 14
};

/* per-pair staging (each pair_cap doubles) */
enum { BDEM_PS_E = 0, BDEM_PS_GI = 1, BDEM_PS_A = 4, BDEM_PS_COUNT = 10 };

enum { BDEM_COLLIDER_HALFSPACE = 0, BDEM_COLLIDER_SPHERE = 1, BDEM_COLLIDER_BOX = 2 };
#define BDEM_MAX_COLLIDERS 8

typedef struct {
  int32_t kind;
  int32_t pad_;
  double a[6]; /* halfspace: n[3], offset; sphere: c[3], r; box: c[3], h[3] */
} bdem_collider_t;

/* reduction scratch: per-block partial sums, then a fixed-order finish */
#define BDEM_RED_BLOCKS 1184 /* 8 x 148 SMs */
enum {
  BDEM_SC_F = 0,        /* objective value                     */
  BDEM_SC_GNORM2 = 1,   /* |z|^2                               */
  BDEM_SC_CNORM2 = 2,   /* |0.5(q.q-1)|^2 over free            */
  BDEM_SC_MAXDEV = 3,   /* max | |q|-1 | over free             */
  BDEM_SC_SLOPE = 4,    /* z . y                               */
  BDEM_SC_FT = 5,       /* trial objective value               */
  BDEM_SC_NSING = 6,    /* singular block-Jacobi blocks        */
  BDEM_SC_EBOND = 7,    /* bond energy                         */
  BDEM_SC_ECOL = 8,     /* collider penalty energy             */
  BDEM_SC_EGRAV = 9,    /* gravity energy -sum m p.g           */
  BDEM_SC_EKIN = 10,    /* kinetic energy                      */
  BDEM_SC_EPAIR = 11,   /* self-contact pair energy            */
  BDEM_SC_COUNT = 32    /* columns 20..26 are PCG partials     */
};

/* PCG device state (doubles), bdem_pcg_* read/write it */
enum {
  BDEM_PCG_RZ = 0,     /* r.z of the current direction           */
  BDEM_PCG_PAP = 1,    /* p.Ap                                    */
  BDEM_PCG_ALPHA = 2,
  BDEM_PCG_BETA = 3,
  BDEM_PCG_RR = 4,     /* |r|^2                                   */
  BDEM_PCG_BNORM = 5,  /* |b|                                     */
  BDEM_PCG_REL = 6,    /* |r|/|b|                                 */
  BDEM_PCG_TOL = 7,
  BDEM_PCG_BOOST = 8,
  BDEM_PCG_APNORM2 = 9, /* |Ap|^2 (breakdown scale)              */
  BDEM_PCG_PNORM2 = 10, /* |p|^2                                  */
  BDEM_PCG_K = 11,      /* iterations of the current run (as double) */
  BDEM_PCG_MAXIT = 12,
  BDEM_PCG_STATE = 13,  /* 0 running, 1 converged, 2 breakdown, 3 max-iterations */
  BDEM_PCG_ROTZERO = 14, /* 1: rotation half of the system identically zero (skipped) */
  BDEM_PCG_COUNT = 16
};

typedef struct {
  /* sizes */
  int64_t n_elem, n_free, n_bond, n_pair, pair_cap;
  int64_t vstride;               /* plane stride of reduced vectors and diag/minv:
                                    n_free rounded up to 32 (256-B aligned planes) */
  int64_t sell_kmax;             /* max i-role slots of any slice               */
  int64_t sell_kjmax;            /* max j-role slots of any slice               */
  /* element data (device) */
  const double *mass, *radius;
  const double *mp_dt2, *mq_dt2; /* m/dt^2, 1.6 m r^2/dt^2; 0 when pinned */
  const double *p_hat, *q_hat;   /* inertial anchors 2x_curr - x_prev   */
  const int32_t *slot;           /* (n_elem) free slot or -1            */
  const int32_t *free_elem;      /* (n_free) element id of each slot    */
  /* bond topology / geometry / state */
  const int32_t *bond_i, *bond_j;
  int8_t *status;                /* INTACT 0, WEAKENED 1, BROKEN 2      */
  const double *geom;            /* BDEM_BG_COUNT planes                */
  double *bstate;                /* BDEM_BS_COUNT planes                */
  /* SELL-32 bond layout.  Every per-bond plane (geometry, state, staging,
   * bond_i/j, status) is indexed by POSITION, not by the caller's bond id.
   * Elements are placed in SELL rows (row_elem / elem_row: a spatially
   * compact Z-order of the initial positions) and rows are cut into slices
   * of 32; slice s owns the positions [slice_base[s], slice_base[s+1]),
   * laid out slot-major (pos = slice_base[s] + 32 k + (row & 31)), slot k =
   * the k-th bond with i == e in ascending bond id (np.add.at order,
   * integrator.py:100-103).  Free slots (reduced-vector indices) are
   * numbered in row order, so the rows of a slice own the consecutive slots
   * [slice_slot[s], slice_slot[s+1]).
   * Padding positions have status BROKEN.  n_bond is the padded length.
   * The j-role lists use the same shape: jpos[jslice_base[s] + 32 k + lane]
   * is the position of the k-th bond with j == e (ascending id), -1 pad. */
  const int32_t *slice_base;     /* (n_slices + 1)                      */
  const int32_t *pos_oslot;      /* (n_bond) free slot of the j end, -1 */
  const int32_t *jslice_base;    /* (n_slices + 1)                      */
  const int32_t *jpos;           /* position of a j-role bond, -1 pad   */
  const int32_t *jslot;          /* free slot of its i end, -1          */
  const int32_t *row_elem;       /* (n_slices * 32) element of a row, -1 pad */
  const int32_t *elem_row;       /* (n_elem) row of an element          */
  const int32_t *slice_slot;     /* (n_slices + 1) first free slot of a slice */
  const int32_t *row_slot;       /* (n_slices * 32) free slot of a row, -1 pinned/pad */
  /* contact pairs (sorted i<j); pairs with i == e are [pi_ptr[e], pi_ptr[e+1]),
   * pairs with j == e are pj_idx[pj_ptr[e] .. pj_ptr[e+1]) ascending */
  const int32_t *pair_i, *pair_j, *pi_ptr, *pj_ptr, *pj_idx;
  /* staging / workspace */
  double *stage;                 /* BDEM_ST_COUNT planes x n_bond      */
  double *scoef;                 /* BDEM_CF_COUNT x n_bond, AoSoA-32    */
  double *pstage;                /* BDEM_PS_COUNT planes x pair_cap    */
  double *diag;                  /* 12 planes x n_free: P sym6, R sym6  */
  double *minv;                  /* 12 planes x n_free: P^-1, R^-1      */
  double *red;                   /* BDEM_RED_BLOCKS x BDEM_SC_COUNT    */
  double *scalars;               /* BDEM_SC_COUNT                      */
  double *pcg;                   /* BDEM_PCG_COUNT                     */
  int32_t *err;                  /* BDEM_ERRSLOT_COUNT                 */
  unsigned int *counter;         /* last-block counters (zeroed)       */
  int32_t *clamp_list;           /* (n_bond) queue of indefinite rotation blocks */
  double *ipart;                 /* BDEM_IP_COUNT planes x n_rows: i-role partial sums */
  int32_t *ikpre;                /* (n_rows) first slot with a staged (i,i) quadrant, -1 */
  double *grad_p, *grad_q;       /* optional (n,3) / (n,4): bdem_element_assemble writes the
                                    ambient gradient of the incremental potential
                                    (ImplicitProblem.value_and_gradient); NULL = off */
  /* physics */
  double gravity[3];
  double k_contact, k_element;
  int32_t n_colliders;
  int32_t asm_flags;             /* BDEM_ASM_* */
  bdem_collider_t colliders[BDEM_MAX_COLLIDERS];
} bdem_system_t;

/* ---- library ----------------------------------------------------------- */
int bdem_abi_version(void);
int64_t bdem_system_size(void); /* sizeof(bdem_system_t), for binding checks */
int64_t bdem_launch_count(void); /* kernels launched by this library so far */
int bdem_device_sm(void); /* compute capability of device 0, e.g. 100 */

/* ---- bonds ------------------------------------------------------------- */

/* Debug ambient evaluation of the listed bonds: energy, ambient gradients and
 * the 6x6 position / 8x8 quaternion Hessians.
 * Replaces BondSet.energy_terms (bonds.py:473-504) = stretch_terms
 * (bonds.py:151-188) + shear_terms (bonds.py:205-264) + bendtwist_terms
 * (bonds.py:282-323).  Outputs are (n_idx, ...) row-major. */
int bdem_bond_eval_ambient(const bdem_system_t *sys, const double *p, const double *q,
                           int64_t n_idx, const int32_t *idx, double *E, double *gpi,
                           double *gpj, double *gqi, double *gqj, double *hpp, double *hqq,
                           int want_hess, void *stream);

/* Fused production bond pass at (p, q): energy, gradient contributions and
 * the SPD-clamped reduced Hessian blocks.  One thread per SELL row walks the
 * row's i-role bonds: coupling coefficients to sys->scoef, the j-role pieces
 * to sys->stage, the i-role pieces summed in order into sys->ipart.
 * Replaces energy_terms(want_hess=True) + spd_project of the position and the
 * G_l-reduced rotation blocks inside build_clamped_pieces (solver.py:141-162). */
int bdem_bond_assemble(const bdem_system_t *sys, const double *p, const double *q,
                       void *stream);

/* Energy-only bond pass (PotentialModel.value bond part, integrator.py:87-89);
 * accumulates into reduction column `col` of sys->red (per-block partials). */
int bdem_bond_energy(const bdem_system_t *sys, const double *p, const double *q, int col,
                     void *stream);

/* Fracture / plasticity update at (p, q): sigma, tau, von Mises yield,
 * weakening, damage, strain and strength breakage; flags[b] = 1 for bonds
 * broken by this call.  Replaces update_bond_states + BondSet.stresses +
 * axial_strain (bonds.py:506-570).  plastic = NULL disables plasticity;
 * otherwise plastic[4] = {fracture_strain, yield_strain, weakening, damage_exponent}
 * (host memory). */
int bdem_bond_update(const bdem_system_t *sys, const double *p, const double *q,
                     double youngs, const double *plastic, uint8_t *flags, void *stream);

/* ---- contact pairs and colliders --------------------------------------- */

/* self_repulsion_terms for the sys->n_pair frozen pairs (contact.py:180-224);
 * clamped pair blocks (spd_project, solver.py:162) into sys->pstage. */
int bdem_pair_assemble(const bdem_system_t *sys, const double *p, int energy_only,
                       void *stream);

/* Ambient contact Hessian blocks at p (PotentialModel.hessian_blocks,
 * integrator.py:111-129): pair_pp (n_pair, 6, 6) = [[a, -a], [-a, a]] with
 * a = k_element (nn - (depth / l)(I - nn)) for touching pairs, else 0
 * (self_repulsion_terms, contact.py:180-224); elem_pp (n_elem, 3, 3) = the
 * sum over colliders of k_contact (grad g grad g^T + g hess g) for
 * penetrating centers (external_repulsion_terms, contact.py:227-248).
 * Row-major; either output may be NULL. */
int bdem_contact_blocks(const bdem_system_t *sys, const double *p, double *pair_pp,
                        double *elem_pp, void *stream);

/* ---- elements ---------------------------------------------------------- */

/* Ordered per-element gradient gather (np.add.at order, integrator.py:95-109),
 * inertia (integrator.py:195-200), colliders (contact.py:227-248), reduced
 * gradient z (solver.py:116-123), diagonal blocks + element terms
 * (solver.py:164-173, 198-248), block-Jacobi inverses (linalg.py:100-128) and
 * the objective / |z| / constraint reductions.  Continues the i-role partial
 * sums of the bdem_bond_assemble call at the same (p, q) (sys->ipart,
 * sys->ikpre) with the j-role pieces it staged: call bdem_bond_assemble (and,
 * with contact pairs, bdem_pair_assemble) first. */
int bdem_element_assemble(const bdem_system_t *sys, const double *p, const double *q,
                          double *z, void *stream);

/* Finish reductions: sums the per-block partials of columns [0, ncol) of
 * sys->red (fixed order) into sys->scalars[col] (max for BDEM_SC_MAXDEV). */
int bdem_reduce_finish(const bdem_system_t *sys, int col0, int ncol, int nblocks,
                       void *stream);

/* Line-search trial point and element part of the objective:
 * p_t = p + alpha dp, q_t = normalize(geodesic(q, alpha dq)) on free rows
 * (solver.py:399-401, quat.py:144-164), then inertia + colliders - gravity
 * partials.  Bond and pair energies are added by bdem_bond_energy /
 * bdem_pair_assemble(energy_only=1). */
int bdem_trial_point(const bdem_system_t *sys, const double *p, const double *q,
                     const double *dp, const double *dq, double alpha, double *p_t,
                     double *q_t, void *stream);

/* Element part of the objective at (p, q) without moving (value()). */
int bdem_element_energy(const bdem_system_t *sys, const double *p, const double *q,
                        int with_inertia, void *stream);

/* Kinetic energy partials (ElementSet.kinetic_energy, elements.py:114-117). */
int bdem_kinetic(const bdem_system_t *sys, const double *v, const double *qdot, void *stream);

/* q[free] = q[free] / |q[free]| (solver.py:516). */
int bdem_normalize_free(const bdem_system_t *sys, double *q, void *stream);

/* Newton direction from the reduced solution: dp = y_pos, dq = G_l(q)^T y_rot
 * (solver.py:409-418); sign = -1 builds the gradient fallback from z. */
int bdem_direction(const bdem_system_t *sys, const double *q, const double *y, double sign,
                   double *dp, double *dq, void *stream);

/* slope = z . y into sys->scalars[BDEM_SC_SLOPE] (solver.py:542). */
int bdem_dot(const bdem_system_t *sys, const double *a, const double *b, int64_t n,
             int sc_col, void *stream);

/* Predictor (integrator.py:268-274) and anchors (integrator.py:153-161,172-174):
 * p_hat = 2p - p_prev, q_hat = 2q - q_prev, p0 = p + dt v, q0 = normalize(
 * geodesic(q, dt qdot)) on free rows, normalize all rows. */
int bdem_predict(const bdem_system_t *sys, const double *p, const double *q,
                 const double *v, const double *qdot, const double *p_prev,
                 const double *q_prev, double dt, double *p_hat, double *q_hat,
                 double *mp_dt2, double *mq_dt2, double *p0, double *q0, void *stream);

/* Velocity update (integrator.py:289-293): v = (p - p_c)/dt,
 * qdot = tangent_project(q, (q - q_c)/dt) on free rows. */
int bdem_finish_step(const bdem_system_t *sys, const double *p, const double *q,
                     const double *p_c, const double *q_c, double dt, double *v,
                     double *qdot, void *stream);

/* ---- reduced linear system --------------------------------------------- */

/* y = A x (+ boost x) with A the reduced Newton matrix held as per-bond
 * clamped blocks + per-element diagonal blocks (assemble_reduced_system,
 * solver.py:198-258, applied as `mat @ v`, solver.py:475).  Also writes the
 * per-block partials of x.y, |y|^2, |x|^2 for PCG. */
int bdem_spmv(const bdem_system_t *sys, const double *x, double *y, void *stream);
/* Rotation-free PCG: when on and the rotation half of the right-hand side
 * is identically zero at bdem_pcg_init (e.g. identity orientations with no
 * rotational load, as on the BASELINE plate), the rotation halves of every
 * PCG vector stay exactly zero (the reduced matrix has no position/rotation
 * coupling), and the SpMV / update kernels skip them: 5 of the 14 SpMV
 * coefficients and 3 of 6 vector components per row.  Bit-identical iterates
 * (up to the sign of zeros).  Default off; BDEM_ROT_SKIP=1 selects it at load
 * time.  Returns the previous setting; any other value only queries. */
int bdem_pcg_set_rot_skip(int on);
/* PCG (linalg.py:40-97) on device state sys->pcg; see pcg_kernels.cu. */
int bdem_pcg_init(const bdem_system_t *sys, const double *b, double sign, double *x,
                  double *r, double *zv, double *pv, double tol, int max_iter, double boost,
                  void *stream);
int bdem_pcg_iterate(const bdem_system_t *sys, double *x, double *r, double *zv, double *pv,
                     double *ap, int n_iter, void *stream);

/* The two halves of one PCG iteration, for callers that time the SpMV
 * separately: Ap = A p (+ boost p) with p.Ap and the breakdown test, then
 * x/r/z updates, r.r, r.z, convergence test and p = z + beta p. */
int bdem_pcg_spmv(const bdem_system_t *sys, const double *pv, double *ap, void *stream);
int bdem_pcg_update(const bdem_system_t *sys, double *x, double *r, double *zv, double *pv,
                    const double *ap, void *stream);

/* Block-Jacobi apply z = M^-1 r (linalg.py:124-126). */
int bdem_precond_apply(const bdem_system_t *sys, const double *r, double *zv, void *stream);

/* ---- broad phase / components ------------------------------------------ */

/* Hash-grid broad phase (contact.py:140-173): sorted unique pairs i<j with
 * |p_j - p_i| < r_i + r_j among points in the 27-cell neighbourhood of cell
 * size `cell`; when labels != NULL only pairs with labels[i] != labels[j]
 * are kept (contact_candidates, solver.py:876-878).
 * Two-phase: call with pairs == NULL to get the count in *n_out (host),
 * then with a buffer of that capacity.  `work` must hold
 * bdem_broadphase_workspace(n) bytes. */
int64_t bdem_broadphase_workspace(int64_t n);
int bdem_broadphase(const double *p, const double *radii, int64_t n, double cell,
                    const int64_t *labels, void *work, int32_t *pairs, int64_t cap,
                    int64_t *n_out, void *stream);

/* The step's frozen self-contact candidates, straight into the system
 * (contact_candidates, solver.py:856-878): radii inflated by dt |v| +
 * dt^2 |g| (dt2g = dt^2 |g| from the host) written to `radii` (n doubles),
 * cell = 2 max(inflated) + 1e-12 formed on the device, the broad phase
 * restricted to labels[i] != labels[j], pairs written to sys->pair_i/pair_j
 * (ascending) and their element adjacency (pi_ptr, pj_ptr, pj_idx).  Sets
 * sys->n_pair and *n_out (host); returns BDEM_ERR_CAPACITY with the needed
 * count in *n_out when it exceeds sys->pair_cap.  Synchronises `stream`
 * twice (grid bounds, pair count).  bp_work: bdem_broadphase_workspace(n);
 * adj_work: bdem_pair_adjacency_workspace(n, pair_cap) bytes. */
int bdem_contact_pairs(bdem_system_t *sys, const double *p, const double *v, double dt,
                       double dt2g, const int64_t *labels, void *bp_work, void *adj_work,
                       double *radii, int64_t *n_out, void *stream);
int64_t bdem_pair_adjacency_workspace(int64_t n, int64_t cap);
/* Install caller-given pairs ((m,2) int32 device array, sorted i<j) and
 * their element adjacency; sets sys->n_pair. */
int bdem_set_pairs(bdem_system_t *sys, const int32_t *pairs, int64_t m, void *work,
                   void *stream);

/* (sigma, tau) of the m flagged bond positions pos[] into out (m x 2): the
 * event records (bond, sigma, tau) of update_bond_states (bonds.py:564-570),
 * pre-update stresses as cached by bdem_bond_update. */
int bdem_event_records(const bdem_system_t *sys, const int32_t *pos, int64_t m, double *out,
                       void *stream);

/* Element rows <-> a packed buffer (m x 14 doubles: p, q, v, qdot) for the
 * listed ids: to_buf=1 gathers (pinned-state backup, solver.py:894-896),
 * to_buf=0 scatters (restore, :910-916; driver rows at t + dt, :898-900). */
int bdem_rows_copy(const int32_t *ids, int64_t m, double *p, double *q, double *v,
                   double *qdot, double *buf, int to_buf, void *stream);
/* Zero the device error words (first-index slots to INT32_MAX). */
int bdem_reset_errors(const bdem_system_t *sys, void *stream);

/* Connected components over non-broken bonds with labels numbered in order of
 * each component's smallest element (label_components, geometry.py:295-310).
 * `work` holds bdem_components_workspace(n) bytes; labels is (n) int64. */
int64_t bdem_components_workspace(int64_t n);
int bdem_components(int64_t n, int64_t n_bond, const int32_t *bi, const int32_t *bj,
                    const int8_t *status, void *work, int64_t *labels, int64_t *n_comp,
                    void *stream);

/* Ascending indices of nonzero flags (the ordered fracture-event list,
 * bonds.py:564-569); *n_out is written to host memory. */
int64_t bdem_select_workspace(int64_t n);
int bdem_select_flagged(const uint8_t *flags, int64_t n, int32_t *out_idx, void *work,
                        int64_t *n_out, void *stream);

/* ---- post-step friction (contact.py:267-350; solver.py:923-925) ---------
 * Replaces apply_friction(elements, pairs, colliders, k_c, k_ec, mu_s, mu_r,
 * dt) (contact.py:303).  Pairs are sys->pair_i/pair_j (the step's frozen
 * candidates, ascending); v (n,3) and qdot (n,4) are corrected in place at
 * the post-step positions p / orientations q.  The sequential pair sweep is
 * executed as dependency waves (bdem_friction_schedule), which reproduces the
 * reference's order of corrections for every element.  `work` holds
 * bdem_friction_workspace(n_elem, pair_cap) bytes; *n_waves (optional) gets
 * the number of waves.  Synchronises `stream` once when pairs are in contact.
 * A no-op when mu_s == mu_r == 0, like the reference. */
int64_t bdem_friction_workspace(int64_t n_elem, int64_t n_pair);
int bdem_friction(const bdem_system_t *sys, const double *p, const double *q, double *v,
                  double *qdot, double mu_s, double mu_r, double dt, void *work,
                  int64_t *n_waves, void *stream);
/* ---- surface reconstruction (reconstruct_surface, geometry.py:313-343) ---
 * Replaces reconstruct_surface(mesh, bonds, labeling, p, q).  Per element:
 * tet_rel (n,4,3) rest tet vertices minus the centroid, bmask (n) bit mask of
 * boundary faces; per bond position: face_i / face_j local face (-1 none).
 * labels (n) fragment ids.  Writes faces ordered by (fragment, element,
 * local face): verts (F,3,3) transported vertices, face_comp (F) fragment.
 * *n_faces = F; when F > cap_faces nothing is written (call again with room).
 * `work` holds bdem_surface_workspace(n_elem) bytes.  Synchronises once. */
int64_t bdem_surface_workspace(int64_t n_elem);
int bdem_surface(const bdem_system_t *sys, const double *p, const double *q,
                 const double *tet_rel, const int32_t *bmask, const int8_t *face_i,
                 const int8_t *face_j, const int64_t *labels, void *work, double *verts,
                 int32_t *face_comp, int64_t cap_faces, int64_t *n_faces, void *stream);

/* Host-only scheduler: pairs (m,2) int32 in sweep order -> wave of each pair
 * = 1 + latest wave of an earlier pair sharing an element.  Writes `order`
 * (m pair indices grouped by wave, ascending within a wave) and `wave_ptr`
 * (depth+1 offsets); returns depth >= 0, or -BDEM_ERR_ARG.  No GPU needed. */
int64_t bdem_friction_schedule(const int32_t *ends, int64_t m, int64_t n_elem, int32_t *order,
                               int32_t *wave_ptr);

#ifdef __cplusplus
}
#endif
#endif /* BDEM_SM100_H */
