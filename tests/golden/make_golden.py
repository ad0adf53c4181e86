"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It imports ``bdem`` read-only from ``/root/reference/pkg/src``, feeds it the
seeded synthetic inputs of ``paper_2308_10459_b200.configs`` (the same
generator the GPU path and the oracle use) and stores inputs + reference
outputs as small ``.npz`` fixtures next to this script.  The fixtures pin the
CPU oracle (``tests/test_oracle_golden.py``) and the CUDA path
(``tests/test_gpu_*.py``).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from bdem import bonds as rb            # noqa: E402
from bdem import contact as rc          # noqa: E402
from bdem import elements as re_        # noqa: E402
from bdem import geometry as rg         # noqa: E402
from bdem import integrator as ri       # noqa: E402
from bdem import linalg as rl           # noqa: E402
from bdem import scenes as rs           # noqa: E402
from bdem import solver as rsv          # noqa: E402
from bdem.quat import quat_normalize    # noqa: E402

from paper_2308_10459_b200 import configs as C   # noqa: E402

BOND_FIELDS = ("i", "j", "rest_length", "radius", "d0", "q0", "frame", "kn", "kt", "k_diag",
               "section", "second_moment", "polar_moment", "tensile_strength",
               "shear_strength", "status", "stiffness_scale", "damage", "plastic_strain",
               "sigma", "tau")
ELEM_FIELDS = ("p", "q", "v", "qdot", "mass", "radius", "pinned")


def ref_bonds(b):
    kw = {f: np.array(getattr(b, f), copy=True) for f in BOND_FIELDS}
    kw["face_i"] = np.zeros(b.n, dtype=np.int64)
    kw["face_j"] = np.zeros(b.n, dtype=np.int64)
    return rb.BondSet(**kw)


def ref_elements(el):
    return re_.ElementSet(*(np.array(getattr(el, f), copy=True) for f in ELEM_FIELDS))


def pack(prefix, obj, fields):
    return {f"{prefix}{f}": np.asarray(getattr(obj, f)) for f in fields}


def dummy_mesh():
    v = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    return rg.TetMesh(v, np.array([[0, 1, 2, 3]]))


def ref_scene(spec, driver=None, colliders=None):
    el = ref_elements(spec.elements)
    return rs.Scene(spec.name, dummy_mesh(), el, ref_bonds(spec.bonds),
                    colliders=ref_colliders(spec.colliders) if colliders is None else list(colliders),
                    gravity=np.array(spec.gravity), dt=spec.dt, youngs=spec.youngs,
                    shear_modulus=spec.shear_modulus, density=spec.density,
                    k_contact=spec.k_contact, k_element=spec.k_element,
                    plastic=spec.plastic, driver=driver, mu_s=spec.mu_s, mu_r=spec.mu_r,
                    surface_flags=np.zeros(el.n, dtype=bool))


def ref_colliders(cols):
    return [rc.HalfSpace(tuple(c.normal), c.offset) for c in cols]


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"  wrote {name}: {os.path.getsize(path) / 1024:.1f} KiB")


# ---------------------------------------------------------------------------

def gold_bond_terms():
    """BondSet.energy_terms (bonds.py:473-504) on random and near-rest states."""
    spec = C.cube(n_side=5, r=0.002, seed=11, random_q=True)
    rng = np.random.default_rng(101)
    b = spec.bonds
    nb = b.n
    b.status[rng.choice(nb, 12, replace=False)] = 2
    b.stiffness_scale[:] = rng.uniform(0.4, 1.0, nb)
    out = pack("b_", b, BOND_FIELDS)
    rbs = ref_bonds(b)
    p = spec.elements.p + 0.02 * 0.002 * rng.normal(size=spec.elements.p.shape)
    cases = {
        "randq": spec.elements.q,
        "nearq": quat_normalize(np.tile([0.0, 0, 0, 1], (spec.elements.n, 1))
                                + 0.05 * rng.normal(size=(spec.elements.n, 4))),
        "ident": np.tile([0.0, 0, 0, 1], (spec.elements.n, 1)),
    }
    for tag, q in cases.items():
        q = np.array(q)
        idx, e, gpi, gpj, gqi, gqj, hpp, hqq = rbs.energy_terms(p, q, want_hess=True)
        out.update({f"{tag}_q": q, f"{tag}_idx": idx, f"{tag}_E": e, f"{tag}_gpi": gpi,
                    f"{tag}_gpj": gpj, f"{tag}_gqi": gqi, f"{tag}_gqj": gqj,
                    f"{tag}_hpp": hpp, f"{tag}_hqq": hqq})
    out["p"] = p
    save("bond_terms.npz", **out)


def gold_block_sample():
    """BASELINE configs[4] (C5: 126^3 jittered block, random unit q, ~12M
    bonds) is too large for a reference step, so its bonds are checked the
    way SURVEY 8(d) asks: the reference's BondSet.energy_terms
    (bonds.py:473-504) on a seeded sample of the block's own bonds, at the
    generator's state (the step-1 predictor with zero velocities)."""
    spec = C.block(random_q=True)
    b = spec.bonds
    rng = np.random.default_rng(5)
    pick = np.sort(rng.choice(b.n, 1000, replace=False))
    sub = rb.BondSet(**{**{f: np.array(getattr(b, f))[pick] for f in BOND_FIELDS},
                        "face_i": np.zeros(pick.size, dtype=np.int64),
                        "face_j": np.zeros(pick.size, dtype=np.int64)})
    el = spec.elements
    idx, e, gpi, gpj, gqi, gqj, hpp, hqq = sub.energy_terms(el.p, el.q, want_hess=True)
    # the elements the sample touches (p, q rows), so the fixture is checkable
    # without regenerating the block
    rows = np.unique(np.r_[sub.i, sub.j])
    save("block_sample.npz", pick=pick, n=el.n, n_bonds=b.n, rows=rows, p_rows=el.p[rows],
         q_rows=el.q[rows], idx=idx, E=e, gpi=gpi, gpj=gpj, gqi=gqi, gqj=gqj, hpp=hpp, hqq=hqq)


def _small_problem(seed=21, random_q=False, qspread=0.05):
    spec = C.cube(n_side=4, r=0.002, seed=seed, random_q=random_q, youngs=3e8,
                  k_contact=1e8)
    rng = np.random.default_rng(seed + 1)
    el = spec.elements
    el.v[:] = 0.05 * rng.normal(size=el.v.shape)
    if not random_q:
        el.q[:] = quat_normalize(el.q + qspread * rng.normal(size=el.q.shape))
    el.qdot[:] = ri.tangent_project(el.q, 2.0 * rng.normal(size=el.q.shape))
    # plane cuts through the top layer so the collider curvature is active
    z_top = float(el.p[:, 2].max())
    cols = [C.HalfSpace((0.0, 0.0, -1.0), -(z_top - 0.3 * 0.002))]
    spec.colliders = cols
    spec.k_element = 1e6
    return spec, rng


def gold_newton_pieces():
    """value_and_gradient, build_clamped_pieces, assemble_reduced_system,
    BlockJacobi, pcg on one ImplicitProblem (integrator.py / solver.py / linalg.py)."""
    out = {}
    for tag, rq in (("near", False), ("rand", True)):
        spec, rng = _small_problem(seed=21 if not rq else 31, random_q=rq)
        sc = ref_scene(spec, colliders=ref_colliders(spec.colliders))
        el = sc.elements
        pairs = rc.broad_phase(el.p, el.radius, 2.0 * float(el.radius.max()) + 1e-12)
        ctx = ri.StepContext(sc.dt, sc.p_prev.copy(), sc.q_prev.copy(), el.p.copy(), el.q.copy())
        model = ri.PotentialModel(el, sc.bonds, pairs, sc.colliders, sc.gravity,
                                  sc.k_contact, sc.k_element)
        prob = ri.ImplicitProblem(model, ctx)
        p, q = ri.predict_state(ctx, el.v, el.qdot, prob.free)
        p = p + 1e-5 * rng.normal(size=p.shape) * prob.free[:, None]
        f, gp, gq = prob.value_and_gradient(p, q)
        z = rsv.reduced_gradient(q, gp, gq, prob.free)
        gnorm = float(np.linalg.norm(z))
        pieces = rsv.build_clamped_pieces(prob, p, q, gq)
        mat, diag = rsv.assemble_reduced_system(pieces, q, prob.free)
        pre = rl.BlockJacobi(diag)
        tol = rl.relative_tolerance(gnorm)
        res = rl.pcg(lambda v: mat @ v, -z, pre.apply, tol, 2000)
        res_tight = rl.pcg(lambda v: mat @ v, -z, pre.apply, 1e-10, 2000)
        out.update(pack(f"{tag}_el_", spec.elements, ELEM_FIELDS))
        out.update(pack(f"{tag}_b_", spec.bonds, BOND_FIELDS))
        hs = spec.colliders[0]
        out.update({
            f"{tag}_dt": sc.dt, f"{tag}_kc": sc.k_contact, f"{tag}_ke": sc.k_element,
            f"{tag}_gravity": sc.gravity, f"{tag}_hs": np.array([*hs.normal, hs.offset]),
            f"{tag}_p_prev": ctx.p_prev, f"{tag}_q_prev": ctx.q_prev,
            f"{tag}_pairs": pairs, f"{tag}_p": p, f"{tag}_q": q,
            f"{tag}_f": f, f"{tag}_gp": gp, f"{tag}_gq": gq, f"{tag}_z": z,
            f"{tag}_gnorm": gnorm,
            f"{tag}_bond_pp": pieces.bond_pp, f"{tag}_bond_qq_red": pieces.bond_qq_red,
            f"{tag}_pair_pp": pieces.pair_pp, f"{tag}_elem_pos": pieces.elem_pos,
            f"{tag}_elem_rot": pieces.elem_rot,
            f"{tag}_A": mat.toarray(), f"{tag}_diag": diag, f"{tag}_minv": pre.inverse_blocks,
            f"{tag}_pcg_x": res.x, f"{tag}_pcg_it": res.iterations, f"{tag}_pcg_tol": tol,
            f"{tag}_pcg_tight_x": res_tight.x, f"{tag}_pcg_tight_it": res_tight.iterations,
            f"{tag}_value": prob.value(p, q),
        })
    save("newton_pieces.npz", **out)


def gold_newton_solve():
    """minimize_second_order (solver.py:511-562) on a well-posed step problem:
    jittered cube with perturbed identity orientations, a plane touching the
    top layer and self-contact candidates; converges in the reference."""
    spec = C.cube(n_side=5, r=0.002, seed=61, random_q=False, youngs=3e8, k_contact=1e7)
    rng = np.random.default_rng(62)
    el = spec.elements
    el.v[:] = 0.02 * rng.normal(size=el.v.shape)
    z_top = float(el.p[:, 2].max())
    spec.colliders = [C.HalfSpace((0.0, 0.0, -1.0), -(z_top - 0.1 * 0.002))]
    # a crack through x = 0 splits the cube into two fragments; the contact
    # candidates are the overlapping pairs across it (contact_candidates)
    b = spec.bonds
    cross = (el.p[b.i, 0] < 0.0) != (el.p[b.j, 0] < 0.0)
    b.status[cross] = 2
    sc = ref_scene(spec)
    pairs = rsv.contact_candidates(sc)
    ctx = ri.StepContext(sc.dt, sc.p_prev.copy(), sc.q_prev.copy(), sc.elements.p.copy(),
                         sc.elements.q.copy())
    model = ri.PotentialModel(sc.elements, sc.bonds, pairs, sc.colliders, sc.gravity,
                              sc.k_contact, sc.k_element)
    prob = ri.ImplicitProblem(model, ctx)
    p0, q0 = ri.predict_state(ctx, sc.elements.v, sc.elements.qdot, prob.free)
    # compressed bonds lose their transverse curvature to the clamp, so this
    # jittered lattice converges linearly; eps 3e-3 (|m g| ~ 8e-4 N per element)
    cfg = rsv.SolverConfig(epsilon=3e-3, max_iterations=200)
    sol = rsv.minimize_second_order(prob, p0, q0, cfg)
    print(f"  newton_solve: converged={sol.converged} it={sol.iterations} "
          f"pcg={sol.pcg_total} gnorm={sol.grad_norm:.2e}")
    assert sol.converged
    hs = spec.colliders[0]
    out = pack("el_", spec.elements, ELEM_FIELDS)
    out.update(pack("b_", spec.bonds, BOND_FIELDS))
    out.update({
        "dt": sc.dt, "kc": sc.k_contact, "ke": sc.k_element, "gravity": sc.gravity,
        "hs": np.array([*hs.normal, hs.offset]), "p_prev": ctx.p_prev, "q_prev": ctx.q_prev,
        "pairs": pairs, "p0": p0, "q0": q0, "epsilon": 3e-3,
        "solve_p": sol.p, "solve_q": sol.q, "solve_iterations": sol.iterations,
        "solve_pcg_total": sol.pcg_total, "solve_gnorm": sol.grad_norm,
        "solve_rec_f": np.array([r.f for r in sol.records]),
        "solve_rec_gnorm": np.array([r.grad_norm for r in sol.records]),
        "solve_rec_alpha": np.array([r.alpha for r in sol.records]),
        "solve_rec_pcg": np.array([r.pcg_iterations for r in sol.records]),
    })
    save("newton_solve.npz", **out)


def gold_colliders():
    """Sphere and box colliders (contact.py:61-133): the collider curvature
    makes the element position blocks indefinite, exercising the 3x3 clamp of
    build_clamped_pieces (solver.py:165-167)."""
    spec = C.cube(n_side=4, r=0.002, seed=71, random_q=False, youngs=3e8, k_contact=1e8)
    rng = np.random.default_rng(72)
    el = spec.elements
    el.v[:] = 0.02 * rng.normal(size=el.v.shape)
    lo, hi = el.p.min(axis=0), el.p.max(axis=0)
    mid = 0.5 * (lo + hi)
    sphere = rc.SphereCollider(tuple(mid + np.array([0.0, 0.0, 0.004])), 0.005)
    box = rc.BoxCollider(tuple(np.array([lo[0], mid[1], mid[2]])), (0.003, 0.02, 0.02))
    sc = ref_scene(spec, colliders=[sphere, box])
    ctx = ri.StepContext(sc.dt, sc.p_prev.copy(), sc.q_prev.copy(), sc.elements.p.copy(),
                         sc.elements.q.copy())
    model = ri.PotentialModel(sc.elements, sc.bonds, np.zeros((0, 2), dtype=np.int64),
                              sc.colliders, sc.gravity, sc.k_contact, sc.k_element)
    prob = ri.ImplicitProblem(model, ctx)
    p, q = ri.predict_state(ctx, sc.elements.v, sc.elements.qdot, prob.free)
    f, gp, gq = prob.value_and_gradient(p, q)
    z = rsv.reduced_gradient(q, gp, gq, prob.free)
    pieces = rsv.build_clamped_pieces(prob, p, q, gq)
    mat, diag = rsv.assemble_reduced_system(pieces, q, prob.free)
    hb = prob.hessian_blocks(p, q)
    n_inside = int(np.count_nonzero(np.abs(hb.elem_pp).sum(axis=(1, 2))))
    n_indef = int(np.count_nonzero(np.linalg.eigvalsh(
        hb.elem_pp + prob.inertia_diag()[0][:, None, None] * np.eye(3)).min(axis=1) < 0))
    print(f"  colliders: {n_inside} elements with collider curvature, {n_indef} indefinite")
    out = pack("el_", spec.elements, ELEM_FIELDS)
    out.update(pack("b_", spec.bonds, BOND_FIELDS))
    out.update({"dt": sc.dt, "kc": sc.k_contact, "ke": sc.k_element, "gravity": sc.gravity,
                "sphere": np.array([*sphere.center, sphere.radius]),
                "box": np.array([*box.center, *box.half_extents]),
                "p_prev": ctx.p_prev, "q_prev": ctx.q_prev, "p": p, "q": q, "f": f, "z": z,
                "elem_pos": pieces.elem_pos, "diag": diag, "A": mat.toarray(),
                "n_indef": n_indef, "value": prob.value(p, q)})
    save("colliders.npz", **out)


def gold_problem_protocol():
    """The ImplicitProblem protocol (integrator.py:24-35, 39-138, 164-210) on a
    scene with every term: bonds (some broken), frozen contact pairs across
    a crack, a half-space, a sphere and a box collider, pinned elements,
    perturbed orientations.  value, value_and_gradient, hessian_blocks,
    inertia_diag and the model's value / energy_breakdown at a state where
    every contact term is active."""
    spec, rng = _small_problem(seed=81)
    el = spec.elements
    lo, hi = el.p.min(axis=0), el.p.max(axis=0)
    mid = 0.5 * (lo + hi)
    z_top = float(hi[2])
    cols = [rc.HalfSpace((0.0, 0.0, -1.0), -(z_top - 0.3 * 0.002)),
            rc.SphereCollider(tuple(mid + np.array([0.0, 0.0, 0.004])), 0.005),
            rc.BoxCollider(tuple(np.array([lo[0], mid[1], mid[2]])), (0.003, 0.02, 0.02))]
    b = spec.bonds
    cross = (el.p[b.i, 0] < mid[0]) != (el.p[b.j, 0] < mid[0])
    b.status[cross] = 2
    sc = ref_scene(spec, colliders=cols)
    e = sc.elements
    pairs = rc.broad_phase(e.p, e.radius, 2.0 * float(e.radius.max()) + 1e-12)
    pairs = pairs[(e.p[pairs[:, 0], 0] < mid[0]) != (e.p[pairs[:, 1], 0] < mid[0])]
    ctx = ri.StepContext(sc.dt, sc.p_prev.copy(), sc.q_prev.copy(), e.p.copy(), e.q.copy())
    model = ri.PotentialModel(e, sc.bonds, pairs, sc.colliders, sc.gravity, sc.k_contact,
                              sc.k_element)
    prob = ri.ImplicitProblem(model, ctx)
    p0, q = ri.predict_state(ctx, e.v, e.qdot, prob.free)
    # push the halves into each other so the pairs overlap
    p = p0 + 1e-5 * rng.normal(size=p0.shape) * prob.free[:, None]
    p[:, 0] += np.where(p[:, 0] < mid[0], 4e-4, -4e-4) * prob.free
    f, gp, gq = prob.value_and_gradient(p, q)
    hb = prob.hessian_blocks(p, q)
    mp, mq = prob.inertia_diag()
    touching = int(np.count_nonzero(np.abs(hb.pair_pp).sum(axis=(1, 2)) > 0))
    inside = int(np.count_nonzero(np.abs(hb.elem_pp).sum(axis=(1, 2)) > 0))
    print(f"  problem protocol: {pairs.shape[0]} pairs ({touching} touching), {inside} elements "
          f"in a collider, {int(np.count_nonzero(cross))} broken bonds")
    out = pack("el_", spec.elements, ELEM_FIELDS)
    out.update(pack("b_", spec.bonds, BOND_FIELDS))
    out.update({
        "dt": sc.dt, "kc": sc.k_contact, "ke": sc.k_element, "gravity": sc.gravity,
        "hs": np.array([*cols[0].normal, cols[0].offset]),
        "sphere": np.array([*cols[1].center, cols[1].radius]),
        "box": np.array([*cols[2].center, *cols[2].half_extents]),
        "pairs": pairs, "p_prev": ctx.p_prev, "q_prev": ctx.q_prev, "p_curr": ctx.p_curr,
        "q_curr": ctx.q_curr, "p": p, "q": q, "f": f, "gp": gp, "gq": gq,
        "value": prob.value(p, q), "model_value": model.value(p, q),
        "eb_bond": model.energy_breakdown(p, q)["bond"],
        "eb_contact": model.energy_breakdown(p, q)["contact"],
        "eb_gravity": model.energy_breakdown(p, q)["gravity"],
        "hb_bond_i": hb.bond_i, "hb_bond_j": hb.bond_j, "hb_bond_pp": hb.bond_pp,
        "hb_bond_qq": hb.bond_qq, "hb_pair_pp": hb.pair_pp, "hb_elem_pp": hb.elem_pp,
        "mp_dt2": mp, "mq_dt2": mq,
    })
    save("problem_protocol.npz", **out)


def gold_runner():
    """run_simulation + _step_with_retries + stats.csv (runner.py:20-164): a
    plain run, a run whose third frame needs dt halving (max_iterations=4),
    and one that gives up (max_iterations=3 -> StepFailure)."""
    import tempfile

    from bdem import runner as rr
    out = {}
    for tag, maxit in (("plain", 300), ("retry", 4)):
        spec = C.cantilever(nx=10, ny=3, nz=3)
        sc = ref_scene(spec)
        d = tempfile.mkdtemp()
        rr.run_simulation(sc, rsv.SolverConfig(epsilon=1e-7, max_iterations=maxit), frames=3,
                          fps=500, outdir=d, write_meshes=False)
        out[f"{tag}_csv"] = np.array(open(os.path.join(d, "stats.csv")).read())
        out[f"{tag}_p"] = sc.elements.p
    spec = C.cantilever(nx=10, ny=3, nz=3)
    sc = ref_scene(spec)
    try:
        rr.run_simulation(sc, rsv.SolverConfig(epsilon=1e-7, max_iterations=3), frames=3,
                          fps=500, write_meshes=False)
        out["fail_msg"] = np.array("")
    except rr.StepFailure as exc:
        out["fail_msg"] = np.array(str(exc))
        out["fail_residuals"] = np.array(exc.residuals)
    save("runner.npz", **out)


def _run_traj(name, spec, steps, eps, driver=None, schedule=None, max_iter=300):
    sc = ref_scene(spec, driver=driver)
    cfg = rsv.SolverConfig(epsilon=eps, max_iterations=max_iter)
    rec = {k: [] for k in ("p", "q", "v", "qdot", "newton", "pcg", "committed", "reason",
                           "pairs", "gnorm", "rec0_f", "rec0_gnorm")}
    events = []
    out = pack("init_el_", spec.elements, ELEM_FIELDS)
    out.update(pack("init_b_", spec.bonds, BOND_FIELDS))
    t0 = time.time()
    for s in range(steps):
        if schedule is not None:
            sc.colliders = ref_colliders(schedule(sc.time + sc.dt))
        rep = rsv.stable_step(sc, cfg)
        el = sc.elements
        for k, v in (("p", el.p), ("q", el.q), ("v", el.v), ("qdot", el.qdot)):
            rec[k].append(v.copy())
        rec["newton"].append(rep.solve.iterations)
        rec["pcg"].append(rep.solve.pcg_total)
        rec["committed"].append(rep.committed)
        rec["reason"].append(rep.solve.reason)
        rec["pairs"].append(rep.contact_pairs)
        rec["gnorm"].append(rep.solve.grad_norm)
        # the first Newton record is evaluated at the predictor (p0, q0):
        # it makes the predictor's retraction observable
        rec["rec0_f"].append(rep.solve.records[0].f)
        rec["rec0_gnorm"].append(rep.solve.records[0].grad_norm)
        events += [(s, b, sg, tu) for (b, sg, tu) in rep.broken]
    out.update({k: np.array(v) for k, v in rec.items()})
    out["events"] = np.array(events, dtype=float).reshape(-1, 4)
    out.update(pack("final_b_", sc.bonds, ("status", "stiffness_scale", "damage",
                                           "plastic_strain", "sigma", "tau")))
    out["labels"] = sc.labels.labels
    out.update({"dt": spec.dt, "youngs": spec.youngs, "epsilon": eps, "k_contact": spec.k_contact,
                "k_element": spec.k_element, "gravity": np.array(spec.gravity),
                "mu_s": spec.mu_s, "mu_r": spec.mu_r})
    if spec.plastic is not None:
        pl = spec.plastic
        out["plastic"] = np.array([pl.fracture_strain, pl.yield_strain, pl.weakening,
                                   pl.damage_exponent])
    print(f"  {name}: {steps} steps in {time.time() - t0:.1f}s; newton {rec['newton']}; "
          f"broken {len(events)}; committed {all(rec['committed'])}")
    save(f"traj_{name}.npz", **out)


def gold_trajectories():
    # BASELINE configs[0] exactly: 40x4x4, eps=1e-8, 20 steps, coordinates
    # centred at the origin; the reference commits all 20 steps.
    spec = C.cantilever()
    _run_traj("cantilever", spec, 20, 1e-8)

    spec = C.rope(n=30, epsilon=1e-5)
    drv = spec.driver
    _run_traj("rope", spec, 6, 1e-5,
              driver=rs.twist_driver(drv.ids, drv.p0, drv.axis_point, drv.rate))

    spec = C.plate(nx=24, ny=14, epsilon=1e-6)
    _run_traj("plate", spec, 6, 1e-6)

    spec = C.cube(n_side=5, random_q=False, seed=3, youngs=3e8, k_contact=1e9, speed=2.0,
                  dt=1e-4)
    sched = spec.collider_schedule
    _run_traj("cube", spec, 6, 1e-6, schedule=sched)


def gold_stall():
    """SURVEY 8(d) (C4 caution): the twist-driven 40x4x4 lattice beam.  The
    reference's clamped Newton iteration stalls at gnorm 1.84e-3 for the whole
    300-iteration budget (alpha = 1 throughout) and stable_step does not
    commit; the GPU path must reproduce the stall (solver.py:511-562, 917-939)."""
    spec = C.twisted_beam()
    drv = spec.driver
    sc = ref_scene(spec, driver=rs.twist_driver(drv.ids, drv.p0, drv.axis_point, drv.rate))
    cfg = rsv.SolverConfig(epsilon=spec.epsilon, max_iterations=300)
    out = pack("init_el_", spec.elements, ELEM_FIELDS)
    out.update(pack("init_b_", spec.bonds, BOND_FIELDS))
    t0 = time.time()
    rep = rsv.stable_step(sc, cfg)
    r = rep.solve
    el = sc.elements
    out.update({"iterations": r.iterations, "pcg_total": r.pcg_total, "committed": rep.committed,
                "reason": r.reason, "grad_norm": r.grad_norm, "converged": r.converged,
                "rec_gnorm": np.array([x.grad_norm for x in r.records]),
                "rec_f": np.array([x.f for x in r.records]),
                "rec_alpha": np.array([x.alpha for x in r.records]),
                "rec_pcg": np.array([x.pcg_iterations for x in r.records]),
                "after_p": el.p.copy(), "after_q": el.q.copy(), "after_v": el.v.copy(),
                "after_qdot": el.qdot.copy(), "time_after": sc.time,
                "dt": spec.dt, "youngs": spec.youngs, "epsilon": spec.epsilon,
                "k_contact": spec.k_contact, "k_element": spec.k_element,
                "gravity": np.array(spec.gravity)})
    print(f"  stall: {r.iterations} Newton / {r.pcg_total} PCG, reason {r.reason}, committed "
          f"{rep.committed}, gnorm {r.grad_norm:.6e} in {time.time() - t0:.1f}s")
    save("stall_beam.npz", **out)


def _subsample_rows(n, stride):
    return np.unique(np.r_[np.arange(0, n, stride), np.arange(max(n - 3, 0), n)])


def gold_rope100k():
    """BASELINE configs[3] at its full size (100,000 spheres, G = 10 E, end
    twisted at 10 rad/s, eps 1e-5): the first 5 implicit steps of the
    reference.  The rotation path (twist driver, quaternion retraction,
    tangent-projected qdot) is the only one that moves q, so every element's
    q and qdot matter; the fixture keeps a strided subsample of rows plus both
    ends and the whole-array norms."""
    spec = C.rope()
    drv = spec.driver
    sc = ref_scene(spec, driver=rs.twist_driver(drv.ids, drv.p0, drv.axis_point, drv.rate))
    cfg = rsv.SolverConfig(epsilon=1e-5, max_iterations=300)
    rows = _subsample_rows(spec.elements.n, 331)
    rec = {k: [] for k in ("p", "q", "v", "qdot", "newton", "pcg", "committed", "gnorm",
                           "q_dev_norm", "qdot_norm", "pcg_per_newton", "reason")}
    t0 = time.time()
    for s in range(5):
        rep = rsv.stable_step(sc, cfg)
        el = sc.elements
        for k, v in (("p", el.p), ("q", el.q), ("v", el.v), ("qdot", el.qdot)):
            rec[k].append(v[rows].copy())
        rec["q_dev_norm"].append(float(np.linalg.norm(el.q - np.array([0.0, 0, 0, 1]))))
        rec["qdot_norm"].append(float(np.linalg.norm(el.qdot)))
        rec["newton"].append(rep.solve.iterations)
        rec["pcg"].append(rep.solve.pcg_total)
        rec["pcg_per_newton"].append([r.pcg_iterations for r in rep.solve.records])
        rec["committed"].append(rep.committed)
        rec["gnorm"].append(rep.solve.grad_norm)
        rec["reason"].append(rep.solve.reason)
        print(f"    step {s}: newton {rep.solve.iterations} pcg {rep.solve.pcg_total} "
              f"{rep.solve.reason} gnorm {rep.solve.grad_norm:.3e} ({time.time() - t0:.0f}s)",
              flush=True)
    out = {k: np.array(v) for k, v in rec.items() if k != "pcg_per_newton"}
    out["pcg_per_newton"] = np.array(sum(rec["pcg_per_newton"], []))
    out.update({"rows": rows, "n": spec.elements.n, "epsilon": 1e-5, "seconds": time.time() - t0})
    save("traj_rope100k.npz", **out)


def gold_cube22():
    """BASELINE configs[1] at its full size (22^3 = 10,648 jittered spheres,
    radii U(0.9r, 1.1r), E = 3e9, PlasticParams(1e-3, 6e-4, 0.5, 2), a rigid
    plane descending at 0.5 m/s, dt = 1e-4) in the identity-q variant SURVEY
    8(d) prescribes for trajectory parity (random q is un-steppable by the
    reference).  The first steps of the reference, eps 1e-6: p, v on a strided
    subsample of rows plus both ends, whole-array norms, counts, the first
    Newton record (predictor) and the fracture / yield state of every bond."""
    spec = C.cube(random_q=False, epsilon=1e-6)
    sched = spec.collider_schedule
    sc = ref_scene(spec)
    cfg = rsv.SolverConfig(epsilon=1e-6, max_iterations=300)
    rows = _subsample_rows(spec.elements.n, 37)
    rec = {k: [] for k in ("p", "v", "newton", "pcg", "committed", "gnorm", "p_norm",
                           "v_norm", "rec0_f", "rec0_gnorm", "n_yielded", "reason")}
    events = []
    t0 = time.time()
    for s in range(int(os.environ.get("CUBE22_STEPS", 4))):
        sc.colliders = ref_colliders(sched(sc.time + sc.dt))
        rep = rsv.stable_step(sc, cfg)
        el = sc.elements
        rec["p"].append(el.p[rows].copy())
        rec["v"].append(el.v[rows].copy())
        rec["p_norm"].append(float(np.linalg.norm(el.p)))
        rec["v_norm"].append(float(np.linalg.norm(el.v)))
        rec["newton"].append(rep.solve.iterations)
        rec["pcg"].append(rep.solve.pcg_total)
        rec["committed"].append(rep.committed)
        rec["gnorm"].append(rep.solve.grad_norm)
        rec["reason"].append(rep.solve.reason)
        rec["rec0_f"].append(rep.solve.records[0].f)
        rec["rec0_gnorm"].append(rep.solve.records[0].grad_norm)
        rec["n_yielded"].append(int(np.count_nonzero(sc.bonds.status == 1)))
        events += [(s, b, sg, tu) for (b, sg, tu) in rep.broken]
        print(f"    step {s}: newton {rep.solve.iterations} pcg {rep.solve.pcg_total} "
              f"{rep.solve.reason} gnorm {rep.solve.grad_norm:.3e} yielded "
              f"{rec['n_yielded'][-1]} broken {len(rep.broken)} ({time.time() - t0:.0f}s)",
              flush=True)
    out = {k: np.array(v) for k, v in rec.items()}
    out["events"] = np.array(events, dtype=float).reshape(-1, 4)
    out.update(pack("final_b_", sc.bonds, ("status", "stiffness_scale", "damage",
                                           "plastic_strain", "sigma", "tau")))
    out.update({"rows": rows, "n": spec.elements.n, "epsilon": 1e-6,
                "seconds": time.time() - t0})
    save("traj_cube22.npz", **out)


def gold_plate600k():
    """The north-star config at full size (BASELINE configs[2], SURVEY 8(d) C3:
    1000x600 plate, 3,591,004 bonds, eps 1e-3): the step-1 problem exactly as
    stable_step builds it (solver.py:902-908) and the first two Newton
    iterations of minimize_second_order (solver.py:511-562).  Kept: the
    iteration records (f, |z|, alpha, PCG counts), the Newton direction y and
    the iterate after each iteration on a strided subsample of rows, and the
    contact-candidate count."""
    spec = C.plate()
    t0 = time.time()
    sc = ref_scene(spec)
    print(f"    scene built in {time.time() - t0:.0f}s", flush=True)
    el = sc.elements
    t1 = time.time()
    pairs = rsv.contact_candidates(sc)
    t_bp = time.time() - t1
    ctx = ri.StepContext(sc.dt, sc.p_prev.copy(), sc.q_prev.copy(), el.p.copy(), el.q.copy())
    model = ri.PotentialModel(el, sc.bonds, pairs, sc.colliders, sc.gravity, sc.k_contact,
                              sc.k_element)
    prob = ri.ImplicitProblem(model, ctx)
    p0, q0 = ri.predict_state(ctx, el.v, el.qdot, prob.free)
    n = el.n
    rows = _subsample_rows(n, 997)
    free_ids = np.nonzero(prob.free)[0]
    slot = np.full(n, -1)
    slot[free_ids] = np.arange(free_ids.size)
    y_idx = (6 * slot[rows][:, None] + np.arange(6)[None, :]).ravel()
    cap = {"y": [], "p": [], "q": [], "t": []}
    orig_nd, orig_ls = rsv._newton_direction, rsv.line_search

    def nd(*a, **k):
        out = orig_nd(*a, **k)
        cap["y"].append(out[0][y_idx].copy())
        return out

    def ls(*a, **k):
        out = orig_ls(*a, **k)
        cap["p"].append(out[1][rows].copy())
        cap["q"].append(out[2][rows].copy())
        cap["t"].append(time.time())
        return out

    rsv._newton_direction, rsv.line_search = nd, ls
    try:
        t2 = time.time()
        sol = rsv.minimize_second_order(prob, p0, q0,
                                        rsv.SolverConfig(epsilon=1e-3, max_iterations=2))
        t_solve = time.time() - t2
    finally:
        rsv._newton_direction, rsv.line_search = orig_nd, orig_ls
    recs = sol.records
    print(f"    2 Newton iterations in {t_solve:.0f}s: gnorm "
          f"{[r.grad_norm for r in recs]} pcg {[r.pcg_iterations for r in recs]} "
          f"alpha {[r.alpha for r in recs]}", flush=True)
    save("plate600k_newton.npz", rows=rows, n=n, n_bonds=sc.bonds.n, n_pairs=pairs.shape[0],
         p0=p0[rows], q0=q0[rows], y=np.array(cap["y"]), p=np.array(cap["p"]),
         q=np.array(cap["q"]), rec_f=np.array([r.f for r in recs]),
         rec_gnorm=np.array([r.grad_norm for r in recs]),
         rec_cnorm=np.array([r.constraint_norm for r in recs]),
         rec_alpha=np.array([r.alpha for r in recs]),
         rec_pcg=np.array([r.pcg_iterations for r in recs]), epsilon=1e-3,
         seconds_solve=t_solve, seconds_broadphase=t_bp)


def _extra_elements(el, rows):
    """Append isolated elements (p, mass, radius) to an ElementSet copy."""
    k = len(rows)
    p = np.concatenate([el.p, np.array([r[0] for r in rows], dtype=float)])
    q = np.concatenate([el.q, np.tile([0.0, 0.0, 0.0, 1.0], (k, 1))])
    return type(el)(p, q, np.concatenate([el.v, np.zeros((k, 3))]),
                    np.concatenate([el.qdot, np.zeros((k, 4))]),
                    np.concatenate([el.mass, [r[1] for r in rows]]),
                    np.concatenate([el.radius, [r[2] for r in rows]]),
                    np.concatenate([el.pinned, np.zeros(k, dtype=bool)]))


def gold_failures():
    """The reference's failure branches, each driven the way it can happen:

    * pcg breakdown / diagonal-boost restart (linalg.py:74-97): the "near"
      Newton system of newton_pieces.npz with every diagonal block shifted by
      -c I (c = lambda_min(A) + delta) -- an indefinite operator; its
      block-Jacobi (linalg.py:100-128) falls back to identity on the blocks
      the shift made singular or indefinite.  One shift the boost cures
      (restarts, then convergence) and one it does not (gives up after 4).
    * BlockJacobi identity fallback in a real solve: a cantilever plus two
      isolated free elements -- one with zero mass (zero 6x6 block) and one
      with zero radius (position block m/dt^2 I, rotation block 0: singular
      as a 6x6 block) -- stepped with stable_step.
    * non-descent fallback (solver.py:542-548): minimize_second_order on the
      newton_solve problem with the linear solve replaced by one returning
      x = -b (an ascent direction); every iteration falls back to -z.
    * reason="line-search" (solver.py:549-556): a random-q cube, whose
      prestressed bonds defeat the line search.
    * DegenerateBondError (bonds.py:163-168) raised through stable_step: a
      two-element bond whose predictor makes its endpoints coincide.
    """
    from bdem import elements as re_
    out = {}
    # -- pcg breakdown -------------------------------------------------------
    d = dict(np.load(os.path.join(HERE, "newton_pieces.npz")))
    A, diag, z = d["near_A"], d["near_diag"], d["near_z"]
    lam0 = float(np.linalg.eigvalsh(A).min())
    for tag, delta in (("cured", 5e-8), ("giveup", 1e3)):
        c = lam0 + delta
        dmod = diag - c * np.eye(6)[None]
        amod = A - c * np.eye(A.shape[0])
        pre = rl.BlockJacobi(dmod)
        res = rl.pcg(lambda v: amod @ v, -z, pre.apply, 1e-8, 2000)
        print(f"  pcg {tag}: lambda_min {float(np.linalg.eigvalsh(amod).min()):.3e} "
              f"restarts {res.restarts} it {res.iterations} converged {res.converged}")
        out.update({f"pcg_{tag}_diag": dmod, f"pcg_{tag}_minv": pre.inverse_blocks,
                    f"pcg_{tag}_x": res.x, f"pcg_{tag}_it": res.iterations,
                    f"pcg_{tag}_restarts": res.restarts,
                    f"pcg_{tag}_converged": res.converged,
                    f"pcg_{tag}_rel": res.relative_residual, f"pcg_{tag}_shift": c})
    out["pcg_tol"] = 1e-8
    # -- singular block-Jacobi in a real solve ---------------------------------
    spec = C.cantilever(nx=6, ny=3, nz=3)
    m0 = float(spec.elements.mass[0])
    el = _extra_elements(spec.elements, [((1.0, 0.0, 0.0), 0.0, 0.005),
                                         ((-1.0, 0.0, 0.0), m0, 0.0)])
    spec.elements = el
    sc = ref_scene(spec)
    cfg = rsv.SolverConfig(epsilon=1e-7, max_iterations=300)
    pk = {k: [] for k in ("p", "q", "newton", "pcg", "committed")}
    import logging
    logging.getLogger("bdem").setLevel(logging.ERROR)
    for _ in range(3):
        rep = rsv.stable_step(sc, cfg)
        pk["p"].append(sc.elements.p.copy())
        pk["q"].append(sc.elements.q.copy())
        pk["newton"].append(rep.solve.iterations)
        pk["pcg"].append(rep.solve.pcg_total)
        pk["committed"].append(rep.committed)
    print(f"  singular: newton {pk['newton']} pcg {pk['pcg']} committed {pk['committed']}")
    out.update(pack("sing_el_", el, ELEM_FIELDS))
    out.update({f"sing_{k}": np.array(v) for k, v in pk.items()})
    # -- non-descent fallback --------------------------------------------------
    g = dict(np.load(os.path.join(HERE, "newton_solve.npz")))
    el = re_.ElementSet(*(g[f"el_{f}"] for f in ELEM_FIELDS))
    bs = rb.BondSet(**{f: g[f"b_{f}"] for f in BOND_FIELDS},
                    face_i=np.zeros(g["b_i"].shape[0], dtype=np.int64),
                    face_j=np.zeros(g["b_i"].shape[0], dtype=np.int64))
    hs = g["hs"]
    ctx = ri.StepContext(float(g["dt"]), g["p_prev"], g["q_prev"], el.p.copy(), el.q.copy())
    model = ri.PotentialModel(el, bs, g["pairs"], [rc.HalfSpace(tuple(hs[:3]), hs[3])],
                              g["gravity"], float(g["kc"]), float(g["ke"]))
    prob = ri.ImplicitProblem(model, ctx)
    orig_pcg = rsv.pcg

    def ascent(apply_a, b, apply_m=None, tol_rel=1e-10, max_iter=None, on_iteration=None):
        return rl.PCGResult(-np.asarray(b, dtype=float), 1, True, 1.0)

    rsv.pcg = ascent
    try:
        sol = rsv.minimize_second_order(prob, g["p0"], g["q0"],
                                        rsv.SolverConfig(epsilon=1e-9, max_iterations=6))
    finally:
        rsv.pcg = orig_pcg
    print(f"  non-descent: {sol.reason} it {sol.iterations} alpha "
          f"{[r.alpha for r in sol.records]}")
    out.update({"nd_p": sol.p, "nd_q": sol.q, "nd_iterations": sol.iterations,
                "nd_reason": np.array(sol.reason),
                "nd_rec_f": np.array([r.f for r in sol.records]),
                "nd_rec_gnorm": np.array([r.grad_norm for r in sol.records]),
                "nd_rec_alpha": np.array([r.alpha for r in sol.records])})
    # -- line-search failure on a random-q cube ------------------------------------
    spec = C.cube(n_side=4, seed=2, random_q=True)
    sc = ref_scene(spec)
    rep = rsv.stable_step(sc, rsv.SolverConfig(epsilon=1e-6, max_iterations=300))
    recs = rep.solve.records
    print(f"  line-search: committed {rep.committed} reason {rep.solve.reason} "
          f"it {rep.solve.iterations} gnorm {rep.solve.grad_norm:.3e}")
    out.update(pack("ls_el_", spec.elements, ELEM_FIELDS))
    out.update(pack("ls_b_", spec.bonds, BOND_FIELDS))
    out.update({"ls_committed": rep.committed, "ls_reason": np.array(rep.solve.reason),
                "ls_iterations": rep.solve.iterations,
                "ls_rec_f": np.array([r.f for r in recs]),
                "ls_rec_gnorm": np.array([r.grad_norm for r in recs]),
                "ls_rec_alpha": np.array([r.alpha for r in recs]),
                "ls_rec_pcg": np.array([r.pcg_iterations for r in recs]),
                "ls_p_after": sc.elements.p, "ls_q_after": sc.elements.q})
    # -- degenerate bond through stable_step ----------------------------------------
    spec = C.cantilever(nx=2, ny=1, nz=1, dt=1e-3)
    el = spec.elements
    el.pinned[:] = False
    el.v[0] = (el.p[1] - el.p[0]) / spec.dt
    sc = ref_scene(spec)
    try:
        rsv.stable_step(sc, rsv.SolverConfig(epsilon=1e-7))
        msg, kind = "", ""
    except Exception as exc:            # noqa: BLE001 - the class is the golden
        msg, kind = str(exc), type(exc).__name__
    print(f"  degenerate: {kind}: {msg}")
    out.update(pack("deg_el_", el, ELEM_FIELDS))
    out.update({"deg_kind": np.array(kind), "deg_msg": np.array(msg)})
    save("failures.npz", **out)


def gold_fracture():
    """update_bond_states (bonds.py:532-570) with plasticity and strengths."""
    spec = C.cube(n_side=5, r=0.002, seed=41, random_q=False, youngs=1e9)
    rng = np.random.default_rng(41)
    el, b = spec.elements, spec.bonds
    nb = b.n
    p = el.p + 0.02 * 0.002 * rng.normal(size=el.p.shape)
    q = quat_normalize(el.q + 0.02 * rng.normal(size=el.q.shape))
    b.status[rng.choice(nb, 10, replace=False)] = 2
    b.status[rng.choice(nb, 10, replace=False)] = 1
    b.stiffness_scale[:] = rng.uniform(0.6, 1.0, nb)
    b.damage[:] = rng.uniform(0.7, 1.0, nb)
    rbs = ref_bonds(b)
    # strengths around the sampled stress distribution so some bonds break
    _, sig, tau = rbs.stresses(p, q)
    # thresholds in the middle of a gap of the sampled stresses, so no bond
    # lies within 1e-6 (relative) of a strength (the parity exclusion band)
    def gap_mid(x, qtl):
        xs = np.sort(x)
        k = int(qtl * (xs.size - 1))
        while xs[k + 1] - xs[k] <= 1e-4 * xs[k + 1]:
            k += 1
        return 0.5 * (xs[k] + xs[k + 1])
    b.tensile_strength[:] = gap_mid(sig, 0.9)
    b.shear_strength[:] = gap_mid(tau, 0.95)
    out = pack("b_", b, BOND_FIELDS)
    out.update({"p": p, "q": q})
    pl = rb.PlasticParams(2e-3, 1e-3, 0.5, 2.0)
    for tag, plastic in (("plastic", pl), ("elastic", None)):
        rbs = ref_bonds(b)
        ev = rb.update_bond_states(rbs, p, q, 1e9, plastic)
        out.update(pack(f"{tag}_out_", rbs, ("status", "stiffness_scale", "damage",
                                             "plastic_strain", "sigma", "tau")))
        out[f"{tag}_events"] = np.array(ev, dtype=float).reshape(-1, 3)
    out["plastic"] = np.array([2e-3, 1e-3, 0.5, 2.0])
    save("fracture.npz", **out)


def gold_friction():
    """apply_friction (contact.py:303-350) on a dense random cloud: long
    dependency chains through shared elements, pinned elements, radial qdot
    components, and all three collider kinds; plus a stacked-blocks
    trajectory through stable_step with mu_s, mu_r > 0 (solver.py:923-925)."""
    rng = np.random.default_rng(81)
    n = 600
    pos = rng.uniform(-0.03, 0.03, size=(n, 3))
    rad = rng.uniform(0.003, 0.006, size=n)
    q = quat_normalize(rng.normal(size=(n, 4)))
    v = rng.normal(size=(n, 3))
    v[rng.random(n) < 0.05] = 0.0
    qdot = rng.normal(size=(n, 4))                   # includes a radial part
    mass = 2500.0 * (4.0 / 3.0) * np.pi * rad**3
    pinned = rng.random(n) < 0.1
    el = re_.ElementSet(pos.copy(), q.copy(), v.copy(), qdot.copy(), mass.copy(), rad.copy(),
                        pinned.copy())
    pairs = rc.broad_phase(pos, rad, 2.0 * rad.max() + 1e-12)
    cols = [rc.HalfSpace((0.0, 0.0, 1.0), -0.02), rc.SphereCollider((0.01, 0.0, 0.0), 0.012),
            rc.BoxCollider((-0.02, 0.01, 0.0), (0.008, 0.01, 0.03))]
    k_c, k_ec, mu_s, mu_r, dt = 3e5, 2e5, 0.3, 0.05, 1e-4
    rc.apply_friction(el, pairs, cols, k_c, k_ec, mu_s, mu_r, dt)
    out = {"p": pos, "q": q, "v": v, "qdot": qdot, "mass": mass, "radius": rad,
           "pinned": pinned, "pairs": pairs, "halfspace": np.array([0.0, 0.0, 1.0, -0.02]),
           "sphere": np.array([0.01, 0.0, 0.0, 0.012]),
           "box": np.array([-0.02, 0.01, 0.0, 0.008, 0.01, 0.03]),
           "k_c": k_c, "k_ec": k_ec, "mu_s": mu_s, "mu_r": mu_r, "dt": dt,
           "v_out": el.v, "qdot_out": el.qdot}
    d = np.linalg.norm(pos[pairs[:, 0]] - pos[pairs[:, 1]], axis=1)
    print(f"  friction: {pairs.shape[0]} pairs, {int((d < rad[pairs[:, 0]] + rad[pairs[:, 1]]).sum())}"
          f" in contact")
    save("friction.npz", **out)
    spec = C.stack()
    _run_traj("stack", spec, spec.steps, spec.epsilon)


def gold_mesh():
    """The reference's tet-mesh scene (scenes.py:239-256, strengths lowered so
    the impact breaks bonds): mesh arrays, elements/bonds with face ids, 10
    implicit steps with friction and fracture, and reconstruct_surface /
    write_surface_obj (geometry.py:313-358) of the initial and final states."""
    import tempfile
    sc = rs.drop_fracture(resolution=1, tensile_strength=3e4, shear_strength=3e4)
    m = sc.mesh
    out = {"mesh_vertices": m.vertices, "mesh_tets": m.tets, "mesh_interior": m.interior,
           "mesh_boundary": m.boundary, "mesh_volumes": m.volumes,
           "mesh_centroids": m.centroids}
    # copies: stepping mutates the scene's arrays in place
    out.update({k: v.copy() for k, v in pack("init_el_", sc.elements, ELEM_FIELDS).items()})
    out.update({k: v.copy() for k, v in
                pack("init_b_", sc.bonds, BOND_FIELDS + ("face_i", "face_j")).items()})

    def surface(tag):
        groups = rg.reconstruct_surface(sc.mesh, sc.bonds, sc.labels, sc.elements.p,
                                        sc.elements.q)
        out[f"{tag}_verts"] = np.concatenate([v for _, v, _ in groups]).reshape(-1, 3)
        out[f"{tag}_counts"] = np.array([v.shape[0] for _, v, _ in groups])
        out[f"{tag}_tris"] = np.concatenate([t for _, _, t in groups]).reshape(-1, 3)
        path = os.path.join(tempfile.mkdtemp(), "s.obj")
        rg.write_surface_obj(path, groups)
        out[f"{tag}_obj"] = np.array(open(path).read())

    surface("surf0")
    cfg = rsv.SolverConfig(epsilon=1e-5, max_iterations=300)
    rec = {k: [] for k in ("p", "q", "v", "qdot", "newton", "committed", "pairs")}
    events = []
    for s in range(10):
        rep = rsv.stable_step(sc, cfg)
        for k, v in (("p", sc.elements.p), ("q", sc.elements.q), ("v", sc.elements.v),
                     ("qdot", sc.elements.qdot)):
            rec[k].append(v.copy())
        rec["newton"].append(rep.solve.iterations)
        rec["committed"].append(rep.committed)
        rec["pairs"].append(rep.contact_pairs)
        events += [(s, b, sg, tu) for (b, sg, tu) in rep.broken]
    out.update({k: np.array(v) for k, v in rec.items()})
    out["events"] = np.array(events, dtype=float).reshape(-1, 4)
    out["final_status"] = sc.bonds.status.copy()
    out["labels"] = sc.labels.labels.copy()
    out["surface_flags"] = sc.surface_flags.copy()
    surface("surf1")
    out.update({"dt": sc.dt, "youngs": sc.youngs, "epsilon": 1e-5, "k_contact": sc.k_contact,
                "k_element": sc.k_element, "mu_s": sc.mu_s, "mu_r": sc.mu_r,
                "gravity": sc.gravity})
    print(f"  mesh: {m.n_tets} tets, {sc.bonds.i.shape[0]} bonds, newton {rec['newton']}, "
          f"broken {len(events)}, components {sc.labels.n_components}")
    save("mesh_drop.npz", **out)


def gold_broadphase_labels():
    rng = np.random.default_rng(51)
    out = {}
    for tag, n in (("a", 300), ("b", 2000)):
        pos = rng.uniform(-0.05, 0.05, size=(n, 3))
        rad = rng.uniform(0.002, 0.006, size=n)
        cell = 2.0 * rad.max() + 1e-12
        out[f"{tag}_pos"], out[f"{tag}_rad"], out[f"{tag}_cell"] = pos, rad, cell
        out[f"{tag}_pairs"] = rc.broad_phase(pos, rad, cell)
    spec = C.cube(n_side=6, seed=52)
    b = spec.bonds
    b.status[rng.random(b.n) < 0.55] = 2
    out.update({"lab_i": b.i, "lab_j": b.j, "lab_status": b.status, "lab_n": spec.elements.n,
                "lab_labels": rg.label_components(spec.elements.n, ref_bonds(b)).labels})
    save("broadphase_labels.npz", **out)


if __name__ == "__main__":
    t = time.time()
    which = sys.argv[1:] or ["bond_terms", "fracture", "broadphase_labels", "newton_pieces",
                             "newton_solve", "colliders", "runner", "trajectories", "friction", "mesh"]
    for name in which:
        globals()[f"gold_{name}"]()
    print(f"done in {time.time() - t:.1f}s")
