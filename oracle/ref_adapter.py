"""The reference ``bdem`` package as a checker and CPU baseline.

TEST / MEASUREMENT INFRASTRUCTURE ONLY: imported by ``tests/`` and by
``bench.py``'s reference / cpu_baseline legs, never by the product path.

``oracle.build_ref.load()`` imports the unmodified reference: its bytecode
build under ``oracle/_ref`` (travels to the GPU box) or, in the build
container, the sources under ``/root/reference``.  The helpers turn the
shared seeded generator's arrays (``paper_2308_10459_b200.configs``) into
reference objects, like ``tests/golden/make_golden.py`` does, and build the
step-1 ``ImplicitProblem`` exactly as ``stable_step`` does
(``solver.py:894-908``).
"""

from __future__ import annotations

import numpy as np

from oracle import build_ref

BOND_FIELDS = ("i", "j", "rest_length", "radius", "d0", "q0", "frame", "kn", "kt", "k_diag",
               "section", "second_moment", "polar_moment", "tensile_strength",
               "shear_strength", "status", "stiffness_scale", "damage", "plastic_strain",
               "sigma", "tau")
ELEM_FIELDS = ("p", "q", "v", "qdot", "mass", "radius", "pinned")


def bdem_or_skip():
    import pytest
    mod = build_ref.load()
    if mod is None:
        pytest.skip("reference bdem unavailable (run build() where /root/reference exists)")
    return mod


def ref_bonds(bdem, b):
    from bdem import bonds as rb
    kw = {f: np.array(getattr(b, f), copy=True) for f in BOND_FIELDS}
    kw["face_i"] = np.zeros(b.n, dtype=np.int64)
    kw["face_j"] = np.zeros(b.n, dtype=np.int64)
    return rb.BondSet(**kw)


def ref_elements(bdem, el):
    from bdem import elements as re_
    return re_.ElementSet(*(np.array(getattr(el, f), copy=True) for f in ELEM_FIELDS))


def dummy_mesh(bdem):
    from bdem import geometry as rg
    v = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    return rg.TetMesh(v, np.array([[0, 1, 2, 3]]))


def ref_driver(bdem, spec):
    from bdem import scenes as rs
    d = spec.driver
    if d is None:
        return None
    if d.kind == "twist":
        return rs.twist_driver(d.ids, d.p0, d.axis_point, d.rate)
    return rs.stretch_driver(d.ids, d.p0, d.speed)


def ref_scene(bdem, spec):
    """A reference ``Scene`` (scenes.py:31-52) holding copies of the spec's arrays."""
    from bdem import contact as rc
    from bdem import scenes as rs
    el = ref_elements(bdem, spec.elements)
    cols = [rc.HalfSpace(tuple(c.normal), c.offset) for c in spec.colliders]
    return rs.Scene(spec.name, dummy_mesh(bdem), el, ref_bonds(bdem, spec.bonds), colliders=cols,
                    gravity=np.array(spec.gravity), dt=spec.dt, youngs=spec.youngs,
                    shear_modulus=spec.shear_modulus, density=spec.density,
                    k_contact=spec.k_contact, k_element=spec.k_element, plastic=spec.plastic,
                    driver=ref_driver(bdem, spec), mu_s=spec.mu_s, mu_r=spec.mu_r,
                    surface_flags=np.zeros(el.n, dtype=bool))


def step_problem(bdem, sc):
    """The step-1 problem of ``stable_step`` (solver.py:894-908): driver rows
    at t + dt, the step context, frozen contact candidates, the potential and
    ``ImplicitProblem``; returns (problem, p0, q0, pairs)."""
    from bdem import integrator as ri
    from bdem import solver as rsv
    el = sc.elements
    if sc.driver is not None:
        sc.driver(el, sc.time + sc.dt)
    ctx = ri.StepContext(sc.dt, sc.p_prev.copy(), sc.q_prev.copy(), el.p.copy(), el.q.copy())
    pairs = rsv.contact_candidates(sc)
    model = ri.PotentialModel(el, sc.bonds, pairs, sc.colliders, sc.gravity, sc.k_contact,
                              sc.k_element)
    prob = ri.ImplicitProblem(model, ctx)
    p0, q0 = ri.predict_state(ctx, el.v, el.qdot, prob.free)
    return prob, p0, q0, pairs
