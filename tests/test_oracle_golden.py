"""Pin the CPU oracle against golden vectors produced by the reference itself.

The fixtures in ``tests/golden`` were written by ``make_golden.py`` running
``/root/reference/pkg/src/bdem`` on the shared seeded generator.  The oracle
restates the same numpy expressions, so agreement is at round-off level
(most checks are bit-exact).  CPU only.
"""

import numpy as np
import pytest

from _fixtures import bonds_from, close, elements_from, load
from oracle import cpu_oracle as O
from paper_2308_10459_b200.colliders import HalfSpace
from paper_2308_10459_b200.scene import TwistDriver
from paper_2308_10459_b200.state import PlasticParams

TIGHT = dict(rtol=1e-13, atol=0.0)


def _assert_close(a, b, rtol, atol, what):
    ok, info = close(a, b, rtol, atol)
    assert ok, f"{what}: got {info[0]!r} want {info[1]!r} at flat index {info[2]}"


@pytest.mark.parametrize("case", ["randq", "nearq", "ident"])
def test_bond_terms(case):
    d = load("bond_terms.npz")
    b = bonds_from(d, "b_")
    ev = O.bond_eval(b, d["p"], d[f"{case}_q"], want_hess=True)
    assert np.array_equal(ev.idx, d[f"{case}_idx"])
    for key, got in (("E", ev.energy), ("gpi", ev.gp_i), ("gpj", ev.gp_j), ("gqi", ev.gq_i),
                     ("gqj", ev.gq_j), ("hpp", ev.h_pp), ("hqq", ev.h_qq)):
        want = d[f"{case}_{key}"]
        _assert_close(got, want, 1e-12, 1e-12 * np.abs(want).max(), f"{case}/{key}")


@pytest.mark.parametrize("mode", ["plastic", "elastic"])
def test_fracture_update(mode):
    d = load("fracture.npz")
    b = bonds_from(d, "b_")
    pl = PlasticParams(*d["plastic"]) if mode == "plastic" else None
    ev = O.fracture_update(b, d["p"], d["q"], 1e9, pl)
    want = d[f"{mode}_events"]
    assert len(ev) == want.shape[0]
    if ev:
        got = np.array(ev)
        assert np.array_equal(got[:, 0], want[:, 0])
        _assert_close(got[:, 1:], want[:, 1:], 1e-13, 0.0, "event stresses")
    for f in ("status", "stiffness_scale", "damage", "plastic_strain", "sigma", "tau"):
        _assert_close(getattr(b, f), d[f"{mode}_out_{f}"], 1e-13, 0.0, f)


def test_broadphase_and_labels():
    d = load("broadphase_labels.npz")
    for tag in ("a", "b"):
        got = O.broad_phase(d[f"{tag}_pos"], d[f"{tag}_rad"], float(d[f"{tag}_cell"]))
        assert np.array_equal(got, d[f"{tag}_pairs"])

    class B:
        pass
    b = B()
    b.i, b.j, b.status = d["lab_i"], d["lab_j"], d["lab_status"]
    assert np.array_equal(O.components(int(d["lab_n"]), b), d["lab_labels"])


def _objective(d, tag):
    el = elements_from(d, f"{tag}_el_")
    b = bonds_from(d, f"{tag}_b_")
    hs = d[f"{tag}_hs"]
    return O.Objective(el, b, d[f"{tag}_pairs"], [HalfSpace(tuple(hs[:3]), hs[3])],
                       d[f"{tag}_gravity"], float(d[f"{tag}_kc"]), float(d[f"{tag}_ke"]),
                       float(d[f"{tag}_dt"]), d[f"{tag}_p_prev"], d[f"{tag}_q_prev"],
                       el.p.copy(), el.q.copy())


@pytest.mark.parametrize("tag", ["near", "rand"])
def test_newton_pieces(tag):
    d = load("newton_pieces.npz")
    obj = _objective(d, tag)
    p, q = d[f"{tag}_p"], d[f"{tag}_q"]
    f, gp, gq = obj.value_and_gradient(p, q)
    assert f == pytest.approx(float(d[f"{tag}_f"]), rel=1e-14)
    _assert_close(gp, d[f"{tag}_gp"], 1e-12, 1e-12 * np.abs(d[f"{tag}_gp"]).max(), "gp")
    _assert_close(gq, d[f"{tag}_gq"], 1e-12, 1e-12 * np.abs(d[f"{tag}_gq"]).max(), "gq")
    z = O.reduced_gradient(q, gp, gq, obj.free)
    _assert_close(z, d[f"{tag}_z"], 1e-12, 1e-12 * np.abs(z).max(), "z")
    pc = O.clamped_pieces(obj, p, q, gq)
    for key, ref in (("bond_pp", "bond_pp"), ("bond_rot", "bond_qq_red"),
                     ("pair_pp", "pair_pp"), ("elem_pos", "elem_pos"), ("elem_rot", "elem_rot")):
        want = d[f"{tag}_{ref}"]
        _assert_close(pc[key], want, 1e-11, 1e-12 * max(np.abs(want).max(), 1e-300), key)
    mat, diag = O.reduced_system(pc, obj.free)
    A = d[f"{tag}_A"]
    _assert_close(mat.toarray(), A, 1e-11, 1e-12 * np.abs(A).max(), "A")
    _assert_close(diag, d[f"{tag}_diag"], 1e-11, 1e-12 * np.abs(A).max(), "diag")
    pre = O.BlockJacobi(diag)
    _assert_close(pre.inv, d[f"{tag}_minv"], 1e-9, 1e-12 * np.abs(pre.inv).max(), "minv")
    tol = O.inner_tolerance(float(np.linalg.norm(z)))
    res = O.pcg(lambda v: mat @ v, -z, pre, tol, 2000)
    assert res.iterations == int(d[f"{tag}_pcg_it"])
    _assert_close(res.x, d[f"{tag}_pcg_x"], 1e-8, 1e-10 * np.abs(res.x).max(), "pcg x")
    assert obj.value(p, q) == pytest.approx(float(d[f"{tag}_value"]), rel=1e-14)


def test_newton_solve():
    d = load("newton_solve.npz")
    el = elements_from(d, "el_")
    b = bonds_from(d, "b_")
    hs = d["hs"]
    obj = O.Objective(el, b, d["pairs"], [HalfSpace(tuple(hs[:3]), hs[3])], d["gravity"],
                      float(d["kc"]), float(d["ke"]), float(d["dt"]), d["p_prev"], d["q_prev"],
                      el.p.copy(), el.q.copy())
    sol = O.newton(obj, d["p0"], d["q0"], O.Config(epsilon=float(d["epsilon"]),
                                                   max_iterations=200))
    assert sol.converged
    assert sol.iterations == int(d["solve_iterations"])
    assert sol.pcg_total == int(d["solve_pcg_total"])
    _assert_close(sol.p, d["solve_p"], 1e-10, 1e-12, "p")
    _assert_close(sol.q, d["solve_q"], 1e-10, 1e-12, "q")
    np.testing.assert_allclose([r.grad_norm for r in sol.records], d["solve_rec_gnorm"],
                               rtol=1e-6, atol=1e-9)


def _oracle_state(d, name, spec_driver=None):
    el = elements_from(d, "init_el_")
    b = bonds_from(d, "init_b_")
    plastic = PlasticParams(*d["plastic"]) if "plastic" in d else None
    cols = []
    if name == "plate":
        cols = [HalfSpace((0.0, 0.0, 1.0), 0.0)]
    if name == "stack":
        from paper_2308_10459_b200 import configs as C
        cols = C.stack().colliders
    return O.OracleState(el, b, float(d["dt"]), float(d["youngs"]), colliders=cols,
                         gravity=d["gravity"], k_contact=float(d["k_contact"]),
                         k_element=float(d["k_element"]), plastic=plastic, driver=spec_driver,
                         mu_s=float(d.get("mu_s", 0.0)), mu_r=float(d.get("mu_r", 0.0)))


@pytest.mark.parametrize("name", ["cantilever", "rope", "plate", "cube", "stack"])
def test_trajectory(name):
    from paper_2308_10459_b200 import configs as C
    d = load(f"traj_{name}.npz")
    driver, schedule = None, None
    if name == "rope":
        spec = C.rope(n=30)
        driver = TwistDriver(spec.driver.ids, spec.driver.p0, spec.driver.axis_point,
                             spec.driver.rate)
    if name == "cube":
        spec = C.cube(n_side=5, random_q=False, seed=3, youngs=3e8, k_contact=1e9, speed=2.0,
                      dt=1e-4)
        schedule = spec.collider_schedule
    st = _oracle_state(d, name, driver)
    cfg = O.Config(epsilon=float(d["epsilon"]), max_iterations=300)
    steps = d["p"].shape[0]
    events = []
    for s in range(steps):
        if schedule is not None:
            st.colliders = schedule(st.time + st.dt)
        out = O.step(st, cfg)
        assert out.committed == bool(d["committed"][s])
        events += [(s, b_, sg, tu) for (b_, sg, tu) in out.broken]
        el = st.elements
        scale = np.abs(d["p"][s]).max()
        _assert_close(el.p, d["p"][s], 1e-8, 1e-9 * scale, f"step {s} p")
        _assert_close(el.q, d["q"][s], 1e-8, 1e-9, f"step {s} q")
    ev = np.array(events, dtype=float).reshape(-1, 4)
    assert np.array_equal(ev[:, :2], d["events"][:, :2])
    assert np.array_equal(st.bonds.status, d["final_b_status"])


def test_sphere_box_colliders():
    from paper_2308_10459_b200.colliders import BoxCollider, SphereCollider
    d = load("colliders.npz")
    el = elements_from(d, "el_")
    b = bonds_from(d, "b_")
    sp, bx = d["sphere"], d["box"]
    cols = [SphereCollider(tuple(sp[:3]), float(sp[3])), BoxCollider(tuple(bx[:3]), tuple(bx[3:]))]
    obj = O.Objective(el, b, np.zeros((0, 2), dtype=np.int64), cols, d["gravity"],
                      float(d["kc"]), float(d["ke"]), float(d["dt"]), d["p_prev"], d["q_prev"],
                      el.p.copy(), el.q.copy())
    p, q = d["p"], d["q"]
    f, gp, gq = obj.value_and_gradient(p, q)
    assert f == pytest.approx(float(d["f"]), rel=1e-14)
    pc = O.clamped_pieces(obj, p, q, gq)
    _assert_close(pc["elem_pos"], d["elem_pos"], 1e-11, 1e-12 * np.abs(d["elem_pos"]).max(),
                  "elem_pos")
    mat, diag = O.reduced_system(pc, obj.free)
    _assert_close(diag, d["diag"], 1e-11, 1e-12 * np.abs(d["diag"]).max(), "diag")
    assert int(d["n_indef"]) > 0


def friction_inputs(d):
    """Host containers for friction.npz (contact.py:303-350 inputs)."""
    from paper_2308_10459_b200.colliders import BoxCollider, SphereCollider
    from paper_2308_10459_b200.state import ElementSet
    el = ElementSet(d["p"].copy(), d["q"].copy(), d["v"].copy(), d["qdot"].copy(),
                    d["mass"].copy(), d["radius"].copy(), d["pinned"].copy())
    hs, sp, bx = d["halfspace"], d["sphere"], d["box"]
    cols = [HalfSpace(tuple(hs[:3]), float(hs[3])), SphereCollider(tuple(sp[:3]), float(sp[3])),
            BoxCollider(tuple(bx[:3]), tuple(bx[3:]))]
    return el, cols


def test_friction_sweep():
    d = load("friction.npz")
    el, cols = friction_inputs(d)
    O.apply_friction(el, d["pairs"], cols, float(d["k_c"]), float(d["k_ec"]), float(d["mu_s"]),
                     float(d["mu_r"]), float(d["dt"]))
    _assert_close(el.v, d["v_out"], 1e-13, 1e-15, "v")
    _assert_close(el.qdot, d["qdot_out"], 1e-13, 1e-15, "qdot")
    assert not np.array_equal(d["v_out"], d["v"])          # the sweep did work
    assert np.array_equal(el.v[el.pinned], d["v"][el.pinned])


def test_mesh_drop_trajectory():
    """The reference's tet-mesh drop scene (friction, fracture) through the oracle."""
    from paper_2308_10459_b200 import configs as C
    d = load("mesh_drop.npz")
    spec = C.drop_fracture(tensile_strength=3e4, shear_strength=3e4)
    st = O.OracleState(spec.elements.copy(), spec.bonds.copy(), spec.dt, spec.youngs,
                       colliders=spec.colliders, gravity=d["gravity"], k_contact=spec.k_contact,
                       k_element=spec.k_element, mu_s=spec.mu_s, mu_r=spec.mu_r)
    cfg = O.Config(epsilon=float(d["epsilon"]), max_iterations=300)
    events = []
    for s in range(d["p"].shape[0]):
        out = O.step(st, cfg)
        assert out.committed == bool(d["committed"][s])
        events += [(s, b) for b, _, _ in out.broken]
        _assert_close(st.elements.p, d["p"][s], 1e-8, 1e-9, f"step {s} p")
        _assert_close(st.elements.q, d["q"][s], 1e-8, 1e-9, f"step {s} q")
    assert events == [(int(a), int(b)) for a, b, _, _ in d["events"]]
    assert np.array_equal(st.bonds.status, d["final_status"])


def test_newton_stall_twisted_beam():
    """The reference's max-iterations stall on the twist-driven lattice beam
    (SURVEY 8(d), C4 caution; stall_beam.npz made by the reference): the oracle
    reproduces the fixed point, the reason and the non-commit."""
    from paper_2308_10459_b200 import configs as C
    d = load("stall_beam.npz")
    drv = C.twisted_beam().driver
    st = _oracle_state(d, "twisted_beam",
                       TwistDriver(drv.ids, drv.p0, drv.axis_point, drv.rate))
    out = O.step(st, O.Config(epsilon=float(d["epsilon"]), max_iterations=300))
    s = out.solve
    assert not out.committed and s.reason == str(d["reason"]) == "max-iterations"
    assert s.iterations == int(d["iterations"])
    gn = np.array([r.grad_norm for r in s.records])
    assert np.all(np.abs(gn - d["rec_gnorm"]) <= 1e-6 * d["rec_gnorm"])
    assert abs(s.pcg_total - int(d["pcg_total"])) <= 2
    assert st.time == 0.0
    assert np.array_equal(st.elements.p, d["after_p"]) and np.array_equal(st.elements.q, d["after_q"])
