"""The reference's ImplicitProblem protocol on the B200 kernels
(``paper_2308_10459_b200.problem``, integrator.py:24-35, 39-138, 164-210).

``problem_protocol.npz`` was made by the reference (``make_golden.py``,
``gold_problem_protocol``) on a scene with every term: bonds (16 broken
across a crack), 9 touching contact pairs across the crack, a half-space, a
sphere and a box collider, pinned elements, perturbed orientations.
"""

from __future__ import annotations

import numpy as np
import pytest

from _fixtures import bonds_from, close, elements_from, load

pytestmark = pytest.mark.gpu


def _assert_close(a, b, rtol, atol, what):
    ok, info = close(a, b, rtol, atol)
    assert ok, f"{what}: got {info[0]!r} want {info[1]!r} at flat index {info[2]}"


def _problem(d):
    from paper_2308_10459_b200 import (BoxCollider, HalfSpace, ImplicitProblem, PotentialModel,
                                       SphereCollider, StepContext)
    el = elements_from(d, "el_")
    b = bonds_from(d, "b_")
    hs, sp, bx = d["hs"], d["sphere"], d["box"]
    cols = [HalfSpace(tuple(hs[:3]), float(hs[3])), SphereCollider(tuple(sp[:3]), float(sp[3])),
            BoxCollider(tuple(bx[:3]), tuple(bx[3:]))]
    model = PotentialModel(el, b, d["pairs"], cols, d["gravity"], float(d["kc"]),
                           float(d["ke"]))
    ctx = StepContext(float(d["dt"]), d["p_prev"], d["q_prev"], d["p_curr"], d["q_curr"])
    return model, ImplicitProblem(model, ctx)


def test_implicit_problem_protocol_vs_reference(cuda_ok):
    d = load("problem_protocol.npz")
    model, prob = _problem(d)
    p, q = d["p"], d["q"]
    assert prob.n == p.shape[0] and prob.free.sum() == (~d["el_pinned"]).sum()
    mp, mq = prob.inertia_diag()
    np.testing.assert_array_equal(mp, d["mp_dt2"])
    _assert_close(mq, d["mq_dt2"], 1e-15, 0.0, "mq_dt2")
    # objective and gradient: the gradient gather is the reference's np.add.at
    # order, so only per-bond arithmetic separates them
    assert prob.value(p, q) == pytest.approx(float(d["value"]), rel=1e-12)
    f, gp, gq = prob.value_and_gradient(p, q)
    assert f == pytest.approx(float(d["f"]), rel=1e-12)
    _assert_close(gp, d["gp"], 1e-9, 1e-11 * np.abs(d["gp"]).max(), "gp")
    _assert_close(gq, d["gq"], 1e-9, 1e-11 * np.abs(d["gq"]).max(), "gq")
    gp2, gq2 = prob.gradient(p, q)
    np.testing.assert_array_equal(gp2, gp)
    assert model.value(p, q) == pytest.approx(float(d["model_value"]), rel=1e-12)
    eb = model.energy_breakdown(p, q)
    for k in ("bond", "contact", "gravity"):
        assert eb[k] == pytest.approx(float(d[f"eb_{k}"]), rel=1e-11, abs=1e-300)
    # ambient Hessian blocks (bonds.py:473-504, contact.py:209-223, 243-247)
    hb = prob.hessian_blocks(p, q)
    np.testing.assert_array_equal(hb.bond_i, d["hb_bond_i"])
    np.testing.assert_array_equal(hb.bond_j, d["hb_bond_j"])
    for k in ("bond_pp", "bond_qq", "pair_pp", "elem_pp"):
        want = d[f"hb_{k}"]
        _assert_close(getattr(hb, k), want, 1e-10, 1e-12 * np.abs(want).max(), k)
    assert np.abs(hb.pair_pp).sum() > 0 and np.abs(hb.elem_pp).sum() > 0
    np.testing.assert_array_equal(hb.pair_i, d["pairs"][:, 0])


def test_reference_minimizer_on_b200_problem(cuda_ok):
    """The reference's own minimize_second_order (solver.py:511-562: its
    clamping, CSR assembly, block-Jacobi PCG and line search on the CPU) run on
    the B200-backed ImplicitProblem, on the converging step problem of
    ``newton_solve.npz`` (jittered cube split by a crack, contact pairs across
    it, a plane, pinned layer): it converges like the reference's own run, to
    the same iterate within the Newton termination bound eps/(m/dt^2), and
    its first iterations see the same gradient norms and PCG counts."""
    from oracle.ref_adapter import bdem_or_skip
    bdem_or_skip()
    from bdem import solver as rsv
    from paper_2308_10459_b200 import HalfSpace, ImplicitProblem, PotentialModel, StepContext
    d = load("newton_solve.npz")
    el = elements_from(d, "el_")
    b = bonds_from(d, "b_")
    hs = d["hs"]
    model = PotentialModel(el, b, d["pairs"], [HalfSpace(tuple(hs[:3]), float(hs[3]))],
                           d["gravity"], float(d["kc"]), float(d["ke"]))
    prob = ImplicitProblem(model, StepContext(float(d["dt"]), d["p_prev"], d["q_prev"],
                                              el.p.copy(), el.q.copy()))
    eps = float(d["epsilon"])
    sol = rsv.minimize_second_order(prob, d["p0"], d["q0"],
                                    rsv.SolverConfig(epsilon=eps, max_iterations=200))
    assert sol.converged
    assert abs(sol.iterations - int(d["solve_iterations"])) <= 10
    m_dt2 = (el.mass / float(d["dt"]) ** 2).min()
    _assert_close(sol.p, d["solve_p"], 1e-8, 10 * eps / m_dt2, "p")
    _assert_close(sol.q, d["solve_q"], 1e-8, 1e-9, "q")
    np.testing.assert_allclose([r.grad_norm for r in sol.records[:3]], d["solve_rec_gnorm"][:3],
                               rtol=1e-8)
    np.testing.assert_array_equal([r.pcg_iterations for r in sol.records[:3]],
                                  d["solve_rec_pcg"][:3])
