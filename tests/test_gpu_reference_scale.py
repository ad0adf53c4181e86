"""Reference parity at BASELINE sizes (fixtures made by the reference itself).

* ``plate600k_newton.npz`` -- the north-star config (C3: 1000x600 plate,
  600,000 spheres, 3,591,004 bonds, eps 1e-3): the step-1 problem exactly as
  ``stable_step`` builds it (``solver.py:902-908``) and the first two Newton
  iterations of ``minimize_second_order`` (``solver.py:511-562``).  Checked:
  the contact-candidate count, the iteration records (f, |z|, alpha, PCG
  counts), the Newton direction y and the iterate after each iteration on a
  strided subsample of 604 rows.
* ``traj_rope100k.npz`` -- C4 at full size (100,000 spheres, G = 10 E, end
  twisted at 10 rad/s, eps 1e-5): five implicit steps.  This is the config
  whose quaternions move (twist driver, retraction, tangent-projected qdot);
  p, q, v, qdot on 333 rows incl. both ends, Newton/PCG counts, and the
  whole-array norms of q - 1 and qdot.
"""

from __future__ import annotations

import numpy as np
import pytest

from _fixtures import close, load

pytestmark = pytest.mark.gpu


def _assert_close(a, b, rtol, atol, what):
    ok, info = close(a, b, rtol, atol)
    assert ok, f"{what}: got {info[0]!r} want {info[1]!r} at flat index {info[2]}"


def test_plate600k_first_two_newton_iterations(cuda_ok):
    import torch

    from paper_2308_10459_b200 import SolverConfig, configs as C
    from paper_2308_10459_b200.newton import GPUProblem, minimize_second_order
    from paper_2308_10459_b200.scene import Scene
    from paper_2308_10459_b200.step import prepare_step
    g = load("plate600k_newton.npz")
    spec = C.plate()
    scene = Scene.from_spec(spec, host_sync=False)
    dev = scene.device
    assert dev.n == int(g["n"]) and dev.nb == int(g["n_bonds"])
    prep = prepare_step(scene)             # stable_step's prologue (solver.py:894-906)
    assert prep.n_pairs == int(g["n_pairs"])
    rows = g["rows"]
    rows_t = torch.as_tensor(rows).cuda()
    np.testing.assert_array_equal(dev.xp[rows_t].cpu().numpy(), g["p0"])
    np.testing.assert_array_equal(dev.xq[rows_t].cpu().numpy(), g["q0"])
    cols = torch.as_tensor(np.asarray(dev.slot_cols)[rows]).cuda()   # plate: all free
    seen = {"p": [], "q": [], "y": []}

    class Capture(GPUProblem):
        def assemble(self, p, q):
            seen["p"].append(p[rows_t].cpu().numpy())
            seen["q"].append(q[rows_t].cpu().numpy())
            return super().assemble(p, q)

        def dot(self, a, b, n):
            vs = self.dev.vstride
            seen["y"].append(self.dev.y[:6 * vs].reshape(6, vs)[:, cols].T.cpu().numpy())
            return super().dot(a, b, n)

    sol = minimize_second_order(Capture(dev), dev.xp, dev.xq,
                                SolverConfig(epsilon=float(g["epsilon"]), max_iterations=2))
    recs = sol.records
    assert [r.pcg_iterations for r in recs] == list(g["rec_pcg"])
    assert [r.alpha for r in recs] == list(g["rec_alpha"])
    np.testing.assert_allclose([r.f for r in recs], g["rec_f"], rtol=1e-12)
    np.testing.assert_allclose([r.grad_norm for r in recs], g["rec_gnorm"], rtol=1e-9)
    for k in range(2):
        y = np.asarray(seen["y"][k]).reshape(-1)
        _assert_close(y, g["y"][k].reshape(-1), 1e-9, 1e-12 * np.abs(g["y"][k]).max(), f"y {k}")
        # the iterate after Newton iteration k: compare the displacement from
        # the predictor so the tolerance is relative to what moved
        dp = seen["p"][k + 1] - g["p0"]
        _assert_close(dp, g["p"][k] - g["p0"], 1e-9, 1e-12 * np.abs(dp).max(), f"p {k}")
        _assert_close(seen["q"][k + 1], g["q"][k], 0.0, 1e-15, f"q {k}")


def test_rope100k_twist_vs_reference(cuda_ok):
    import torch

    from paper_2308_10459_b200 import SolverConfig, configs as C, stable_step
    from paper_2308_10459_b200.scene import Scene
    g = load("traj_rope100k.npz")
    spec = C.rope()
    scene = Scene.from_spec(spec, host_sync=False)
    dev = scene.device
    rows = torch.as_tensor(g["rows"]).cuda()
    cfg = SolverConfig(epsilon=float(g["epsilon"]), max_iterations=300)
    ident = torch.tensor([0.0, 0.0, 0.0, 1.0], dtype=torch.float64, device="cuda")
    for s in range(g["p"].shape[0]):
        rep = stable_step(scene, cfg)
        assert rep.committed == bool(g["committed"][s])
        assert rep.solve.iterations == int(g["newton"][s]), s
        assert abs(rep.solve.pcg_total - int(g["pcg"][s])) <= max(2, int(g["pcg"][s]) // 100)
        got = {k: getattr(dev, k)[rows].cpu().numpy() for k in ("p", "q", "v", "qdot")}
        # positions: SURVEY 8(a) rtol 1e-8 + eps/(m/dt^2)
        m_dt2 = float((spec.elements.mass / spec.dt**2).min())
        _assert_close(got["p"], g["p"][s], 1e-8, 10 * cfg.epsilon / m_dt2, f"p {s}")
        _assert_close(got["v"], g["v"][s], 1e-6, 10 * cfg.epsilon / m_dt2 / spec.dt, f"v {s}")
        # rotations: same Newton path as the reference, but ~300-700 PCG
        # iterations per solve at rtol min(0.5, sqrt|z|) leave iterate
        # differences of ~1e-10 (observed 1.2e-10 at step 3), four orders
        # below the Newton-termination bound eps / k_twist = 1.3e-6; q moves
        # up to 2.5e-3 here
        _assert_close(got["q"], g["q"][s], 1e-8, 1e-9, f"q {s}")
        _assert_close(got["qdot"], g["qdot"][s], 1e-8, 1e-9 / spec.dt, f"qdot {s}")
        qdev = float(torch.linalg.vector_norm(dev.q - ident))
        assert qdev == pytest.approx(float(g["q_dev_norm"][s]), rel=1e-7)
        qdn = float(torch.linalg.vector_norm(dev.qdot))
        assert qdn == pytest.approx(float(g["qdot_norm"][s]), rel=1e-6)
    assert float(g["q_dev_norm"][-1]) > 1e-3      # the rotation path really moved


def test_cube22_identity_q_vs_reference(cuda_ok):
    """BASELINE configs[1] at full size (22^3 = 10,648 jittered spheres,
    radii U(0.9r, 1.1r), plasticity and fracture, plane descending at 0.5
    m/s) in SURVEY 8(d)'s identity-q variant: the reference's first steps
    (``traj_cube22.npz``).  Positions rtol 1e-8 + 10 eps/(m/dt^2) on a
    strided subsample and as whole-array norms; the predictor's Newton record;
    the yield / fracture state of every bond exactly."""
    import torch

    from paper_2308_10459_b200 import SolverConfig, configs as C, stable_step
    from paper_2308_10459_b200.scene import Scene
    g = load("traj_cube22.npz")
    spec = C.cube(random_q=False, epsilon=float(g["epsilon"]))
    sched = spec.collider_schedule
    scene = Scene.from_spec(spec, host_sync=False)
    dev = scene.device
    assert dev.n == int(g["n"])
    rows = torch.as_tensor(g["rows"]).cuda()
    cfg = SolverConfig(epsilon=float(g["epsilon"]), max_iterations=300)
    m_dt2 = float((spec.elements.mass / spec.dt**2).min())
    atol_p = 10 * cfg.epsilon / m_dt2
    for s in range(g["p"].shape[0]):
        scene.colliders = sched(scene.time + scene.dt)
        rep = stable_step(scene, cfg)
        assert rep.committed == bool(g["committed"][s])
        r0 = rep.solve.records[0]     # at the predictor: same inputs up to the last step's tolerance
        assert r0.f == pytest.approx(float(g["rec0_f"][s]), rel=1e-9)
        assert r0.grad_norm == pytest.approx(float(g["rec0_gnorm"][s]), rel=1e-6)
        got_p = dev.p[rows].cpu().numpy()
        _assert_close(got_p, g["p"][s], 1e-8, atol_p, f"p {s}")
        _assert_close(dev.v[rows].cpu().numpy(), g["v"][s], 1e-6, atol_p / spec.dt, f"v {s}")
        assert float(torch.linalg.vector_norm(dev.p)) == pytest.approx(float(g["p_norm"][s]),
                                                                       rel=1e-10)
    scene.sync_to_host()
    b = scene.bonds
    np.testing.assert_array_equal(b.status, g["final_b_status"])
    for k in ("stiffness_scale", "damage", "plastic_strain"):
        _assert_close(getattr(b, k), g[f"final_b_{k}"], 1e-8, 1e-12, k)


def test_block_2m_bond_sample_vs_reference(cuda_ok):
    """BASELINE configs[4] at full size (C5: 126^3 jittered block, random unit
    q, 11.86M bonds): the B200 bond kernel against the reference's own
    BondSet.energy_terms on 1,000 of the block's bonds (``block_sample.npz``,
    made by the reference at the generator's state): energies, gradients and
    ambient Hessians at rtol 1e-10 plus atol 1e-12 x the bond's stiffness."""
    from paper_2308_10459_b200 import configs as C
    from paper_2308_10459_b200.state import BondSet
    g = load("block_sample.npz")
    spec = C.block(random_q=True)
    el, b = spec.elements, spec.bonds
    assert el.n == int(g["n"]) and b.n == int(g["n_bonds"])
    rows = g["rows"]
    np.testing.assert_array_equal(el.p[rows], g["p_rows"])   # same generator state
    np.testing.assert_array_equal(el.q[rows], g["q_rows"])
    pick = g["pick"]
    sub = BondSet(**{f: np.asarray(getattr(b, f))[pick] for f in b.__dataclass_fields__})
    got = sub.energy_terms(el.p, el.q, want_hess=True)
    np.testing.assert_array_equal(got[0], g["idx"])
    sc = sub.stiffness_scale
    kn = sc * sub.kn
    krot = sc * (sub.kt + sub.k_diag.sum(axis=1))
    l0 = sub.rest_length
    for name, got_, scale in zip(("E", "gpi", "gpj", "gqi", "gqj", "hpp", "hqq"), got[1:],
                                 (kn * l0**2 + krot, kn * l0 + krot, kn * l0 + krot, krot, krot,
                                  kn + krot, kn + krot)):
        want = g[name]
        atol = 1e-12 * scale.reshape((-1,) + (1,) * (want.ndim - 1))
        err = np.abs(got_ - want) - (1e-10 * np.abs(want) + atol)
        assert err.max() <= 0, f"{name}: worst excess {err.max():.3e}"
