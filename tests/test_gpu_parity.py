"""GPU parity: the CUDA path against the reference's golden vectors and the
CPU oracle on identical seeded inputs.  All calls go through the C ABI.

Tolerances (north star): per-bond energy/gradient/Hessian rtol 1e-10 with an
absolute floor of 1e-12 x the bond's stiffness scale (cancellation near
rest); trajectories rtol 1e-8 with atol >= eps/(m/dt^2) (Newton termination);
broken-bond sets bit-exact away from thresholds.
"""

import numpy as np
import pytest

from _fixtures import bonds_from, close, elements_from, load

pytestmark = pytest.mark.gpu


def _assert_close(a, b, rtol, atol, what):
    ok, info = close(a, b, rtol, atol)
    assert ok, f"{what}: got {info[0]!r} want {info[1]!r} at flat index {info[2]}"


def _bond_scales(b, idx):
    sc = b.stiffness_scale[idx]
    kn = sc * b.kn[idx]
    krot = sc * (b.kt[idx] + b.k_diag[idx].sum(axis=1))
    l0 = b.rest_length[idx]
    return kn, krot, l0


# ---------------------------------------------------------------------------
# per-bond kernels (bonds.py:151-323, 473-504)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("case", ["randq", "nearq", "ident"])
def test_bond_terms_vs_golden(cuda_ok, case):
    d = load("bond_terms.npz")
    b = bonds_from(d, "b_")
    got = b.energy_terms(d["p"], d[f"{case}_q"], want_hess=True)
    idx = d[f"{case}_idx"]
    assert np.array_equal(got[0], idx)
    kn, krot, l0 = _bond_scales(b, idx)
    e_sc = kn * l0**2 + krot
    g_sc = np.maximum(kn * l0, krot)
    h_sc = np.maximum(kn, krot)
    names = ("E", "gpi", "gpj", "gqi", "gqj", "hpp", "hqq")
    scales = (e_sc, g_sc, g_sc, g_sc, g_sc, h_sc, h_sc)
    for k, (name, sc) in enumerate(zip(names, scales)):
        want = d[f"{case}_{name}"]
        atol = 1e-12 * sc.reshape((-1,) + (1,) * (want.ndim - 1))
        err = np.abs(got[k + 1] - want) - (1e-10 * np.abs(want) + atol)
        assert err.max() <= 0, f"{case}/{name}: worst excess {err.max():.3e}"


def test_bond_terms_closed_forms(cuda_ok):
    """Known answers from the reference's tests (tests/test_bonds.py):
    1% stretch energy, shear 1/2 k phi^2, pure twist 1/2 k sin^2(phi/2)."""
    from paper_2308_10459_b200 import configs as C
    from paper_2308_10459_b200 import quat as Q
    pos = np.array([[0.0, 0.0, 0.0], [0.1, 0.0, 0.0]])
    rad = np.array([0.02, 0.02])
    b = C.build_bonds(pos, rad, np.array([[0, 1]]), 1e7, 4e6)
    kn, kt, ktw = b.kn[0], b.kt[0], b.k_diag[0, 0]
    # stretch 1%
    p = np.array([[0.0, 0, 0], [0.101, 0, 0]])
    q = np.tile(Q.IDENTITY, (2, 1))
    e = b.energy_terms(p, q)[1][0]
    assert e == pytest.approx(0.5 * kn * (0.01 * 0.1) ** 2, rel=1e-12)
    # shear: common rotation about an axis perpendicular to d0
    for phi in (0.05, 0.3, 1.2):
        qq = np.tile(Q.axis_angle([0, 1, 0], phi), (2, 1))
        e = b.energy_terms(pos, qq)[1][0]
        assert e == pytest.approx(0.5 * kt * phi**2, rel=1e-10)
    # pure relative twist about the bond axis: the mean rotation is a twist
    # too, so the shear term vanishes and E = 1/2 k_twist sin^2(phi/2)
    for phi in (0.1, 0.6, 1.5):
        qq = np.stack([Q.axis_angle([1, 0, 0], phi), Q.IDENTITY])
        e = b.energy_terms(pos, qq)[1][0]
        assert e == pytest.approx(0.5 * ktw * np.sin(phi / 2) ** 2, rel=1e-10)


def test_degenerate_and_antipodal_raise(cuda_ok):
    from paper_2308_10459_b200 import DegenerateBondError, DegenerateShearError
    from paper_2308_10459_b200 import configs as C
    from paper_2308_10459_b200 import quat as Q
    pos = np.array([[0.0, 0.0, 0.0], [0.1, 0.0, 0.0]])
    b = C.build_bonds(pos, np.array([0.02, 0.02]), np.array([[0, 1]]), 1e7, 4e6)
    q = np.tile(Q.IDENTITY, (2, 1))
    with pytest.raises(DegenerateBondError):
        b.energy_terms(np.zeros((2, 3)), q)
    qa = np.array([[0.1, 0.2, 0.3, 0.9], [-0.1, -0.2, -0.3, -0.9]])
    with pytest.raises(DegenerateShearError):
        b.energy_terms(pos, qa)


def test_bond_terms_large_random_vs_oracle(cuda_ok):
    """Full C2-size batch (22^3 jittered cube, random q) against the oracle."""
    from oracle import cpu_oracle as O
    from paper_2308_10459_b200 import configs as C
    spec = C.cube()
    rng = np.random.default_rng(9)
    b = spec.bonds
    b.stiffness_scale[:] = rng.uniform(0.3, 1.0, b.n)
    p = spec.elements.p + 1e-5 * rng.normal(size=spec.elements.p.shape)
    q = spec.elements.q
    got = b.energy_terms(p, q, want_hess=True)
    ref = O.bond_eval(b, p, q, want_hess=True)
    kn, krot, l0 = _bond_scales(b, ref.idx)
    for g, r, sc in zip(got[1:], (ref.energy, ref.gp_i, ref.gp_j, ref.gq_i, ref.gq_j, ref.h_pp,
                                  ref.h_qq),
                        (kn * l0**2 + krot, kn * l0 + krot, kn * l0 + krot, krot, krot,
                         kn + krot, kn + krot)):
        atol = 1e-12 * sc.reshape((-1,) + (1,) * (r.ndim - 1))
        err = np.abs(g - r) - (1e-10 * np.abs(r) + atol)
        assert err.max() <= 0, f"worst excess {err.max():.3e}"


# ---------------------------------------------------------------------------
# assembly, clamp, block-Jacobi, SpMV, PCG (solver.py:116-258, linalg.py)
# ---------------------------------------------------------------------------

def _gpu_problem(d, tag):
    import torch
    from paper_2308_10459_b200.colliders import HalfSpace
    from paper_2308_10459_b200.device import DeviceSystem
    from paper_2308_10459_b200.newton import GPUProblem
    el = elements_from(d, f"{tag}_el_")
    b = bonds_from(d, f"{tag}_b_")
    dev = DeviceSystem(elements=el, bonds=b)
    hs = d[f"{tag}_hs"]
    dev.set_physics(d[f"{tag}_gravity"], float(d[f"{tag}_kc"]), float(d[f"{tag}_ke"]),
                    [HalfSpace(tuple(hs[:3]), hs[3])])
    dev.p_prev.copy_(torch.from_numpy(d[f"{tag}_p_prev"]))
    dev.q_prev.copy_(torch.from_numpy(d[f"{tag}_q_prev"]))
    dev.set_pairs(torch.as_tensor(d[f"{tag}_pairs"].astype(np.int32)).cuda().reshape(-1, 2))
    dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(),
             dev.qdot.data_ptr(), dev.p_prev.data_ptr(), dev.q_prev.data_ptr(),
             float(d[f"{tag}_dt"]), dev.p_hat.data_ptr(), dev.q_hat.data_ptr(),
             dev.mp_dt2.data_ptr(), dev.mq_dt2.data_ptr(), dev.tp.data_ptr(), dev.tq.data_ptr(),
             dev.stream)
    dev.xp.copy_(torch.from_numpy(d[f"{tag}_p"]))
    dev.xq.copy_(torch.from_numpy(d[f"{tag}_q"]))
    return dev, GPUProblem(dev)


def _aos(t, dev):
    """Reduced device vector (6 planes of stride vstride, slots in SELL row
    order) -> 6 per free element in ascending id (the oracle's order)."""
    vs = dev.vstride
    return t[:6 * vs].reshape(6, vs)[:, dev.slot_cols].T.reshape(-1).cpu().numpy()


def _soa(a, dev):
    import torch
    vs, nf = dev.vstride, dev.nf
    out = np.zeros((6, vs))
    out[:, dev.slot_cols] = a.reshape(nf, 6).T
    return torch.from_numpy(out).reshape(-1).cuda()


def _sym6_to_mat(s):
    m = np.empty(s.shape[:-1] + (3, 3))
    idx = [(0, 0, 0), (1, 0, 1), (2, 0, 2), (3, 1, 1), (4, 1, 2), (5, 2, 2)]
    for t, r, c in idx:
        m[..., r, c] = s[..., t]
        m[..., c, r] = s[..., t]
    return m


@pytest.mark.parametrize("tag", ["near", "rand"])
def test_assembly_vs_golden(cuda_ok, tag):
    import torch
    from paper_2308_10459_b200 import _lib as L
    d = load("newton_pieces.npz")
    dev, prob = _gpu_problem(d, tag)
    # production path: i-role pieces summed by the bond pass's row threads
    f0, g0, _, _ = prob.assemble(dev.xp, dev.xq)
    kpre = dev.ikpre[:dev.n].clone()
    ref = [t.clone() for t in (dev.z, dev.diag, dev.minv)]
    if tag == "rand":   # random q: every rotation block goes through the eigen-clamp
        assert int(dev.counter[5]) > 0
        assert bool((kpre[(dev.ipart[L.IP["E"], :dev.n] != 0)] >= 0).all())
    # every (i,i) quadrant staged (ikpre = 0) so the blocks can be read back;
    # the element pass then sums them itself: same bits
    dev.sys.asm_flags = L.ASM_STAGE_ALL_A
    f, gnorm, cnorm, _ = prob.assemble(dev.xp, dev.xq)
    dev.sys.asm_flags = 0
    assert (f, gnorm) == (f0, g0)
    for a, b_ in zip(ref, (dev.z, dev.diag, dev.minv)):
        assert torch.equal(a, b_)
    assert f == pytest.approx(float(d[f"{tag}_f"]), rel=1e-12)
    assert gnorm == pytest.approx(float(d[f"{tag}_gnorm"]), rel=1e-10)
    z = _aos(dev.z, dev)
    _assert_close(z, d[f"{tag}_z"], 1e-9, 1e-11 * np.abs(z).max(), "z")
    # clamped bond blocks against build_clamped_pieces (active bonds)
    b = bonds_from(d, f"{tag}_b_")
    act = np.nonzero(b.status != 2)[0]
    st = dev.stage.cpu().numpy()[:, dev.sell.pos_of_bond]
    cf = dev.coef_planes().cpu().numpy()[:, dev.sell.pos_of_bond]   # AoSoA-32 -> planes
    n = cf[L.CF["N"]:L.CF["N"] + 3].T[act]
    al, be = cf[L.CF["ALPHA"]][act], cf[L.CF["BETA"]][act]
    apos = al[:, None, None] * n[:, :, None] * n[:, None, :] + be[:, None, None] * np.eye(3)
    want_pp = d[f"{tag}_bond_pp"]
    hs = np.abs(want_pp).max()
    _assert_close(apos, want_pp[:, :3, :3], 1e-10, 1e-12 * hs, "a+ (ii)")
    _assert_close(-apos, want_pp[:, :3, 3:], 1e-10, 1e-12 * hs, "-a+ (ij)")
    rot = d[f"{tag}_bond_qq_red"]
    hr = np.abs(rot).max()
    A = _sym6_to_mat(st[L.ST["A"]:L.ST["A"] + 6].T[act])
    D = _sym6_to_mat(st[L.ST["D"]:L.ST["D"] + 6].T[act])
    Cb = cf[L.CF["C"]:L.CF["C"] + 9].T[act].reshape(-1, 3, 3)
    _assert_close(A, rot[:, :3, :3], 1e-9, 1e-11 * hr, "rot (ii)")
    _assert_close(D, rot[:, 3:, 3:], 1e-9, 1e-11 * hr, "rot (jj)")
    _assert_close(Cb, rot[:, :3, 3:], 1e-9, 1e-11 * hr, "rot (ij)")
    # diagonal blocks and block-Jacobi inverses
    diag = dev.diag[:, dev.slot_cols].cpu().numpy().T
    P, R = _sym6_to_mat(diag[:, :6]), _sym6_to_mat(diag[:, 6:])
    want = d[f"{tag}_diag"]
    sc = np.abs(want).max()
    _assert_close(P, want[:, :3, :3], 1e-9, 1e-11 * sc, "diag pos")
    _assert_close(R, want[:, 3:, 3:], 1e-9, 1e-11 * sc, "diag rot")
    minv = dev.minv[:, dev.slot_cols].cpu().numpy().T
    wm = d[f"{tag}_minv"]
    _assert_close(_sym6_to_mat(minv[:, :6]), wm[:, :3, :3], 1e-7, 1e-9 * np.abs(wm).max(), "Pinv")
    _assert_close(_sym6_to_mat(minv[:, 6:]), wm[:, 3:, 3:], 1e-7, 1e-9 * np.abs(wm).max(), "Rinv")
    # SpMV against the reference's assembled CSR (as dense)
    Adense = d[f"{tag}_A"]
    rng = np.random.default_rng(3)
    x = rng.normal(size=Adense.shape[0])
    xd = _soa(x, dev)
    yd = torch.zeros_like(xd)
    dev.call("bdem_spmv", dev.sysp, xd.data_ptr(), yd.data_ptr(), dev.stream)
    want_y = Adense @ x
    _assert_close(_aos(yd, dev), want_y, 1e-9, 1e-11 * np.abs(want_y).max(), "A x")
    # PCG at the reference's inner tolerance
    res = prob.solve_pcg(float(d[f"{tag}_pcg_tol"]), 2000)
    assert abs(res.iterations - int(d[f"{tag}_pcg_it"])) <= 1
    y = _aos(dev.y, dev)
    if res.iterations == int(d[f"{tag}_pcg_it"]):
        _assert_close(y, d[f"{tag}_pcg_x"], 1e-6, 1e-8 * np.abs(y).max(), "pcg x")
    # tight solve is path independent: compare to the exact solution
    res = prob.solve_pcg(1e-10, 2000)
    y = _aos(dev.y, dev)
    _assert_close(y, d[f"{tag}_pcg_tight_x"], 1e-7, 1e-9 * np.abs(y).max(), "tight pcg x")
    # objective value at the iterate
    val = prob.value(dev.xp, dev.xq)
    assert val == pytest.approx(float(d[f"{tag}_value"]), rel=1e-12)


def test_newton_solve_vs_golden(cuda_ok):
    """A full minimize_second_order (96 Newton iterations, contact pairs across
    a crack, a plane, pinned layer) against the reference's solution: final
    iterates agree to the Newton termination tolerance eps/(m/dt^2)."""
    import torch
    from paper_2308_10459_b200 import HalfSpace, SolverConfig, minimize_second_order
    from paper_2308_10459_b200.device import DeviceSystem
    from paper_2308_10459_b200.newton import GPUProblem
    d = load("newton_solve.npz")
    el = elements_from(d, "el_")
    b = bonds_from(d, "b_")
    dev = DeviceSystem(elements=el, bonds=b)
    hs = d["hs"]
    dev.set_physics(d["gravity"], float(d["kc"]), float(d["ke"]),
                    [HalfSpace(tuple(hs[:3]), hs[3])])
    dev.p_prev.copy_(torch.from_numpy(d["p_prev"]))
    dev.q_prev.copy_(torch.from_numpy(d["q_prev"]))
    dev.set_pairs(torch.as_tensor(d["pairs"].astype(np.int32)).cuda().reshape(-1, 2))
    dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(),
             dev.qdot.data_ptr(), dev.p_prev.data_ptr(), dev.q_prev.data_ptr(),
             float(d["dt"]), dev.p_hat.data_ptr(), dev.q_hat.data_ptr(),
             dev.mp_dt2.data_ptr(), dev.mq_dt2.data_ptr(), dev.tp.data_ptr(), dev.tq.data_ptr(),
             dev.stream)
    # the predictor kernel reproduces predict_state exactly
    _assert_close(dev.tp.cpu().numpy(), d["p0"], 1e-15, 0.0, "p0")
    _assert_close(dev.tq.cpu().numpy(), d["q0"], 1e-15, 1e-16, "q0")
    sol = minimize_second_order(GPUProblem(dev), torch.from_numpy(d["p0"]).cuda(),
                                torch.from_numpy(d["q0"]).cuda(),
                                SolverConfig(epsilon=float(d["epsilon"]), max_iterations=200))
    assert sol.converged
    assert abs(sol.iterations - int(d["solve_iterations"])) <= 10
    m_dt2 = (el.mass / float(d["dt"]) ** 2).min()
    atol = 10 * float(d["epsilon"]) / m_dt2
    _assert_close(sol.p.cpu().numpy(), d["solve_p"], 1e-8, atol, "p")
    _assert_close(sol.q.cpu().numpy(), d["solve_q"], 1e-8, 1e-9, "q")
    # the first Newton iterations see identical inputs: same PCG counts and gnorm
    gn = [r.grad_norm for r in sol.records[:3]]
    np.testing.assert_allclose(gn, d["solve_rec_gnorm"][:3], rtol=1e-8)


# ---------------------------------------------------------------------------
# step level (solver.py:881-939)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["cantilever", "rope", "plate", "cube", "stack"])
def test_trajectory_vs_golden(cuda_ok, name):
    from paper_2308_10459_b200 import HalfSpace, PlasticParams, Scene, SolverConfig, stable_step
    from paper_2308_10459_b200 import configs as C
    from paper_2308_10459_b200.scene import TwistDriver
    d = load(f"traj_{name}.npz")
    el = elements_from(d, "init_el_")
    b = bonds_from(d, "init_b_")
    driver, sched, cols = None, None, []
    if name == "rope":
        spec = C.rope(n=30)
        driver = TwistDriver(spec.driver.ids, spec.driver.p0, spec.driver.axis_point,
                             spec.driver.rate)
    if name == "cube":
        spec = C.cube(n_side=5, random_q=False, seed=3, youngs=3e8, k_contact=1e9, speed=2.0,
                      dt=1e-4)
        sched = spec.collider_schedule
    if name == "plate":
        cols = [HalfSpace((0.0, 0.0, 1.0), 0.0)]
    if name == "stack":
        cols = C.stack().colliders
    plastic = PlasticParams(*d["plastic"]) if "plastic" in d else None
    scene = Scene(name, None, el, b, colliders=cols, gravity=d["gravity"], dt=float(d["dt"]),
                  youngs=float(d["youngs"]), k_contact=float(d["k_contact"]),
                  k_element=float(d["k_element"]), plastic=plastic, driver=driver,
                  mu_s=float(d.get("mu_s", 0.0)), mu_r=float(d.get("mu_r", 0.0)))
    cfg = SolverConfig(epsilon=float(d["epsilon"]), max_iterations=300)
    # positions rtol 1e-8 with atol >= eps / (min m / dt^2) to
    # absorb Newton-termination differences.  Rotations:
    # * cantilever / plate / cube: q stays exactly identity -- equal;
    # * rope (twist driver, the rotating config): GPU and reference take the
    #   same Newton path (same iteration and PCG counts every step), so q is
    #   held to rtol 1e-8 + atol 1e-10 (q moves 5e-4 per step) and qdot to
    #   rtol 1e-8 + atol 1e-10 / dt;
    # * stack (friction, spinning blocks): the Newton path diverges at the
    #   termination tolerance after a few steps (PCG 105 vs 91 at step 6), so
    #   the honest bound is eps over the smallest rotational Hessian stiffness
    #   (bend/twist k_diag + inertia), not the rotational inertia alone.
    dt = float(d["dt"])
    eps = float(d["epsilon"])
    m_dt2 = (el.mass / dt**2).min()
    atol_p = max(10 * eps / m_dt2, 1e-12)
    if name == "rope":
        atol_q, rtol_q = 1e-10, 1e-8
    elif name == "stack":
        k_rot = float(np.min(b.k_diag)) + float((1.6 * el.mass * el.radius**2 / dt**2).min())
        atol_q, rtol_q = 10 * eps / k_rot, 1e-8
    else:
        atol_q, rtol_q = 0.0, 0.0
    events = []
    n_newton = []
    for s in range(d["p"].shape[0]):
        if sched is not None:
            scene.colliders = sched(scene.time + scene.dt)
        rep = stable_step(scene, cfg)
        assert rep.committed == bool(d["committed"][s])
        n_newton.append(rep.solve.iterations)
        # the first Newton record is evaluated at the predictor (p0, q0): it
        # pins the predictor's retraction, which the converged state cannot
        # see (Newton erases its starting point)
        # (rope: same Newton path, 1e-10 -- a 1e-9 perturbation of the
        # predictor's retraction step fails it, profiles/r02/README.md;
        # cantilever/plate/cube: the previous step's converged state differs
        # at its Newton tolerance, ~2e-9 relative in the predictor gradient;
        # stack: the Newton path diverges, ~4e-8)
        r0 = rep.solve.records[0]
        rt = {"rope": 1e-10, "stack": 1e-6}.get(name, 1e-8)
        g0 = float(d["rec0_gnorm"][s])
        assert abs(r0.grad_norm - g0) <= rt * abs(g0), (s, r0.grad_norm, g0)
        events += [(s, bb) for (bb, _, _) in rep.broken]
        _assert_close(scene.elements.p, d["p"][s], 1e-8, atol_p, f"step {s} p")
        _assert_close(scene.elements.q, d["q"][s], rtol_q, atol_q, f"step {s} q")
        _assert_close(scene.elements.v, d["v"][s], 1e-6, atol_p / dt, f"step {s} v")
        _assert_close(scene.elements.qdot, d["qdot"][s], rtol_q, atol_q / dt, f"step {s} qdot")
    if name in ("cantilever", "rope", "plate", "cube"):
        assert n_newton == [int(k) for k in d["newton"]]
    assert [tuple(e) for e in events] == [(int(a), int(bb)) for a, bb, _, _ in d["events"]]
    assert np.array_equal(scene.bonds.status, d["final_b_status"])


@pytest.mark.parametrize("mode", ["plastic", "elastic"])
def test_fracture_vs_golden(cuda_ok, mode):
    from paper_2308_10459_b200 import PlasticParams, update_bond_states
    d = load("fracture.npz")
    b = bonds_from(d, "b_")
    pl = PlasticParams(*d["plastic"]) if mode == "plastic" else None
    ev = update_bond_states(b, d["p"], d["q"], 1e9, pl)
    want = d[f"{mode}_events"]
    assert [e[0] for e in ev] == [int(x) for x in want[:, 0]]
    if ev:
        _assert_close(np.array([e[1:] for e in ev]), want[:, 1:], 1e-12, 0.0, "event stresses")
    for f in ("stiffness_scale", "damage", "plastic_strain", "sigma", "tau"):
        _assert_close(getattr(b, f), d[f"{mode}_out_{f}"], 1e-12, 0.0, f)
    assert np.array_equal(b.status, d[f"{mode}_out_status"])


def test_broadphase_and_components_vs_golden(cuda_ok):
    from paper_2308_10459_b200 import broad_phase, label_components
    d = load("broadphase_labels.npz")
    for tag in ("a", "b"):
        got = broad_phase(d[f"{tag}_pos"], d[f"{tag}_rad"], float(d[f"{tag}_cell"]))
        assert np.array_equal(got, d[f"{tag}_pairs"])

    class B:
        pass
    b = B()
    b.i, b.j, b.status = d["lab_i"], d["lab_j"], d["lab_status"]
    lab = label_components(int(d["lab_n"]), b)
    assert np.array_equal(lab.labels, d["lab_labels"])


def test_reference_minimizers_adapter(cuda_ok):
    """integration.minimize_reference_problem accepts the reference's
    ImplicitProblem shape (solver.py:834-840 MINIMIZERS seam) and reproduces
    the reference's solution of the golden solve."""
    from paper_2308_10459_b200 import HalfSpace, SolverConfig
    from paper_2308_10459_b200.integration import minimize_reference_problem
    d = load("newton_solve.npz")
    el = elements_from(d, "el_")
    b = bonds_from(d, "b_")
    hs = d["hs"]
    dt = float(d["dt"])

    class Model:                      # PotentialModel fields (integrator.py:46-54)
        pass
    model = Model()
    model.elements, model.bonds, model.pairs = el, b, d["pairs"]
    model.colliders = [HalfSpace(tuple(hs[:3]), hs[3])]
    model.gravity, model.k_contact, model.k_element = d["gravity"], float(d["kc"]), float(d["ke"])

    class Ctx:                        # StepContext (integrator.py:141-161)
        pass
    ctx = Ctx()
    ctx.p_hat = 2.0 * el.p - d["p_prev"]
    ctx.q_hat = 2.0 * el.q - d["q_prev"]

    class Problem:                    # ImplicitProblem (integrator.py:164-210)
        free = ~el.pinned

        def inertia_diag(self):
            mp = np.where(self.free, el.mass / dt**2, 0.0)
            mq = np.where(self.free, 1.6 * el.mass * el.radius**2 / dt**2, 0.0)
            return mp, mq
    prob = Problem()
    prob.model, prob.ctx = model, ctx
    res = minimize_reference_problem(prob, d["p0"], d["q0"],
                                     SolverConfig(epsilon=float(d["epsilon"]),
                                                  max_iterations=200))
    assert res.converged and isinstance(res.p, np.ndarray)
    atol = 10 * float(d["epsilon"]) / (el.mass / dt**2).min()
    _assert_close(res.p, d["solve_p"], 1e-8, atol, "p")


def test_spmv_matches_oracle_csr_random_q(cuda_ok):
    """Reduced matrix-vector product on a 22^3 random-q cube (every rotation
    block indefinite -> Jacobi clamp) against the oracle's assembled CSR."""
    import torch
    from oracle import cpu_oracle as O
    from paper_2308_10459_b200 import configs as C
    from paper_2308_10459_b200.device import DeviceSystem
    from paper_2308_10459_b200.newton import GPUProblem
    spec = C.cube(seed=13, random_q=True)
    el, b = spec.elements, spec.bonds
    rng = np.random.default_rng(13)
    el.v[:] = 0.05 * rng.normal(size=el.v.shape)
    dev = DeviceSystem(elements=el, bonds=b)
    dev.set_physics(spec.gravity, spec.k_contact, 0.0, spec.colliders)
    p_prev = el.p - spec.dt * el.v
    dev.p_prev.copy_(torch.from_numpy(p_prev))
    dev.q_prev.copy_(torch.from_numpy(el.q))
    dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(),
             dev.qdot.data_ptr(), dev.p_prev.data_ptr(), dev.q_prev.data_ptr(), spec.dt,
             dev.p_hat.data_ptr(), dev.q_hat.data_ptr(), dev.mp_dt2.data_ptr(),
             dev.mq_dt2.data_ptr(), dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream)
    prob = GPUProblem(dev)
    f, gnorm, _, _ = prob.assemble(dev.xp, dev.xq)
    obj = O.Objective(el, b, np.zeros((0, 2), dtype=np.int64), spec.colliders, spec.gravity,
                      spec.k_contact, 0.0, spec.dt, p_prev, el.q.copy(), el.p.copy(), el.q.copy())
    p, q = dev.xp.cpu().numpy(), dev.xq.cpu().numpy()
    fo, gp, gq = obj.value_and_gradient(p, q)
    assert f == pytest.approx(fo, rel=1e-11)
    pc = O.clamped_pieces(obj, p, q, gq)
    mat, _ = O.reduced_system(pc, obj.free)
    x = rng.normal(size=mat.shape[0])
    xd = _soa(x, dev)
    yd = torch.zeros_like(xd)
    dev.call("bdem_spmv", dev.sysp, xd.data_ptr(), yd.data_ptr(), dev.stream)
    want = mat @ x
    _assert_close(_aos(yd, dev), want, 1e-9, 1e-10 * np.abs(want).max(), "A x (random q)")


def test_sphere_box_colliders_vs_golden(cuda_ok):
    """Sphere and box penalties (contact.py:61-133, 227-248): values, gradient
    and the clamped element position blocks (8 of them indefinite before the
    clamp), diagonal blocks and A x against the reference."""
    import torch
    from paper_2308_10459_b200 import BoxCollider, SphereCollider
    from paper_2308_10459_b200.device import DeviceSystem
    from paper_2308_10459_b200.newton import GPUProblem
    d = load("colliders.npz")
    el = elements_from(d, "el_")
    b = bonds_from(d, "b_")
    dev = DeviceSystem(elements=el, bonds=b)
    sp, bx = d["sphere"], d["box"]
    dev.set_physics(d["gravity"], float(d["kc"]), float(d["ke"]),
                    [SphereCollider(tuple(sp[:3]), float(sp[3])),
                     BoxCollider(tuple(bx[:3]), tuple(bx[3:]))])
    dev.p_prev.copy_(torch.from_numpy(d["p_prev"]))
    dev.q_prev.copy_(torch.from_numpy(d["q_prev"]))
    dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(),
             dev.qdot.data_ptr(), dev.p_prev.data_ptr(), dev.q_prev.data_ptr(), float(d["dt"]),
             dev.p_hat.data_ptr(), dev.q_hat.data_ptr(), dev.mp_dt2.data_ptr(),
             dev.mq_dt2.data_ptr(), dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream)
    _assert_close(dev.xp.cpu().numpy(), d["p"], 1e-15, 0.0, "p0")
    prob = GPUProblem(dev)
    f, gnorm, _, _ = prob.assemble(dev.xp, dev.xq)
    assert f == pytest.approx(float(d["f"]), rel=1e-12)
    _assert_close(_aos(dev.z, dev), d["z"], 1e-9, 1e-11 * np.abs(d["z"]).max(), "z")
    diag = dev.diag[:, dev.slot_cols].cpu().numpy().T
    want = d["diag"]
    sc = np.abs(want).max()
    _assert_close(_sym6_to_mat(diag[:, :6]), want[:, :3, :3], 1e-9, 1e-11 * sc, "diag pos")
    x = np.random.default_rng(4).normal(size=want.shape[0] * 6)
    xd = _soa(x, dev)
    yd = torch.zeros_like(xd)
    dev.call("bdem_spmv", dev.sysp, xd.data_ptr(), yd.data_ptr(), dev.stream)
    wy = d["A"] @ x
    _assert_close(_aos(yd, dev), wy, 1e-9, 1e-11 * np.abs(wy).max(), "A x")
    assert prob.value(dev.xp, dev.xq) == pytest.approx(float(d["value"]), rel=1e-12)


@pytest.mark.parametrize("tag,maxit", [("plain", 300), ("retry", 4)])
def test_runner_stats_vs_golden(cuda_ok, tmp_path, tag, maxit):
    """run_simulation with dt-halving retries and the bdem-stats-1 CSV
    (runner.py:20-164) against the reference's own stats.csv."""
    import io

    from paper_2308_10459_b200 import SolverConfig, configs
    from paper_2308_10459_b200.runner import read_stats_csv, run_simulation
    from paper_2308_10459_b200.scene import Scene
    d = load("runner.npz")
    scene = Scene.from_spec(configs.cantilever(nx=10, ny=3, nz=3))
    run_simulation(scene, SolverConfig(epsilon=1e-7, max_iterations=maxit), frames=3, fps=500,
                   outdir=tmp_path, write_meshes=False)
    ref_path = tmp_path / "ref.csv"
    ref_path.write_text(str(d[f"{tag}_csv"]))
    got = read_stats_csv(tmp_path / "stats.csv")
    want = read_stats_csv(ref_path)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g["frame"] == w["frame"] and g["time"] == w["time"]      # same dt sums, exact
        assert g["intact_bonds"] == w["intact_bonds"] and g["bonds_broken"] == w["bonds_broken"]
        assert abs(g["newton_iterations"] - w["newton_iterations"]) <= 1
        for k in ("kinetic", "bond_energy", "gravity_energy"):
            assert g[k] == pytest.approx(w[k], rel=1e-6, abs=1e-15)
    _assert_close(scene.elements.p, d[f"{tag}_p"], 1e-8, 1e-9, "final p")


def test_runner_step_failure(cuda_ok):
    from paper_2308_10459_b200 import SolverConfig, configs
    from paper_2308_10459_b200.runner import StepFailure, run_simulation
    from paper_2308_10459_b200.scene import Scene
    d = load("runner.npz")
    scene = Scene.from_spec(configs.cantilever(nx=10, ny=3, nz=3))
    with pytest.raises(StepFailure) as exc:
        run_simulation(scene, SolverConfig(epsilon=1e-7, max_iterations=3), frames=3, fps=500,
                       write_meshes=False)
    assert str(exc.value) == str(d["fail_msg"])


# ---------------------------------------------------------------------------
# post-step friction (contact.py:303-350) through the C-ABI
# ---------------------------------------------------------------------------

def test_friction_sweep_vs_golden(cuda_ok):
    import torch

    from paper_2308_10459_b200 import Scene
    from paper_2308_10459_b200 import configs as C
    from test_oracle_golden import friction_inputs
    d = load("friction.npz")
    el, cols = friction_inputs(d)
    b = C.build_bonds(el.p, el.radius, np.zeros((0, 2), dtype=np.int64), 1e7, 4e6)
    scene = Scene("friction", None, el, b, colliders=cols, k_contact=float(d["k_c"]),
                  k_element=float(d["k_ec"]), host_sync=False)
    dev = scene.device
    dev.set_physics(scene.gravity, scene.k_contact, scene.k_element, cols)
    dev.set_pairs(torch.as_tensor(d["pairs"], dtype=torch.int32, device="cuda"))
    before = dev.lib.bdem_launch_count()
    waves = dev.friction(float(d["mu_s"]), float(d["mu_r"]), float(d["dt"]))
    torch.cuda.synchronize()
    assert dev.lib.bdem_launch_count() > before
    assert 1 < waves < d["pairs"].shape[0]            # chained, yet parallel
    _assert_close(dev.v.cpu().numpy(), d["v_out"], 1e-12, 1e-14, "v")
    _assert_close(dev.qdot.cpu().numpy(), d["qdot_out"], 1e-12, 1e-14, "qdot")
    # mu = 0 is a no-op, like the reference
    v0 = dev.v.clone()
    dev.friction(0.0, 0.0, float(d["dt"]))
    assert torch.equal(v0, dev.v)


def test_friction_large_wave_path_vs_oracle(cuda_ok):
    """A contact set whose first wave exceeds the single-CTA threshold
    (kWaveBig = 8192 pairs), so the grid-wide wave launch runs as well as the
    single-CTA runs of small waves."""
    import ctypes

    import torch

    from oracle import cpu_oracle as O
    from paper_2308_10459_b200 import Scene
    from paper_2308_10459_b200 import configs as C
    from paper_2308_10459_b200.colliders import HalfSpace
    from paper_2308_10459_b200.state import ElementSet
    rng = np.random.default_rng(91)
    n = 40_000
    pos = rng.uniform(-2e-4, 2e-4, size=(n, 3))        # every listed pair touches
    rad = np.full(n, 0.001)
    el = ElementSet(pos, O.unit(rng.normal(size=(n, 4))), rng.normal(size=(n, 3)),
                    rng.normal(size=(n, 4)) * 0.1, np.full(n, 1e-5), rad, rng.random(n) < 0.02)
    k = np.arange(n // 2)
    pairs = np.concatenate([np.stack([2 * k, 2 * k + 1], 1), np.stack([k, k + n // 2], 1)])
    pairs = pairs[np.lexsort((pairs[:, 1], pairs[:, 0]))].astype(np.int32)
    cols = [HalfSpace((0.0, 0.0, 1.0), 0.0)]
    ref = el.copy()
    O.apply_friction(ref, pairs, cols, 1e5, 1e5, 0.4, 0.1, 1e-4)
    b = C.build_bonds(pos, rad, np.zeros((0, 2), dtype=np.int64), 1e7, 4e6)
    scene = Scene("cluster", None, el, b, colliders=cols, k_contact=1e5, k_element=1e5,
                  host_sync=False)
    dev = scene.device
    order = np.zeros(pairs.shape[0], dtype=np.int32)
    wptr = np.zeros(pairs.shape[0] + 1, dtype=np.int32)
    depth = dev.lib.bdem_friction_schedule(pairs.ctypes.data_as(ctypes.c_void_p), pairs.shape[0],
                                           n, order.ctypes.data_as(ctypes.c_void_p),
                                           wptr.ctypes.data_as(ctypes.c_void_p))
    assert np.diff(wptr[:depth + 1]).max() >= 8192 and depth > 2
    dev.set_physics(scene.gravity, 1e5, 1e5, cols)
    dev.set_pairs(torch.as_tensor(pairs, device="cuda"))
    assert dev.friction(0.4, 0.1, 1e-4) == depth
    _assert_close(dev.v.cpu().numpy(), ref.v, 1e-12, 1e-14, "v")
    _assert_close(dev.qdot.cpu().numpy(), ref.qdot, 1e-12, 1e-14, "qdot")


# ---------------------------------------------------------------------------
# PCG execution paths (rotation-free) against the default path
# ---------------------------------------------------------------------------

def _assembled(spec, k_element=None):
    from paper_2308_10459_b200.newton import GPUProblem
    from paper_2308_10459_b200.scene import Scene
    from paper_2308_10459_b200.step import prepare_step
    scene = Scene.from_spec(spec, host_sync=False)
    if k_element is not None:
        scene.k_element = k_element
    prepare_step(scene)
    dev = scene.device
    GPUProblem(dev).assemble(dev.xp, dev.xq)
    return dev


@pytest.mark.parametrize("case", ["plate", "rope"])
def test_rot_skip_bit_identical(cuda_ok, case):
    """Rotation-free PCG (bdem_pcg_set_rot_skip): on the plate (identity
    orientations, centre-based contact: the rotation half of every Newton
    right-hand side is exactly zero) the skipped solve gives bit-identical
    trajectories; on the twisted rope the rotation half is non-zero, the
    flag stays off and the results are the same path."""
    from paper_2308_10459_b200 import SolverConfig, stable_step
    from paper_2308_10459_b200 import _lib as L
    from paper_2308_10459_b200 import configs as C
    from paper_2308_10459_b200.scene import Scene
    lib = L.load()
    eps = 1e-6 if case == "plate" else 1e-5
    out = []
    for skip in (0, 1):
        prev = lib.bdem_pcg_set_rot_skip(skip)
        try:
            # a fresh spec per run: the scene steps the spec's arrays in place
            spec = C.plate(nx=60, ny=36, epsilon=1e-6) if case == "plate" else C.rope(n=200)
            scene = Scene.from_spec(spec)
            recs, flags = [], []
            for _ in range(4):
                rep = stable_step(scene, SolverConfig(epsilon=eps, max_iterations=200))
                recs.append((rep.committed, rep.solve.iterations, rep.solve.pcg_total))
                flags.append(float(scene.device.pcg_state[L.PCG["ROTZERO"]].item()))
        finally:
            lib.bdem_pcg_set_rot_skip(prev)
        out.append((recs, flags, scene.elements.p.copy(), scene.elements.q.copy(),
                    scene.elements.v.copy()))
    (r0, f0, p0, q0, v0), (r1, f1, p1, q1, v1) = out
    assert r0 == r1 and sum(r[2] for r in r0) > 0
    assert np.array_equal(p0, p1) and np.array_equal(q0, q1) and np.array_equal(v0, v1)
    assert all(f == 0.0 for f in f0)
    assert all(f == (1.0 if case == "plate" else 0.0) for f in f1)


def test_rot_skip_with_fracture(cuda_ok):
    """Rotation-free PCG on the identity-q cube crushed by a descending plane
    (bonds break): the same trajectory, fracture events and Newton/PCG counts,
    bit for bit, as the default path."""
    from paper_2308_10459_b200 import SolverConfig, stable_step
    from paper_2308_10459_b200 import _lib as L
    from paper_2308_10459_b200 import configs as C
    from paper_2308_10459_b200.scene import Scene
    lib = L.load()
    out = []
    for skip in (0, 1):
        prev_s = lib.bdem_pcg_set_rot_skip(skip)
        try:
            spec = C.cube(n_side=6, random_q=False, seed=3, youngs=3e8, k_contact=1e9, speed=2.0,
                          dt=1e-4)
            scene = Scene.from_spec(spec)
            recs, events, flags = [], [], []
            for _ in range(6):
                scene.colliders = spec.collider_schedule(scene.time + scene.dt)
                rep = stable_step(scene, SolverConfig(epsilon=1e-6, max_iterations=300))
                recs.append((rep.committed, rep.solve.iterations, rep.solve.pcg_total))
                events.append([b for (b, _, _) in rep.broken])
                flags.append(float(scene.device.pcg_state[L.PCG["ROTZERO"]].item()))
        finally:
            lib.bdem_pcg_set_rot_skip(prev_s)
        out.append((recs, events, scene.elements.p.copy(), scene.elements.q.copy(), flags))
    (r0, e0, p0, q0, f0), (r1, e1, p1, q1, f1) = out
    assert r0 == r1 and e0 == e1
    assert np.array_equal(p0, p1) and np.array_equal(q0, q1)
    # the run exercised what it is named for: bonds broke and the rotation
    # half was skipped
    assert sum(len(e) for e in e0) > 0
    assert all(f == 0.0 for f in f0) and all(f == 1.0 for f in f1)


def test_assembly_rows_with_mixed_clamp(cuda_ok):
    """Rows whose first i-role blocks pass the PSD certificate and a later one
    goes through the eigen-clamp (ikpre > 0): the bond pass folds the PSD
    prefix into the row sums and stages the rest, the element pass continues
    the sum.  Identity orientations with every third element turned to a
    random orientation give such rows; z, diag and minv must be bit-identical
    to the run that stages every (i,i) quadrant (ikpre = 0)."""
    import torch
    from paper_2308_10459_b200 import _lib as L
    from paper_2308_10459_b200 import configs as C
    spec = C.cube(n_side=5, random_q=False, seed=5)
    rng = np.random.default_rng(5)
    q = spec.elements.q
    turned = np.arange(0, q.shape[0], 3)
    r = rng.normal(size=(turned.size, 4))
    q[turned] = r / np.linalg.norm(r, axis=1, keepdims=True)
    dev = _assembled(spec)
    from paper_2308_10459_b200.newton import GPUProblem
    prob = GPUProblem(dev)
    f0, g0, _, _ = prob.assemble(dev.xp, dev.xq)
    kpre = dev.ikpre[:dev.n].cpu().numpy()
    assert int(dev.counter[5]) > 0
    assert (kpre > 0).sum() > 0 and (kpre < 0).sum() > 0, np.bincount(kpre + 1)
    ref = [t.clone() for t in (dev.z, dev.diag, dev.minv)]
    dev.sys.asm_flags = L.ASM_STAGE_ALL_A
    try:
        f1, g1, _, _ = prob.assemble(dev.xp, dev.xq)
    finally:
        dev.sys.asm_flags = 0
    assert (f0, g0) == (f1, g1)
    for a, b_ in zip(ref, (dev.z, dev.diag, dev.minv)):
        assert torch.equal(a, b_)
