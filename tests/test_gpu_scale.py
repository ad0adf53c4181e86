"""Full-size GPU checks (BASELINE configs C3 at 600K and C5 at 2M spheres)
through size-independent properties, plus sampled kernel parity at C5 scale.

* the reduced Newton operator is symmetric and positive definite
  (sum of clamped PSD blocks + mass terms, solver.py:141-258);
* the reduced gradient z matches a central finite difference of the
  incremental potential along a random position direction (integrator.py:191-200);
* one full implicit step commits with Armijo-monotone objective values
  (solver.py:387-406, 511-562);
* C5 (random q): a 1e5-bond sample of the batched bond terms matches the
  oracle at the per-bond tolerance (SURVEY §8(d) "sampled kernel parity").
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _predicted_system(spec, k_element=None):
    import torch

    from paper_2308_10459_b200.scene import Scene
    from paper_2308_10459_b200.step import prepare_step
    scene = Scene.from_spec(spec, host_sync=False)
    if k_element is not None:
        scene.k_element = k_element
    prep = prepare_step(scene)            # stable_step's prologue: predictor in xp, xq
    torch.cuda.synchronize()
    return scene, scene.device, prep.problem


def _operator_checks(dev, seed):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    n6 = 6 * dev.vstride
    mask = torch.zeros(6, dev.vstride, dtype=torch.float64, device="cuda")
    mask[:, :dev.nf] = 1.0
    mask = mask.reshape(-1)
    x1 = torch.randn(n6, generator=g, dtype=torch.float64, device="cuda") * mask
    x2 = torch.randn(n6, generator=g, dtype=torch.float64, device="cuda") * mask
    y1, y2 = torch.zeros_like(x1), torch.zeros_like(x2)
    dev.call("bdem_spmv", dev.sysp, x1.data_ptr(), y1.data_ptr(), dev.stream)
    dev.call("bdem_spmv", dev.sysp, x2.data_ptr(), y2.data_ptr(), dev.stream)
    a = float(torch.dot(x2, y1))
    b = float(torch.dot(x1, y2))
    scale = float(torch.linalg.vector_norm(x1) * torch.linalg.vector_norm(y2))
    assert abs(a - b) <= 1e-12 * scale, (a, b)
    assert float(torch.dot(x1, y1)) > 0.0 and float(torch.dot(x2, y2)) > 0.0


def test_plate_600k_operator_and_gradient(cuda_ok):
    import torch

    from paper_2308_10459_b200 import configs
    spec = configs.plate(epsilon=1e-3)
    scene, dev, prob = _predicted_system(spec)
    assert dev.n == 600_000 and dev.nb == 3_591_004
    f0, gnorm, _, _ = prob.assemble(dev.xp, dev.xq)
    assert np.isfinite(f0) and gnorm > 0
    _operator_checks(dev, 1)
    # z . d  vs  (f(p + h d) - f(p - h d)) / 2h along a random position direction
    g = torch.Generator(device="cuda").manual_seed(2)
    dp = torch.randn(dev.n, 3, generator=g, dtype=torch.float64, device="cuda") * 1e-3
    dq = torch.zeros(dev.n, 4, dtype=torch.float64, device="cuda")
    y = torch.zeros(6, dev.vstride, dtype=torch.float64, device="cuda")
    free = torch.as_tensor(dev.free_ids_np, device="cuda")
    slot = torch.as_tensor(dev.slot_np[dev.free_ids_np], device="cuda").long()
    y[:3, slot] = dp[free].T
    slope = prob.dot(dev.z, y.reshape(-1), 6 * dev.vstride)
    h = 1e-6
    fp = prob.trial_value(dev.xp, dev.xq, dp, dq, h, dev.tp, dev.tq)
    fm = prob.trial_value(dev.xp, dev.xq, dp, dq, -h, dev.tp, dev.tq)
    fd = (fp - fm) / (2 * h)
    assert fd == pytest.approx(slope, rel=1e-5)


def test_plate_600k_step_commits_monotone(cuda_ok):
    from paper_2308_10459_b200 import SolverConfig, configs, stable_step
    from paper_2308_10459_b200.scene import Scene
    spec = configs.plate(epsilon=1e-3)
    scene = Scene.from_spec(spec, host_sync=False)
    rep = stable_step(scene, SolverConfig(epsilon=1e-3, max_iterations=300))
    assert rep.committed and rep.solve.converged
    fs = [r.f for r in rep.solve.records]
    assert all(b <= a + 8 * np.finfo(float).eps * abs(a) for a, b in zip(fs, fs[1:]))
    assert rep.solve.records[-1].grad_norm < 1e-3
    scene.sync_to_host()
    assert np.all(np.isfinite(scene.elements.p))
    # identity orientations stay exactly identity
    assert np.array_equal(scene.elements.q, np.tile([0.0, 0.0, 0.0, 1.0], (dev_n(scene), 1)))


def dev_n(scene):
    return scene.elements.n


def test_block_2m_random_q_operator_and_sampled_parity(cuda_ok):
    from oracle import cpu_oracle as O
    from paper_2308_10459_b200 import configs
    from paper_2308_10459_b200.state import BondSet
    spec = configs.block(random_q=True)
    scene, dev, prob = _predicted_system(spec, k_element=0.0)
    assert dev.n == 126**3 and dev.nb > 11_000_000
    f0, gnorm, _, _ = prob.assemble(dev.xp, dev.xq)
    assert np.isfinite(f0)
    _operator_checks(dev, 3)
    # sampled kernel parity: 1e5 bonds of the block against the oracle
    rng = np.random.default_rng(5)
    b = spec.bonds
    pick = np.sort(rng.choice(b.n, 100_000, replace=False))
    sub = BondSet(**{f: np.asarray(getattr(b, f))[pick] for f in b.__dataclass_fields__})
    p = dev.xp.cpu().numpy()
    q = dev.xq.cpu().numpy()
    got = sub.energy_terms(p, q, want_hess=True)
    ref = O.bond_eval(sub, p, q, want_hess=True)
    sc = sub.stiffness_scale
    kn = sc * sub.kn
    krot = sc * (sub.kt + sub.k_diag.sum(axis=1))
    l0 = sub.rest_length
    for g_, r_, s_ in zip(got[1:], (ref.energy, ref.gp_i, ref.gp_j, ref.gq_i, ref.gq_j,
                                    ref.h_pp, ref.h_qq),
                          (kn * l0**2 + krot, kn * l0 + krot, kn * l0 + krot, krot, krot,
                           kn + krot, kn + krot)):
        atol = 1e-12 * s_.reshape((-1,) + (1,) * (r_.ndim - 1))
        err = np.abs(g_ - r_) - (1e-10 * np.abs(r_) + atol)
        assert err.max() <= 0, f"worst excess {err.max():.3e}"
