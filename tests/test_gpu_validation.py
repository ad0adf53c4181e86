"""The reference's system-level validation battery (pkg/src/bdem/validate.py,
the only checks it has for solver.py / linalg.py / integrator.py)
restated on the CUDA path:

* manifold-gradient-direction (validate.py:308-331): the reduced gradient z
  paired with a reduced direction equals the central difference of the
  objective along the geodesics of that direction, h = 1e-6, tolerance 1e-6;
* manifold-hessian-quadratic (validate.py:334-360): y . A y of the assembled
  reduced operator equals the geodesic second difference, h = 1e-4, tolerance
  1e-3 -- on a state where the SPD clamps change the operator by far less
  than that (every bond in tension: the stretch clamp is inactive; rotations
  of 1e-5: the eigen-clamp only removes negative eigenvalues of relative size
  ~theta), so that the clamped operator is the Riemannian Hessian to 1e-5;
* pcg-vs-dense (validate.py:375-386) and the reduced Newton direction
  (validate.py:363-372): the device PCG against a dense solve of the operator
  read out column by column with bdem_spmv, tolerance 1e-8.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _system(spec, dp_noise, dq_noise, seed, dilate=0.0):
    """The step-1 problem of `spec` at a perturbed point (validate._small_problem)."""
    import torch

    from paper_2308_10459_b200.scene import Scene
    from paper_2308_10459_b200.step import prepare_step
    scene = Scene.from_spec(spec, host_sync=False)
    prob = prepare_step(scene).problem
    dev = scene.device
    g = torch.Generator(device="cuda").manual_seed(seed)
    free = torch.as_tensor(dev.free_np, device="cuda")
    rn = lambda *s: torch.randn(*s, generator=g, dtype=torch.float64, device="cuda")  # noqa: E731
    if dilate:
        c = dev.xp.mean(dim=0, keepdim=True)
        # pinned rows too: they only enter as the fixed ends of their bonds
        dev.xp.copy_(c + (1.0 + dilate) * (dev.xp - c))
    dev.xp.add_(dp_noise * rn(dev.n, 3) * free[:, None])
    dev.xq.add_(dq_noise * rn(dev.n, 4) * free[:, None])
    dev.xq.div_(dev.xq.norm(dim=1, keepdim=True))
    torch.cuda.synchronize()
    return scene, dev, prob, g


def _unit_direction(dev, g):
    """A reduced direction with unit position and unit rotation blocks on every
    free element (so every geodesic step is well above the retraction's
    small-step shortcut, as in the reference's check)."""
    import torch
    y = torch.zeros(6, dev.vstride, dtype=torch.float64, device="cuda")
    a = torch.randn(3, dev.nf, generator=g, dtype=torch.float64, device="cuda")
    b = torch.randn(3, dev.nf, generator=g, dtype=torch.float64, device="cuda")
    y[:3, :dev.nf] = a / a.norm(dim=0, keepdim=True)
    y[3:, :dev.nf] = b / b.norm(dim=0, keepdim=True)
    return y.reshape(-1)


def test_manifold_gradient_direction(cuda_ok):
    from paper_2308_10459_b200 import configs
    scene, dev, prob, g = _system(configs.cube(n_side=6), 0.002 * 0.002, 0.02, seed=3)
    prob.assemble(dev.xp, dev.xq)
    n6 = 6 * dev.vstride
    h, worst = 1e-6, 0.0
    for _ in range(24):
        y = _unit_direction(dev, g)
        an = prob.dot(dev.z, y, n6)
        prob.direction(dev.xq, y, 1.0)
        fp = prob.trial_value(dev.xp, dev.xq, dev.dp, dev.dq, h, dev.tp, dev.tq)
        fm = prob.trial_value(dev.xp, dev.xq, dev.dp, dev.dq, -h, dev.tp, dev.tq)
        fd = (fp - fm) / (2.0 * h)
        worst = max(worst, abs(fd - an) / max(abs(fd), 1e-9))
    assert worst < 1e-6, worst


def test_manifold_hessian_quadratic_where_clamps_are_negligible(cuda_ok):
    import torch

    from paper_2308_10459_b200 import configs
    # every bond stretched by 0.1% (c / l > 0: the stretch clamp is inactive),
    # rotations of 1e-5 rad (clamped eigenvalues are ~1e-5 of the block)
    spec = configs.cube(n_side=6, random_q=False)
    scene, dev, prob, g = _system(spec, 0.0, 1e-5, seed=4, dilate=1e-3)
    prob.assemble(dev.xp, dev.xq)
    kc = dev.stage[0]                                  # BDEM_ST_KC = k c per bond position
    live = dev.status != 2
    assert bool((kc[live] > 0).all())
    n6 = 6 * dev.vstride
    f0 = prob.value(dev.xp, dev.xq)
    h, worst = 1e-4, 0.0
    ay = torch.zeros(n6, dtype=torch.float64, device="cuda")
    # scale the unit blocks to the lattice: steps of h x 1e-3 x spacing keep
    # every bond in tension along the whole stencil
    r = float(spec.elements.radius.mean())
    for _ in range(16):
        y = _unit_direction(dev, g)
        y.view(6, -1)[:3] *= 1e-3 * r
        dev.call("bdem_spmv", dev.sysp, y.data_ptr(), ay.data_ptr(), dev.stream)
        quad = float(torch.dot(y, ay))
        prob.direction(dev.xq, y, 1.0)
        fp = prob.trial_value(dev.xp, dev.xq, dev.dp, dev.dq, h, dev.tp, dev.tq)
        fm = prob.trial_value(dev.xp, dev.xq, dev.dp, dev.dq, -h, dev.tp, dev.tq)
        fd = (fp - 2.0 * f0 + fm) / (h * h)
        worst = max(worst, abs(fd - quad) / max(abs(fd), 1e-9))
    assert worst < 1e-3, worst


def _dense_operator(dev):
    """The assembled reduced operator, column by column through bdem_spmv."""
    import torch
    nf, vs = dev.nf, dev.vstride
    idx = (torch.arange(6, device="cuda")[:, None] * vs + torch.arange(nf, device="cuda")[None, :])
    idx = idx.reshape(-1)                               # reduced index -> padded plane index
    m = idx.numel()
    a = torch.zeros(m, m, dtype=torch.float64, device="cuda")
    x = torch.zeros(6 * vs, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
    for k in range(m):
        x[idx[k]] = 1.0
        dev.call("bdem_spmv", dev.sysp, x.data_ptr(), y.data_ptr(), dev.stream)
        a[:, k] = y[idx]
        x[idx[k]] = 0.0
    torch.cuda.synchronize()
    return a.cpu().numpy(), idx


@pytest.mark.parametrize("name", ["cube_random_q", "rope"])
def test_pcg_and_newton_direction_vs_dense_solve(cuda_ok, name):
    from paper_2308_10459_b200 import configs
    spec = {"cube_random_q": lambda: configs.cube(n_side=5),
            "rope": lambda: configs.rope(n=120)}[name]()
    scene, dev, prob, g = _system(spec, 0.0, 0.02 if name == "rope" else 0.0, seed=6)
    prob.assemble(dev.xp, dev.xq)
    a, idx = _dense_operator(dev)
    assert np.abs(a - a.T).max() <= 1e-12 * np.abs(a).max()
    assert np.linalg.eigvalsh(a).min() > 0.0            # sum of clamped PSD pieces + inertia
    res = prob.solve_pcg(1e-10, 20 * a.shape[0])
    assert res.converged
    b = -dev.z[idx].cpu().numpy()
    exact = np.linalg.solve(a, b)
    got = dev.y[idx].cpu().numpy()
    assert np.linalg.norm(got - exact) / np.linalg.norm(exact) < 1e-8
