"""Drop-in adapters for code that still drives the reference package.

The reference's only registry is ``bdem.solver.MINIMIZERS``
(``/root/reference/pkg/src/bdem/solver.py:834-840``): ``stable_step`` calls
``MINIMIZERS[method](problem, p0, q0, cfg)`` with a numpy
``ImplicitProblem`` (``integrator.py:164-210``).  ``minimize_reference_problem``
accepts exactly that call, runs the Newton solve on the GPU and returns an
object with the reference ``SolveResult`` fields (numpy ``p``/``q``), so

    import bdem.solver
    from paper_2308_10459_b200.integration import register
    register(bdem.solver)
    bdem.solver.stable_step(scene, cfg, method="b200")

runs the reference orchestration with the B200 solve.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .device import DeviceSystem
from .newton import GPUProblem, minimize_second_order


@dataclass
class ReferenceSolveResult:
    """Field-for-field mirror of solver.py:63-73 with host arrays."""

    p: np.ndarray
    q: np.ndarray
    converged: bool
    iterations: int
    grad_norm: float
    records: list = field(default_factory=list)
    pcg_total: int = 0
    max_unit_dev: float = 0.0
    reason: str = "converged"


_CACHE: dict = {}


def _device_for(model):
    """One DeviceSystem per (bond set, element count); bond state refreshed."""
    key = (id(model.bonds), model.elements.n)
    dev = _CACHE.get(key)
    if dev is None:
        dev = DeviceSystem(elements=model.elements, bonds=model.bonds)
        _CACHE.clear()
        _CACHE[key] = dev
    else:
        dev.upload_elements(model.elements)
    dev.upload_bond_state(model.bonds)
    return dev


def minimize_reference_problem(problem, p0, q0, cfg):
    """``MINIMIZERS``-compatible GPU solve of a reference ``ImplicitProblem``."""
    model, ctx = problem.model, problem.ctx
    dev = _device_for(model)
    dev.set_physics(model.gravity, model.k_contact, model.k_element, model.colliders)
    dd = dev.device
    dev.p_hat.copy_(torch.from_numpy(np.ascontiguousarray(ctx.p_hat, dtype=np.float64)))
    dev.q_hat.copy_(torch.from_numpy(np.ascontiguousarray(ctx.q_hat, dtype=np.float64)))
    mp, mq = problem.inertia_diag()
    dev.mp_dt2.copy_(torch.from_numpy(np.ascontiguousarray(mp, dtype=np.float64)))
    dev.mq_dt2.copy_(torch.from_numpy(np.ascontiguousarray(mq, dtype=np.float64)))
    pairs = np.asarray(model.pairs, dtype=np.int32).reshape(-1, 2)
    dev.set_pairs(torch.from_numpy(pairs).to(dd))
    dev.reset_errors()
    res = minimize_second_order(GPUProblem(dev), torch.from_numpy(np.asarray(p0, float)).to(dd),
                                torch.from_numpy(np.asarray(q0, float)).to(dd), cfg)
    return ReferenceSolveResult(res.p.cpu().numpy(), res.q.cpu().numpy(), res.converged,
                                res.iterations, res.grad_norm, res.records, res.pcg_total,
                                res.max_unit_dev, res.reason)


def register(solver_module, name: str = "b200"):
    """Install the GPU solve into a reference ``MINIMIZERS`` registry."""
    solver_module.MINIMIZERS[name] = minimize_reference_problem
    return name
