"""The reference's incremental-potential protocol on the GPU.

``PotentialModel``, ``StepContext``, ``ImplicitProblem`` and
``PotentialBlocks`` mirror ``/root/reference/pkg/src/bdem/integrator.py``
(lines 24-35, 39-138, 141-161, 164-210): numpy arrays in and out, the same
names, shapes and semantics, so any minimizer written against the
reference's protocol (``problem.free``, ``.n``, ``value``,
``value_and_gradient``, ``gradient``, ``hessian_blocks``, ``inertia_diag``;
e.g. ``bdem.solver.minimize_second_order`` itself) runs on the B200 kernels
unchanged.  Every evaluation is a kernel of this library:

* ``value``               -> ``bdem_element_energy`` + ``bdem_bond_energy`` +
                             ``bdem_pair_assemble(energy_only)``
* ``value_and_gradient``  -> ``bdem_bond_assemble`` + ``bdem_element_assemble``
                             with ``sys->grad_p/grad_q`` set (the ordered
                             ``np.add.at`` gather, integrator.py:95-109, 195-200)
* ``hessian_blocks``      -> ``bdem_bond_eval_ambient`` (6x6 / 8x8 per bond) +
                             ``bdem_contact_blocks`` (pairs, colliders)

The state is uploaded on every call and the bond state (status, stiffness
scale) is re-read from the ``BondSet``, like the reference reads its arrays
live; this is the host-array protocol, not the device-resident production
path (``stable_step`` / ``newton.GPUProblem``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .bond_api import energy_terms

F64 = torch.float64


@dataclass
class PotentialBlocks:
    """integrator.py:24-35: second-derivative blocks keyed by element ids."""

    bond_i: np.ndarray
    bond_j: np.ndarray
    bond_pp: np.ndarray          # (nb, 6, 6) positions of (i, j)
    bond_qq: np.ndarray          # (nb, 8, 8) quaternions of (i, j)
    pair_i: np.ndarray
    pair_j: np.ndarray
    pair_pp: np.ndarray          # (np, 6, 6) self-contact position blocks
    elem_pp: np.ndarray          # (n, 3, 3) collider contact blocks


class PotentialModel:
    """integrator.py:39-138: bonds + frozen contact pairs + colliders + gravity."""

    def __init__(self, elements, bonds, pairs, colliders, gravity, k_contact: float,
                 k_element: float):
        from .device import DeviceSystem
        self.elements = elements
        self.bonds = bonds
        self.pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
        self.colliders = list(colliders)
        self.gravity = np.asarray(gravity, dtype=float)
        self.k_contact = k_contact
        self.k_element = k_element
        self.dev = dev = DeviceSystem(elements=elements, bonds=bonds)
        dev.set_physics(self.gravity, k_contact, k_element, self.colliders)
        dev.set_pairs(torch.as_tensor(self.pairs.astype(np.int32)).to(dev.device).reshape(-1, 2))
        n = dev.n
        self._zero_n = np.zeros(n)
        self._grad_p = torch.zeros((n, 3), dtype=F64, device=dev.device)
        self._grad_q = torch.zeros((n, 4), dtype=F64, device=dev.device)

    # -- device state for one evaluation
    def _load(self, p, q, mp_dt2, mq_dt2, p_hat, q_hat):
        d = self.dev
        for name, arr in (("xp", p), ("xq", q), ("mp_dt2", mp_dt2), ("mq_dt2", mq_dt2),
                          ("p_hat", p_hat), ("q_hat", q_hat)):
            getattr(d, name).copy_(torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)))
        if d.nb:
            d.upload_bond_state(self.bonds)
        d.reset_errors()

    def _value(self, p, q, mp_dt2, mq_dt2, p_hat, q_hat) -> float:
        self._load(p, q, mp_dt2, mq_dt2, p_hat, q_hat)
        d = self.dev
        s, st = d.sysp, d.stream
        d.call("bdem_element_energy", s, d.xp.data_ptr(), d.xq.data_ptr(), 1, st)
        d.call("bdem_bond_energy", s, d.xp.data_ptr(), d.xq.data_ptr(), L.SC["EBOND"], st)
        d.call("bdem_pair_assemble", s, d.xp.data_ptr(), 1, st)
        d.call("bdem_reduce_finish", s, L.SC["FT"], 7, L.RED_BLOCKS, st)
        d.eval_pq = (d.xp, d.xq)
        sc = d.read_scalars()
        return float(sc[L.SC["FT"]]) + (((float(sc[L.SC["EBOND"]]) + float(sc[L.SC["EPAIR"]]))
                                         + float(sc[L.SC["ECOL"]])) + float(sc[L.SC["EGRAV"]]))

    def _value_and_gradient(self, p, q, mp_dt2, mq_dt2, p_hat, q_hat):
        self._load(p, q, mp_dt2, mq_dt2, p_hat, q_hat)
        d = self.dev
        s, st = d.sysp, d.stream
        d.sys.grad_p, d.sys.grad_q = self._grad_p.data_ptr(), self._grad_q.data_ptr()
        try:
            if d.nb:
                d.call("bdem_bond_assemble", s, d.xp.data_ptr(), d.xq.data_ptr(), st)
            if d.n_pair:
                d.call("bdem_pair_assemble", s, d.xp.data_ptr(), 0, st)
            d.call("bdem_element_assemble", s, d.xp.data_ptr(), d.xq.data_ptr(), d.z.data_ptr(),
                   st)
            d.call("bdem_reduce_finish", s, 0, 7, L.RED_BLOCKS, st)
            d.eval_pq = (d.xp, d.xq)
            sc = d.read_scalars()
        finally:
            d.sys.grad_p = d.sys.grad_q = None
        return float(sc[L.SC["F"]]), self._grad_p.cpu().numpy(), self._grad_q.cpu().numpy()

    # -- the reference's PotentialModel API (no inertia)
    def value(self, p, q) -> float:
        z = self._zero_n
        return self._value(p, q, z, z, p, q)

    def value_and_gradient(self, p, q):
        z = self._zero_n
        return self._value_and_gradient(p, q, z, z, p, q)

    def gradient(self, p, q):
        _, gp, gq = self.value_and_gradient(p, q)
        return gp, gq

    def hessian_blocks(self, p, q) -> PotentialBlocks:
        d = self.dev
        if d.nb:
            d.upload_bond_state(self.bonds)
        idx, _, _, _, _, _, hpp, hqq = energy_terms(self.bonds, p, q, want_hess=True, dev=d)
        n = d.n
        pd = torch.from_numpy(np.ascontiguousarray(p, dtype=np.float64)).to(d.device)
        m = int(self.pairs.shape[0])
        pair_pp = torch.zeros((m, 6, 6), dtype=F64, device=d.device)
        elem_pp = torch.zeros((n, 3, 3), dtype=F64, device=d.device)
        d.call("bdem_contact_blocks", d.sysp, pd.data_ptr(), pair_pp.data_ptr() if m else None,
               elem_pp.data_ptr() if self.colliders else None, d.stream)
        return PotentialBlocks(
            bond_i=np.asarray(self.bonds.i)[idx], bond_j=np.asarray(self.bonds.j)[idx],
            bond_pp=hpp if hpp is not None else np.zeros((0, 6, 6)),
            bond_qq=hqq if hqq is not None else np.zeros((0, 8, 8)),
            pair_i=self.pairs[:, 0], pair_j=self.pairs[:, 1],
            pair_pp=pair_pp.cpu().numpy(), elem_pp=elem_pp.cpu().numpy())

    def energy_breakdown(self, p, q):
        """integrator.py:131-138."""
        self._load(p, q, self._zero_n, self._zero_n, p, q)
        d = self.dev
        s, st = d.sysp, d.stream
        d.call("bdem_element_energy", s, d.xp.data_ptr(), d.xq.data_ptr(), 0, st)
        d.call("bdem_bond_energy", s, d.xp.data_ptr(), d.xq.data_ptr(), L.SC["EBOND"], st)
        d.call("bdem_pair_assemble", s, d.xp.data_ptr(), 1, st)
        d.call("bdem_reduce_finish", s, L.SC["FT"], 7, L.RED_BLOCKS, st)
        d.eval_pq = (d.xp, d.xq)
        sc = d.read_scalars()
        return {"bond": float(sc[L.SC["EBOND"]]),
                "contact": float(sc[L.SC["EPAIR"]]) + float(sc[L.SC["ECOL"]]),
                "gravity": float(sc[L.SC["EGRAV"]])}


@dataclass
class StepContext:
    """integrator.py:141-161: two-point history of one implicit step."""

    dt: float
    p_prev: np.ndarray
    q_prev: np.ndarray
    p_curr: np.ndarray
    q_curr: np.ndarray
    p_hat: np.ndarray = field(default=None)
    q_hat: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.dt <= 0.0:
            raise ValueError("dt must be positive")
        if self.p_hat is None:
            self.p_hat = 2.0 * self.p_curr - self.p_prev
        if self.q_hat is None:
            self.q_hat = 2.0 * self.q_curr - self.q_prev


class ImplicitProblem:
    """integrator.py:164-210: incremental potential of the right-point rule
    over the free elements, evaluated by the B200 kernels."""

    def __init__(self, model: PotentialModel, ctx: StepContext):
        self.model = model
        self.ctx = ctx
        elements = model.elements
        self.free = ~np.asarray(elements.pinned, dtype=bool)
        dt2 = ctx.dt * ctx.dt
        self.mp_dt2 = np.where(self.free, elements.mass / dt2, 0.0)
        self.mq_dt2 = np.where(self.free, elements.rot_mass / dt2, 0.0)

    @property
    def n(self) -> int:
        return self.model.elements.n

    def _check(self, p, q):
        if p.shape != self.ctx.p_curr.shape or q.shape != self.ctx.q_curr.shape:
            raise ValueError("state dimension mismatch with the step context")

    def value(self, p, q) -> float:
        self._check(p, q)
        return self.model._value(p, q, self.mp_dt2, self.mq_dt2, self.ctx.p_hat, self.ctx.q_hat)

    def value_and_gradient(self, p, q):
        self._check(p, q)
        return self.model._value_and_gradient(p, q, self.mp_dt2, self.mq_dt2, self.ctx.p_hat,
                                               self.ctx.q_hat)

    def gradient(self, p, q):
        _, gp, gq = self.value_and_gradient(p, q)
        return gp, gq

    def hessian_blocks(self, p, q) -> PotentialBlocks:
        return self.model.hessian_blocks(p, q)

    def inertia_diag(self):
        return self.mp_dt2, self.mq_dt2


def incremental_potential(p_next, q_next, problem: ImplicitProblem) -> float:
    """integrator.py:213-215."""
    return problem.value(p_next, q_next)
