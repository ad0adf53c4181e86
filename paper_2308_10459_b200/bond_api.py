"""Per-bond energy / gradient / Hessian entry point on the GPU.

``energy_terms`` replaces ``BondSet.energy_terms``
(``/root/reference/pkg/src/bdem/bonds.py:473-504``) with the same return
tuple ``(idx, energy, gp_i, gp_j, gq_i, gq_j, h_pp, h_qq)``, computed by
``bdem_bond_eval_ambient`` (ambient 6x6 / 8x8 Hessians, the debug form of
the fused production kernel).
"""

from __future__ import annotations

import numpy as np
import torch

from .state import BROKEN, ElementSet


def energy_terms(bonds, p, q, want_hess=False, want_grad=True, dev=None):
    from .device import DeviceSystem
    p = np.ascontiguousarray(p, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    idx = np.nonzero(np.asarray(bonds.status) != BROKEN)[0]
    m = idx.size
    if m == 0:
        z3, z4 = np.zeros((0, 3)), np.zeros((0, 4))
        return idx, np.zeros(0), z3, z3, z4, z4, None, None
    if dev is None:
        n = p.shape[0]
        el = ElementSet(p, q, np.zeros((n, 3)), np.zeros((n, 4)), np.ones(n), np.ones(n))
        dev = DeviceSystem(elements=el, bonds=bonds)
    dd = dev.device
    pd = torch.as_tensor(p).to(dd)
    qd = torch.as_tensor(q).to(dd)
    idx_d = torch.as_tensor(dev.sell.pos_of_bond[idx].astype(np.int32)).to(dd)
    out = {k: torch.empty((m,) + s, dtype=torch.float64, device=dd)
           for k, s in (("E", ()), ("gpi", (3,)), ("gpj", (3,)), ("gqi", (4,)), ("gqj", (4,)))}
    hpp = torch.empty((m, 6, 6), dtype=torch.float64, device=dd) if want_hess else None
    hqq = torch.empty((m, 8, 8), dtype=torch.float64, device=dd) if want_hess else None
    dev.reset_errors()
    dev.call("bdem_bond_eval_ambient", dev.sysp, pd.data_ptr(), qd.data_ptr(), m,
             idx_d.data_ptr(), out["E"].data_ptr(), out["gpi"].data_ptr(), out["gpj"].data_ptr(),
             out["gqi"].data_ptr(), out["gqj"].data_ptr(),
             hpp.data_ptr() if want_hess else None, hqq.data_ptr() if want_hess else None,
             int(bool(want_hess)), dev.stream)
    dev.eval_pq = (pd, qd)
    dev.read_scalars()  # synchronises and raises DegenerateBondError / DegenerateShearError
    h = {k: v.cpu().numpy() for k, v in out.items()}
    if not (want_grad or want_hess):
        return idx, h["E"], None, None, None, None, None, None
    return (idx, h["E"], h["gpi"], h["gpj"], h["gqi"], h["gqj"],
            hpp.cpu().numpy() if want_hess else None, hqq.cpu().numpy() if want_hess else None)
