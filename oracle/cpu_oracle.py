"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference's per-Newton-iteration hot path
(arXiv 2308.10459 reference package ``bdem``).  It exists to CHECK the CUDA
path: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product
(``paper_2308_10459_b200``) never imports, links or executes anything here.

Parity of this restatement is PINNED against golden vectors produced by the
reference itself (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src/bdem`` in the build container and writes
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this module
against them).

Every function cites the reference lines it restates
(``src/X.py`` = ``/root/reference/pkg/src/bdem/X.py``).  Arithmetic order
follows the reference's numpy expressions so results agree to round-off.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy import sparse

INTACT, WEAKENED, BROKEN = 0, 1, 2
_EYE3 = np.eye(3)
_EYE4 = np.eye(4)


class DegenerateBondError(ValueError):
    pass


class DegenerateShearError(ValueError):
    pass


class LineSearchError(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# quaternion primitives  (src/quat.py)
# ---------------------------------------------------------------------------

def skew(t):
    m = np.zeros(t.shape[:-1] + (3, 3))
    m[..., 0, 1], m[..., 0, 2] = -t[..., 2], t[..., 1]
    m[..., 1, 0], m[..., 1, 2] = t[..., 2], -t[..., 0]
    m[..., 2, 0], m[..., 2, 1] = -t[..., 1], t[..., 0]
    return m


def gl(q):
    """G_l(q) = [s I - [t]x, -t]  (src/quat.py:81-93)."""
    out = np.zeros(q.shape[:-1] + (3, 4))
    out[..., :3, :3] = q[..., 3, None, None] * _EYE3 - skew(q[..., :3])
    out[..., :, 3] = -q[..., :3]
    return out


def unit(q):
    """quat_normalize (src/quat.py:159-164)."""
    nrm = np.linalg.norm(q, axis=-1, keepdims=True)
    if np.any(nrm < 1e-300):
        raise ValueError("cannot normalize a zero quaternion")
    return q / nrm


def retract(q, dq):
    """geodesic_step (src/quat.py:144-156), step below 1e-8 keeps q."""
    nrm = np.linalg.norm(dq, axis=-1, keepdims=True)
    tiny = nrm < 1e-8
    den = np.where(tiny, 1.0, nrm)
    return np.where(tiny, q, q * np.cos(nrm) + dq / den * np.sin(nrm))


def tangent(q, v):
    """tangent_project (src/quat.py:173-177)."""
    return v - np.sum(q * v, axis=-1, keepdims=True) * q


# ---------------------------------------------------------------------------
# bond potentials  (src/bonds.py:151-323)
# ---------------------------------------------------------------------------

def stretch(pi, pj, l0, k, want_hess):
    """Rest-length spring (src/bonds.py:151-188).  Returns E, g_j, H(6x6)."""
    d = pj - pi
    ln = np.linalg.norm(d, axis=-1)
    bad = ln < 1e-12 * l0
    if np.any(bad):
        raise DegenerateBondError(f"coincident bond endpoints at indices "
                                  f"{np.nonzero(np.atleast_1d(bad))[0].tolist()}")
    c = ln - l0
    e = 0.5 * k * c**2
    nvec = d / ln[..., None]
    gj = (k * c)[..., None] * nvec
    hess = None
    if want_hess:
        nn = nvec[..., :, None] * nvec[..., None, :]
        blk = k[..., None, None] * (nn + (c / ln)[..., None, None] * (_EYE3 - nn))
        hess = np.zeros(e.shape + (6, 6))
        hess[..., :3, :3] = blk
        hess[..., 3:, 3:] = blk
        hess[..., :3, 3:] = -blk
        hess[..., 3:, :3] = -blk
    return e, gj, hess


def _angle_derivs(theta, k):
    """dV/drho, d2V/drho2 of k/2 arccos(rho)^2 with the theta<1e-4 series
    (src/bonds.py:191-202)."""
    s = np.sin(theta)
    small = theta < 1e-4
    s_safe = np.where(small, 1.0, s)
    d1 = np.where(small, -(1.0 + theta**2 / 6.0), -theta / s_safe)
    d2 = np.where(small, (1.0 + 2.0 * theta**2 / 5.0) / 3.0,
                  (s - theta * np.cos(theta)) / s_safe**3)
    return k * d1, k * d2


def shear(qi, qj, d0, k, want_hess):
    """Shear of the common rotation (src/bonds.py:205-264).  Returns E, g, H(8x8)."""
    u = qi + qj
    un2 = np.sum(u * u, axis=-1)
    bad = un2 < 1e-8**2
    if np.any(bad):
        raise DegenerateShearError(f"antipodal quaternion pairs at indices "
                                   f"{np.nonzero(np.atleast_1d(bad))[0].tolist()}")
    ut, us = u[..., :3], u[..., 3]
    proj = np.sum(d0 * ut, axis=-1)
    rho = (2.0 * proj**2 - np.sum(ut * ut, axis=-1) + us**2) / un2
    theta = np.arccos(np.clip(rho, -1.0 + 1e-12, 1.0))
    e = 0.5 * k * theta**2
    su = np.concatenate([2.0 * proj[..., None] * d0 - ut, u[..., 3:]], axis=-1)
    d1, d2 = _angle_derivs(theta, k)
    drho = 2.0 * (su - rho[..., None] * u) / un2[..., None]
    g = d1[..., None] * drho
    hess = None
    if want_hess:
        smat = np.zeros(un2.shape + (4, 4))
        smat[..., :3, :3] = 2.0 * d0[..., :, None] * d0[..., None, :] - _EYE3
        smat[..., 3, 3] = 1.0
        gu = drho[..., :, None] * u[..., None, :]
        h_rho = (2.0 / un2[..., None, None]) * (smat - rho[..., None, None] * _EYE4
                                                 - gu - np.swapaxes(gu, -1, -2))
        hu = d2[..., None, None] * drho[..., :, None] * drho[..., None, :] \
            + d1[..., None, None] * h_rho
        hess = np.zeros(un2.shape + (8, 8))
        hess[..., :4, :4] = hu
        hess[..., :4, 4:] = hu
        hess[..., 4:, :4] = hu
        hess[..., 4:, 4:] = hu
    return e, g, hess


def _right_pure(w):
    """Right-multiplication matrix of (w, 0) (src/bonds.py:267-279)."""
    m = np.zeros(w.shape[:-1] + (4, 4))
    m[..., 0, 1], m[..., 0, 2] = w[..., 2], -w[..., 1]
    m[..., 1, 0], m[..., 1, 2] = -w[..., 2], w[..., 0]
    m[..., 2, 0], m[..., 2, 1] = w[..., 1], -w[..., 0]
    m[..., :3, 3] = w
    m[..., 3, :3] = -w
    return m


def bendtwist(qi, qj, frame, kd, want_hess):
    """Bend/twist of the relative rotation (src/bonds.py:282-323)."""
    ai = frame @ gl(qj)
    t = np.einsum("...ij,...j->...i", ai, qi)
    kt = kd * t
    e = 0.5 * np.sum(t * kt, axis=-1)
    aj = -frame @ gl(qi)
    gi = np.einsum("...ij,...i->...j", ai, kt)
    gj = np.einsum("...ij,...i->...j", aj, kt)
    hess = None
    if want_hess:
        ait = np.swapaxes(ai, -1, -2)
        hii = ait @ (kd[..., :, None] * ai)
        hjj = np.swapaxes(aj, -1, -2) @ (kd[..., :, None] * aj)
        hij = ait @ (kd[..., :, None] * aj) + _right_pure(np.einsum("...ji,...j->...i", frame, kt))
        hess = np.zeros(e.shape + (8, 8))
        hess[..., :4, :4] = hii
        hess[..., 4:, 4:] = hjj
        hess[..., :4, 4:] = hij
        hess[..., 4:, :4] = np.swapaxes(hij, -1, -2)
    return e, gi, gj, hess


@dataclass
class BondEval:
    idx: np.ndarray
    energy: np.ndarray
    gp_i: np.ndarray = None
    gp_j: np.ndarray = None
    gq_i: np.ndarray = None
    gq_j: np.ndarray = None
    h_pp: np.ndarray = None
    h_qq: np.ndarray = None


def bond_eval(b, p, q, want_hess=False, want_grad=True) -> BondEval:
    """Batched active-bond evaluation (src/bonds.py:473-504)."""
    idx = np.nonzero(b.status != BROKEN)[0]
    if idx.size == 0:
        z3, z4 = np.zeros((0, 3)), np.zeros((0, 4))
        return BondEval(idx, np.zeros(0), z3, z3, z4, z4)
    ii, jj = b.i[idx], b.j[idx]
    sc = b.stiffness_scale[idx]
    e_s, gpj, hpp = stretch(p[ii], p[jj], b.rest_length[idx], sc * b.kn[idx], want_hess)
    e_h, g_h, hqq_h = shear(q[ii], q[jj], b.d0[idx], sc * b.kt[idx], want_hess)
    e_b, gi_b, gj_b, hqq_b = bendtwist(q[ii], q[jj], b.frame[idx],
                                       sc[:, None] * b.k_diag[idx], want_hess)
    out = BondEval(idx, e_s + e_h + e_b)
    if want_grad or want_hess:
        out.gp_i, out.gp_j = -gpj, gpj
        out.gq_i, out.gq_j = g_h + gi_b, g_h + gj_b
    if want_hess:
        out.h_pp, out.h_qq = hpp, hqq_h + hqq_b
    return out


# ---------------------------------------------------------------------------
# contact  (src/contact.py:38-248)
# ---------------------------------------------------------------------------

def collider_sdf(col, p):
    kind = type(col).__name__
    if kind == "HalfSpace":
        return p @ np.asarray(col.normal) - col.offset
    if kind == "SphereCollider":
        return np.linalg.norm(p - np.asarray(col.center), axis=-1) - col.radius
    if kind == "BoxCollider":
        d = np.abs(p - np.asarray(col.center)) - np.asarray(col.half_extents)
        return np.linalg.norm(np.maximum(d, 0.0), axis=-1) + np.minimum(np.max(d, axis=-1), 0.0)
    raise TypeError(kind)


def collider_grad_hess(col, p):
    """SDF gradient/Hessian (src/contact.py:52-58, 76-84, 103-133)."""
    kind = type(col).__name__
    if kind == "HalfSpace":
        return np.broadcast_to(np.asarray(col.normal), p.shape).copy(), np.zeros(p.shape[:-1] + (3, 3))
    if kind == "SphereCollider":
        d = p - np.asarray(col.center)
        r = np.maximum(np.linalg.norm(d, axis=-1), 1e-12)
        nv = d / r[..., None]
        return nv, (_EYE3 - nv[..., :, None] * nv[..., None, :]) / r[..., None, None]
    if kind == "BoxCollider":
        loc = p - np.asarray(col.center)
        d = np.abs(loc) - np.asarray(col.half_extents)
        sign = np.where(loc >= 0.0, 1.0, -1.0)
        pos = np.maximum(d, 0.0)
        on = np.linalg.norm(pos, axis=-1)
        out = on > 0.0
        g_out = sign * pos / np.maximum(on, 1e-300)[..., None]
        g_in = np.zeros_like(loc)
        np.put_along_axis(g_in, np.argmax(d, axis=-1)[..., None], 1.0, axis=-1)
        grad = np.where(out[..., None], g_out, g_in * sign)
        h = np.zeros(loc.shape[:-1] + (3, 3))
        if np.any(out):
            nn = g_out[..., :, None] * g_out[..., None, :]
            h_out = ((pos > 0.0).astype(float)[..., :, None] * _EYE3 - nn) \
                / np.maximum(on, 1e-300)[..., None, None]
            h = np.where(out[..., None, None], h_out, h)
        return grad, h
    raise TypeError(kind)


def collider_terms(p, col, k, want_hess):
    """external_repulsion_terms (src/contact.py:227-248)."""
    g = collider_sdf(col, p)
    inside = g < 0.0
    e = np.where(inside, 0.5 * k * g**2, 0.0)
    dg, hg = collider_grad_hess(col, p)
    grad = np.where(inside[..., None], k * g[..., None] * dg, 0.0)
    hess = None
    if want_hess:
        hess = np.where(inside[..., None, None],
                        k * (dg[..., :, None] * dg[..., None, :] + g[..., None, None] * hg), 0.0)
    return e, grad, hess


def pair_terms(pi, pj, ri, rj, k, want_hess):
    """self_repulsion_terms (src/contact.py:180-224).  Returns E, g_i, H."""
    d = pj - pi
    ln = np.linalg.norm(d, axis=-1)
    depth = np.maximum(0.0, ri + rj - ln)
    e = 0.5 * k * depth**2
    coinc = ln < 1e-12
    nv = np.where(coinc[..., None], np.array([1.0, 0.0, 0.0]),
                  d / np.maximum(ln, 1e-300)[..., None])
    touch = depth > 0.0
    gi = np.where(touch[..., None], (k * depth)[..., None] * nv, 0.0)
    hess = None
    if want_hess:
        nn = nv[..., :, None] * nv[..., None, :]
        blk = k * (nn - (depth / np.maximum(ln, 1e-300))[..., None, None] * (_EYE3 - nn))
        blk = np.where(touch[..., None, None], blk, 0.0)
        hess = np.zeros(e.shape + (6, 6))
        hess[..., :3, :3] = blk
        hess[..., 3:, 3:] = blk
        hess[..., :3, 3:] = -blk
        hess[..., 3:, :3] = -blk
    return e, gi, hess


def broad_phase(p, radii, cell):
    """Spatial-hash candidate pairs, sorted, i<j, overlap-filtered
    (src/contact.py:140-173)."""
    if radii.size and cell < 2.0 * float(np.max(radii)):
        raise ValueError("cell_size must be at least twice the largest radius")
    keys = np.floor(p / cell).astype(np.int64)
    buckets: dict = {}
    for e, key in enumerate(map(tuple, keys)):
        buckets.setdefault(key, []).append(e)
    found = set()
    for key, members in buckets.items():
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    other = buckets.get((key[0] + dx, key[1] + dy, key[2] + dz))
                    if other is None:
                        continue
                    for a in members:
                        for c in other:
                            if a < c:
                                found.add((a, c))
    if not found:
        return np.zeros((0, 2), dtype=np.int64)
    cand = np.array(sorted(found), dtype=np.int64)
    dist = np.linalg.norm(p[cand[:, 1]] - p[cand[:, 0]], axis=1)
    return cand[dist < radii[cand[:, 0]] + radii[cand[:, 1]]]


# ---------------------------------------------------------------------------
# incremental potential  (src/integrator.py:38-210)
# ---------------------------------------------------------------------------

class Objective:
    """PotentialModel + ImplicitProblem restated (src/integrator.py:38-210)."""

    def __init__(self, el, bonds, pairs, colliders, gravity, k_contact, k_element,
                 dt, p_prev, q_prev, p_curr, q_curr):
        self.el, self.bonds = el, bonds
        self.pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
        self.colliders = list(colliders)
        self.gravity = np.asarray(gravity, dtype=float)
        self.kc, self.ke = k_contact, k_element
        self.dt = dt
        self.p_curr, self.q_curr = p_curr, q_curr
        self.p_hat = 2.0 * p_curr - p_prev          # integrator.py:157
        self.q_hat = 2.0 * q_curr - q_prev          # integrator.py:161
        self.free = ~el.pinned
        dt2 = dt * dt
        self.mp_dt2 = np.where(self.free, el.mass / dt2, 0.0)                      # :173
        self.mq_dt2 = np.where(self.free, 1.6 * el.mass * el.radius**2 / dt2, 0.0)  # :174

    @property
    def n(self):
        return self.el.p.shape[0]

    # -- contact pieces (integrator.py:56-85)
    def _contacts(self, p, want_grad, want_hess):
        e = 0.0
        gc = np.zeros_like(p) if (want_grad or want_hess) else None
        pair_h, elem_h = None, None
        r = self.el.radius
        if self.pairs.shape[0]:
            a, b = self.pairs[:, 0], self.pairs[:, 1]
            ep, gi, hp = pair_terms(p[a], p[b], r[a], r[b], self.ke, want_hess)
            e += float(np.sum(ep))
            if gc is not None:
                np.add.at(gc, a, gi)
                np.add.at(gc, b, -gi)
            pair_h = hp
        if self.colliders:
            if want_hess:
                elem_h = np.zeros((p.shape[0], 3, 3))
            for col in self.colliders:
                ec, gcol, hcol = collider_terms(p, col, self.kc, want_hess)
                e += float(np.sum(ec))
                if gc is not None:
                    gc += gcol
                if want_hess:
                    elem_h += hcol
        return e, gc, pair_h, elem_h

    def _gravity_energy(self, p):
        return float(np.sum(self.el.mass * (p @ self.gravity)))

    def _inertia(self, p, q):
        dp, dq = p - self.p_hat, q - self.q_hat
        return 0.5 * float(np.sum(self.mp_dt2 * np.sum(dp * dp, axis=1))) \
            + 0.5 * float(np.sum(self.mq_dt2 * np.sum(dq * dq, axis=1)))

    def potential(self, p, q):
        """PotentialModel.value (integrator.py:87-93)."""
        ev = bond_eval(self.bonds, p, q, want_grad=False)
        e = float(np.sum(ev.energy))
        e += self._contacts(p, False, False)[0]
        return e - self._gravity_energy(p)

    def value(self, p, q):
        """ImplicitProblem.value (integrator.py:191-193)."""
        return self._inertia(p, q) + self.potential(p, q)

    def value_and_gradient(self, p, q):
        """ImplicitProblem.value_and_gradient (integrator.py:95-109, 195-200)."""
        gp = np.zeros_like(p)
        gq = np.zeros((p.shape[0], 4))
        ev = bond_eval(self.bonds, p, q)
        if ev.idx.size:
            bi, bj = self.bonds.i[ev.idx], self.bonds.j[ev.idx]
            np.add.at(gp, bi, ev.gp_i)
            np.add.at(gp, bj, ev.gp_j)
            np.add.at(gq, bi, ev.gq_i)
            np.add.at(gq, bj, ev.gq_j)
        ec, gc, _, _ = self._contacts(p, True, False)
        gp += gc
        gp -= self.el.mass[:, None] * self.gravity
        e = float(np.sum(ev.energy)) + ec
        e -= self._gravity_energy(p)
        gp = gp + self.mp_dt2[:, None] * (p - self.p_hat)
        gq = gq + self.mq_dt2[:, None] * (q - self.q_hat)
        return e + self._inertia(p, q), gp, gq

    def hessian_blocks(self, p, q):
        """PotentialModel.hessian_blocks (integrator.py:115-129)."""
        ev = bond_eval(self.bonds, p, q, want_hess=True)
        _, _, pair_h, elem_h = self._contacts(p, True, True)
        n = p.shape[0]
        return dict(
            bond_i=self.bonds.i[ev.idx], bond_j=self.bonds.j[ev.idx],
            bond_pp=ev.h_pp if ev.h_pp is not None else np.zeros((0, 6, 6)),
            bond_qq=ev.h_qq if ev.h_qq is not None else np.zeros((0, 8, 8)),
            pair_i=self.pairs[:, 0], pair_j=self.pairs[:, 1],
            pair_pp=pair_h if pair_h is not None else np.zeros((0, 6, 6)),
            elem_pp=elem_h if elem_h is not None else np.zeros((n, 3, 3)),
        )

    def energy_breakdown(self, p, q):
        """integrator.py:131-138."""
        ev = bond_eval(self.bonds, p, q)
        return {"bond": float(np.sum(ev.energy)),
                "contact": self._contacts(p, False, False)[0],
                "gravity": -self._gravity_energy(p)}


# ---------------------------------------------------------------------------
# Newton pieces  (src/solver.py, src/linalg.py)
# ---------------------------------------------------------------------------

def psd_clamp(blocks):
    """spd_project (src/solver.py:89-113): symmetrise, eigh, clamp at 0."""
    blocks = np.asarray(blocks, dtype=float)
    sym = 0.5 * (blocks + np.swapaxes(blocks, -1, -2))
    if sym.shape[0] == 0:
        return sym
    w, v = np.linalg.eigh(sym)
    return (v * np.maximum(w, 0.0)[:, None, :]) @ np.swapaxes(v, 1, 2)


def reduced_gradient(q, gp, gq, free):
    """z = [gp; G_l(q) gq] per free element (src/solver.py:116-123)."""
    z = np.zeros((int(np.count_nonzero(free)), 6))
    z[:, :3] = gp[free]
    z[:, 3:] = np.einsum("bij,bj->bi", gl(q[free]), gq[free])
    return z.reshape(-1)


def clamped_pieces(obj: Objective, p, q, gq):
    """build_clamped_pieces (src/solver.py:141-180)."""
    hb = obj.hessian_blocks(p, q)
    G = gl(q)
    nb = hb["bond_i"].shape[0]
    pp = psd_clamp(hb["bond_pp"])
    if nb:
        T = np.zeros((nb, 6, 8))
        T[:, :3, :4] = G[hb["bond_i"]]
        T[:, 3:, 4:] = G[hb["bond_j"]]
        rot = psd_clamp((T @ hb["bond_qq"]) @ np.swapaxes(T, 1, 2))
    else:
        rot = np.zeros((0, 6, 6))
    pair = psd_clamp(hb["pair_pp"])
    if np.any(hb["elem_pp"]):
        elem_pos = psd_clamp(hb["elem_pp"] + obj.mp_dt2[:, None, None] * _EYE3)
    else:
        elem_pos = obj.mp_dt2[:, None, None] * _EYE3
    elem_rot = np.maximum(obj.mq_dt2 + (-np.sum(q * gq, axis=1)), 0.0)
    elem_rot[~obj.free] = 0.0
    return dict(bond_i=hb["bond_i"], bond_j=hb["bond_j"], bond_pp=pp, bond_rot=rot,
                pair_i=hb["pair_i"], pair_j=hb["pair_j"], pair_pp=pair,
                elem_pos=elem_pos, elem_rot=elem_rot)


def reduced_system(pc, free):
    """assemble_reduced_system (src/solver.py:183-258): COO -> CSR with
    duplicate summation, plus the (m,6,6) diagonal blocks."""
    slot = np.full(free.shape[0], -1, dtype=np.int64)
    slot[free] = np.arange(int(np.count_nonzero(free)))
    m = int(np.count_nonzero(free))
    R, C, V = [], [], []
    pos_d = np.zeros((m, 3, 3))
    rot_d = np.zeros((m, 3, 3))

    def scatter(ei, ej, blocks, off, dacc):
        if ei.shape[0] == 0:
            return
        si, sj = slot[ei], slot[ej]
        idx6 = np.full((ei.shape[0], 6), -1, dtype=np.int64)
        for c in range(3):
            idx6[:, c] = np.where(si >= 0, 6 * si + off + c, -1)
            idx6[:, 3 + c] = np.where(sj >= 0, 6 * sj + off + c, -1)
        rows = np.broadcast_to(idx6[:, :, None], blocks.shape)
        cols = np.broadcast_to(idx6[:, None, :], blocks.shape)
        ok = (rows >= 0) & (cols >= 0)
        R.append(rows[ok])
        C.append(cols[ok])
        V.append(blocks[ok])
        np.add.at(dacc, si[si >= 0], blocks[si >= 0][:, :3, :3])
        np.add.at(dacc, sj[sj >= 0], blocks[sj >= 0][:, 3:, 3:])

    scatter(pc["bond_i"], pc["bond_j"], pc["bond_pp"], 0, pos_d)
    scatter(pc["bond_i"], pc["bond_j"], pc["bond_rot"], 3, rot_d)
    scatter(pc["pair_i"], pc["pair_j"], pc["pair_pp"], 0, pos_d)
    fid = np.nonzero(free)[0]
    pos_d += pc["elem_pos"][fid]
    rot_d += pc["elem_rot"][fid, None, None] * _EYE3
    diag = np.zeros((m, 6, 6))
    diag[:, :3, :3] = pos_d
    diag[:, 3:, 3:] = rot_d
    base0 = 6 * slot[fid]
    for off, blk in ((0, pc["elem_pos"][fid]), (3, pc["elem_rot"][fid, None, None] * _EYE3)):
        b = (base0 + off)[:, None, None]
        R.append(np.broadcast_to(b + np.arange(3)[None, :, None], blk.shape).ravel())
        C.append(np.broadcast_to(b + np.arange(3)[None, None, :], blk.shape).ravel())
        V.append(blk.ravel())
    mat = sparse.coo_matrix((np.concatenate(V), (np.concatenate(R), np.concatenate(C))),
                            shape=(6 * m, 6 * m)).tocsr()
    return mat, diag


class BlockJacobi:
    """Block-diagonal inverse with identity fallback (src/linalg.py:100-128)."""

    def __init__(self, diag):
        diag = np.asarray(diag, dtype=float)
        m, k, _ = diag.shape
        self.k = k
        sym = 0.5 * (diag + np.swapaxes(diag, 1, 2))
        inv = np.empty_like(sym)
        if m:
            lam = np.linalg.eigvalsh(sym)
            bad = lam.min(axis=1) <= 1e-12 * np.maximum(np.abs(lam).max(axis=1), 1e-300)
        else:
            bad = np.zeros(0, dtype=bool)
        if np.any(~bad):
            inv[~bad] = np.linalg.inv(sym[~bad])
        inv[bad] = np.eye(k)
        self.inv = inv
        self.n_singular = int(bad.sum())

    def __call__(self, x):
        m = self.inv.shape[0]
        return np.einsum("bij,bj->bi", self.inv, x.reshape(m, self.k)).reshape(-1)


@dataclass
class PCGOut:
    x: np.ndarray
    iterations: int
    converged: bool
    relative_residual: float
    restarts: int = 0


def inner_tolerance(gnorm):
    """relative_tolerance (src/linalg.py:29-37)."""
    return min(0.5, math.sqrt(gnorm))


def pcg(apply_a, b, apply_m, tol, max_iter):
    """PCG with breakdown restarts (src/linalg.py:40-97)."""
    n = b.shape[0]
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return PCGOut(np.zeros(n), 0, True, 0.0)
    boost, restarts = 0.0, 0
    while True:
        x = np.zeros(n)
        r = b.copy()
        z = apply_m(r)
        d = z.copy()
        rz = float(r @ z)
        broke, k, rel = False, 0, 1.0
        while k < max_iter:
            ad = apply_a(d)
            if boost:
                ad = ad + boost * d
            dad = float(d @ ad)
            if dad <= 0.0:
                broke = True
                ratio = float(np.linalg.norm(ad)) / max(float(np.linalg.norm(d)), 1e-300)
                boost = max(boost * 100.0, 1e-10 * max(ratio, 1.0))
                break
            a = rz / dad
            x += a * d
            r -= a * ad
            k += 1
            rel = float(np.linalg.norm(r)) / bn
            if rel <= tol:
                return PCGOut(x, k, True, rel, restarts)
            z = apply_m(r)
            rz_new = float(r @ z)
            d = z + (rz_new / rz) * d
            rz = rz_new
        if not broke:
            return PCGOut(x, k, False, rel, restarts)
        restarts += 1
        if restarts > 3:
            return PCGOut(x, k, False, rel, restarts)


def direction_from_reduced(y, q, free):
    """dp = y_pos, dq = G_l(q)^T y_rot on free elements (src/solver.py:409-418)."""
    m = int(np.count_nonzero(free))
    yb = y.reshape(m, 6)
    dp = np.zeros((q.shape[0], 3))
    dq = np.zeros((q.shape[0], 4))
    dp[free] = yb[:, :3]
    dq[free] = np.einsum("bji,bj->bi", gl(q[free]), yb[:, 3:])
    return dp, dq


def line_search(obj, p, q, dp, dq, f0, slope, cfg, free, alpha0=1.0):
    """Armijo backtracking with geodesic retraction (src/solver.py:387-406)."""
    alpha = alpha0
    noise = 8.0 * np.finfo(float).eps * abs(f0)
    trials = 0
    while alpha >= cfg.min_alpha:
        pt = p + alpha * dp
        qt = q.copy()
        qt[free] = unit(retract(q[free], alpha * dq[free]))
        ft = obj.value(pt, qt)
        trials += 1
        if np.isfinite(ft) and ft <= f0 + cfg.armijo * alpha * slope + noise:
            return alpha, pt, qt, ft, trials
        alpha *= cfg.shrink
    raise LineSearchError(f"line search failed below alpha={cfg.min_alpha}")


@dataclass
class Config:
    """SolverConfig defaults (src/solver.py:38-49)."""
    epsilon: float = 1e-6
    max_iterations: int = 100
    armijo: float = 1e-4
    shrink: float = 0.5
    min_alpha: float = 1e-12
    pcg_max_iterations: int = 2000


@dataclass
class IterRec:
    index: int
    f: float
    grad_norm: float
    constraint_norm: float
    alpha: float = 0.0
    pcg_iterations: int = 0
    ls_trials: int = 0


@dataclass
class Solve:
    p: np.ndarray
    q: np.ndarray
    converged: bool
    iterations: int
    grad_norm: float
    records: list
    pcg_total: int = 0
    max_unit_dev: float = 0.0
    reason: str = "converged"


def _max_dev(q, free):
    nr = np.linalg.norm(q[free], axis=1)
    return float(np.max(np.abs(nr - 1.0))) if nr.size else 0.0


def newton(obj: Objective, p0, q0, cfg) -> Solve:
    """minimize_second_order (src/solver.py:511-562), PCG linear mode."""
    free = obj.free
    p, q = p0.copy(), q0.copy()
    q[free] = unit(q[free])
    recs, pcg_total, gnorm = [], 0, np.inf
    dev = _max_dev(q, free)
    for it in range(cfg.max_iterations):
        f, gp, gq = obj.value_and_gradient(p, q)
        z = reduced_gradient(q, gp, gq, free)
        gnorm = float(np.linalg.norm(z))
        cnorm = float(np.linalg.norm(0.5 * (np.sum(q[free] * q[free], axis=-1) - 1.0)))
        dev = max(dev, _max_dev(q, free))
        if gnorm < cfg.epsilon:
            recs.append(IterRec(it, f, gnorm, cnorm))
            return Solve(p, q, True, it, gnorm, recs, pcg_total, dev)
        pc = clamped_pieces(obj, p, q, gq)
        mat, diag = reduced_system(pc, free)
        pre = BlockJacobi(diag)
        res = pcg(lambda v: mat @ v, -z, pre, inner_tolerance(gnorm), cfg.pcg_max_iterations)
        y = res.x
        pcg_total += res.iterations
        slope = float(z @ y)
        dp, dq = direction_from_reduced(y, q, free)
        if not np.isfinite(slope) or slope >= 0.0:
            dp, dq = direction_from_reduced(-z, q, free)
            slope = -gnorm * gnorm
        try:
            alpha, p, q, f, trials = line_search(obj, p, q, dp, dq, f, slope, cfg, free)
        except LineSearchError:
            recs.append(IterRec(it, f, gnorm, cnorm, pcg_iterations=res.iterations))
            return Solve(p, q, False, it, gnorm, recs, pcg_total, dev, "line-search")
        recs.append(IterRec(it, f, gnorm, cnorm, alpha, res.iterations, trials))
        dev = max(dev, _max_dev(q, free))
    return Solve(p, q, False, cfg.max_iterations, gnorm, recs, pcg_total, dev, "max-iterations")


# ---------------------------------------------------------------------------
# step level  (src/integrator.py:268-293, src/solver.py:856-939,
#              src/bonds.py:506-570, src/geometry.py:264-310)
# ---------------------------------------------------------------------------

def predictor(el, dt, free):
    """predict_state (src/integrator.py:268-274)."""
    p0, q0 = el.p.copy(), el.q.copy()
    p0[free] += dt * el.v[free]
    q0[free] = retract(el.q[free], dt * el.qdot[free])
    return p0, unit(q0)


def fracture_update(b, p, q, youngs, plastic):
    """update_bond_states with BondSet.stresses/axial_strain
    (src/bonds.py:506-570).  Mutates ``b``; returns ascending events."""
    idx = np.nonzero(b.status != BROKEN)[0]
    if idx.size == 0:
        return []
    ii, jj = b.i[idx], b.j[idx]
    sc = b.stiffness_scale[idx]
    ln = np.linalg.norm(p[jj] - p[ii], axis=-1)
    fn = sc * b.kn[idx] * np.abs(ln - b.rest_length[idx])
    t = np.einsum("bij,bj->bi", b.frame[idx], np.einsum("bij,bj->bi", gl(q[jj]), q[ii]))
    kt = sc[:, None] * b.k_diag[idx] * t
    mt = np.abs(kt[:, 0])
    mb = np.hypot(kt[:, 1], kt[:, 2])
    sigma = fn / (b.damage[idx] * b.section[idx]) + mb * b.radius[idx] / b.second_moment[idx]
    tau = mt * b.radius[idx] / b.polar_moment[idx]
    b.sigma[idx] = sigma
    b.tau[idx] = tau
    broke = np.zeros(idx.size, dtype=bool)
    if plastic is not None:
        strain = (ln - b.rest_length[idx]) / b.rest_length[idx]
        sy = youngs * plastic.yield_strain
        vm = np.sqrt(sigma**2 + 3.0 * tau**2)
        yl = vm > sy
        if np.any(yl):
            sub = idx[yl]
            b.stiffness_scale[sub] = np.minimum(b.stiffness_scale[sub],
                                                1.0 - plastic.weakening * (1.0 - sy / vm[yl]))
            ep = np.maximum(0.0, strain[yl] - plastic.yield_strain)
            b.plastic_strain[sub] = np.maximum(b.plastic_strain[sub], ep)
            b.damage[sub] = np.minimum(b.damage[sub], np.exp(-ep**plastic.damage_exponent))
            b.status[sub] = np.maximum(b.status[sub], WEAKENED)
        broke |= strain > plastic.fracture_strain
    broke |= (sigma > b.tensile_strength[idx]) | (tau > b.shear_strength[idx])
    if not np.any(broke):
        return []
    sub = idx[broke]
    b.status[sub] = BROKEN
    return [(int(x), float(s), float(t_)) for x, s, t_ in zip(sub, sigma[broke], tau[broke])]


def components(n, b):
    """label_components: union-find keeping the smaller root, labels in order of
    each component's smallest element (src/geometry.py:264-310)."""
    parent = list(range(n))

    def find(a):
        r = a
        while parent[r] != r:
            r = parent[r]
        while parent[a] != r:
            parent[a], a = r, parent[a]
        return r

    for k in np.nonzero(b.status != BROKEN)[0]:
        ra, rb = find(int(b.i[k])), find(int(b.j[k]))
        if ra != rb:
            lo, hi = (ra, rb) if ra < rb else (rb, ra)
            parent[hi] = lo
    roots = [find(e) for e in range(n)]
    order: dict = {}
    for r in roots:
        order.setdefault(r, len(order))
    return np.array([order[r] for r in roots], dtype=np.int64)


def candidates(st, labels):
    """contact_candidates (src/solver.py:856-878)."""
    el = st.elements
    if st.k_element <= 0.0 or el.n < 2:
        return np.zeros((0, 2), dtype=np.int64)
    travel = st.dt * np.linalg.norm(el.v, axis=1)
    travel += st.dt**2 * float(np.linalg.norm(st.gravity))
    infl = el.radius + travel
    pairs = broad_phase(el.p, infl, 2.0 * float(np.max(infl)) + 1e-12)
    if pairs.shape[0] == 0:
        return pairs
    return pairs[labels[pairs[:, 0]] != labels[pairs[:, 1]]]


# ---------------------------------------------------------------------------
# friction  (src/contact.py:267-350, src/quat.py:41-49, 116-140)
# ---------------------------------------------------------------------------

def qmul(a, b):
    """Hamilton product, scalar last (src/quat.py:41-49)."""
    at, asc = a[..., :3], a[..., 3:]
    bt, bsc = b[..., :3], b[..., 3:]
    vec = asc * bt + bsc * at + np.cross(at, bt)
    return np.concatenate([vec, asc * bsc - np.sum(at * bt, axis=-1, keepdims=True)], axis=-1)


def angular_velocity(q, qdot):
    """2 tangent(qdot) * conj(q), vector part (src/quat.py:116-134)."""
    radial = np.sum(q * qdot, axis=-1, keepdims=True)
    conj = np.concatenate([-q[..., :3], q[..., 3:]], axis=-1)
    return (2.0 * qmul(qdot - radial * q, conj))[..., :3]


def quat_rate(q, w):
    """0.5 (w, 0) * q (src/quat.py:137-141)."""
    return 0.5 * qmul(np.concatenate([w, np.zeros(w.shape[:-1] + (1,))], axis=-1), q)


def _friction_delta(rel, own, fn, coeff, scale, dt):
    """src/contact.py:267-282."""
    own_n = np.linalg.norm(own)
    rel_n = np.linalg.norm(rel)
    if own_n == 0.0 or rel_n == 0.0 or fn == 0.0:
        return np.zeros(3)
    factor = min(1.0, coeff * fn * dt / (scale * rel_n))
    direction = own / own_n
    along = min(0.0, max(float(np.dot(-factor * rel, direction)), -own_n))
    return along * direction


def apply_friction(el, pairs, colliders, k_c, k_ec, mu_s, mu_r, dt):
    """Sequential post-step friction sweep (src/contact.py:303-350): pairs in
    ascending order correcting both sides, then colliders in order, ascending
    elements; quaternion rates of touched elements rebuilt from w."""
    if mu_s == 0.0 and mu_r == 0.0:
        return
    p, v = el.p, el.v
    w = angular_velocity(el.q, el.qdot)
    touched = np.zeros(el.n, dtype=bool)
    inertia = 0.4 * el.mass * el.radius**2

    def correct(k, v_rel, w_rel, nrm, fn):
        if el.pinned[k]:
            return
        v_t = v_rel - float(np.dot(v_rel, nrm)) * nrm
        v[k] += _friction_delta(v_t, v[k], fn, mu_s, el.mass[k], dt)
        w[k] += _friction_delta(w_rel, w[k], fn, mu_r, inertia[k] / el.radius[k]**3, dt)
        touched[k] = True

    for a, b in np.asarray(pairs).reshape(-1, 2):
        d = p[a] - p[b]
        dist = np.linalg.norm(d)
        if dist >= el.radius[a] + el.radius[b]:
            continue
        nrm = d / dist if dist > 1e-12 else np.array([1.0, 0.0, 0.0])
        fn = k_ec * dist
        correct(a, v[a] - v[b], w[a] - w[b], nrm, fn)
        correct(b, v[b] - v[a], w[b] - w[a], -nrm, fn)
    for col in colliders:
        g = collider_sdf(col, p)
        inside = np.nonzero(g < 0.0)[0]
        if inside.size == 0:
            continue
        grads, _ = collider_grad_hess(col, p[inside])
        for row, k in enumerate(inside):
            correct(int(k), v[k], w[k], grads[row], k_c * abs(g[k]) * np.linalg.norm(grads[row]))
    upd = np.nonzero(touched)[0]
    if upd.size:
        el.qdot[upd] = quat_rate(el.q[upd], w[upd])


@dataclass
class OracleState:
    """Minimal scene state the step needs (src/scenes.py:32-77 fields)."""
    elements: object
    bonds: object
    dt: float
    youngs: float
    colliders: list = field(default_factory=list)
    gravity: np.ndarray = field(default_factory=lambda: np.array([0.0, 0.0, -9.81]))
    k_contact: float = 1e6
    k_element: float = 1e6
    mu_s: float = 0.0
    mu_r: float = 0.0
    plastic: object = None
    driver: object = None
    time: float = 0.0
    p_prev: np.ndarray = None
    q_prev: np.ndarray = None
    labels: np.ndarray = None

    def __post_init__(self):
        if self.labels is None:
            self.labels = components(self.elements.n, self.bonds)
        if self.p_prev is None:
            self.bootstrap()

    def bootstrap(self):
        """Scene.bootstrap_history (src/scenes.py:64-68)."""
        el = self.elements
        self.p_prev = el.p - self.dt * el.v
        self.q_prev = unit(retract(el.q, -self.dt * el.qdot))


@dataclass
class StepOut:
    solve: Solve
    broken: list
    contact_pairs: int
    energies: dict
    committed: bool


def step(st: OracleState, cfg) -> StepOut:
    """stable_step (src/solver.py:881-939) with step_right_point
    (src/integrator.py:277-293)."""
    el = st.elements
    pin = np.nonzero(el.pinned)[0]
    saved = (el.p[pin].copy(), el.q[pin].copy(), el.v[pin].copy(), el.qdot[pin].copy())
    t_next = st.time + st.dt
    if st.driver is not None:
        st.driver(el, t_next)
    p_curr, q_curr = el.p.copy(), el.q.copy()
    pairs = candidates(st, st.labels)
    obj = Objective(el, st.bonds, pairs, st.colliders, st.gravity, st.k_contact,
                    st.k_element, st.dt, st.p_prev.copy(), st.q_prev.copy(), p_curr, q_curr)
    free = obj.free
    p0, q0 = predictor(el, st.dt, free)
    res = newton(obj, p0, q0, cfg)
    v = (res.p - p_curr) / st.dt
    qd = tangent(res.q, (res.q - q_curr) / st.dt)
    v[~free] = el.v[~free]
    qd[~free] = el.qdot[~free]
    if not res.converged:
        el.p[pin], el.q[pin], el.v[pin], el.qdot[pin] = saved
        return StepOut(res, [], int(pairs.shape[0]), {"kinetic": _kinetic(el)}, False)
    el.p[:], el.q[:], el.v[:], el.qdot[:] = res.p, res.q, v, qd
    if st.mu_s > 0.0 or st.mu_r > 0.0:                 # src/solver.py:923-925
        apply_friction(el, pairs, st.colliders, st.k_contact, st.k_element, st.mu_s,
                       st.mu_r, st.dt)
    events = fracture_update(st.bonds, el.p, el.q, st.youngs, st.plastic)
    if events:
        st.labels = components(el.n, st.bonds)
    st.p_prev, st.q_prev = p_curr, q_curr
    st.time = t_next
    en = obj.energy_breakdown(el.p, el.q)
    en["kinetic"] = _kinetic(el)
    return StepOut(res, events, int(pairs.shape[0]), en, True)


def _kinetic(el):
    lin = 0.5 * np.sum(el.mass * np.sum(el.v**2, axis=1))
    rot = 0.5 * np.sum(1.6 * el.mass * el.radius**2 * np.sum(el.qdot**2, axis=1))
    return float(lin + rot)
