"""Host-side quaternion helpers used for scene setup (not on the Newton path).

Storage is scalar-last ``(x, y, z, w)`` like the reference
(``/root/reference/pkg/src/bdem/quat.py:1-7``).  Only what scene construction
and the drivers need lives here; the per-iteration quaternion math (nullspace
operator, geodesic retraction, normalisation) runs inside the CUDA kernels
(``csrc/bdem_math.cuh``).
"""

from __future__ import annotations

import numpy as np

IDENTITY = np.array([0.0, 0.0, 0.0, 1.0])
GEODESIC_EPS = 1e-8  # quat.py:16


class ZeroQuaternionError(ValueError):
    """Normalisation of a (near-)zero quaternion (quat.py:19-20)."""


def _skew(v: np.ndarray) -> np.ndarray:
    out = np.zeros(v.shape[:-1] + (3, 3))
    out[..., 0, 1], out[..., 0, 2] = -v[..., 2], v[..., 1]
    out[..., 1, 0], out[..., 1, 2] = v[..., 2], -v[..., 0]
    out[..., 2, 0], out[..., 2, 1] = -v[..., 1], v[..., 0]
    return out


def g_left(q: np.ndarray) -> np.ndarray:
    """3x4 tangent operator G_l(q) = [s I - [t]x | -t]  (quat.py:81-93)."""
    q = np.asarray(q, dtype=float)
    s = q[..., 3]
    g = np.empty(q.shape[:-1] + (3, 4))
    g[..., :, :3] = s[..., None, None] * np.eye(3) - _skew(q[..., :3])
    g[..., :, 3] = -q[..., :3]
    return g


def g_right(q: np.ndarray) -> np.ndarray:
    """Right counterpart [s I + [t]x | -t]  (quat.py:96-103)."""
    q = np.asarray(q, dtype=float)
    s = q[..., 3]
    g = np.empty(q.shape[:-1] + (3, 4))
    g[..., :, :3] = s[..., None, None] * np.eye(3) + _skew(q[..., :3])
    g[..., :, 3] = -q[..., :3]
    return g


def normalize(q: np.ndarray) -> np.ndarray:
    q = np.asarray(q, dtype=float)
    nrm = np.linalg.norm(q, axis=-1, keepdims=True)
    if np.any(nrm < 1e-300):
        raise ZeroQuaternionError("cannot normalize a zero quaternion")
    return q / nrm


def hamilton(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Hamilton product a*b (quat.py:41-49)."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    av, aw = a[..., :3], a[..., 3:]
    bv, bw = b[..., :3], b[..., 3:]
    return np.concatenate([aw * bv + bw * av + np.cross(av, bv),
                           aw * bw - np.sum(av * bv, axis=-1, keepdims=True)], axis=-1)


def axis_angle(axis, angle) -> np.ndarray:
    """Unit quaternion of a rotation by ``angle`` about ``axis`` (quat.py:180-188)."""
    axis = np.asarray(axis, dtype=float)
    axis = axis / np.linalg.norm(axis)
    half = 0.5 * float(angle)
    return np.concatenate([axis * np.sin(half), [np.cos(half)]])


def rate_from_omega(q: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Tangent rate 0.5 (w,0) * q for world angular velocity w (quat.py:137-141)."""
    w = np.asarray(w, dtype=float)
    w4 = np.concatenate([w, np.zeros(w.shape[:-1] + (1,))], axis=-1)
    return 0.5 * hamilton(w4, q)


def geodesic(q: np.ndarray, dq: np.ndarray) -> np.ndarray:
    """Great-circle step on S^3; identity below GEODESIC_EPS (quat.py:144-156)."""
    q = np.asarray(q, dtype=float)
    dq = np.asarray(dq, dtype=float)
    nrm = np.linalg.norm(dq, axis=-1, keepdims=True)
    tiny = nrm < GEODESIC_EPS
    safe = np.where(tiny, 1.0, nrm)
    return np.where(tiny, q, q * np.cos(nrm) + dq / safe * np.sin(nrm))


def min_rotation(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Vectorised shortest-arc rotation taking unit ``a`` onto each row of ``b``.

    Same branches as the reference's scalar ``shortest_arc``
    (quat.py:202-219): the antipodal case is a half turn about
    ``normalize(a x helper)`` with helper e_z (e_y when |a_z| > 0.9).
    """
    a = np.asarray(a, dtype=float)
    b = np.atleast_2d(np.asarray(b, dtype=float))
    dot = b @ a
    out = np.empty((b.shape[0], 4))
    anti = dot < -1.0 + 1e-12
    reg = ~anti
    if np.any(reg):
        raw = np.concatenate([np.cross(a, b[reg]), (1.0 + dot[reg])[:, None]], axis=1)
        out[reg] = normalize(raw)
    if np.any(anti):
        helper = np.array([0.0, 1.0, 0.0]) if abs(a[2]) > 0.9 else np.array([0.0, 0.0, 1.0])
        ax = np.cross(a, helper)
        ax = ax / np.linalg.norm(ax)
        out[anti] = np.concatenate([ax, [0.0]])
    return out


def rest_frames(q0: np.ndarray) -> np.ndarray:
    """World->local bond frames G_l(q0) G_r(q0)^T (bonds.py:106-114, geometry.py:219)."""
    return g_left(q0) @ np.swapaxes(g_right(q0), -1, -2)
