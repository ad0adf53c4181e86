"""Static colliders (signed-distance penalties on element centers).

Mirrors ``/root/reference/pkg/src/bdem/contact.py:25-133``: ``HalfSpace``
(``normal . p < offset`` is inside), ``SphereCollider`` and ``BoxCollider``.
The objects here are plain parameter holders; the penalty energy, gradient
and the clamped curvature are evaluated on the GPU by the element kernel
(``csrc/element_kernels.cu``), which receives each collider as a
``bdem_collider_t`` record (``include/bdem_sm100.h``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

COLLIDER_HALFSPACE = 0
COLLIDER_SPHERE = 1
COLLIDER_BOX = 2


class Collider:
    kind: int = -1

    def packed(self) -> tuple:
        """(kind, a0..a5) for the device record."""
        raise NotImplementedError


@dataclass(frozen=True)
class HalfSpace(Collider):
    normal: tuple
    offset: float
    kind = COLLIDER_HALFSPACE

    def __post_init__(self):
        n = np.asarray(self.normal, dtype=float)
        object.__setattr__(self, "normal", tuple(n / np.linalg.norm(n)))

    def sdf(self, p):
        return np.asarray(p, dtype=float) @ np.asarray(self.normal) - self.offset

    def packed(self):
        n = self.normal
        return (self.kind, n[0], n[1], n[2], float(self.offset), 0.0, 0.0)


@dataclass(frozen=True)
class SphereCollider(Collider):
    center: tuple
    radius: float
    kind = COLLIDER_SPHERE

    def packed(self):
        c = tuple(float(x) for x in self.center)
        return (self.kind, c[0], c[1], c[2], float(self.radius), 0.0, 0.0)


@dataclass(frozen=True)
class BoxCollider(Collider):
    center: tuple
    half_extents: tuple
    kind = COLLIDER_BOX

    def packed(self):
        c = tuple(float(x) for x in self.center)
        h = tuple(float(x) for x in self.half_extents)
        return (self.kind, c[0], c[1], c[2], h[0], h[1], h[2])
