"""Host mirrors of the reference's struct-of-arrays state.

Field names, shapes, dtypes and defaults follow the reference so that code
written against ``bdem`` can hand its arrays over unchanged:

* ``ElementSet``   -- ``/root/reference/pkg/src/bdem/elements.py:79-123``
* ``BondSet``      -- ``/root/reference/pkg/src/bdem/bonds.py:418-463``
* ``PlasticParams``-- ``/root/reference/pkg/src/bdem/bonds.py:129-144``

These are host (numpy) containers.  The Newton path never computes on them:
``paper_2308_10459_b200.device.DeviceSystem`` uploads them once into HBM and
every kernel works on the device copy.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

INTACT = 0     # bonds.py:26
WEAKENED = 1   # bonds.py:27
BROKEN = 2     # bonds.py:28


class DegenerateBondError(ValueError):
    """Bond endpoints are (numerically) coincident (bonds.py:35-36)."""


class DegenerateShearError(ValueError):
    """Endpoint quaternions are antipodal (bonds.py:39-40)."""


class BrokenBondError(ValueError):
    """Stress was requested for a broken bond (bonds.py:43-44)."""


@dataclass(frozen=True)
class PlasticParams:
    """Yield/damage parameters (bonds.py:129-144), same validation."""

    fracture_strain: float
    yield_strain: float
    weakening: float = 1.0
    damage_exponent: float = 1.0

    def __post_init__(self):
        if not 0.0 < self.yield_strain < self.fracture_strain:
            raise ValueError("need 0 < yield_strain < fracture_strain")
        if not 0.0 <= self.weakening <= 1.0:
            raise ValueError("weakening must lie in [0, 1]")
        if self.damage_exponent <= 0.0:
            raise ValueError("damage_exponent must be positive")


@dataclass
class ElementSet:
    """Per-element state, reference layout: p (n,3), q (n,4) scalar-last."""

    p: np.ndarray
    q: np.ndarray
    v: np.ndarray
    qdot: np.ndarray
    mass: np.ndarray
    radius: np.ndarray
    pinned: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.pinned is None:
            self.pinned = np.zeros(self.p.shape[0], dtype=bool)

    @property
    def n(self) -> int:
        return self.p.shape[0]

    @property
    def rot_mass(self) -> np.ndarray:
        """Quaternion-coordinate mass 1.6 m r^2 (elements.py:104-107)."""
        return 1.6 * self.mass * self.radius**2

    @property
    def inertia(self) -> np.ndarray:
        return 0.4 * self.mass * self.radius**2

    def kinetic_energy(self) -> float:
        """Translational + quaternion-form rotational KE (elements.py:114-117)."""
        lin = 0.5 * np.sum(self.mass * np.sum(self.v**2, axis=1))
        rot = 0.5 * np.sum(self.rot_mass * np.sum(self.qdot**2, axis=1))
        return float(lin + rot)

    def copy(self) -> "ElementSet":
        return ElementSet(self.p.copy(), self.q.copy(), self.v.copy(), self.qdot.copy(),
                          self.mass.copy(), self.radius.copy(), self.pinned.copy())


@dataclass
class BondSet:
    """Per-bond arrays; broken bonds stay in place behind ``status``."""

    i: np.ndarray
    j: np.ndarray
    rest_length: np.ndarray
    radius: np.ndarray
    d0: np.ndarray
    q0: np.ndarray
    frame: np.ndarray
    kn: np.ndarray
    kt: np.ndarray
    k_diag: np.ndarray
    section: np.ndarray
    second_moment: np.ndarray
    polar_moment: np.ndarray
    tensile_strength: np.ndarray
    shear_strength: np.ndarray
    face_i: np.ndarray = field(default=None)
    face_j: np.ndarray = field(default=None)
    status: np.ndarray = field(default=None)
    stiffness_scale: np.ndarray = field(default=None)
    damage: np.ndarray = field(default=None)
    plastic_strain: np.ndarray = field(default=None)
    sigma: np.ndarray = field(default=None)
    tau: np.ndarray = field(default=None)

    def __post_init__(self):
        nb = self.i.shape[0]
        defaults = {
            "face_i": lambda: np.full(nb, -1, dtype=np.int64),
            "face_j": lambda: np.full(nb, -1, dtype=np.int64),
            "status": lambda: np.full(nb, INTACT, dtype=np.int8),
            "stiffness_scale": lambda: np.ones(nb),
            "damage": lambda: np.ones(nb),
            "plastic_strain": lambda: np.zeros(nb),
            "sigma": lambda: np.zeros(nb),
            "tau": lambda: np.zeros(nb),
        }
        for name, make in defaults.items():
            if getattr(self, name) is None:
                setattr(self, name, make())

    @property
    def n(self) -> int:
        return self.i.shape[0]

    @property
    def active(self) -> np.ndarray:
        return self.status != BROKEN

    def energy_terms(self, p, q, want_hess=False, want_grad=True):
        """GPU evaluation with the reference's return tuple (bonds.py:473-504)."""
        from .bond_api import energy_terms
        return energy_terms(self, p, q, want_hess, want_grad)

    # mutable per-bond state that the fracture update writes (bonds.py:532-570)
    STATE_FIELDS = ("status", "stiffness_scale", "damage", "plastic_strain", "sigma", "tau")

    def copy(self) -> "BondSet":
        kw = {f: np.array(getattr(self, f), copy=True) for f in self.__dataclass_fields__}
        return BondSet(**kw)
