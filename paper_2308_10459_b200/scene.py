"""Scene container and the pinned-element drivers.

``Scene`` mirrors ``/root/reference/pkg/src/bdem/scenes.py:32-77`` (same
attribute names; ``mesh`` is optional because lattice scenes have none).
The Newton path keeps its state in HBM (``DeviceSystem``); the numpy arrays
of ``scene.elements`` / ``scene.bonds`` are the host view.  ``stable_step``
keeps the two in step according to ``scene.host_sync``:

* ``host_sync=True`` (default, drop-in semantics): every step uploads the
  host state before and downloads it after, exactly like calling the
  reference on numpy arrays;
* ``host_sync=False`` (device-resident): state stays in HBM between steps;
  call ``scene.sync_to_host()`` to refresh the numpy view.

Drivers mirror ``scenes.py:146-176``.  They only touch the (few) driven
rows, so the device path evaluates them on the host and scatters the rows.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import quat as Q
from .state import BondSet, ElementSet, PlasticParams

GRAVITY = np.array([0.0, 0.0, -9.81])


@dataclass
class FragmentLabeling:
    """Connected components over intact bonds (geometry.py:285-292)."""

    labels: np.ndarray

    @property
    def components(self) -> list:
        order = np.argsort(self.labels, kind="stable")
        cuts = np.flatnonzero(np.diff(self.labels[order])) + 1
        return [list(map(int, c)) for c in np.split(order, cuts)] if self.labels.size else []

    @property
    def n_components(self) -> int:
        return int(self.labels.max()) + 1 if self.labels.size else 0


class StretchDriver:
    """Constant-velocity axial motion of the driven rows (scenes.py:146-155)."""

    def __init__(self, ids, p0, speed):
        self.ids = np.asarray(ids, dtype=np.int64)
        self.p0 = np.asarray(p0, dtype=float)
        self.velocity = np.array([float(speed), 0.0, 0.0])

    def rows(self, t):
        n = self.ids.size
        return (self.p0 + t * self.velocity, np.tile(self.velocity, (n, 1)),
                np.tile(Q.IDENTITY, (n, 1)), np.zeros((n, 4)))

    def __call__(self, elements, t):
        p, v, q, qd = self.rows(t)
        elements.p[self.ids], elements.v[self.ids] = p, v
        elements.q[self.ids], elements.qdot[self.ids] = q, qd


class TwistDriver:
    """Constant-rate rotation of the driven rows about +x (scenes.py:158-176)."""

    def __init__(self, ids, p0, axis_point, rate):
        self.ids = np.asarray(ids, dtype=np.int64)
        self.p0 = np.asarray(p0, dtype=float)
        self.axis_point = np.asarray(axis_point, dtype=float)
        self.rate = float(rate)

    def rows(self, t):
        ex = np.array([1.0, 0.0, 0.0])
        w = self.rate * ex
        rot = Q.axis_angle(ex, self.rate * t)
        arm0 = self.p0 - self.axis_point
        c, s = np.cos(self.rate * t), np.sin(self.rate * t)
        arm = np.stack([arm0[:, 0], c * arm0[:, 1] - s * arm0[:, 2],
                        s * arm0[:, 1] + c * arm0[:, 2]], axis=1)
        n = self.ids.size
        q = np.broadcast_to(rot, (n, 4))
        return (self.axis_point + arm, np.cross(w, arm), q.copy(), Q.rate_from_omega(q, w))

    def __call__(self, elements, t):
        p, v, q, qd = self.rows(t)
        elements.p[self.ids], elements.v[self.ids] = p, v
        elements.q[self.ids], elements.qdot[self.ids] = q, qd


def stretch_driver(ids, p0, speed):
    return StretchDriver(ids, p0, speed)


def twist_driver(ids, p0, axis_point, rate):
    return TwistDriver(ids, p0, axis_point, rate)


def driver_from_spec(spec):
    if spec is None:
        return None
    if spec.kind == "stretch":
        return StretchDriver(spec.ids, spec.p0, spec.speed)
    if spec.kind == "twist":
        return TwistDriver(spec.ids, spec.p0, spec.axis_point, spec.rate)
    raise ValueError(spec.kind)


class Scene:
    """Scene state (scenes.py:32-77); attribute names follow the reference."""

    def __init__(self, name, mesh, elements: ElementSet, bonds: BondSet, colliders=None,
                 gravity=None, dt=1.0 / 60.0, youngs=1e7, shear_modulus=4e6, density=2500.0,
                 k_contact=1e6, k_element=1e6, mu_s=0.0, mu_r=0.0,
                 plastic: PlasticParams | None = None, driver=None, time=0.0, p_prev=None,
                 q_prev=None, labels=None, surface_flags=None, *, host_sync=True):
        """Positional and keyword order of the reference dataclass
        (scenes.py:31-52: name, mesh, elements, bonds, colliders, gravity, dt,
        youngs, shear_modulus, density, k_contact, k_element, mu_s, mu_r,
        plastic, driver, time, p_prev, q_prev, labels, surface_flags); ``mesh``
        may be None (lattice scenes), ``host_sync`` is keyword-only."""
        self.name, self.mesh = name, mesh
        self.elements, self.bonds = elements, bonds
        self.colliders = list(colliders or [])
        self.gravity = np.array(GRAVITY if gravity is None else gravity, dtype=float)
        self.dt, self.youngs, self.shear_modulus, self.density = dt, youngs, shear_modulus, density
        self.k_contact, self.k_element = k_contact, k_element
        self.mu_s, self.mu_r = mu_s, mu_r
        self.plastic, self.driver, self.time = plastic, driver, time
        self.p_prev, self.q_prev = p_prev, q_prev
        if surface_flags is None:                       # scenes.py:59-60
            if mesh is not None:
                from .mesh import mark_surface_elements
                surface_flags = mark_surface_elements(mesh)
            else:
                surface_flags = np.zeros(elements.n, dtype=bool)
        self.surface_flags = surface_flags
        self.host_sync = host_sync
        self._labels = labels
        self._device = None
        if self.p_prev is None:
            self.bootstrap_history()

    # -- reference API ------------------------------------------------------
    def bootstrap_history(self):
        """Seed the two-point history from the velocities (scenes.py:64-68)."""
        if self._device is not None and not self.host_sync:
            self._device.bootstrap_history(self.dt)
            return
        el = self.elements
        self.p_prev = el.p - self.dt * el.v
        self.q_prev = Q.normalize(Q.geodesic(el.q, -self.dt * el.qdot))

    def force_scale(self) -> float:
        g = float(np.linalg.norm(self.gravity))
        if g == 0.0:
            return 1.0
        return float(np.sqrt(np.sum((self.elements.mass * g) ** 2)))

    def default_epsilon(self) -> float:
        """'auto' tolerance 1e-4 |m g| (scenes.py:76-77)."""
        return 1e-4 * self.force_scale()

    @property
    def labels(self) -> FragmentLabeling:
        if self._labels is None:
            from .step import label_components
            self._labels = label_components(self.elements.n, self.bonds, scene=self)
        return self._labels

    @labels.setter
    def labels(self, value):
        self._labels = value

    # -- device residency ---------------------------------------------------
    @property
    def device(self):
        if self._device is None:
            from .device import DeviceSystem
            self._device = DeviceSystem(self)
            if self.mesh is not None:
                self._device.set_mesh(self.mesh, self.bonds)
        return self._device

    def reconstruct_surface(self):
        """reconstruct_surface(mesh, bonds, labels, p, q) of the current state
        (geometry.py:313-343), computed on the GPU."""
        from .step import label_components
        dev = self.device
        if getattr(dev, "labels", None) is None:
            label_components(dev.n, self.bonds, self)
        return dev.surface(dev.labels)

    def sync_to_host(self):
        if self._device is not None:
            self._device.download_state(self)

    @classmethod
    def from_spec(cls, spec, host_sync=True) -> "Scene":
        return cls(spec.name, spec.mesh, spec.elements, spec.bonds, colliders=spec.colliders,
                   gravity=spec.gravity, dt=spec.dt, youngs=spec.youngs,
                   shear_modulus=spec.shear_modulus, density=spec.density,
                   k_contact=spec.k_contact, k_element=spec.k_element, plastic=spec.plastic,
                   driver=driver_from_spec(spec.driver), mu_s=spec.mu_s, mu_r=spec.mu_r,
                   host_sync=host_sync)
