"""Seeded synthetic scenes for the five BASELINE.json configurations.

One generator feeds every consumer (the GPU path, the CPU oracle, and --
in this container only -- the reference itself when golden vectors are
made), so all of them see bit-identical arrays.  The rules are SURVEY.md
§8(d):

* element mass = rho (4/3) pi r^3; bond radius r0 = min(r_i, r_j);
  S = pi r0^2, I = pi r0^4 / 4, J = pi r0^4 / 2,
  kn = E S / l0, kt = G S / l0, k_diag = [G J, E I, E I] / l0
  (the per-bond formulas of ``geometry.py:210-225``);
* q0 = shortest_arc(e_x, d0), frame = G_l(q0) G_r(q0)^T (``geometry.py:215-219``);
* G = E / (2 (1 + nu)), nu = 0.25 and rho = 2500 when unstated
  (``scenes.py:43-44``); gravity (0, 0, -9.81) (``scenes.py:29``);
* ``np.random.default_rng(seed)`` for every random draw; coordinates are
  centred near the origin (gradient noise floor).

No public dataset is involved: BASELINE.json's configs are themselves
synthetic lattices, restated here with their stated sizes and parameters.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import quat as Q
from .colliders import HalfSpace
from .state import BondSet, ElementSet, PlasticParams

GRAVITY = (0.0, 0.0, -9.81)


@dataclass
class DriverSpec:
    kind: str                    # "stretch" | "twist"
    ids: np.ndarray
    p0: np.ndarray
    speed: float = 0.0           # stretch: m/s along +x
    axis_point: np.ndarray = None
    rate: float = 0.0            # twist: rad/s about +x


@dataclass
class SceneSpec:
    name: str
    elements: ElementSet
    bonds: BondSet
    dt: float
    youngs: float
    shear_modulus: float
    density: float
    colliders: list = field(default_factory=list)
    gravity: tuple = GRAVITY
    k_contact: float = 1e6
    k_element: float = 1e6
    plastic: PlasticParams | None = None
    driver: DriverSpec | None = None
    mu_s: float = 0.0            # sliding friction (scenes.py:46-47)
    mu_r: float = 0.0            # rolling friction
    mesh: object = None          # TetMesh for scenes built from tets (surface output)
    epsilon: float = 1e-6
    steps: int = 1
    seed: int = 0
    # per-step collider schedule (C2's descending plane): t -> list of colliders
    collider_schedule: object = None
    notes: str = ""


def sphere_mass(radius: np.ndarray, density: float) -> np.ndarray:
    return density * (4.0 / 3.0) * math.pi * radius**3


def build_bonds(pos: np.ndarray, radius: np.ndarray, pairs: np.ndarray, youngs: float,
                shear_modulus: float, tensile: float = math.inf,
                shear: float = math.inf) -> BondSet:
    """Bond arrays for sorted (i<j) pairs with the SURVEY §8(d) rules."""
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    i, j = pairs[:, 0].copy(), pairs[:, 1].copy()
    delta = pos[j] - pos[i]
    l0 = np.linalg.norm(delta, axis=1)
    d0 = delta / l0[:, None]
    r0 = np.minimum(radius[i], radius[j])
    section = math.pi * r0**2
    second = math.pi * r0**4 / 4.0
    polar = math.pi * r0**4 / 2.0
    q0 = Q.min_rotation(np.array([1.0, 0.0, 0.0]), d0)
    frame = Q.rest_frames(q0)
    k_diag = np.stack([shear_modulus * polar, youngs * second, youngs * second], axis=1) / l0[:, None]
    nb = i.shape[0]
    return BondSet(
        i=i, j=j, rest_length=l0, radius=r0, d0=d0, q0=q0, frame=frame,
        kn=youngs * section / l0, kt=shear_modulus * section / l0, k_diag=k_diag,
        section=section, second_moment=second, polar_moment=polar,
        tensile_strength=np.full(nb, float(tensile)), shear_strength=np.full(nb, float(shear)),
    )


def _pairs_within(pos: np.ndarray, cutoff: float) -> np.ndarray:
    from scipy.spatial import cKDTree
    pairs = cKDTree(pos).query_pairs(cutoff, output_type="ndarray").astype(np.int64)
    pairs.sort(axis=1)
    order = np.lexsort((pairs[:, 1], pairs[:, 0]))
    return pairs[order]


def _elements(pos, q, radius, density, pinned=None, v=None) -> ElementSet:
    n = pos.shape[0]
    return ElementSet(
        p=np.ascontiguousarray(pos, dtype=float), q=np.ascontiguousarray(q, dtype=float),
        v=np.zeros((n, 3)) if v is None else np.ascontiguousarray(v, dtype=float),
        qdot=np.zeros((n, 4)),
        mass=sphere_mass(radius, density), radius=np.ascontiguousarray(radius, dtype=float),
        pinned=np.zeros(n, dtype=bool) if pinned is None else pinned,
    )


def _random_unit_quats(rng, n):
    return Q.normalize(rng.normal(size=(n, 4)))


# ---------------------------------------------------------------------------
# C1: cantilever beam (trajectory-parity config #1)
# ---------------------------------------------------------------------------

def cantilever(nx=40, ny=4, nz=4, h=0.01, r=0.005, youngs=1e7, nu=0.3, density=1000.0,
               dt=1e-3, steps=20, epsilon=1e-8) -> SceneSpec:
    """40x4x4 simple-cubic beam, 6-neighbour bonds, x=0 face pinned (BASELINE configs[0])."""
    g = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1)
    g = g.reshape(-1, 3)
    # centred on the origin in all three axes: eps = 1e-8 sits
    # on this beam's gradient noise floor (~1.15e-8 at step 2), so the last
    # bits of the coordinates decide whether the reference commits: with the
    # mean subtracted it commits 20/20 (128 Newton / 3,174 PCG); uncentred,
    # or centred as h (k - (n-1)/2), it stalls from step 2
    pos = h * g.astype(float)
    pos -= pos.mean(axis=0)
    n = pos.shape[0]
    radius = np.full(n, r)
    G = youngs / (2.0 * (1.0 + nu))
    pairs = _pairs_within(pos, 1.01 * h)
    pinned = g[:, 0] == 0
    el = _elements(pos, np.tile(Q.IDENTITY, (n, 1)), radius, density, pinned)
    bonds = build_bonds(pos, radius, pairs, youngs, G)
    return SceneSpec("cantilever", el, bonds, dt, youngs, G, density, k_element=0.0,
                     epsilon=epsilon, steps=steps,
                     notes="SC lattice, cutoff 1.01h, pinned x=0 face, no fracture")


def twisted_beam(nx=40, ny=4, nz=4, rate=10.0, epsilon=1e-8, **kw) -> SceneSpec:
    """The cantilever lattice with its x = max face pinned and twist-driven at
    `rate` rad/s about the beam axis.  SURVEY 8(d) (C4 caution): the
    reference's clamped Newton iteration stalls on this scene (gnorm stuck
    above epsilon, alpha = 1, one PCG iteration per Newton iteration, residual
    in the rotation DOFs next to the driven layer) and the step is not
    committed; the GPU path has to reproduce the stall, not fix it."""
    spec = cantilever(nx=nx, ny=ny, nz=nz, epsilon=epsilon, **kw)
    el = spec.elements
    x = el.p[:, 0]
    ids = np.nonzero(x > x.max() - 1e-9)[0]
    el.pinned[ids] = True
    spec.driver = DriverSpec("twist", ids, el.p[ids].copy(), axis_point=np.zeros(3), rate=rate)
    spec.name = "twisted_beam"
    spec.notes = "cantilever lattice, x = max face twist-driven; the reference stalls"
    return spec


# ---------------------------------------------------------------------------
# C2: jittered cube compressed by a descending plane
# ---------------------------------------------------------------------------

def cube(n_side=22, r=0.002, youngs=3e9, nu=0.25, density=2500.0, seed=2,
         random_q=True, speed=0.5, k_contact=1e9, dt=1e-4, steps=50,
         epsilon=1e-6) -> SceneSpec:
    """Jittered 22^3 lattice, bonds where d < 1.05 (r_i + r_j), plastic fracture."""
    rng = np.random.default_rng(seed)
    g = np.stack(np.meshgrid(*(np.arange(n_side),) * 3, indexing="ij"), -1).reshape(-1, 3)
    pos = 2.0 * r * g.astype(float)
    pos += rng.uniform(-0.05 * r, 0.05 * r, size=pos.shape)
    n = pos.shape[0]
    radius = rng.uniform(0.9 * r, 1.1 * r, size=n)
    q = _random_unit_quats(rng, n) if random_q else np.tile(Q.IDENTITY, (n, 1))
    centre = np.array([pos[:, 0].mean(), pos[:, 1].mean(), 0.0])
    pos -= centre
    cand = _pairs_within(pos, 1.05 * 2.0 * radius.max())
    dist = np.linalg.norm(pos[cand[:, 1]] - pos[cand[:, 0]], axis=1)
    pairs = cand[dist < 1.05 * (radius[cand[:, 0]] + radius[cand[:, 1]])]
    pinned = pos[:, 2] < 0.5 * r
    G = youngs / (2.0 * (1.0 + nu))
    el = _elements(pos, q, radius, density, pinned)
    bonds = build_bonds(pos, radius, pairs, youngs, G)
    z_top = float(pos[:, 2].max())

    def plane(t):
        return [HalfSpace((0.0, 0.0, -1.0), -(z_top - speed * t))]

    return SceneSpec("cube", el, bonds, dt, youngs, G, density, colliders=plane(0.0),
                     k_contact=k_contact, plastic=PlasticParams(1e-3, 6e-4, 0.5, 2.0),
                     epsilon=epsilon, steps=steps, seed=seed, collider_schedule=plane,
                     notes=("random q" if random_q else "identity q")
                     + "; descending HalfSpace at 0.5 m/s; bottom layer pinned")


# ---------------------------------------------------------------------------
# friction scenario (apply_friction, contact.py:303-350)
# ---------------------------------------------------------------------------

def stack(n=4, r=0.002, youngs=1e7, nu=0.25, density=2500.0, mu_s=0.3, mu_r=0.05,
          slide=0.3, spin=40.0, k_contact=1e6, k_element=1e6, dt=1e-4, seed=7,
          steps=8, epsilon=1e-5) -> SceneSpec:
    """Two unbonded lattice blocks: an n x n x 2 block sunk slightly into a
    floor HalfSpace and an (n-1) x (n-1) x 2 block nested into the hollows of its top layer,
    sliding along +x and spinning, with sliding and rolling friction (the
    regime of scenes.py:239-256's drop-fracture: mu_s 0.2-0.3, mu_r 0.05)."""
    rng = np.random.default_rng(seed)
    h = 2.0 * r

    def lattice(nx, nz, origin):
        g = np.stack(np.meshgrid(np.arange(nx), np.arange(nx), np.arange(nz), indexing="ij"), -1)
        return origin + h * g.reshape(-1, 3).astype(float)

    lo = lattice(n, 2, np.array([0.0, 0.0, 0.0]))
    up = lattice(n - 1, 2, np.array([0.5 * h, 0.5 * h, 1.0 * h + 0.69 * h]))
    pos = np.concatenate([lo, up]) + rng.uniform(-0.02 * r, 0.02 * r, size=(lo.shape[0] + up.shape[0], 3))
    n_lo = lo.shape[0]
    npt = pos.shape[0]
    radius = np.full(npt, r)
    q = np.tile(Q.IDENTITY, (npt, 1))
    el = _elements(pos, q, radius, density)
    el.v[n_lo:, 0] = slide
    w = np.zeros((npt, 3))
    w[n_lo:] = spin * rng.normal(size=(npt - n_lo, 3))
    el.qdot[:] = Q.rate_from_omega(q, w)
    pairs = np.concatenate([_pairs_within(pos[:n_lo], 1.05 * h),
                            n_lo + _pairs_within(pos[n_lo:], 1.05 * h)])
    G = youngs / (2.0 * (1.0 + nu))
    bonds = build_bonds(pos, radius, pairs, youngs, G)
    floor = [HalfSpace((0.0, 0.0, 1.0), 0.05 * r)]
    return SceneSpec("stack", el, bonds, dt, youngs, G, density, colliders=floor,
                     k_contact=k_contact, k_element=k_element, mu_s=mu_s, mu_r=mu_r,
                     epsilon=epsilon, steps=steps, seed=seed,
                     notes="two unbonded blocks, floor contact, sliding + rolling friction")


# ---------------------------------------------------------------------------
# tet-mesh scene of the reference (scenes.py:239-256)
# ---------------------------------------------------------------------------

def drop_fracture(resolution=1, youngs=1e9, density=2500.0, speed=4.0, tensile_strength=3e5,
                  shear_strength=3e5, dt=0.002, steps=10, epsilon=1e-5) -> SceneSpec:
    """The reference's drop-fracture scene: a (4r x 4r x 1) cube-grid plate of
    Kuhn tets (cell 0.4/(4r), bottom at z=0.05) falling at ``speed`` onto a
    floor, sliding/rolling friction 0.2/0.05, contact stiffness 2e7."""
    from .mesh import build_elements_and_bonds, grid_tet_mesh
    n = 4 * resolution
    h = 0.4 / n
    G = youngs / 2.5
    mesh = grid_tet_mesh(n, n, 1, h, origin=(0.0, 0.0, 0.05))
    el, bonds = build_elements_and_bonds(mesh, density, youngs, G, tensile_strength,
                                         shear_strength)
    el.v[:, 2] = -speed
    return SceneSpec("drop-fracture", el, bonds, dt, youngs, G, density,
                     colliders=[HalfSpace((0.0, 0.0, 1.0), 0.0)], k_contact=2e7, k_element=2e7,
                     mu_s=0.2, mu_r=0.05, mesh=mesh, epsilon=epsilon, steps=steps,
                     notes="tet-mesh plate (one element per tet, one bond per interior face)")


# ---------------------------------------------------------------------------
# C3: ceramic plate impact (north star)
# ---------------------------------------------------------------------------

def plate(nx=1000, ny=600, r=0.25e-3, youngs=3e11, nu=0.25, density=3900.0,
          tilt_deg=10.0, v0=5.0, k_contact=1e9, dt=5e-6, steps=200,
          epsilon=1e-3) -> SceneSpec:
    """One triangular (HCP) layer, bonds to first+second shell (cutoff 1.8a).

    At 1000x600 this gives 3,591,004 bonds (11.97 per particle).
    Tilted 10 degrees about y with the lowest centre at z = 1e-7 m, falling
    at 5 m/s onto HalfSpace((0,0,1), 0).
    """
    a = 2.0 * r
    iy, ix = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    x = a * (ix + 0.5 * (iy % 2)).astype(float)
    y = a * (math.sqrt(3.0) / 2.0) * iy.astype(float)
    pos = np.stack([x.ravel(), y.ravel(), np.zeros(nx * ny)], axis=1)
    pos[:, 0] -= 0.5 * (pos[:, 0].max() + pos[:, 0].min())
    pos[:, 1] -= 0.5 * (pos[:, 1].max() + pos[:, 1].min())
    n = pos.shape[0]
    pairs = _pairs_within(pos, 1.8 * a)
    th = math.radians(tilt_deg)
    rot = np.array([[math.cos(th), 0.0, math.sin(th)], [0.0, 1.0, 0.0],
                    [-math.sin(th), 0.0, math.cos(th)]])
    pos = pos @ rot.T
    pos[:, 2] += 1e-7 - pos[:, 2].min()
    radius = np.full(n, r)
    G = youngs / (2.0 * (1.0 + nu))
    v = np.tile([0.0, 0.0, -v0], (n, 1))
    el = _elements(pos, np.tile(Q.IDENTITY, (n, 1)), radius, density, v=v)
    bonds = build_bonds(pos, radius, pairs, youngs, G)
    return SceneSpec("plate", el, bonds, dt, youngs, G, density,
                     colliders=[HalfSpace((0.0, 0.0, 1.0), 0.0)], k_contact=k_contact,
                     plastic=PlasticParams(2e-4, 1.5e-4, 0.5, 2.0), epsilon=epsilon,
                     steps=steps,
                     notes=f"{nx}x{ny} triangular layer, a=2r, cutoff 1.8a, tilt {tilt_deg} deg")


# ---------------------------------------------------------------------------
# C4: shear-stiff rope with a twist driver
# ---------------------------------------------------------------------------

def rope(n=100_000, r=1e-3, youngs=1e9, shear_ratio=10.0, density=2500.0, rate=10.0,
         eps_c=5e-3, dt=1e-4, steps=100, epsilon=1e-5) -> SceneSpec:
    """1D chain, nearest-neighbour bonds, G = 10 E, end twisted at 10 rad/s."""
    pos = np.zeros((n, 3))
    pos[:, 0] = 2.0 * r * np.arange(n)
    pos[:, 0] -= 0.5 * pos[-1, 0]
    radius = np.full(n, r)
    pairs = np.stack([np.arange(n - 1), np.arange(1, n)], axis=1)
    pinned = np.zeros(n, dtype=bool)
    pinned[[0, n - 1]] = True
    G = shear_ratio * youngs
    strength = youngs * eps_c
    el = _elements(pos, np.tile(Q.IDENTITY, (n, 1)), radius, density, pinned)
    bonds = build_bonds(pos, radius, pairs, youngs, G, tensile=strength, shear=strength)
    ids = np.array([n - 1])
    drv = DriverSpec("twist", ids, pos[ids].copy(), axis_point=np.zeros(3), rate=rate)
    return SceneSpec("rope", el, bonds, dt, youngs, G, density, driver=drv,
                     epsilon=epsilon, steps=steps,
                     notes="G = 10 E; strengths = E eps_c; last element twist-driven")


# ---------------------------------------------------------------------------
# C5: 2M-sphere scale block
# ---------------------------------------------------------------------------

_BLOCK_OFFSETS = np.array([[1, 0, 0], [0, 1, 0], [0, 0, 1],
                           [1, 1, 0], [1, 0, 1], [0, 1, 1]])


def block(n_side=126, r=1e-3, youngs=1e10, nu=0.25, density=2500.0, seed=5, speed=1.0,
          dt=1e-5, steps=20, epsilon=1e-6, random_q=True) -> SceneSpec:
    """Jittered n^3 lattice with 12 neighbours per interior particle.

    Bond rule (fixed here, SURVEY §8(d) leaves it to the generator): lattice
    offsets +-x, +-y, +-z, +-(1,1,0), +-(1,0,1), +-(0,1,1), giving ~6 bonds
    per particle (≈12.0M bonds at 126^3).
    """
    rng = np.random.default_rng(seed)
    m = n_side
    g = np.stack(np.meshgrid(*(np.arange(m),) * 3, indexing="ij"), -1).reshape(-1, 3)
    pos = 2.0 * r * g.astype(float)
    pos += rng.uniform(-0.05 * r, 0.05 * r, size=pos.shape)
    pos -= pos.mean(axis=0)
    n = pos.shape[0]
    radius = rng.uniform(0.9 * r, 1.1 * r, size=n)
    q = _random_unit_quats(rng, n) if random_q else np.tile(Q.IDENTITY, (n, 1))
    lin = np.arange(n).reshape(m, m, m)
    chunks = []
    for off in _BLOCK_OFFSETS:
        a = lin[: m - off[0], : m - off[1], : m - off[2]].ravel()
        b = lin[off[0]:, off[1]:, off[2]:].ravel()
        chunks.append(np.stack([a, b], axis=1))
    pairs = np.concatenate(chunks)
    order = np.lexsort((pairs[:, 1], pairs[:, 0]))
    pairs = pairs[order]
    drive_ids = np.nonzero(g[:, 0] == m - 1)[0]
    pinned = (g[:, 0] == 0) | (g[:, 0] == m - 1)
    G = youngs / (2.0 * (1.0 + nu))
    el = _elements(pos, q, radius, density, pinned)
    bonds = build_bonds(pos, radius, pairs, youngs, G)
    drv = DriverSpec("stretch", drive_ids, pos[drive_ids].copy(), speed=speed)
    return SceneSpec("block", el, bonds, dt, youngs, G, density, driver=drv,
                     plastic=PlasticParams(5e-4, 3e-4), epsilon=epsilon, steps=steps,
                     seed=seed, notes="12-neighbour jittered lattice, random q, x-min pinned, "
                                      "x-max stretch-driven")


CONFIGS = {"cantilever": cantilever, "cube": cube, "plate": plate, "rope": rope,
           "block": block}
