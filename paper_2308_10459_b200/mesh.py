"""Tetrahedral scene format: mesh, element/bond construction, surface output.

Host-side data formats on either side of the GPU path:
the reference builds every scene from a tet mesh -- one element per tet, one
bond per interior face (``geometry.py:33-245``) -- and writes one surface OBJ
per frame (``geometry.py:313-358``, ``runner.py:124-127``).  Face adjacency is
built with array sorts instead of a Python dict, with the reference's
orderings (interior faces ``(tet_a, local_a, tet_b, local_b)`` and boundary
faces ``(tet, local)`` ascending), so element and bond indices match the
reference's for the same mesh.  The per-frame reconstruction itself runs on
the GPU (``DeviceSystem.surface``, ``bdem_surface``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import quat as Q
from .state import BondSet, ElementSet

# local faces, outward for a positively oriented tet (a, b, c, d) (geometry.py:23)
FACE_VERTS = np.array([(0, 2, 1), (0, 1, 3), (1, 2, 3), (0, 3, 2)], dtype=np.int64)
DEGENERATE_REL_VOLUME = 1e-12
# the six monotone lattice paths splitting a cube along its main diagonal (scenes.py:84)
KUHN_PATHS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))


class MeshError(ValueError):
    """Malformed or inconsistent tetrahedral mesh input (geometry.py:29-30)."""


@dataclass
class TetMesh:
    """Validated tetrahedral mesh with face adjacency (geometry.py:33-97)."""

    vertices: np.ndarray
    tets: np.ndarray
    volumes: np.ndarray = field(default=None)
    centroids: np.ndarray = field(default=None)
    interior: np.ndarray = field(default=None)   # (tet_a, local_a, tet_b, local_b), a < b
    boundary: np.ndarray = field(default=None)   # (tet, local)

    def __post_init__(self):
        self.vertices = np.asarray(self.vertices, dtype=float)
        self.tets = np.asarray(self.tets, dtype=np.int64)
        if self.volumes is None:
            self._build()

    def _build(self):
        v, t = self.vertices, self.tets
        a, b, c, d = (v[t[:, k]] for k in range(4))
        signed = np.einsum("ij,ij->i", b - a, np.cross(c - a, d - a)) / 6.0
        bad = np.nonzero(signed <= 0.0)[0]
        if bad.size:
            raise MeshError(f"inverted or flat tets at indices {bad.tolist()}")
        mean_vol = float(np.mean(signed))
        bad = np.nonzero(signed < DEGENERATE_REL_VOLUME * mean_vol)[0]
        if bad.size:
            raise MeshError(f"degenerate tets at indices {bad.tolist()}")
        self.volumes = signed
        self.centroids = (a + b + c + d) / 4.0
        nt = t.shape[0]
        tri = t[:, FACE_VERTS]                          # (nt, 4, 3)
        key = np.sort(tri.reshape(-1, 3), axis=1)       # faces by vertex set
        owner = np.arange(4 * nt)                       # = 4 tet + local
        order = np.lexsort((owner, key[:, 2], key[:, 1], key[:, 0]))
        ks = key[order]
        start = np.ones(ks.shape[0], dtype=bool)
        start[1:] = np.any(ks[1:] != ks[:-1], axis=1)
        gid = np.cumsum(start) - 1
        count = np.bincount(gid)
        if np.any(count > 2):
            g = int(np.nonzero(count > 2)[0][0])
            raise MeshError(f"non-manifold face {tuple(ks[start][g].tolist())} shared by "
                            f"{int(count[g])} tets")
        first = order[start]                            # lowest (tet, local) of each face
        pair = count == 2
        second = order[np.nonzero(start)[0][pair] + 1]
        fa, fb = first[pair], second
        interior = np.stack([fa // 4, fa % 4, fb // 4, fb % 4], axis=1)
        single = first[~pair]
        boundary = np.stack([single // 4, single % 4], axis=1)
        self.interior = interior[np.lexsort(interior.T[::-1])].reshape(-1, 4)
        self.boundary = boundary[np.lexsort(boundary.T[::-1])].reshape(-1, 2)

    @property
    def n_tets(self) -> int:
        return self.tets.shape[0]

    def face_vertices(self, tet: int, local: int) -> np.ndarray:
        """Vertex indices of a local face, outward for that tet (geometry.py:91-94)."""
        return self.tets[tet, FACE_VERTS[local]]

    def total_volume(self) -> float:
        return float(np.sum(self.volumes))


def grid_tet_mesh(nx: int, ny: int, nz: int, h: float, origin=(0.0, 0.0, 0.0)) -> TetMesh:
    """Cube grid, six Kuhn tets per cube, cubes in (i, j, k) order and paths in
    KUHN_PATHS order; a negatively oriented tet swaps its last two corners
    (scenes.py:87-119)."""
    origin = np.asarray(origin, dtype=float)
    shape = np.array([nx + 1, ny + 1, nz + 1])
    g = np.stack(np.meshgrid(np.arange(shape[0]), np.arange(shape[1]), np.arange(shape[2]),
                             indexing="ij"), axis=-1).reshape(-1, 3)
    vertices = origin + h * g
    base = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"),
                    axis=-1).reshape(-1, 1, 1, 3)
    steps = np.zeros((len(KUHN_PATHS), 4, 3), dtype=np.int64)
    for p, path in enumerate(KUHN_PATHS):
        for m, axis in enumerate(path):
            steps[p, m + 1:, axis] += 1
    corners = (base + steps[None]).reshape(-1, 4, 3)
    ids = (corners[..., 0] * shape[1] + corners[..., 1]) * shape[2] + corners[..., 2]
    a, b, c, d = (vertices[ids[:, k]] for k in range(4))
    vol = np.einsum("ij,ij->i", b - a, np.cross(c - a, d - a))
    neg = vol < 0.0
    ids[neg, 2], ids[neg, 3] = ids[neg, 3].copy(), ids[neg, 2].copy()
    return TetMesh(vertices, ids)


def build_elements_and_bonds(mesh: TetMesh, density: float, youngs: float,
                             shear_modulus: float, tensile_strength: float = math.inf,
                             shear_strength: float = math.inf):
    """One element per tet (mass ρV, volume-equivalent radius), one bond per
    interior face with the face area as section (geometry.py:165-245)."""
    n = mesh.n_tets
    elements = ElementSet(
        p=mesh.centroids.copy(), q=np.tile(Q.IDENTITY, (n, 1)), v=np.zeros((n, 3)),
        qdot=np.zeros((n, 4)), mass=density * mesh.volumes,
        radius=(3.0 * mesh.volumes / (4.0 * math.pi)) ** (1.0 / 3.0),
        pinned=np.zeros(n, dtype=bool))
    it = mesh.interior
    nb = it.shape[0]
    i_arr, j_arr = it[:, 0].copy(), it[:, 2].copy()
    delta = mesh.centroids[j_arr] - mesh.centroids[i_arr]
    l0 = np.linalg.norm(delta, axis=1)
    if np.any(l0 < 1e-14):
        raise MeshError("coincident tet centroids across a shared face")
    d0 = delta / l0[:, None]
    fv = mesh.vertices[mesh.tets[i_arr[:, None], FACE_VERTS[it[:, 1]]]]   # (nb, 3, 3)
    areas = 0.5 * np.linalg.norm(np.cross(fv[:, 1] - fv[:, 0], fv[:, 2] - fv[:, 0]), axis=1)
    r0 = np.sqrt(areas / math.pi)
    second = math.pi * r0**4 / 4.0
    polar = math.pi * r0**4 / 2.0
    q0 = Q.min_rotation(np.array([1.0, 0.0, 0.0]), d0) if nb else np.zeros((0, 4))
    frame = Q.rest_frames(q0) if nb else np.zeros((0, 3, 3))
    k_diag = np.stack([shear_modulus * polar, youngs * second, youngs * second],
                      axis=1) / l0[:, None] if nb else np.zeros((0, 3))
    bonds = BondSet(
        i=i_arr, j=j_arr, rest_length=l0, radius=r0, d0=d0, q0=q0, frame=frame,
        kn=youngs * areas / l0, kt=shear_modulus * areas / l0, k_diag=k_diag, section=areas,
        second_moment=second, polar_moment=polar,
        tensile_strength=np.full(nb, float(tensile_strength)),
        shear_strength=np.full(nb, float(shear_strength)),
        face_i=it[:, 1].copy(), face_j=it[:, 3].copy())
    return elements, bonds


def mark_surface_elements(mesh: TetMesh) -> np.ndarray:
    """Every tet owning a boundary face (geometry.py:248-253)."""
    flags = np.zeros(mesh.n_tets, dtype=bool)
    if mesh.boundary.size:
        flags[mesh.boundary[:, 0]] = True
    return flags


def boundary_masks(mesh: TetMesh) -> np.ndarray:
    """Per-tet bit mask of its boundary faces (bit = local face index)."""
    mask = np.zeros(mesh.n_tets, dtype=np.int32)
    if mesh.boundary.size:
        np.bitwise_or.at(mask, mesh.boundary[:, 0], (1 << mesh.boundary[:, 1]).astype(np.int32))
    return mask


def reconstruct_surface(mesh: TetMesh, bonds: BondSet, labeling, p: np.ndarray,
                        q: np.ndarray):
    """Triangle soup per fragment with rigidly transported tet vertices
    (geometry.py:313-343), computed on the GPU from host arrays: each
    boundary face once, each broken bond's face once per side."""
    import torch

    from .device import DeviceSystem
    n = mesh.n_tets
    el = ElementSet(np.ascontiguousarray(p, dtype=float), np.ascontiguousarray(q, dtype=float),
                    np.zeros((n, 3)), np.zeros((n, 4)), np.ones(n), np.ones(n))
    dev = DeviceSystem(elements=el, bonds=bonds)
    dev.set_mesh(mesh, bonds)
    labels = torch.as_tensor(np.asarray(labeling.labels, dtype=np.int64), device=dev.device)
    return dev.surface(labels)


def write_surface_obj(path, groups):
    """``g component_<id>``, ``v x y z`` (repr) and 1-based ``f`` lines per
    group, vertex indices continuing across groups (geometry.py:346-358)."""
    lines = []
    offset = 0
    for comp_id, verts, tris in groups:
        lines.append(f"g component_{comp_id}")
        lines += [f"v {x!r} {y!r} {z!r}" for x, y, z in np.asarray(verts, dtype=float).tolist()]
        t = np.asarray(tris, dtype=np.int64) + 1 + offset
        lines += [f"f {a} {b} {c}" for a, b, c in t.tolist()]
        offset += len(verts)
    Path(path).write_text("\n".join(lines) + "\n")
