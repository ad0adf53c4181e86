"""Tet-mesh scene format on the host: mesh adjacency,
element/bond construction, the tetmesh text format and the OBJ writer,
against the reference's own arrays and text (tests/golden/mesh_drop.npz,
written by the reference's drop_fracture scene, scenes.py:239-256)."""

import numpy as np
import pytest

from _fixtures import BOND_FIELDS, load
from paper_2308_10459_b200 import mesh as M


@pytest.fixture(scope="module")
def gold():
    return load("mesh_drop.npz")


def test_grid_mesh_matches_reference(gold):
    m = M.grid_tet_mesh(4, 4, 1, 0.1, origin=(0.0, 0.0, 0.05))
    assert np.array_equal(m.vertices, gold["mesh_vertices"])
    assert np.array_equal(m.tets, gold["mesh_tets"])
    assert np.array_equal(m.interior, gold["mesh_interior"])
    assert np.array_equal(m.boundary, gold["mesh_boundary"])
    assert np.array_equal(m.volumes, gold["mesh_volumes"])
    assert np.array_equal(m.centroids, gold["mesh_centroids"])


def test_drop_scene_elements_and_bonds(gold):
    from paper_2308_10459_b200 import configs as C
    spec = C.drop_fracture(tensile_strength=3e4, shear_strength=3e4)
    el, b = spec.elements, spec.bonds
    for f in ("p", "q", "v", "mass", "radius"):
        np.testing.assert_allclose(getattr(el, f), gold["init_el_" + f], rtol=1e-15, atol=0)
    for f in ("i", "j", "face_i", "face_j", "status"):
        assert np.array_equal(getattr(b, f), gold["init_b_" + f]), f
    for f in BOND_FIELDS:
        if f in ("i", "j", "status"):
            continue
        a, r = np.asarray(getattr(b, f), dtype=float), gold["init_b_" + f].astype(float)
        fin = np.isfinite(r)
        assert np.array_equal(fin, np.isfinite(a)), f
        np.testing.assert_allclose(a[fin], r[fin], rtol=1e-14, atol=1e-300, err_msg=f)
    assert np.array_equal(M.mark_surface_elements(spec.mesh),
                          M.boundary_masks(spec.mesh) != 0)


def test_non_manifold_face():
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, -1], [1, 1, 1.0]])
    tets = np.array([[0, 1, 2, 3], [0, 2, 1, 4], [0, 1, 2, 5]])
    tets[2] = [0, 1, 2, 5] if np.dot(np.cross(v[1] - v[0], v[2] - v[0]), v[5] - v[0]) > 0 \
        else [0, 2, 1, 5]
    with pytest.raises(M.MeshError, match="non-manifold"):
        M.TetMesh(v, tets)


def reference_obj_text(gold, tag):
    """The reference's OBJ text with numpy 2's scalar repr undone: its
    ``f"{x!r}"`` prints ``np.float64(0.05)`` under numpy >= 2 (the
    installed 2.3) and ``0.05`` under the numpy 1.x its pyproject allows;
    the plain form is the OBJ format it means to write."""
    import re
    return re.sub(r"np\.float64\(([^)]*)\)", r"\1", str(gold[f"{tag}_obj"]))


@pytest.mark.parametrize("tag", ["surf0", "surf1"])
def test_obj_writer_matches_reference_text(gold, tag, tmp_path):
    """write_surface_obj on the reference's own groups reproduces its bytes
    (modulo numpy 2's scalar repr, see reference_obj_text)."""
    counts = gold[f"{tag}_counts"]
    verts, tris = gold[f"{tag}_verts"], gold[f"{tag}_tris"]
    groups, v0, t0 = [], 0, 0
    for c, k in enumerate(counts):
        groups.append((c, verts[v0:v0 + k], tris[t0:t0 + k // 3]))
        v0 += k
        t0 += k // 3
    path = tmp_path / "s.obj"
    M.write_surface_obj(path, groups)
    assert path.read_text() == reference_obj_text(gold, tag)
