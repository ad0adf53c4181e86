"""Tet-mesh scenes on the GPU against the reference's drop-fracture scene
(tests/golden/mesh_drop.npz; scenes.py:239-256 with strengths 3e4): the
implicit trajectory with friction and fracture, and the per-frame surface
reconstruction (reconstruct_surface / write_surface_obj, geometry.py:313-358)
-- bit-identical vertices and OBJ text on the reference's own states."""

import numpy as np
import pytest

from _fixtures import bonds_from, close, load
from test_mesh import reference_obj_text

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    return load("mesh_drop.npz")


def _spec():
    from paper_2308_10459_b200 import configs as C
    return C.drop_fracture(tensile_strength=3e4, shear_strength=3e4)


@pytest.mark.parametrize("tag", ["surf0", "surf1"])
def test_surface_bit_exact_on_reference_state(cuda_ok, gold, tag, tmp_path):
    from paper_2308_10459_b200 import mesh as M
    from paper_2308_10459_b200.scene import FragmentLabeling
    spec = _spec()
    b = bonds_from(gold, "init_b_")
    b.face_i, b.face_j = gold["init_b_face_i"], gold["init_b_face_j"]
    if tag == "surf0":
        p, q = gold["init_el_p"], gold["init_el_q"]
        labels = np.zeros(spec.mesh.n_tets, dtype=np.int64)
    else:
        p, q = gold["p"][-1], gold["q"][-1]
        b.status = gold["final_status"].copy()
        labels = gold["labels"]
    groups = M.reconstruct_surface(spec.mesh, b, FragmentLabeling(labels), p, q)
    assert [g[0] for g in groups] == list(range(len(gold[f"{tag}_counts"])))
    assert [g[1].shape[0] for g in groups] == gold[f"{tag}_counts"].tolist()
    assert np.array_equal(np.concatenate([g[1] for g in groups]), gold[f"{tag}_verts"])
    assert np.array_equal(np.concatenate([g[2] for g in groups]), gold[f"{tag}_tris"])
    path = tmp_path / "s.obj"
    M.write_surface_obj(path, groups)
    assert path.read_text() == reference_obj_text(gold, tag)


def test_drop_trajectory_and_surface_vs_reference(cuda_ok, gold):
    from paper_2308_10459_b200 import Scene, SolverConfig, stable_step
    spec = _spec()
    scene = Scene.from_spec(spec)
    cfg = SolverConfig(epsilon=float(gold["epsilon"]), max_iterations=300)
    m_dt2 = (spec.elements.mass / spec.dt**2).min()
    atol_p = 10 * float(gold["epsilon"]) / m_dt2
    mq_dt2 = (1.6 * spec.elements.mass * spec.elements.radius**2 / spec.dt**2).min()
    atol_q = 10 * float(gold["epsilon"]) / mq_dt2
    events = []
    for s in range(gold["p"].shape[0]):
        rep = stable_step(scene, cfg)
        assert rep.committed == bool(gold["committed"][s])
        assert rep.contact_pairs == int(gold["pairs"][s])
        events += [(s, bb) for bb, _, _ in rep.broken]
        ok, info = close(scene.elements.p, gold["p"][s], 1e-8, atol_p)
        assert ok, (s, info)
        ok, info = close(scene.elements.q, gold["q"][s], 1e-8, atol_q)
        assert ok, (s, info)
    assert events == [(int(a), int(b)) for a, b, _, _ in gold["events"]]
    assert np.array_equal(scene.bonds.status, gold["final_status"])
    assert np.array_equal(scene.labels.labels, gold["labels"])
    assert np.array_equal(scene.surface_flags, gold["surface_flags"])
    groups = scene.reconstruct_surface()
    assert [g[1].shape[0] for g in groups] == gold["surf1_counts"].tolist()
    ok, info = close(np.concatenate([g[1] for g in groups]), gold["surf1_verts"], 1e-8,
                     atol_p + 0.1 * atol_q)
    assert ok, info


def test_runner_writes_one_obj_per_frame(cuda_ok, tmp_path):
    from paper_2308_10459_b200 import SolverConfig
    from paper_2308_10459_b200.runner import run_simulation
    from paper_2308_10459_b200.scene import Scene
    scene = Scene.from_spec(_spec())
    stats = run_simulation(scene, SolverConfig(epsilon=1e-5, max_iterations=300), frames=2,
                           fps=500.0, outdir=tmp_path)
    assert len(stats.rows) == 2
    for k in range(2):
        text = (tmp_path / f"frame_{k:05d}.obj").read_text().splitlines()
        assert text[0] == "g component_0"
        nv = sum(ln.startswith("v ") for ln in text)
        nf = sum(ln.startswith("f ") for ln in text)
        assert nv == 3 * nf > 0
