"""The reference's quaternion tests (pkg/tests/test_quat.py: TestNullspace,
TestGeodesic, TestNormalize) restated for the kernels of the Newton path that
carry those operations: bdem_direction (dq = G_l(q)^T y_rot, solver.py:409-418,
quat.py:81-93), bdem_trial_point (q_t = normalize(geodesic(q, alpha dq)),
solver.py:399-401, quat.py:144-164) and bdem_normalize_free (solver.py:516).
Values are also compared with the host mirror of quat.py."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 1000


@pytest.fixture(scope="module")
def rope_system(cuda_ok):
    import torch

    from paper_2308_10459_b200 import configs
    from paper_2308_10459_b200.scene import Scene
    from paper_2308_10459_b200.step import prepare_step
    scene = Scene.from_spec(configs.rope(n=N), host_sync=False)
    prepare_step(scene)
    torch.cuda.synchronize()
    return scene.device


def _random_unit(rng, n):
    q = rng.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _direction(dev, q, y_rot, y_pos=None, sign=1.0):
    import torch
    y = torch.zeros(6, dev.vstride, dtype=torch.float64, device="cuda")
    free = np.nonzero(dev.free_np)[0]
    if y_pos is not None:
        y[:3, :dev.nf] = torch.from_numpy(np.ascontiguousarray(y_pos[free].T)).cuda()
    y[3:, :dev.nf] = torch.from_numpy(np.ascontiguousarray(y_rot[free].T)).cuda()
    qd = torch.from_numpy(q).cuda()
    dev.dp.zero_(); dev.dq.zero_()
    dev.call("bdem_direction", dev.sysp, qd.data_ptr(), y.reshape(-1).data_ptr(), float(sign),
             dev.dp.data_ptr(), dev.dq.data_ptr(), dev.stream)
    torch.cuda.synchronize()
    return dev.dp.cpu().numpy(), dev.dq.cpu().numpy()


def _trial(dev, p, q, dp, dq, alpha):
    import torch
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    pd, qd, dpd, dqd = t(p), t(q), t(dp), t(dq)
    pt, qt = torch.empty_like(pd), torch.empty_like(qd)
    dev.call("bdem_trial_point", dev.sysp, pd.data_ptr(), qd.data_ptr(), dpd.data_ptr(),
             dqd.data_ptr(), float(alpha), pt.data_ptr(), qt.data_ptr(), dev.stream)
    torch.cuda.synchronize()
    return pt.cpu().numpy(), qt.cpu().numpy()


class TestNullspaceDirection:
    """G_l(q)^T maps a reduced rotation 3-vector to a tangent of the sphere at q."""

    def test_annihilates_base_quaternion(self, rope_system):
        dev = rope_system
        rng = np.random.default_rng(11)
        q, y = _random_unit(rng, N), rng.normal(size=(N, 3))
        _, dq = _direction(dev, q, y)
        free = dev.free_np
        assert np.abs(np.einsum("ij,ij->i", q, dq))[free].max() < 1e-15 * 4
        assert np.all(dq[~free] == 0.0)          # pinned rows are not written

    def test_rows_orthonormal_norm_preserved(self, rope_system):
        dev = rope_system
        rng = np.random.default_rng(12)
        q, y = _random_unit(rng, N), rng.normal(size=(N, 3))
        _, dq = _direction(dev, q, y)
        free = dev.free_np
        np.testing.assert_allclose(np.linalg.norm(dq, axis=1)[free],
                                   np.linalg.norm(y, axis=1)[free], rtol=1e-14)

    def test_identity_reduces_to_selector(self, rope_system):
        from paper_2308_10459_b200 import quat as Q
        dev = rope_system
        rng = np.random.default_rng(13)
        y = rng.normal(size=(N, 3))
        _, dq = _direction(dev, np.tile(Q.IDENTITY, (N, 1)), y)
        free = dev.free_np
        assert np.array_equal(dq[free, :3], y[free]) and np.all(dq[free, 3] == 0.0)

    def test_matches_host_mirror_and_sign(self, rope_system):
        from paper_2308_10459_b200 import quat as Q
        dev = rope_system
        rng = np.random.default_rng(14)
        q, y, yp = _random_unit(rng, N), rng.normal(size=(N, 3)), rng.normal(size=(N, 3))
        dp, dq = _direction(dev, q, y, yp, sign=-1.0)
        free = dev.free_np
        ref = -np.einsum("nij,ni->nj", Q.g_left(q), y)
        np.testing.assert_allclose(dq[free], ref[free], rtol=0, atol=4e-16 * np.abs(y).max())
        assert np.array_equal(dp[free], -yp[free])


class TestGeodesicTrialPoint:
    def test_zero_step(self, rope_system):
        dev = rope_system
        rng = np.random.default_rng(21)
        q, p = _random_unit(rng, N), rng.normal(size=(N, 3))
        pt, qt = _trial(dev, p, q, np.zeros((N, 3)), np.zeros((N, 4)), 1.0)
        assert np.array_equal(pt, p)
        # below GEODESIC_EPS the base point is returned, then normalised
        np.testing.assert_allclose(qt, q, rtol=0, atol=2.3e-16)

    def test_quarter_turn_lands_on_pole(self, rope_system):
        from paper_2308_10459_b200 import quat as Q
        dev = rope_system
        q = np.tile(Q.IDENTITY, (N, 1))
        dq = np.tile([np.pi / 2, 0.0, 0.0, 0.0], (N, 1))
        _, qt = _trial(dev, np.zeros((N, 3)), q, np.zeros((N, 3)), dq, 1.0)
        free = dev.free_np
        np.testing.assert_allclose(qt[free], np.tile([1.0, 0.0, 0.0, 0.0], (int(free.sum()), 1)),
                                   rtol=0, atol=1e-15)
        assert np.array_equal(qt[~free], q[~free])      # pinned rows do not move

    def test_stays_on_sphere(self, rope_system):
        dev = rope_system
        rng = np.random.default_rng(23)
        q = _random_unit(rng, N)
        w = rng.normal(size=(N, 4))
        dq = w - q * np.einsum("ij,ij->i", q, w)[:, None]      # tangent_project
        _, qt = _trial(dev, np.zeros((N, 3)), q, np.zeros((N, 3)), dq, 0.7)
        assert np.abs(np.linalg.norm(qt, axis=1) - 1.0).max() < 1e-12

    @pytest.mark.parametrize("alpha", [1.0, 0.25, 1e-9])
    def test_matches_host_mirror(self, rope_system, alpha):
        from paper_2308_10459_b200 import quat as Q
        dev = rope_system
        rng = np.random.default_rng(24)
        q, p = _random_unit(rng, N), rng.normal(size=(N, 3))
        w, dp = rng.normal(size=(N, 4)), rng.normal(size=(N, 3))
        dq = w - q * np.einsum("ij,ij->i", q, w)[:, None]
        pt, qt = _trial(dev, p, q, dp, dq, alpha)
        free = dev.free_np
        ref = Q.normalize(Q.geodesic(q, alpha * dq))
        # a few ulps: the device and numpy sin / cos are each within 1 ulp, not equal
        np.testing.assert_allclose(qt[free], ref[free], rtol=0, atol=2e-15)
        np.testing.assert_allclose(pt, p + alpha * dp, rtol=0, atol=1e-15 * np.abs(p).max())


class TestNormalizeFree:
    def test_scales_to_unit_scale_invariant_unit_unchanged(self, rope_system):
        import torch
        dev = rope_system
        rng = np.random.default_rng(31)
        q = _random_unit(rng, N)
        scaled = q * rng.uniform(0.1, 7.0, size=(N, 1))
        free = dev.free_np
        outs = []
        for arr in (q, scaled):
            t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
            dev.call("bdem_normalize_free", dev.sysp, t.data_ptr(), dev.stream)
            torch.cuda.synchronize()
            outs.append(t.cpu().numpy())
        assert np.abs(np.linalg.norm(outs[1], axis=1)[free] - 1.0).max() < 4e-16
        np.testing.assert_allclose(outs[1][free], q[free], rtol=0, atol=4e-16)
        np.testing.assert_allclose(outs[0][free], q[free], rtol=0, atol=2.3e-16)
        assert np.array_equal(outs[1][~free], scaled[~free])   # pinned rows untouched
