"""The real drop-in: the UNMODIFIED reference orchestration with the B200 solve.

``register(bdem.solver)`` installs ``MINIMIZERS["b200"]``
(``/root/reference/pkg/src/bdem/solver.py:834-840``); then
``bdem.solver.stable_step(scene, cfg, "b200")`` (``solver.py:881-939``) runs
the reference's own predictor, broad phase, fracture update and history roll
around the GPU Newton solve.  Each scene is stepped twice from identical
arrays -- once with the reference's ``"second-order"`` minimizer on the CPU,
once with ``"b200"`` -- and the trajectories are compared step by step
(rtol 1e-8; identical Newton counts, commit flags and breaks).
The reference is imported from ``oracle/_ref`` (bytecode build that travels
to the GPU box) or ``/root/reference`` (build container).
"""

from __future__ import annotations

import numpy as np
import pytest

from paper_2308_10459_b200 import configs as C
from _fixtures import close
from oracle.ref_adapter import bdem_or_skip, ref_scene

pytestmark = pytest.mark.gpu


def _cases():
    return {
        "cantilever": (C.cantilever(nx=10, ny=3, nz=3), 4, 1e-7, None),
        "rope_twist": (C.rope(n=30), 6, 1e-5, None),
        "cube_fracture": (C.cube(n_side=5, random_q=False, seed=3, youngs=3e8, k_contact=1e9,
                                 speed=2.0, dt=1e-4), 6, 1e-6, "schedule"),
    }


@pytest.mark.parametrize("name", ["cantilever", "rope_twist", "cube_fracture"])
def test_reference_stable_step_with_b200_minimizer(cuda_ok, name):
    bdem = bdem_or_skip()
    from bdem import contact as rc
    from bdem import solver as rsv

    from paper_2308_10459_b200.integration import register
    assert register(rsv) == "b200"
    spec, steps, eps, sched = _cases()[name]
    cpu, gpu = ref_scene(bdem, spec), ref_scene(bdem, spec)
    cfg = rsv.SolverConfig(epsilon=eps, max_iterations=300)
    moved_q = 0.0
    for s in range(steps):
        if sched:
            for sc in (cpu, gpu):
                sc.colliders = [rc.HalfSpace(tuple(c.normal), c.offset)
                                for c in spec.collider_schedule(sc.time + sc.dt)]
        rc_ = rsv.stable_step(cpu, cfg, "second-order")
        rg_ = rsv.stable_step(gpu, cfg, "b200")
        assert rg_.committed == rc_.committed, (s, rg_.solve.reason, rc_.solve.reason)
        assert rg_.solve.iterations == rc_.solve.iterations, s
        assert abs(rg_.solve.pcg_total - rc_.solve.pcg_total) <= rc_.solve.iterations, s
        assert [b for b, _, _ in rg_.broken] == [b for b, _, _ in rc_.broken], s
        assert rg_.contact_pairs == rc_.contact_pairs
        m_dt2 = (cpu.elements.mass / cpu.dt**2).min()
        atol_p = max(10 * eps / m_dt2, 1e-13)
        for k, rtol, atol in (("p", 1e-8, atol_p), ("q", 1e-8, 1e-10),
                              ("v", 1e-6, atol_p / cpu.dt), ("qdot", 1e-6, 1e-6)):
            ok, info = close(getattr(gpu.elements, k), getattr(cpu.elements, k), rtol, atol)
            assert ok, (name, s, k, info)
        moved_q = max(moved_q, float(np.abs(cpu.elements.q - np.array([0.0, 0, 0, 1])).max()))
    assert np.array_equal(gpu.bonds.status, cpu.bonds.status)
    if name == "rope_twist":
        assert moved_q > 1e-4        # the rotation path is really exercised
