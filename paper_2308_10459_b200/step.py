"""Step orchestration: the drop-in ``stable_step`` and its per-step pieces.

``stable_step`` follows ``/root/reference/pkg/src/bdem/solver.py:881-939``
(call stack B of SURVEY.md §3) with every array operation on the device:
driver rows -> predictor/anchors kernel -> contact broad phase -> Newton
solve -> velocity kernel -> fracture kernel + ordered event compaction ->
components (only when bonds broke) -> energy reductions.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .newton import GPUProblem, SolverConfig, minimize_second_order
from .scene import FragmentLabeling

MINIMIZERS = {"second-order": minimize_second_order}


@dataclass
class StepReport:
    """solver.py:847-853."""

    solve: object
    broken: list
    contact_pairs: int
    energies: dict
    committed: bool


# ---------------------------------------------------------------------------
# broad phase and components
# ---------------------------------------------------------------------------

def _device_broadphase(dev, p, radii, cell, labels=None):
    lib = dev.lib
    n = int(p.shape[0])
    if n < 2:
        return torch.zeros((0, 2), dtype=torch.int32, device=p.device)
    need = int(lib.bdem_broadphase_workspace(n))
    if dev._bp_work is None or dev._bp_work.numel() < need:
        dev._bp_work = torch.empty(need, dtype=torch.uint8, device=p.device)
    cnt = C.c_int64(0)
    lab = 0 if labels is None else labels.data_ptr()
    st = torch.cuda.current_stream(p.device).cuda_stream
    L.check(lib.bdem_broadphase(p.data_ptr(), radii.data_ptr(), n, float(cell), lab,
                                dev._bp_work.data_ptr(), None, 0, C.byref(cnt), st),
            "bdem_broadphase(count)")
    m = int(cnt.value)
    out = torch.empty((max(m, 1), 2), dtype=torch.int32, device=p.device)
    if m:
        L.check(lib.bdem_broadphase(p.data_ptr(), radii.data_ptr(), n, float(cell), lab,
                                    dev._bp_work.data_ptr(), out.data_ptr(), m, C.byref(cnt), st),
                "bdem_broadphase(write)")
    dev.launches += 2
    return out[:m]


class _Scratch:
    """Minimal holder for workspaces when no DeviceSystem exists."""

    def __init__(self):
        self.lib = L.load()
        self._bp_work = None
        self._cc_work = None
        self.launches = 0


def broad_phase(positions, radii, cell_size):
    """Sorted overlapping pairs i<j (contact.py:140-173), computed on the GPU.

    Accepts numpy arrays (returns an (m,2) int64 numpy array like the
    reference) or CUDA tensors (returns an (m,2) int32 CUDA tensor).
    """
    on_host = isinstance(positions, np.ndarray)
    p = torch.as_tensor(np.ascontiguousarray(positions, dtype=np.float64)).cuda() if on_host \
        else positions.contiguous()
    r = torch.as_tensor(np.ascontiguousarray(radii, dtype=np.float64)).cuda() if on_host \
        else radii.contiguous()
    if r.numel() and cell_size < 2.0 * float(r.max()):
        raise ValueError("cell_size must be at least twice the largest radius")
    out = _device_broadphase(_Scratch(), p, r, cell_size)
    return out.cpu().numpy().astype(np.int64) if on_host else out


def _components(lib, n, bi, bj, status, work_holder):
    need = int(lib.bdem_components_workspace(n))
    if work_holder._cc_work is None or work_holder._cc_work.numel() < need:
        work_holder._cc_work = torch.empty(need, dtype=torch.uint8, device=bi.device)
    labels = torch.empty(max(n, 1), dtype=torch.int64, device=bi.device)
    nc = C.c_int64(0)
    st = torch.cuda.current_stream(bi.device).cuda_stream
    L.check(lib.bdem_components(n, int(bi.numel()), bi.data_ptr(), bj.data_ptr(),
                                status.data_ptr(), work_holder._cc_work.data_ptr(),
                                labels.data_ptr(), C.byref(nc), st), "bdem_components")
    return labels[:n], int(nc.value)


def label_components(n_elements, bonds, scene=None) -> FragmentLabeling:
    """Connected components over non-broken bonds, numbered by smallest element
    (geometry.py:295-310), on the GPU."""
    if scene is not None and scene._device is not None:
        dev = scene._device
        labels, _ = _components(dev.lib, dev.n, dev.bond_i, dev.bond_j, dev.status, dev)
        dev.labels = labels
        return FragmentLabeling(labels.cpu().numpy())
    bi = torch.as_tensor(np.asarray(bonds.i, dtype=np.int32)).cuda()
    bj = torch.as_tensor(np.asarray(bonds.j, dtype=np.int32)).cuda()
    stt = torch.as_tensor(np.asarray(bonds.status, dtype=np.int8)).cuda()
    labels, _ = _components(L.load(), int(n_elements), bi, bj, stt, _Scratch())
    return FragmentLabeling(labels.cpu().numpy())


def _candidates_into_system(scene) -> int:
    """contact_candidates (solver.py:856-878) straight into the device pair
    arrays: inflated radii, cell size, labelled broad phase and the element
    adjacency all in the library (bdem_contact_pairs).  Returns the count."""
    dev = scene.device
    if scene.k_element <= 0.0 or dev.n < 2:
        dev.set_pairs(torch.zeros((0, 2), dtype=torch.int32, device=dev.device))
        return 0
    if getattr(dev, "labels", None) is None:
        label_components(dev.n, scene.bonds, scene)
    dt2g = scene.dt**2 * float(np.linalg.norm(scene.gravity))
    return dev.contact_pairs(scene.dt, dt2g, dev.labels)


def contact_candidates(scene):
    """Frozen self-contact candidates of one step (solver.py:856-878): broad
    phase on radii inflated by dt|v| + dt^2|g|, restricted to element pairs
    in different fragments.  Installs them in the scene's device system and
    returns them as an (m,2) int32 CUDA tensor."""
    _candidates_into_system(scene)
    return scene.device.pair_array()


# ---------------------------------------------------------------------------
# fracture update
# ---------------------------------------------------------------------------

def _device_bond_update(dev, youngs, plastic):
    """bdem_bond_update + ordered event compaction -> [(bond, sigma, tau)]."""
    if dev.nb == 0:
        return []
    st = dev.stream
    if getattr(dev, "_flags", None) is None:
        dev._flags = torch.empty(dev.npos, dtype=torch.uint8, device=dev.device)
        dev._ev_idx = torch.empty(dev.npos, dtype=torch.int32, device=dev.device)
        dev._ev_rec = torch.empty((dev.npos, 2), dtype=torch.float64, device=dev.device)
        dev._sel_work = torch.empty(int(dev.lib.bdem_select_workspace(dev.npos)),
                                    dtype=torch.uint8, device=dev.device)
    pl = None
    if plastic is not None:
        arr = (C.c_double * 4)(plastic.fracture_strain, plastic.yield_strain, plastic.weakening,
                               plastic.damage_exponent)
        pl = C.cast(arr, C.c_void_p)
    dev.call("bdem_bond_update", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), float(youngs), pl,
             dev._flags.data_ptr(), st)
    cnt = C.c_int64(0)
    L.check(dev.lib.bdem_select_flagged(dev._flags.data_ptr(), dev.npos, dev._ev_idx.data_ptr(),
                                        dev._sel_work.data_ptr(), C.byref(cnt), st),
            "bdem_select_flagged")
    dev.launches += 1
    m = int(cnt.value)
    if m == 0:
        return []
    dev.call("bdem_event_records", dev.sysp, dev._ev_idx.data_ptr(), m, dev._ev_rec.data_ptr(), st)
    pos = dev._ev_idx[:m].cpu().numpy()
    rec = dev._ev_rec[:m].cpu().numpy()
    ids = dev.sell.bond_of_pos[pos]
    order = np.argsort(ids, kind="stable")       # ascending bond id (bonds.py:564-569)
    return [(int(ids[k]), float(rec[k, 0]), float(rec[k, 1])) for k in order]


def update_bond_states(bonds, p, q, youngs, plastic=None, scene=None):
    """update_bond_states (bonds.py:532-570) on the GPU.

    With ``scene`` the scene's device state is used (no transfers); otherwise
    the host arrays are uploaded, updated in HBM and written back in place.
    """
    from .device import DeviceSystem
    from .state import ElementSet
    if scene is not None:
        return _device_bond_update(scene.device, youngs, plastic)
    n = np.asarray(p).shape[0]
    el = ElementSet(np.asarray(p, dtype=float), np.asarray(q, dtype=float), np.zeros((n, 3)),
                    np.zeros((n, 4)), np.ones(n), np.ones(n))
    dev = DeviceSystem(elements=el, bonds=bonds)
    events = _device_bond_update(dev, youngs, plastic)
    dev.download_bond_state(bonds)
    return events


# ---------------------------------------------------------------------------
# the step
# ---------------------------------------------------------------------------

def _apply_driver(scene, dev, t):
    """Driver rows at t + dt (solver.py:898-900, scenes.py:146-176): the few
    driven rows are formed on the host, copied once and scattered by
    bdem_rows_copy."""
    drv = scene.driver
    if drv is None:
        return
    if hasattr(drv, "rows") and hasattr(drv, "ids"):
        p, v, q, qd = drv.rows(t)
        m = len(drv.ids)
        cache = getattr(dev, "_drv_cache", None)
        if cache is None or cache[0] is not drv:
            ids = torch.as_tensor(np.asarray(drv.ids, dtype=np.int32)).to(dev.device)
            host = torch.zeros((m, 14), dtype=torch.float64).pin_memory()
            cache = dev._drv_cache = (drv, ids, host, torch.empty((m, 14), dtype=torch.float64,
                                                                  device=dev.device))
        _, ids, host, buf = cache
        torch.cuda.current_stream(dev.device).synchronize()   # host buffer reuse
        h = host.numpy()
        h[:, 0:3], h[:, 3:7], h[:, 7:10], h[:, 10:14] = p, q, v, qd
        buf.copy_(host, non_blocking=True)
        dev.rows_copy(ids, buf, to_buf=False)
        return
    # arbitrary reference-style callable: run it on a host view of the state
    el = scene.elements
    for name in ("p", "q", "v", "qdot"):
        getattr(el, name)[:] = getattr(dev, name).cpu().numpy()
    drv(el, t)
    pin = torch.as_tensor(np.nonzero(el.pinned)[0], device=dev.device)
    for name in ("p", "q", "v", "qdot"):
        src = torch.as_tensor(getattr(el, name)[el.pinned], dtype=torch.float64,
                              device=dev.device)
        getattr(dev, name)[pin] = src


@dataclass
class PreparedStep:
    """The step-1..6 prologue of stable_step (solver.py:894-906): what the
    minimizer and the epilogue need."""

    problem: GPUProblem
    n_pairs: int
    t_next: float


def prepare_step(scene) -> PreparedStep:
    """Everything stable_step does before the minimizer (solver.py:894-906,
    integrator.py:141-161, 268-274): state upload, pinned backups, driver rows
    at t + dt, the step context, frozen contact candidates and the predictor
    (p0, q0 in ``dev.xp`` / ``dev.xq``)."""
    dev = scene.device
    if scene.host_sync:
        dev.upload_elements(scene.elements, scene.p_prev, scene.q_prev)
        dev.upload_bond_state(scene.bonds)
    elif not getattr(dev, "_history_uploaded", False):
        dev.upload_elements(scene.elements, scene.p_prev, scene.q_prev)
    dev._history_uploaded = True
    dev.set_physics(scene.gravity, scene.k_contact, scene.k_element, scene.colliders)
    st = dev.stream

    dev.rows_copy(dev.pinned_ids, dev.pin_buf, to_buf=True)     # pinned backup
    t_next = scene.time + scene.dt
    _apply_driver(scene, dev, t_next)

    dev.p_cur.copy_(dev.p)
    dev.q_cur.copy_(dev.q)
    n_pairs = _candidates_into_system(scene)
    dev.reset_errors()
    dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(),
             dev.qdot.data_ptr(), dev.p_prev.data_ptr(), dev.q_prev.data_ptr(), float(scene.dt),
             dev.p_hat.data_ptr(), dev.q_hat.data_ptr(), dev.mp_dt2.data_ptr(),
             dev.mq_dt2.data_ptr(), dev.xp.data_ptr(), dev.xq.data_ptr(), st)
    return PreparedStep(GPUProblem(dev), n_pairs, t_next)


def stable_step(scene, cfg: SolverConfig, method: str = "second-order") -> StepReport:
    """Advance ``scene`` by one implicit step on the GPU (solver.py:881-939)."""
    if method not in MINIMIZERS:
        raise ValueError(f"the GPU path implements {sorted(MINIMIZERS)}, got {method!r}")
    prep = prepare_step(scene)
    dev, problem, n_pairs, t_next = scene.device, prep.problem, prep.n_pairs, prep.t_next
    st = dev.stream
    result = MINIMIZERS[method](problem, dev.xp, dev.xq, cfg)

    if not result.converged:
        dev.rows_copy(dev.pinned_ids, dev.pin_buf, to_buf=False)   # restore pinned rows
        energies = {"kinetic": _kinetic(dev)}
        if scene.host_sync:
            dev.download_state(scene)
        return StepReport(result, [], n_pairs, energies, False)

    dev.call("bdem_finish_step", dev.sysp, result.p.data_ptr(), result.q.data_ptr(),
             dev.p_cur.data_ptr(), dev.q_cur.data_ptr(), float(scene.dt), dev.v.data_ptr(),
             dev.qdot.data_ptr(), st)
    dev.p.copy_(result.p)
    dev.q.copy_(result.q)
    if scene.mu_s > 0.0 or scene.mu_r > 0.0:         # solver.py:923-925
        dev.friction(scene.mu_s, scene.mu_r, scene.dt)

    events = _device_bond_update(dev, scene.youngs, scene.plastic)
    if events:
        flags = scene.surface_flags
        bi = np.asarray(scene.bonds.i)
        bj = np.asarray(scene.bonds.j)
        for b, _, _ in events:                      # geometry.py:257-261
            flags[bi[b]] = True
            flags[bj[b]] = True
        scene.labels = label_components(dev.n, scene.bonds, scene)

    dev.p_prev, dev.p_cur = dev.p_cur, dev.p_prev
    dev.q_prev, dev.q_cur = dev.q_cur, dev.q_prev
    scene.time = t_next

    energies = problem.energy_breakdown(dev.p, dev.q)
    if scene.host_sync:
        dev.download_state(scene)
    return StepReport(result, events, n_pairs, energies, True)


def _kinetic(dev):
    dev.call("bdem_kinetic", dev.sysp, dev.v.data_ptr(), dev.qdot.data_ptr(), dev.stream)
    dev.call("bdem_reduce_finish", dev.sysp, L.SC["EKIN"], 1, L.RED_BLOCKS, dev.stream)
    return float(dev.read_scalars()[L.SC["EKIN"]])
