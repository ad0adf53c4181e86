"""HBM-resident system state and the typed handles the kernels see.

``DeviceSystem`` owns every device buffer (torch tensors used purely as
allocations) and one ``bdem_system_t`` struct that points into them.  It is
built once per scene; topology (bond list, element->bond adjacency) is fixed
for the scene's lifetime -- broken bonds keep their slots and the kernels
skip them by status -- so nothing is re-allocated inside a step.

Memory layout (HBM):
  elements  p (n,3), q (n,4) [scalar-last, 32-byte rows], v, qdot,
            p_prev, q_prev, p_hat, q_hat, mass, radius, m/dt^2, mq/dt^2
  bonds     i, j (int32), status (int8), 24 geometry planes, 5 state planes
            (structure-of-arrays, one plane = n_bond doubles)
  staging   17 planes x n_bond (j-end pieces) + 14 AoSoA coupling coefficients
            per bond + 20 row partial-sum planes, written by the bond pass
  reduced   z, y, r, zv, pv, Ap (6 doubles per free element), diag and
            block-Jacobi inverses (12 doubles per free element)
"""

from __future__ import annotations

import ctypes as C
import logging
import weakref

import numpy as np
import torch

from . import _lib as L
from .state import DegenerateBondError, DegenerateShearError

logger = logging.getLogger(__name__)

F64 = torch.float64
I32 = torch.int32


def _t(arr, dtype=F64, device="cuda"):
    return torch.as_tensor(np.ascontiguousarray(arr), dtype=dtype).to(device)


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def row_order(el) -> np.ndarray:
    """SELL row order: the caller's element order.  On lattices the neighbour
    offsets are then constant, so the SpMV's j-role and x gathers are
    shift-coalesced (Z-order and strip-major orders were measured for the
    tiled SpMV variants and lost, profiles/r01/README.md)."""
    return np.arange(int(el.p.shape[0]), dtype=np.int64)


class SellLayout:
    """SELL-32 placement of the bonds (see bdem_system_t in the header).

    Elements are placed in rows (``rows[r]`` = element of row r) and rows are
    cut into slices of 32.  Each slice owns a slot-major block of positions:
    slot k of lane l holds the k-th bond with i == rows[32 s + l] in
    ascending bond id (the order np.add.at accumulates in,
    integrator.py:100-103).  A warp that owns a slice therefore reads slot k
    of 32 rows as one contiguous 256-byte segment per plane.  The j-role
    lists (bonds with j == e, ascending id) use the same shape and hold
    positions.  Padding positions carry status BROKEN and zero data.
    """

    def __init__(self, bi: np.ndarray, bj: np.ndarray, n: int, slot: np.ndarray,
                 rows: np.ndarray | None = None):
        nb = bi.shape[0]
        self.n_slices = ns = max((n + 31) // 32, 1)
        rows = np.arange(n, dtype=np.int64) if rows is None else np.asarray(rows, dtype=np.int64)
        self.rows = rows
        self.elem_row = np.empty(n, dtype=np.int64)
        self.elem_row[rows] = np.arange(n)
        self.row_elem = np.full(ns * 32, -1, dtype=np.int32)
        self.row_elem[:n] = rows
        ri = self.elem_row[bi]
        rj = self.elem_row[bj]
        self.slice_base, rank_i, self.kmax = self._slices(ri, n, ns)
        self.n_pos = int(self.slice_base[-1])
        self.pos_of_bond = self.slice_base[ri // 32] + 32 * rank_i + (ri % 32)
        self.bond_of_pos = np.full(self.n_pos, -1, dtype=np.int64)
        self.bond_of_pos[self.pos_of_bond] = np.arange(nb)
        self.pos_oslot = np.full(self.n_pos, -1, dtype=np.int32)
        self.pos_oslot[self.pos_of_bond] = slot[bj]
        self.jslice_base, rank_j, self.kjmax = self._slices(rj, n, ns)
        self.n_jpos = int(self.jslice_base[-1])
        jidx = self.jslice_base[rj // 32] + 32 * rank_j + (rj % 32)
        self.jpos = np.full(self.n_jpos, -1, dtype=np.int32)
        self.jpos[jidx] = self.pos_of_bond
        self.jslot = np.full(self.n_jpos, -1, dtype=np.int32)
        self.jslot[jidx] = slot[bi]
        free_row = np.zeros(ns * 32, dtype=np.int64)
        free_row[:n] = slot[rows] >= 0
        self.row_slot = np.full(ns * 32, -1, dtype=np.int32)
        self.row_slot[:n] = slot[rows]
        self.slice_slot = np.zeros(ns + 1, dtype=np.int64)
        np.cumsum(free_row.reshape(ns, 32).sum(axis=1), out=self.slice_slot[1:])

    @staticmethod
    def _slices(key, n, ns):
        """Slot rank of every bond within its row (ascending bond id), the
        slice base offsets (32 x max slots per slice) and the max slots."""
        nb = key.shape[0]
        cnt = np.bincount(key, minlength=n)
        order = np.argsort(key, kind="stable")
        start = np.cumsum(cnt) - cnt
        rank = np.empty(nb, dtype=np.int64)
        rank[order] = np.arange(nb) - start[key[order]]
        padded = np.zeros(ns * 32, dtype=np.int64)
        padded[:n] = cnt
        kmax = padded.reshape(ns, 32).max(axis=1)
        base = np.zeros(ns + 1, dtype=np.int64)
        np.cumsum(32 * kmax, out=base[1:])
        return base, rank, int(kmax.max()) if kmax.size else 0

    def to_positions(self, arr, fill=0):
        """Scatter a per-bond array (..., nb) into positions (..., n_pos)."""
        arr = np.asarray(arr)
        out = np.full(arr.shape[:-1] + (max(self.n_pos, 1),), fill, dtype=arr.dtype)
        out[..., self.pos_of_bond] = arr
        return out

    def to_bonds(self, arr):
        """Gather a per-position array back into caller bond order."""
        return np.asarray(arr)[..., self.pos_of_bond]


def bond_geometry_planes(b) -> np.ndarray:
    nb = b.i.shape[0]
    g = np.empty((L.BG["COUNT"], nb))
    g[L.BG["L0"]] = b.rest_length
    g[L.BG["D0"]:L.BG["D0"] + 3] = np.asarray(b.d0).T
    g[L.BG["FRAME"]:L.BG["FRAME"] + 9] = np.asarray(b.frame).reshape(nb, 9).T
    g[L.BG["KN"]] = b.kn
    g[L.BG["KT"]] = b.kt
    g[L.BG["KDIAG"]:L.BG["KDIAG"] + 3] = np.asarray(b.k_diag).T
    g[L.BG["RADIUS"]] = b.radius
    g[L.BG["SECTION"]] = b.section
    g[L.BG["SECOND"]] = b.second_moment
    g[L.BG["POLAR"]] = b.polar_moment
    g[L.BG["TENSILE"]] = b.tensile_strength
    g[L.BG["SHEAR"]] = b.shear_strength
    return g


class DeviceSystem:
    """Device mirror of one scene (elements, bonds, colliders, workspaces)."""

    def __init__(self, scene=None, *, elements=None, bonds=None, device="cuda"):
        if not torch.cuda.is_available():
            raise RuntimeError("DeviceSystem needs a CUDA device (B200, sm_100a)")
        self.lib = L.load()
        self.device = torch.device(device)
        el = scene.elements if scene is not None else elements
        b = scene.bonds if scene is not None else bonds
        self.n = n = int(el.p.shape[0])
        self.nb = nb = int(b.i.shape[0])
        pinned = np.asarray(el.pinned, dtype=bool)
        self.free_np = ~pinned
        # SELL rows; free slots numbered in row order (contiguous per slice)
        rows = row_order(el)
        slot = np.full(n, -1, dtype=np.int32)
        free_rows = rows[self.free_np[rows]]
        slot[free_rows] = np.arange(free_rows.size, dtype=np.int32)
        self.free_ids_np = np.nonzero(self.free_np)[0]
        self.slot_np = slot
        # slot of the k-th free element in ascending element id (oracle order)
        self.slot_cols = slot[self.free_ids_np].astype(np.int64)
        self.nf = nf = int(self.free_ids_np.size)
        dev = self.device

        # element constants
        self.mass = _t(el.mass, device=dev)
        self.radius = _t(el.radius, device=dev)
        self.slot = _t(slot, I32, dev)
        self.free_elem = _t(free_rows.astype(np.int32), I32, dev)
        # element state + step context
        z3 = lambda: torch.zeros((n, 3), dtype=F64, device=dev)  # noqa: E731
        z4 = lambda: torch.zeros((n, 4), dtype=F64, device=dev)  # noqa: E731
        self.p, self.q, self.v, self.qdot = z3(), z4(), z3(), z4()
        self.p_prev, self.q_prev = z3(), z4()
        self.p_hat, self.q_hat = z3(), z4()
        self.p_cur, self.q_cur = z3(), z4()
        self.mp_dt2 = torch.zeros(n, dtype=F64, device=dev)
        self.mq_dt2 = torch.zeros(n, dtype=F64, device=dev)
        # Newton iterate, trial point, direction (pinned rows of dp/dq stay 0)
        self.xp, self.xq, self.tp, self.tq = z3(), z4(), z3(), z4()
        self.dp, self.dq = z3(), z4()
        # bonds, placed by SELL-32 position
        bi64 = np.asarray(b.i, dtype=np.int64)
        bj64 = np.asarray(b.j, dtype=np.int64)
        self.sell = sell = SellLayout(bi64, bj64, n, slot, rows)
        self.npos = npos = max(sell.n_pos, 1)
        self.bond_i = _t(sell.to_positions(bi64.astype(np.int32)), I32, dev)
        self.bond_j = _t(sell.to_positions(bj64.astype(np.int32)), I32, dev)
        self.status = _t(sell.to_positions(np.asarray(b.status, dtype=np.int8), fill=2),
                         torch.int8, dev)
        self.geom = _t(sell.to_positions(bond_geometry_planes(b)), device=dev)
        self.bstate = torch.zeros((L.BS["COUNT"], npos), dtype=F64, device=dev)
        self.slice_base = _t(sell.slice_base.astype(np.int32), I32, dev)
        self.pos_oslot = _t(np.append(sell.pos_oslot, -1).astype(np.int32), I32, dev)
        self.jslice_base = _t(sell.jslice_base.astype(np.int32), I32, dev)
        self.jpos = _t(np.append(sell.jpos, -1).astype(np.int32), I32, dev)
        self.jslot = _t(np.append(sell.jslot, -1).astype(np.int32), I32, dev)
        self.row_elem = _t(sell.row_elem, I32, dev)
        self.elem_row = _t(np.append(sell.elem_row, -1).astype(np.int32), I32, dev)
        self.slice_slot = _t(sell.slice_slot.astype(np.int32), I32, dev)
        self.row_slot = _t(sell.row_slot, I32, dev)
        self.pos_of_bond_d = torch.as_tensor(sell.pos_of_bond).to(dev)
        # staging / reduced system
        self.stage = torch.zeros((L.ST["COUNT"], npos), dtype=F64, device=dev)
        npos32 = (npos + 31) // 32 * 32
        self.scoef = torch.zeros(L.CF["COUNT"] * npos32, dtype=F64, device=dev)
        # reduced vectors / diagonal blocks: planes of stride vstride (n_free
        # rounded up to 32 -> 256-byte aligned planes, zero padding)
        self.vstride = vs = max(32, (nf + 31) // 32 * 32)
        self.diag = torch.zeros((12, vs), dtype=F64, device=dev)
        self.minv = torch.zeros((12, vs), dtype=F64, device=dev)
        v6 = lambda: torch.zeros(6 * vs, dtype=F64, device=dev)  # noqa: E731
        self.z, self.y, self.r, self.zv, self.pv, self.ap = v6(), v6(), v6(), v6(), v6(), v6()
        self.red = torch.zeros((L.SC["COUNT"], L.RED_BLOCKS), dtype=F64, device=dev)
        self.scalars = torch.zeros(L.SC["COUNT"], dtype=F64, device=dev)
        self.pcg_state = torch.zeros(L.PCG["COUNT"], dtype=F64, device=dev)
        self.err = torch.zeros(L.ERRSLOT_COUNT, dtype=I32, device=dev)
        self.counter = torch.zeros(L.N_COUNTERS, dtype=torch.int32, device=dev)
        self.clamp_list = torch.zeros(npos, dtype=I32, device=dev)
        # i-role partial sums of the bond pass, one column per SELL row
        nrow = int(sell.row_elem.shape[0])
        self.ipart = torch.zeros((L.IP["COUNT"], nrow), dtype=F64, device=dev)
        self.ikpre = torch.zeros(nrow, dtype=I32, device=dev)
        # host staging for scalar read-backs
        self.h_scalars = torch.zeros(L.SC["COUNT"], dtype=F64).pin_memory()
        self.h_pcg = torch.zeros(L.PCG["COUNT"], dtype=F64).pin_memory()
        self.h_err = torch.zeros(L.ERRSLOT_COUNT, dtype=I32).pin_memory()
        self._bp_work = None
        self._bp_need = int(self.lib.bdem_broadphase_workspace(max(n, 1)))
        # pinned rows: ids and the packed backup of stable_step (p, q, v, qdot)
        self.pinned_ids = torch.as_tensor(np.nonzero(pinned)[0].astype(np.int32)).to(dev)
        self.pin_buf = torch.zeros((max(int(self.pinned_ids.numel()), 1), 14), dtype=F64,
                                   device=dev)
        self._cc_work = None
        self._sel_work = None
        self.launches = 0
        self.labels = None
        self._bi_np, self._bj_np = bi64, bj64   # caller bond order (error messages)
        self.eval_pq = None   # (p, q) of the last evaluation (error messages)
        self.timer = None   # optional timing.KernelTimer picked up by GPUProblem
        self._pins = {}

        self.sys = L.System()
        s = self.sys
        s.n_elem, s.n_free, s.n_bond = n, nf, (sell.n_pos if nb else 0)
        s.vstride = self.vstride
        s.sell_kmax, s.sell_kjmax = sell.kmax, sell.kjmax
        s.mass, s.radius = _ptr(self.mass), _ptr(self.radius)
        s.mp_dt2, s.mq_dt2 = _ptr(self.mp_dt2), _ptr(self.mq_dt2)
        s.p_hat, s.q_hat = _ptr(self.p_hat), _ptr(self.q_hat)
        s.slot, s.free_elem = _ptr(self.slot), _ptr(self.free_elem)
        s.bond_i, s.bond_j, s.status = _ptr(self.bond_i), _ptr(self.bond_j), _ptr(self.status)
        s.geom, s.bstate = _ptr(self.geom), _ptr(self.bstate)
        s.slice_base, s.pos_oslot = _ptr(self.slice_base), _ptr(self.pos_oslot)
        s.jslice_base, s.jpos, s.jslot = (_ptr(self.jslice_base), _ptr(self.jpos),
                                          _ptr(self.jslot))
        s.row_elem, s.elem_row = _ptr(self.row_elem), _ptr(self.elem_row)
        s.slice_slot, s.row_slot = _ptr(self.slice_slot), _ptr(self.row_slot)
        s.stage, s.diag, s.minv = _ptr(self.stage), _ptr(self.diag), _ptr(self.minv)
        s.scoef = _ptr(self.scoef)
        s.red, s.scalars, s.pcg = _ptr(self.red), _ptr(self.scalars), _ptr(self.pcg_state)
        s.err, s.counter = _ptr(self.err), _ptr(self.counter)
        s.clamp_list = _ptr(self.clamp_list)
        s.ipart, s.ikpre = _ptr(self.ipart), _ptr(self.ikpre)
        self.sysp = C.pointer(s)
        # contact pairs (capacity grows on demand)
        self.n_pair = 0
        self._alloc_pairs(1024)
        self.reset_errors()

        if scene is not None:
            self.set_physics(scene.gravity, scene.k_contact, scene.k_element, scene.colliders)
        self.upload_elements(el)
        self.upload_bond_state(b)

    # ------------------------------------------------------------------ setup
    @property
    def stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def set_physics(self, gravity, k_contact, k_element, colliders):
        s = self.sys
        for c in range(3):
            s.gravity[c] = float(gravity[c])
        s.k_contact, s.k_element = float(k_contact), float(k_element)
        self.set_colliders(colliders)

    def set_colliders(self, colliders):
        cols = list(colliders or [])
        if len(cols) > L.MAX_COLLIDERS:
            raise ValueError(f"at most {L.MAX_COLLIDERS} colliders are supported")
        s = self.sys
        s.n_colliders = len(cols)
        for k, col in enumerate(cols):
            kind, *a = _pack_collider(col)
            s.colliders[k].kind = kind
            for t in range(6):
                s.colliders[k].a[t] = a[t]

    def _pinned(self, key, shape, dtype=F64):
        """Reusable page-locked host staging buffer."""
        buf = self._pins.get(key)
        if buf is None or tuple(buf.shape) != tuple(shape):
            buf = torch.empty(shape, dtype=dtype).pin_memory()
            self._pins[key] = buf
        return buf

    def _host_view(self, arr, dtype):
        """Torch view of a caller's numpy array in page-locked memory.

        The array is registered with the CUDA driver once (cudaHostRegister),
        so host<->HBM copies run directly on the caller's memory at PCIe
        speed with no staging memcpy; registration is dropped when the array
        is garbage collected.  Returns None for arrays that cannot be viewed
        (wrong dtype, non-contiguous) -- callers then stage."""
        if not isinstance(arr, np.ndarray) or arr.dtype != dtype or \
                not arr.flags["C_CONTIGUOUS"] or arr.nbytes == 0:
            return None
        key = (arr.ctypes.data, arr.nbytes)
        if key not in _REGISTERED:
            rt = torch.cuda.cudart()
            if int(rt.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)) != 0:
                return None
            _REGISTERED[key] = True
            weakref.finalize(arr.base if arr.base is not None else arr, _unregister, key)
        return torch.from_numpy(arr)

    def _h2d(self, dst, src_np, key):
        src = np.asarray(src_np)
        view = self._host_view(src, np.float64 if dst.dtype == F64 else np.int8)
        if view is not None and tuple(view.shape) == tuple(dst.shape):
            dst.copy_(view, non_blocking=True)
            return
        st = self._pinned(key, dst.shape, dst.dtype)
        st.numpy()[...] = src
        dst.copy_(st, non_blocking=True)

    def _d2h_into(self, dst_np, src):
        """Queue an HBM -> host copy into the caller's array (synchronise later)."""
        view = self._host_view(dst_np, np.float64 if src.dtype == F64 else np.int8)
        if view is not None and tuple(view.shape) == tuple(src.shape):
            view.copy_(src, non_blocking=True)
            return None
        st = self._pinned(("out",) + tuple(src.shape) + (str(src.dtype),), src.shape, src.dtype)
        st.copy_(src, non_blocking=True)
        return (dst_np, st)

    def _d2h(self, src, key):
        st = self._pinned(key, src.shape, src.dtype)
        st.copy_(src, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return st.numpy()

    def upload_elements(self, el, p_prev=None, q_prev=None):
        """Host -> HBM copy of the element state (caller arrays page-locked)."""
        for name in ("p", "q", "v", "qdot"):
            self._h2d(getattr(self, name), getattr(el, name), name)
        if p_prev is not None:
            self._h2d(self.p_prev, p_prev, "p_prev")
            self._h2d(self.q_prev, q_prev, "q_prev")

    _BSTATE = (("stiffness_scale", "SCALE"), ("damage", "DAMAGE"),
               ("plastic_strain", "PLASTIC"), ("sigma", "SIGMA"), ("tau", "TAU"))

    def upload_bond_state(self, b):
        """Host -> HBM copy of the mutable bond state, scattered to SELL positions."""
        if self.nb == 0:
            return
        if getattr(self, "_bs_stage", None) is None:
            self._bs_stage = torch.empty((L.BS["COUNT"], self.nb), dtype=F64, device=self.device)
            self._st_stage = torch.empty(self.nb, dtype=torch.int8, device=self.device)
        for name, plane in self._BSTATE:
            self._h2d(self._bs_stage[L.BS[plane]], getattr(b, name), "bs_" + name)
        self._h2d(self._st_stage, np.asarray(b.status, dtype=np.int8), "bs_status")
        pos = self.pos_of_bond_d
        self.bstate[:, pos] = self._bs_stage
        self.status[pos] = self._st_stage

    def download_bond_state(self, b, sync=True):
        if self.nb == 0:
            return []
        pos = self.pos_of_bond_d
        if getattr(self, "_bs_stage", None) is None:
            self._bs_stage = torch.empty((L.BS["COUNT"], self.nb), dtype=F64, device=self.device)
            self._st_stage = torch.empty(self.nb, dtype=torch.int8, device=self.device)
        torch.index_select(self.bstate, 1, pos, out=self._bs_stage)
        torch.index_select(self.status, 0, pos, out=self._st_stage)
        pending = [self._d2h_into(getattr(b, name), self._bs_stage[L.BS[plane]])
                   for name, plane in self._BSTATE]
        pending.append(self._d2h_into(b.status, self._st_stage))
        if sync:
            self._finish(pending)
            return []
        return pending

    def _finish(self, pending):
        torch.cuda.current_stream(self.device).synchronize()
        for item in pending:
            if item is not None:
                dst, st = item
                dst[...] = st.numpy()

    def download_state(self, scene):
        """HBM -> host copy of element and bond state into the caller's arrays."""
        el = scene.elements
        pending = [self._d2h_into(getattr(el, name), getattr(self, name))
                   for name in ("p", "q", "v", "qdot")]
        if not isinstance(scene.p_prev, np.ndarray) or scene.p_prev.shape != (self.n, 3):
            scene.p_prev = np.empty((self.n, 3))
            scene.q_prev = np.empty((self.n, 4))
        pending.append(self._d2h_into(scene.p_prev, self.p_prev))
        pending.append(self._d2h_into(scene.q_prev, self.q_prev))
        pending += self.download_bond_state(scene.bonds, sync=False)
        self._finish(pending)

    def bootstrap_history(self, dt):
        """p_prev = p - dt v, q_prev = normalize(geodesic(q, -dt qdot))
        (scenes.py:64-68), via the predictor kernel with -dt."""
        # predictor: p0 = p + dt' v, q0 = normalize(geodesic(q, dt' qdot)) on free rows.
        # The reference applies it to every row, so run it with a temporary
        # all-free view is not possible; pinned rows use the same formula:
        p = self.p.cpu().numpy()
        q = self.q.cpu().numpy()
        v = self.v.cpu().numpy()
        qd = self.qdot.cpu().numpy()
        from . import quat as Q
        self.p_prev.copy_(torch.from_numpy(p - dt * v))
        self.q_prev.copy_(torch.from_numpy(Q.normalize(Q.geodesic(q, -dt * qd))))

    # ----------------------------------------------------------- contact pairs
    def _alloc_pairs(self, cap):
        dev = self.device
        self.pair_cap = int(cap)
        self.pstage = torch.zeros((L.PS["COUNT"], self.pair_cap), dtype=F64, device=dev)
        self.pi_ptr = torch.zeros(self.n + 1, dtype=I32, device=dev)
        self.pj_ptr = torch.zeros(self.n + 1, dtype=I32, device=dev)
        self.pj_idx = torch.zeros(self.pair_cap, dtype=I32, device=dev)
        s = self.sys
        s.pair_cap = self.pair_cap
        s.pstage = _ptr(self.pstage)
        self._pair_i = torch.zeros(self.pair_cap, dtype=I32, device=dev)
        self._pair_j = torch.zeros(self.pair_cap, dtype=I32, device=dev)
        s.pair_i, s.pair_j = _ptr(self._pair_i), _ptr(self._pair_j)
        s.pi_ptr, s.pj_ptr, s.pj_idx = _ptr(self.pi_ptr), _ptr(self.pj_ptr), _ptr(self.pj_idx)
        self._adj_work = torch.empty(int(self.lib.bdem_pair_adjacency_workspace(self.n, cap)),
                                     dtype=torch.uint8, device=dev)

    def set_pairs(self, pairs: torch.Tensor):
        """Install the frozen self-contact candidates of this step ((m,2) int32,
        sorted, i<j) and their element adjacency."""
        m = int(pairs.shape[0])
        if m > self.pair_cap:
            self._alloc_pairs(max(m, 2 * self.pair_cap))
        pairs = pairs.to(device=self.device, dtype=I32).contiguous() if m else pairs
        L.check(self.lib.bdem_set_pairs(self.sysp, pairs.data_ptr() if m else None, m,
                                        self._adj_work.data_ptr(), self.stream),
                "bdem_set_pairs")
        self.launches += 1
        self.n_pair = m

    def contact_pairs(self, dt: float, dt2g: float, labels) -> int:
        """The step's frozen self-contact candidates straight into the pair
        arrays (bdem_contact_pairs: inflated radii, device-side cell size,
        labelled broad phase, CUB adjacency); returns their count."""
        if self._bp_work is None or self._bp_work.numel() < self._bp_need:
            self._bp_work = torch.empty(self._bp_need, dtype=torch.uint8, device=self.device)
        if getattr(self, "_radii_buf", None) is None:
            self._radii_buf = torch.empty(max(self.n, 1), dtype=F64, device=self.device)
        cnt = C.c_int64(0)
        lab = 0 if labels is None else labels.data_ptr()
        for _ in range(2):
            rc = self.lib.bdem_contact_pairs(self.sysp, self.p.data_ptr(), self.v.data_ptr(),
                                             float(dt), float(dt2g), lab, self._bp_work.data_ptr(),
                                             self._adj_work.data_ptr(), self._radii_buf.data_ptr(),
                                             C.byref(cnt), self.stream)
            if rc != L.ERR_CAPACITY:
                break
            self._alloc_pairs(max(int(cnt.value), 2 * self.pair_cap))
        L.check(rc, "bdem_contact_pairs")
        self.launches += 1
        self.n_pair = int(cnt.value)
        return self.n_pair

    def pair_array(self) -> torch.Tensor:
        """The installed pairs as an (m, 2) int32 tensor (a view for callers
        of the reference's (m, 2) API; not used on the step path)."""
        m = self.n_pair
        return torch.stack([self._pair_i[:m], self._pair_j[:m]], dim=1)

    # ----------------------------------------------------------------- errors
    def reset_errors(self):
        L.check(self.lib.bdem_reset_errors(self.sysp, self.stream), "bdem_reset_errors")

    # ------------------------------------------------------- element rows
    def rows_copy(self, ids: torch.Tensor, buf: torch.Tensor, to_buf: bool):
        """Pinned/driven element rows <-> packed (m, 14) buffer (bdem_rows_copy)."""
        m = int(ids.numel())
        if m:
            L.check(self.lib.bdem_rows_copy(ids.data_ptr(), m, self.p.data_ptr(), self.q.data_ptr(),
                                            self.v.data_ptr(), self.qdot.data_ptr(), buf.data_ptr(),
                                            int(to_buf), self.stream), "bdem_rows_copy")
            self.launches += 1

    def bond_id(self, pos: int) -> int:
        """Caller bond index of a SELL position."""
        return int(self.sell.bond_of_pos[pos]) if 0 <= pos < self.sell.n_pos else -1

    def raise_errors(self, host_err):
        """Re-raise a kernel's data error as the reference exception.

        The message lists, like ``stretch_terms`` / ``shear_terms``
        (bonds.py:163-168, 222-227), the offending indices into the ACTIVE
        bond list of ``energy_terms`` (bonds.py:482-490), evaluated at the
        state the kernel saw (``self.eval_pq``, set by the caller before the
        read-back).  Error path only: the state is read back and the
        indices are recovered on the host."""
        deg = host_err[L.ERRSLOT_DEG_COUNT] > 0
        if not deg and host_err[L.ERRSLOT_ANTI_COUNT] <= 0:
            return
        first = self.bond_id(int(host_err[L.ERRSLOT_DEG_FIRST if deg
                                           else L.ERRSLOT_ANTI_FIRST]))
        self.reset_errors()
        idx = [first]
        if self.eval_pq is not None:
            idx = self._offending_active(*self.eval_pq, deg)
        if deg:
            raise DegenerateBondError(f"coincident bond endpoints at indices {idx}")
        raise DegenerateShearError(f"antipodal quaternion pairs at indices {idx}")

    def _offending_active(self, p, q, degenerate: bool) -> list:
        pos = self.sell.pos_of_bond
        status = self.status.cpu().numpy()[pos]
        act = np.nonzero(status != 2)[0]
        i, j = self._bi_np[act], self._bj_np[act]
        if degenerate:
            pp = p.cpu().numpy()
            l0 = self.geom[L.BG["L0"]].cpu().numpy()[pos][act]
            bad = np.linalg.norm(pp[j] - pp[i], axis=-1) < 1e-12 * l0
        else:
            qq = q.cpu().numpy()
            u = qq[i] + qq[j]
            bad = np.sum(u * u, axis=-1) < 1e-8**2
        return np.nonzero(bad)[0].tolist()

    def read_scalars(self):
        """Synchronise once and return (scalars, err) host arrays."""
        self.h_scalars.copy_(self.scalars, non_blocking=True)
        self.h_err.copy_(self.err, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        err = self.h_err.numpy()
        if err[L.ERRSLOT_COINCIDENT]:
            # contact.py:200-203: evaluated with the +x fallback normal, and logged
            logger.warning("coincident contact centers; using +x fallback normal")
            self.err[L.ERRSLOT_COINCIDENT] = 0
        if err[L.ERRSLOT_DEG_COUNT] or err[L.ERRSLOT_ANTI_COUNT]:
            self.raise_errors(err.copy())
        return self.h_scalars.numpy()

    # ---------------------------------------------------------------- kernels
    # ------------------------------------------------------------- surfaces
    def set_mesh(self, mesh, bonds):
        """Static inputs of the surface reconstruction: rest tet vertices about
        the centroid, boundary-face masks, and each bond's local faces."""
        from .mesh import boundary_masks
        rel = mesh.vertices[mesh.tets] - mesh.centroids[:, None, :]       # (n, 4, 3)
        self.tet_rel = _t(np.ascontiguousarray(rel), device=self.device)
        self.bmask = _t(boundary_masks(mesh), I32, self.device)
        fi = np.asarray(bonds.face_i, dtype=np.int8)
        fj = np.asarray(bonds.face_j, dtype=np.int8)
        self.face_i = _t(self.sell.to_positions(fi, fill=-1), torch.int8, self.device)
        self.face_j = _t(self.sell.to_positions(fj, fill=-1), torch.int8, self.device)

    def surface(self, labels: torch.Tensor):
        """reconstruct_surface (geometry.py:313-343) of the device state:
        [(component, verts (3F,3), tris (F,3))] in the reference's order."""
        if getattr(self, "tet_rel", None) is None:
            raise ValueError("surface reconstruction needs a tet mesh (Scene(mesh=...))")
        need = int(self.lib.bdem_surface_workspace(self.n))
        if getattr(self, "_surf_work", None) is None or self._surf_work.numel() < need:
            self._surf_work = torch.empty(need, dtype=torch.uint8, device=self.device)
        cap = getattr(self, "_surf_cap", 0)
        nf = C.c_int64(0)
        for _ in range(2):
            if cap > 0 and getattr(self, "_surf_verts", None) is not None:
                vp, cp_ = self._surf_verts.data_ptr(), self._surf_comp.data_ptr()
            else:
                vp = cp_ = None
            self.call("bdem_surface", self.sysp, self.p.data_ptr(), self.q.data_ptr(),
                      self.tet_rel.data_ptr(), self.bmask.data_ptr(), self.face_i.data_ptr(),
                      self.face_j.data_ptr(), labels.data_ptr(), self._surf_work.data_ptr(),
                      vp, cp_, cap, C.byref(nf), self.stream)
            if int(nf.value) <= cap:
                break
            cap = max(int(nf.value), 2 * cap)
            self._surf_cap = cap
            self._surf_verts = torch.empty((cap, 3, 3), dtype=F64, device=self.device)
            self._surf_comp = torch.empty(cap, dtype=I32, device=self.device)
        F = int(nf.value)
        verts = self._surf_verts[:F].reshape(-1, 3).cpu().numpy() if F else np.zeros((0, 3))
        comp = self._surf_comp[:F].cpu().numpy() if F else np.zeros(0, dtype=np.int32)
        n_comp = int(labels.max()) + 1 if labels.numel() else 0
        counts = np.bincount(comp, minlength=n_comp)
        groups, start = [], 0
        for c in range(n_comp):
            k = int(counts[c])
            v = verts[3 * start:3 * (start + k)]
            tris = np.arange(3 * k, dtype=np.int64).reshape(-1, 3)
            groups.append((c, v, tris))
            start += k
        return groups

    def coef_planes(self) -> torch.Tensor:
        """The AoSoA-32 SpMV coefficients as (BDEM_CF_COUNT, n_pos) planes."""
        npos32 = self.scoef.numel() // L.CF["COUNT"]
        k = L.CF["COUNT"]
        # record per 32 positions: coefficient pair j, lane l, member m at 64 j + 2 l + m
        v = self.scoef.view(npos32 // 32, k // 2, 32, 2).permute(1, 3, 0, 2)
        return v.reshape(k, npos32)[:, :self.npos]

    def friction(self, mu_s: float, mu_r: float, dt: float) -> int:
        """apply_friction (contact.py:303-350) on the device state in place;
        returns the number of dependency waves the pair sweep used."""
        need = int(self.lib.bdem_friction_workspace(self.n, self.pair_cap))
        work = getattr(self, "_fric_work", None)
        if work is None or work.numel() < need:
            work = self._fric_work = torch.empty(max(need, 1), dtype=torch.uint8,
                                                 device=self.device)
        waves = C.c_int64(0)
        self.call("bdem_friction", self.sysp, self.p.data_ptr(), self.q.data_ptr(),
                  self.v.data_ptr(), self.qdot.data_ptr(), float(mu_s), float(mu_r), float(dt),
                  work.data_ptr(), C.byref(waves), self.stream)
        return int(waves.value)

    def call(self, name, *args):
        rc = getattr(self.lib, name)(*args)
        self.launches += 1
        if rc != 0:
            raise L.BdemLibraryError(f"{name} failed with status {rc}")


_REGISTERED: dict = {}


def _unregister(key):
    if _REGISTERED.pop(key, None):
        try:
            torch.cuda.cudart().cudaHostUnregister(key[0])
        except Exception:
            pass


def _host(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))


def _pack_collider(col):
    kind = type(col).__name__
    if kind == "HalfSpace":
        n = np.asarray(col.normal, dtype=float)
        return (0, n[0], n[1], n[2], float(col.offset), 0.0, 0.0)
    if kind == "SphereCollider":
        c = np.asarray(col.center, dtype=float)
        return (1, c[0], c[1], c[2], float(col.radius), 0.0, 0.0)
    if kind == "BoxCollider":
        c = np.asarray(col.center, dtype=float)
        h = np.asarray(col.half_extents, dtype=float)
        return (2, c[0], c[1], c[2], h[0], h[1], h[2])
    raise TypeError(f"unsupported collider {kind}")
