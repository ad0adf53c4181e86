"""Manifold Newton solve of the incremental potential on the GPU.

Host control flow mirrors ``minimize_second_order``
(``/root/reference/pkg/src/bdem/solver.py:511-562``), ``line_search``
(``:387-406``), ``_newton_direction`` (``:462-508``) and ``pcg``
(``linalg.py:40-97``) line by line; every array operation is a kernel of
``libbdem_sm100.so`` and the host only reads back the scalars the control
flow branches on (f, |z|, PCG state per chunk, slope, f_t).
"""

from __future__ import annotations

import logging
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L

# the reference logs its solver's recoveries (linalg.py:95,118, solver.py:545);
# same messages here
logger = logging.getLogger(__name__)

EPS = float(np.finfo(float).eps)


@dataclass
class SolverConfig:
    """Same fields and defaults as the reference (solver.py:38-49)."""

    epsilon: float = 1e-6
    max_iterations: int = 100
    armijo: float = 1e-4
    shrink: float = 0.5
    min_alpha: float = 1e-12
    pcg_max_iterations: int = 2000
    linear_mode: str = "pcg"
    compare_projector: bool = False
    workers: int = 1
    penalty_kappa: float = 1e8


@dataclass
class IterationRecord:
    """solver.py:52-60 (+ ls_trials: line-search energy evaluations)."""

    index: int
    f: float
    grad_norm: float
    constraint_norm: float
    alpha: float = 0.0
    pcg_iterations: int = 0
    direction_gap: float = 0.0
    ls_trials: int = 0


@dataclass
class SolveResult:
    """solver.py:63-73; p, q are device tensors (``.cpu().numpy()`` for host)."""

    p: object
    q: object
    converged: bool
    iterations: int
    grad_norm: float
    records: list = field(default_factory=list)
    pcg_total: int = 0
    max_unit_dev: float = 0.0
    reason: str = "converged"


@dataclass
class PCGResult:
    """linalg.py:20-26 (x lives in DeviceSystem.y)."""

    iterations: int
    converged: bool
    relative_residual: float
    restarts: int = 0


class LineSearchError(RuntimeError):
    pass


def relative_tolerance(grad_norm: float) -> float:
    """min(0.5, sqrt(|g|)) (linalg.py:29-37)."""
    if grad_norm < 0.0:
        raise ValueError("gradient norm must be non-negative")
    return min(0.5, math.sqrt(grad_norm))


class GPUProblem:
    """The step objective on the device (ImplicitProblem, integrator.py:164-210).

    Wraps a ``DeviceSystem`` whose step context (p_hat, q_hat, m/dt^2,
    colliders, frozen pairs) has been prepared by the predictor.
    """

    def __init__(self, dev, timer=None):
        self.dev = dev
        self.free = dev.free_np
        # optional KernelTimer: CUDA events around the fused bond kernel and
        # every SpMV launch (bench.py's live roofline measurement)
        self.timer = timer if timer is not None else getattr(dev, "timer", None)

    @property
    def n(self):
        return self.dev.n

    # -- assembly: value, gradient, reduced gradient and clamped blocks
    def assemble(self, p, q):
        d = self.dev
        s, st = d.sysp, d.stream
        if d.nb:
            tm = self.timer
            if tm is not None:
                tm.begin("bond_assemble")
            d.call("bdem_bond_assemble", s, p.data_ptr(), q.data_ptr(), st)
            if tm is not None:
                tm.end("bond_assemble")
        if d.n_pair:
            d.call("bdem_pair_assemble", s, p.data_ptr(), 0, st)
        tm = self.timer
        if tm is not None:
            tm.begin("element_assemble")
        d.call("bdem_element_assemble", s, p.data_ptr(), q.data_ptr(), d.z.data_ptr(), st)
        if tm is not None:
            tm.end("element_assemble")
        d.call("bdem_reduce_finish", s, 0, 7, L.RED_BLOCKS, st)
        d.eval_pq = (p, q)
        sc = d.read_scalars()
        nsing = int(sc[L.SC["NSING"]])
        if nsing:
            logger.warning("block-jacobi: %d singular blocks fall back to identity", nsing)
        f = float(sc[L.SC["F"]])
        gnorm = math.sqrt(float(sc[L.SC["GNORM2"]]))
        cnorm = math.sqrt(float(sc[L.SC["CNORM2"]]))
        return f, gnorm, cnorm, float(sc[L.SC["MAXDEV"]])

    # -- objective at a trial point (ImplicitProblem.value)
    def trial_value(self, p, q, dp, dq, alpha, pt, qt):
        d = self.dev
        s, st = d.sysp, d.stream
        d.call("bdem_trial_point", s, p.data_ptr(), q.data_ptr(), dp.data_ptr(), dq.data_ptr(),
               float(alpha), pt.data_ptr(), qt.data_ptr(), st)
        return self._energy_tail(pt, qt)

    def value(self, p, q):
        d = self.dev
        d.call("bdem_element_energy", d.sysp, p.data_ptr(), q.data_ptr(), 1, d.stream)
        return self._energy_tail(p, q)

    def _energy_tail(self, p, q):
        d = self.dev
        s, st = d.sysp, d.stream
        d.call("bdem_bond_energy", s, p.data_ptr(), q.data_ptr(), L.SC["EBOND"], st)
        d.call("bdem_pair_assemble", s, p.data_ptr(), 1, st)
        d.call("bdem_reduce_finish", s, L.SC["FT"], 7, L.RED_BLOCKS, st)
        d.eval_pq = (p, q)
        sc = d.read_scalars()
        # inertia + (bonds + contacts - gravity)   (integrator.py:87-93, 191-193)
        return float(sc[L.SC["FT"]]) + (((float(sc[L.SC["EBOND"]]) + float(sc[L.SC["EPAIR"]]))
                                         + float(sc[L.SC["ECOL"]])) + float(sc[L.SC["EGRAV"]]))

    def energy_breakdown(self, p, q):
        """PotentialModel.energy_breakdown (integrator.py:131-138)."""
        d = self.dev
        s, st = d.sysp, d.stream
        d.call("bdem_element_energy", s, p.data_ptr(), q.data_ptr(), 0, st)
        d.call("bdem_bond_energy", s, p.data_ptr(), q.data_ptr(), L.SC["EBOND"], st)
        d.call("bdem_pair_assemble", s, p.data_ptr(), 1, st)
        d.call("bdem_kinetic", s, d.v.data_ptr(), d.qdot.data_ptr(), st)
        d.call("bdem_reduce_finish", s, L.SC["FT"], 7, L.RED_BLOCKS, st)
        sc = d.read_scalars()
        return {"bond": float(sc[L.SC["EBOND"]]),
                "contact": float(sc[L.SC["EPAIR"]]) + float(sc[L.SC["ECOL"]]),
                "gravity": float(sc[L.SC["EGRAV"]]),
                "kinetic": float(sc[L.SC["EKIN"]])}

    # -- PCG on the reduced system: A y = -z   (linalg.py:40-97)
    def solve_pcg(self, tol, max_iter, chunk0=4, chunk_max=16) -> PCGResult:
        d = self.dev
        s, st = d.sysp, d.stream
        ptrs = (d.y.data_ptr(), d.r.data_ptr(), d.zv.data_ptr(), d.pv.data_ptr())
        boost, restarts = 0.0, 0
        while True:
            d.call("bdem_pcg_init", s, d.z.data_ptr(), -1.0, *ptrs, float(tol), int(max_iter),
                   float(boost), st)
            chunk = chunk0
            tm = self.timer
            k_before = 0
            hist = []
            while True:
                if tm is None:
                    d.call("bdem_pcg_iterate", s, *ptrs, d.ap.data_ptr(), int(chunk), st)
                else:
                    for _ in range(chunk):
                        tm.begin("spmv")
                        d.call("bdem_pcg_spmv", s, ptrs[3], d.ap.data_ptr(), st)
                        tm.end("spmv")
                        d.call("bdem_pcg_update", s, *ptrs, d.ap.data_ptr(), st)
                d.h_pcg.copy_(d.pcg_state, non_blocking=True)
                torch.cuda.current_stream(d.device).synchronize()
                h = d.h_pcg.numpy()
                state = int(h[L.PCG["STATE"]])
                if tm is not None:
                    # SpMV launches after the solve stopped exited early: drop them
                    k_now = int(h[L.PCG["K"]])
                    worked = k_now - k_before + (1 if state == L.PCG_BREAKDOWN else 0)
                    tm.drop_last("spmv", chunk - min(worked, chunk))
                    k_before = k_now
                if state == L.PCG_RUNNING:
                    chunk = self._next_chunk(chunk, chunk_max, h, hist)
                    continue
                break
            k = int(h[L.PCG["K"]])
            rel = float(h[L.PCG["REL"]])
            if state == L.PCG_BREAKDOWN:
                restarts += 1
                boost = float(h[L.PCG["BOOST"]])
                logger.warning("pcg breakdown; restarting with diagonal boost %.3e", boost)
                if restarts > 3:
                    return PCGResult(k, False, rel, restarts)
                continue
            return PCGResult(k, state == L.PCG_CONVERGED, rel, restarts)

    @staticmethod
    def _next_chunk(chunk, chunk_max, h, hist):
        """Iterations to enqueue before the next read-back.  Kernels past
        convergence exit at once, so a chunk only trades early-exit launches
        against read-back bubbles; once two read-backs show the residual's
        geometric rate, the chunk is sized to the iterations it predicts
        (plus one), else it doubles up to ``chunk_max``."""
        k, rel, tol = float(h[L.PCG["K"]]), float(h[L.PCG["REL"]]), float(h[L.PCG["TOL"]])
        hist.append((k, rel))
        if len(hist) >= 2:
            (k0, r0), (k1, r1) = hist[-2], hist[-1]
            if k1 > k0 and 0.0 < r1 < r0 and tol > 0.0:
                rate = (r1 / r0) ** (1.0 / (k1 - k0))
                if rate < 1.0:
                    need = math.log(tol / r1) / math.log(rate)
                    if math.isfinite(need):
                        return int(min(max(math.ceil(need) + 1, 4), 4 * chunk_max))
        return min(chunk * 2, chunk_max)

    def dot(self, a, b, n):
        d = self.dev
        d.call("bdem_dot", d.sysp, a.data_ptr(), b.data_ptr(), int(n), L.SC["SLOPE"], d.stream)
        return float(d.read_scalars()[L.SC["SLOPE"]])

    def direction(self, q, vec, sign):
        d = self.dev
        d.call("bdem_direction", d.sysp, q.data_ptr(), vec.data_ptr(), float(sign),
               d.dp.data_ptr(), d.dq.data_ptr(), d.stream)


def minimize_second_order(problem: GPUProblem, p0, q0, cfg: SolverConfig) -> SolveResult:
    """Newton on the manifold (solver.py:511-562) with device-resident arrays.

    ``p0``/``q0`` are device tensors; they are copied into the iterate.
    """
    if cfg.linear_mode != "pcg":
        raise NotImplementedError("the GPU path implements linear_mode='pcg'")
    d = problem.dev
    p, q, pt, qt = d.xp, d.xq, d.tp, d.tq
    if p0.data_ptr() != p.data_ptr():
        p.copy_(p0)
    if q0.data_ptr() != q.data_ptr():
        q.copy_(q0)
    d.call("bdem_normalize_free", d.sysp, q.data_ptr(), d.stream)
    records = []
    pcg_total = 0
    gnorm = math.inf
    max_dev = 0.0
    nf6 = 6 * d.vstride
    last_checked = True
    for it in range(cfg.max_iterations):
        f, gnorm, cnorm, dev_it = problem.assemble(p, q)
        max_dev = max(max_dev, dev_it)
        last_checked = True
        if gnorm < cfg.epsilon:
            records.append(IterationRecord(it, f, gnorm, cnorm))
            return SolveResult(p, q, True, it, gnorm, records, pcg_total, max_dev)
        res = problem.solve_pcg(relative_tolerance(gnorm), cfg.pcg_max_iterations)
        pcg_total += res.iterations
        slope = problem.dot(d.z, d.y, nf6)
        problem.direction(q, d.y, 1.0)
        if not math.isfinite(slope) or slope >= 0.0:
            logger.warning("newton direction not a descent direction; "
                           "falling back to the gradient")
            problem.direction(q, d.z, -1.0)
            slope = -gnorm * gnorm
        # line search (solver.py:387-406)
        alpha = 1.0
        noise = 8.0 * EPS * abs(f)
        trials = 0
        accepted = False
        while alpha >= cfg.min_alpha:
            ft = problem.trial_value(p, q, d.dp, d.dq, alpha, pt, qt)
            trials += 1
            if math.isfinite(ft) and ft <= f + cfg.armijo * alpha * slope + noise:
                accepted = True
                break
            alpha *= cfg.shrink
        if not accepted:
            records.append(IterationRecord(it, f, gnorm, cnorm, pcg_iterations=res.iterations,
                                           ls_trials=trials))
            return SolveResult(p, q, False, it, gnorm, records, pcg_total, max_dev, "line-search")
        p, pt = pt, p
        q, qt = qt, q
        f = ft
        last_checked = False
        records.append(IterationRecord(it, f, gnorm, cnorm, alpha=alpha,
                                       pcg_iterations=res.iterations, ls_trials=trials))
    # the reference also folds in the deviation of the final iterate
    if not last_checked:
        _, _, _, dev_last = problem.assemble(p, q)
        max_dev = max(max_dev, dev_last)
    return SolveResult(p, q, False, cfg.max_iterations, gnorm, records, pcg_total, max_dev,
                       "max-iterations")
