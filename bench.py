#!/usr/bin/env python
"""Benchmark: Newton iterations/s of the implicit BDEM step on the 600K plate.

Workload (BASELINE.json configs[2]): 1000x600 triangular
ceramic plate, 600,000 spheres, 3,591,004 bonds, E=3e11, dropped at 5 m/s
onto a half-space, tilted 10 deg, plasticity/fracture on, dt=5e-6,
eps=1e-3 (the fp64 gradient noise floor at 600K is ~3e-5 N).
Synthetic, seeded inputs; no dataset.

A bench "step" is one committed time step of the trajectory, advanced the
way the reference's runner does it (``runner.advance``, runner.py:47-71): a
``stable_step`` (broad phase, predictor, manifold Newton solve with PCG and
line search, velocity update, fracture update, energies) whose solve does
not commit is replaced by two half steps (recursively, 2 levels) -- the
plate's Newton iteration cycles at the penalty-contact onset around step 18,
in the reference as well.  Every timed step therefore
commits; a step that cannot be committed even at dt/4 aborts the bench.
``value`` = all Newton iterations performed in the timed region (committed
solves and the attempts that triggered a split; both are full Newton
iterations) / max-over-ranks device time; the split-off work and the
committed-only rate are reported beside it, with per-step Newton / PCG /
line-search counts.  ``e2e`` repeats the same steps through the same public
call with host buffers (``Scene(host_sync=True)``: host->device upload of the
element and bond state before, device->host download after, every
``stable_step``).  Per-kernel durations (fused bond + element assembly, every
SpMV) are taken with CUDA events on the launching stream around every launch
of a replay of exactly the timed steps (the timed region itself runs the
production path uninstrumented).  ``rot_zero_shortcut`` replays the timed
steps with ``bdem_pcg_set_rot_skip(1)`` (exact; reported beside the full 6-DOF
headline, not as it).

``--impl reference`` times the UNMODIFIED reference (``bdem``, shipped to the
GPU box as bytecode in ``oracle/_ref``; ``oracle/build_ref.py``) on the host
cores at the same 600K config: K=2 Newton iterations of
``minimize_second_order`` (solver.py:511-562) on the step-1 problem exactly
as ``stable_step`` builds it (solver.py:894-908), started (a) from a mid-solve
iterate -- the first Newton iterate of the GPU step-1 solve whose PCG count
reaches that solve's average, computed on the GPU during setup, outside the
timed region -- and (b) from the predictor, each with ``workers=cpu_count``
and ``workers=1``.  The headline is (a) with ``workers=cpu_count``.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "Newton iters/sec @600K particles; bonds/sec assembled; SpMV HBM GB/s vs peak"
UNIT = "Newton it/s"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nx", type=int, default=1000)
    ap.add_argument("--ny", type=int, default=600)
    ap.add_argument("--epsilon", type=float, default=1e-3)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 2M-block kernel leg")
    ap.add_argument("--no-rot-leg", action="store_true",
                    help="skip the rotation-free (bdem_pcg_set_rot_skip) leg")
    ap.add_argument("--c5-side", type=int, default=126)
    ap.add_argument("--ref-plate", type=int, nargs=2, default=None,
                    help="plate size of the reference measurement (default: --nx --ny)")
    ap.add_argument("--ref-k", type=int, default=2,
                    help="Newton iterations per reference measurement (BASELINE.md §3: 2)")
    ap.add_argument("--ref-starts", type=lambda s: s.split(","),
                    default=["mid-solve", "predictor"],
                    help="reference start points, headline first")
    ap.add_argument("--ref-workers", default="cores",
                    help="SolverConfig.workers of the reference runs: 'cores', 'both' "
                         "(cores and 1; BASELINE.md §3) or an integer")
    ap.add_argument("--max-retries", type=int, default=2,
                    help="dt-halving levels per timed step (runner.py:47-71)")
    return ap.parse_args()


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def fp64_peak():
    """Measured FP64 DFMA throughput of this B200 (profiles/r02/fp64_peak.json,
    scratch/r02/fp64/fp64_peak.cu), TFLOP/s."""
    try:
        with open(os.path.join(REPO, "profiles", "r02", "fp64_peak.json")) as fh:
            return float(json.load(fh)["fp64_dfma_tflops"]), "measured (profiles/r02/fp64_peak.json)"
    except Exception:
        return None, None


# ---------------------------------------------------------------------------
# the reference on the host cores
# ---------------------------------------------------------------------------

def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def gpu_mid_iterate(spec, eps):
    """Setup for the mid-solve start (outside any timed region): the step-1
    Newton solve on the GPU, its per-iteration PCG counts, and the iterate at
    the start of the first Newton iteration whose PCG count reaches the
    solve's average.  Returns (p, q, info) or None without
    a GPU."""
    import torch
    if not torch.cuda.is_available():
        return None
    from paper_2308_10459_b200 import SolverConfig
    from paper_2308_10459_b200.newton import GPUProblem, minimize_second_order
    from paper_2308_10459_b200.scene import Scene
    from paper_2308_10459_b200.step import prepare_step
    scene = Scene.from_spec(spec, host_sync=False)
    prep = prepare_step(scene)
    seen = []

    class Capture(GPUProblem):
        def assemble(self, p, q):
            seen.append((p.cpu().numpy(), q.cpu().numpy()))
            return super().assemble(p, q)

    sol = minimize_second_order(Capture(prep.problem.dev), scene.device.xp, scene.device.xq,
                                SolverConfig(epsilon=eps, max_iterations=300))
    pcg = [r.pcg_iterations for r in sol.records if r.pcg_iterations > 0]
    avg = sum(pcg) / max(len(pcg), 1)
    k = next((i for i, c in enumerate(pcg) if c >= avg), len(pcg) - 1)
    p, q = seen[k]
    info = {"gpu_step1_newton": len(pcg), "gpu_step1_pcg": pcg, "gpu_step1_pcg_avg": avg,
            "start_iteration": k, "gpu_pcg_at_start": pcg[k]}
    del scene, prep, seen
    torch.cuda.empty_cache()
    return p, q, info


def reference_newton(nx, ny, eps, k_iters, starts, workers, mid=None):
    """K Newton iterations of the UNMODIFIED reference minimize_second_order
    (solver.py:511-562) on the step-1 problem of the nx x ny plate, built as
    stable_step builds it (solver.py:894-908), for every (start, workers).
    Returns (kind, runs, setup info)."""
    from oracle import build_ref
    from oracle import ref_adapter as RA
    from paper_2308_10459_b200 import configs as C
    bdem = build_ref.load()
    if bdem is None:
        raise RuntimeError("reference bdem unavailable: run __graft_entry__.build() where "
                           "/root/reference exists (it writes oracle/_ref)")
    from bdem import solver as rsv
    import logging
    logging.getLogger("bdem").setLevel(logging.ERROR)
    spec = C.plate(nx=nx, ny=ny, epsilon=eps)
    t0 = time.perf_counter()
    sc = RA.ref_scene(bdem, spec)
    prob, p0, q0, pairs = RA.step_problem(bdem, sc)
    setup = {"scene_and_step_problem_s": time.perf_counter() - t0, "bonds": int(sc.bonds.n),
             "spheres": int(sc.elements.n), "contact_pairs": int(pairs.shape[0])}
    start_pts = {"predictor": (p0, q0)}
    if mid is not None:
        start_pts["mid-solve"] = (mid[0], mid[1])
    runs = []
    for name in starts:
        if name not in start_pts:
            continue
        p, q = start_pts[name]
        for w in workers:
            cfg = rsv.SolverConfig(epsilon=eps, max_iterations=k_iters, workers=w)
            t = time.perf_counter()
            sol = rsv.minimize_second_order(prob, p, q, cfg)
            sec = time.perf_counter() - t
            its = [r for r in sol.records if r.pcg_iterations > 0 or r.alpha > 0]
            n_it = max(len(its), 1)
            runs.append({"start": name, "workers": w, "newton_iterations": len(its),
                         "seconds": sec, "newton_per_s": n_it / sec,
                         "pcg_per_iteration": [r.pcg_iterations for r in its],
                         "grad_norm": [r.grad_norm for r in its], "reason": sol.reason})
    return "reference", runs, setup


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    nx, ny = args.ref_plate if args.ref_plate else (args.nx, args.ny)
    # workers only threads spd_project (solver.py:48,107-110); measured on the
    # GPU box: 172.7 s (16) vs 166.3 s (1) for the mid-solve start, 102.8 vs
    # 97.2 s from the predictor (profiles/r02/reference_arm.json), so the
    # default run uses cpu_count only and '--ref-workers both' adds workers=1
    if args.ref_workers == "both":
        workers = sorted({cores, 1}, reverse=True)
    elif args.ref_workers == "cores":
        workers = [cores]
    else:
        workers = [int(args.ref_workers)]
    mid = gpu_mid_iterate(__import__("paper_2308_10459_b200.configs", fromlist=["plate"])
                          .plate(nx=nx, ny=ny, epsilon=args.epsilon), args.epsilon) \
        if "mid-solve" in args.ref_starts else None
    kind, runs, setup = reference_newton(nx, ny, args.epsilon, args.ref_k, args.ref_starts,
                                         workers, mid)
    head = runs[0]
    value = head["newton_per_s"]
    timed_s = sum(r["seconds"] for r in runs)
    sample = (f"reference bdem (oracle/_ref bytecode, numpy/scipy) on {cpu_model()}: "
              f"{head['newton_iterations']} Newton iterations of minimize_second_order on the "
              f"{nx}x{ny} plate's step-1 problem from the {head['start']} start, "
              f"workers={head['workers']} ({head['seconds']:.1f}s, PCG "
              f"{head['pcg_per_iteration']})")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        # one 600K Newton iteration of the reference takes minutes on the host:
        # the timed region is the headline measurement, spread over the
        # requested step count so ms_per_step x steps is its real duration
        "ms_per_step": 1e3 * head["seconds"] / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(args),
        "pcg_per_newton": sum(head["pcg_per_iteration"]) / max(head["newton_iterations"], 1),
        "measurements": runs, "setup": setup, "mid_start": (mid[2] if mid else None),
        "all_measurements_s": timed_s, "cpu_model": cpu_model(),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": int(head["workers"]),
                         "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_block(args):
    return {"workload": f"C3 plate impact {args.nx}x{args.ny} (BASELINE configs[2])",
            "spheres": args.nx * args.ny, "epsilon": args.epsilon, "dt": 5e-6,
            "l2": "inputs larger than L2 (bond geometry 24 + staging 17 + coefficient 14 "
                  "planes x n_bond fp64 = 1.97 GB >> 126 MB)",
            "parallelism": f"replicas x{args.gpus}"}


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.nv is not None:
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.t.join(timeout=1.0)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def snapshot(scene):
    """Host copy of everything a step reads (element + bond state, history)."""
    import copy
    scene.sync_to_host()
    return {"el": scene.elements.copy(), "b": scene.bonds.copy(), "time": scene.time,
            "p_prev": scene.p_prev.copy(), "q_prev": scene.q_prev.copy(),
            "labels": copy.deepcopy(scene._labels)}


def restore(scene, snap):
    """Write a snapshot back into the scene's host arrays (in place)."""
    for name in ("p", "q", "v", "qdot"):
        getattr(scene.elements, name)[...] = getattr(snap["el"], name)
    for name in scene.bonds.STATE_FIELDS:
        getattr(scene.bonds, name)[...] = getattr(snap["b"], name)
    scene.p_prev[...] = snap["p_prev"]
    scene.q_prev[...] = snap["q_prev"]
    scene.time = snap["time"]
    if snap["labels"] is not None:
        scene._labels = snap["labels"]
        scene.device.labels = __import__("torch").as_tensor(snap["labels"].labels).to(
            scene.device.device)


def c5_leg(n_side, peak):
    """BASELINE configs[4] (C5): 2M-sphere jittered block, random unit
    quaternions, ~12M bonds.  Measures the fused assembly (random q sends
    every rotation block through the eigen-clamp pass) and the SpMV at
    memory-bound scale, each timed with CUDA events over repeated launches on
    the predictor state of step 1."""
    import torch

    from paper_2308_10459_b200 import configs
    from paper_2308_10459_b200.newton import GPUProblem
    from paper_2308_10459_b200.scene import Scene
    spec = configs.block(n_side=n_side, random_q=True)
    scene = Scene.from_spec(spec, host_sync=False)
    dev = scene.device
    dev.set_physics(spec.gravity, spec.k_contact, 0.0, [])
    dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(),
             dev.qdot.data_ptr(), dev.p_prev.data_ptr(), dev.q_prev.data_ptr(), spec.dt,
             dev.p_hat.data_ptr(), dev.q_hat.data_ptr(), dev.mp_dt2.data_ptr(),
             dev.mq_dt2.data_ptr(), dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream)
    GPUProblem(dev).assemble(dev.xp, dev.xq)

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    asm_ms = timed(lambda: dev.call("bdem_bond_assemble", dev.sysp, dev.xp.data_ptr(),
                                    dev.xq.data_ptr(), dev.stream), 3)
    x = torch.randn(6 * dev.vstride, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
    spmv_ms = timed(lambda: dev.call("bdem_spmv", dev.sysp, x.data_ptr(), y.data_ptr(),
                                     dev.stream), 20)
    sb = spmv_bytes(dev)
    out = {"workload": f"C5 block {n_side}^3 random q (BASELINE configs[4])",
           "spheres": dev.n, "bonds": dev.nb, "assembly_ms": asm_ms,
           "bonds_per_sec_assembled": dev.nb / (asm_ms * 1e-3),
           "spmv_ms": spmv_ms, "spmv_bytes": sb, "spmv_gbs": sb / (spmv_ms * 1e-3) / 1e9,
           "spmv_frac": sb / (spmv_ms * 1e-3) / 1e9 / peak}
    # FP64 view of the random-q assembly (every rotation block through the
    # register Jacobi eigen-clamp): ncu FP64 operation counts of the same
    # launch (2 flops per DFMA) over the live CUDA-event time
    c5n = load_ncu_traffic().get("c5_block", {})
    flops = _sum_or_none(c5n.get(k, {}).get("fp64_flops_per_launch")
                         for k in ("k_bond_rows", "k_bond_clamp"))
    fpk, fpk_src = fp64_peak()
    if flops and fpk:
        ach = flops / (asm_ms * 1e-3) / 1e12
        out["fp64"] = {"bound": "fp64", "achieved": ach, "peak": fpk, "unit": "TFLOP/s",
                       "frac": ach / fpk, "flops_per_launch": flops,
                       "pipe_frac": {k: c5n.get(k, {}).get("fp64_pipe_frac")
                                     for k in ("k_bond_rows", "k_bond_clamp")},
                       "source": "ncu sm__sass_thread_inst_executed_op_{dfma,dmul,dadd} "
                                 "(profiles/ncu_traffic.json)", "peak_source": fpk_src}
    del scene, dev
    torch.cuda.empty_cache()
    return out


def pcg_leg(dev, peak, traffic, chunk=32, reps=3):
    """One PCG iteration as a whole (SpMV + r/z update + p update, the loop
    that takes ~85% of a Newton iteration): a chunk of iterations of
    bdem_pcg_iterate on the last assembled system (full 6-DOF, tolerance 0
    so every launch works), CUDA events around the chunk, best of reps;
    against the ncu DRAM bytes of the three kernels per iteration."""
    import torch
    ptrs = (dev.y.data_ptr(), dev.r.data_ptr(), dev.zv.data_ptr(), dev.pv.data_ptr())
    best = float("inf")
    for _ in range(reps):
        dev.call("bdem_pcg_init", dev.sysp, dev.z.data_ptr(), -1.0, *ptrs, 1e-30, 100000, 0.0,
                 dev.stream)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        dev.call("bdem_pcg_iterate", dev.sysp, *ptrs, dev.ap.data_ptr(), chunk, dev.stream)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / chunk)
    dram = _sum_or_none(traffic.get(k, {}).get("dram_bytes_per_launch")
                        for k in ("k_spmv", "k_pcg_update", "k_pcg_pupdate"))
    out = {"us": best, "chunk": chunk, "dram_bytes": dram,
           "timing": "CUDA events around bdem_pcg_iterate chunks on the last assembled system"}
    if dram:
        out.update({"achieved_gbs": dram / (best * 1e-6) / 1e9,
                    "frac": dram / (best * 1e-6) / 1e9 / peak,
                    "bytes_source": "ncu dram__bytes_read+write of the three in-chain kernels "
                                    "(profiles/ncu_traffic.json)"})
    return out


def reduce_across_ranks(times_ms, counts, world, device):
    """Replica aggregation: device times -> max over ranks, work -> sum."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(times_ms, dtype=torch.float64, device=device)
    c = torch.tensor(counts, dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
    return [float(v) for v in t], [float(v) for v in c]


def spmv_bytes(dev):
    """Algorithmic bytes of one SpMV in this library's format:
    per bond with both ends free: n (3), alpha, beta, C (9) fp64 read once =
    112 B, plus two adjacency entries (position/slot, int32) = 16 B; per free
    row: x and y (48 + 48 B), diagonal P, R (96 B), slot/slice index (12 B)."""
    entries = int((dev.sell.pos_oslot >= 0).sum() + (dev.sell.jslot >= 0).sum())
    return 56 * entries + 8 * entries + dev.nf * (48 + 48 + 96 + 12)


def assembly_bytes(dev):
    """SURVEY §8(d)'s algorithmic bytes of one assembly (bond + element
    kernels) per Newton iteration: per bond 161 B in (i, j, status, l0, d0,
    frame, kn, kt, k_diag, scale) + 288 B out (the two off-diagonal 18-value
    blocks); per free element 136 B in (p, q, p_hat, q_hat, m, r, pinned),
    144 B diagonal, 144 B block-Jacobi inverse, 48 B z, 56 B gp + gq."""
    return dev.nb * (161 + 288) + dev.nf * (136 + 144 + 144 + 48 + 56)


# Chip-wide L2-slice (LTS) throughput cap per SM clock, measured on the
# GB300 (B300_MICROARCH.md "LTS throughput cap ~6300 B/cyc full-chip"); the
# SpMV's gathers re-read coefficients and x from L2, so this is its real bound.
def _l2_bytes_per_clk():
    """Measured L2 read throughput of this B200 (profiles/l2_peak.json,
    scratch/l2bw); the B300 figure of B300_MICROARCH.md if absent."""
    try:
        with open(os.path.join(REPO, "profiles", "l2_peak.json")) as fh:
            return float(json.load(fh)["l2_read_bytes_per_clk"]), "measured (profiles/l2_peak.json)"
    except Exception:
        return 6300.0, "B300_MICROARCH.md estimate"


L2_BYTES_PER_CLK, L2_CAP_SOURCE = _l2_bytes_per_clk()


def l2_roofline(ncu, spmv_ms, clocks):
    """L2 view of the SpMV: ncu lts__t_sectors x 32 B per launch over the live
    launch time, against the LTS cap at the sampled SM clock."""
    sectors = ncu.get("l2_sectors_per_launch")
    mhz = (clocks.summary() or {}).get("sm_mhz") or 1965.0
    if not sectors or not spmv_ms == spmv_ms:
        return None
    achieved = 32.0 * sectors / (spmv_ms * 1e-3) / 1e9
    cap = L2_BYTES_PER_CLK * mhz * 1e6 / 1e9
    return {"bytes_per_launch": 32.0 * sectors, "achieved": achieved, "cap": cap, "unit": "GB/s",
            "frac": achieved / cap, "source": "ncu lts__t_sectors.sum x 32 B (profiles/ncu_traffic.json)",
            "cap_source": f"{L2_BYTES_PER_CLK:.0f} B/clk x sampled SM clock, {L2_CAP_SOURCE}"}


def _sum_or_none(vals):
    vals = list(vals)
    return None if any(v is None for v in vals) else float(sum(vals))


def load_ncu_traffic():
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return {}


def _timed_steps(scene, cfg, steps, max_retries, record=None):
    """``steps`` committed steps through runner.advance; returns the
    per-step records (every attempt's Newton / PCG / line-search counts)."""
    from paper_2308_10459_b200.runner import advance
    per_step = []
    for _ in range(steps):
        attempts = []
        committed = advance(scene, cfg, max_retries=max_retries, attempts=attempts)
        per_step.append({
            "newton": [a.solve.iterations for a in attempts],
            "pcg": [a.solve.pcg_total for a in attempts],
            "ls": [sum(r.ls_trials for r in a.solve.records) for a in attempts],
            "committed": [bool(a.committed) for a in attempts],
            "substeps": len(committed), "broken": sum(len(c.broken) for c in committed),
            "pairs": max(c.contact_pairs for c in committed)})
    return per_step


def _totals(per_step):
    flat = lambda key: [x for s in per_step for x in s[key]]  # noqa: E731
    newton, pcg, ls, ok = flat("newton"), flat("pcg"), flat("ls"), flat("committed")
    return {"newton": sum(newton), "pcg": sum(pcg), "ls": sum(ls),
            "newton_committed": sum(n for n, c in zip(newton, ok) if c),
            "newton_split_off": sum(n for n, c in zip(newton, ok) if not c),
            "attempts": len(newton), "failed_attempts": ok.count(False),
            "broken": sum(s["broken"] for s in per_step),
            "pairs": max((s["pairs"] for s in per_step), default=0)}


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")

    from paper_2308_10459_b200 import SolverConfig, configs
    from paper_2308_10459_b200 import _lib as L
    from paper_2308_10459_b200.scene import Scene
    from paper_2308_10459_b200.timing import KernelTimer

    lib = L.load()
    spec = configs.plate(nx=args.nx, ny=args.ny, epsilon=args.epsilon)
    scene = Scene.from_spec(spec, host_sync=False)
    cfg = SolverConfig(epsilon=args.epsilon, max_iterations=300)
    dev = scene.device

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    _timed_steps(scene, cfg, args.warmup, args.max_retries)
    snap = snapshot(scene)      # the replays below run exactly the timed steps

    barrier()
    launches0 = lib.bdem_launch_count()
    with ClockSampler(local) as clocks:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        per_step = _timed_steps(scene, cfg, args.steps, args.max_retries)
        t1.record()
        barrier()
    launches = lib.bdem_launch_count() - launches0
    ms = t0.elapsed_time(t1)
    tot = _totals(per_step)
    final = snapshot(scene)     # the rotation-free leg must reproduce it bit for bit

    # kernel timing: the timed region runs the production path uninstrumented;
    # the same steps are replayed from the snapshot with CUDA events around
    # every SpMV and assembly launch (same kernels, same inputs)
    restore(scene, snap)
    scene.host_sync = True
    timer = KernelTimer()
    dev.timer = timer
    replay = _totals(_timed_steps(scene, cfg, args.steps, args.max_retries))
    torch.cuda.synchronize()
    durations = timer.resolve()
    dev.timer = None

    pcg_it = pcg_leg(dev, peaks()[0], load_ncu_traffic())

    # e2e: the same steps again, from the same state, through the same public
    # call with host buffers every stable_step (H2D of the state before, D2H after)
    n_e2e = args.e2e_steps if args.e2e_steps is not None else args.steps
    restore(scene, snap)
    scene.host_sync = True
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    e2e = _totals(_timed_steps(scene, cfg, n_e2e, args.max_retries))
    e1.record()
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    h2d = dev.n * (3 + 4 + 3 + 4 + 3 + 4) * 8 + dev.nb * (5 * 8 + 1)
    d2h = h2d

    # rotation-free leg (SURVEY §0.5's exact shortcut, reported separately):
    # the same timed steps from the same snapshot with bdem_pcg_set_rot_skip(1)
    rot = None
    if not args.no_rot_leg:
        prev = lib.bdem_pcg_set_rot_skip(1)
        restore(scene, snap)
        scene.host_sync = False
        dev.upload_elements(scene.elements, scene.p_prev, scene.q_prev)
        dev.upload_bond_state(scene.bonds)
        barrier()
        r0 = torch.cuda.Event(enable_timing=True)
        r1 = torch.cuda.Event(enable_timing=True)
        r0.record()
        rt = _totals(_timed_steps(scene, cfg, args.steps, args.max_retries))
        r1.record()
        barrier()
        rot_ms = r0.elapsed_time(r1)
        skipped = float(dev.pcg_state[L.PCG["ROTZERO"]].item()) == 1.0
        lib.bdem_pcg_set_rot_skip(prev)
        scene.sync_to_host()
        same = all(np.array_equal(getattr(scene.elements, k), getattr(final["el"], k))
                   for k in ("p", "q", "v", "qdot"))
        rot = {"value": rt["newton_committed"] / (rot_ms * 1e-3), "unit": UNIT,
               "ms_per_step": rot_ms / args.steps, "newton_iterations": rt["newton"],
               "newton_committed": rt["newton_committed"],
               "pcg_per_newton": rt["pcg"] / max(rt["newton"], 1),
               "rotation_half_skipped": skipped, "bit_identical_final_state": bool(same),
               "note": "bdem_pcg_set_rot_skip(1): the rotation half of every Newton "
                       "system is exactly zero on this config, so the PCG kernels skip it "
                       "(exact; reported separately from the full 6-DOF headline)"}

    # headline work = Newton iterations of COMMITTED solves; the time also
    # covers the attempts that were split (their iterations are reported beside)
    (ms_max, e2e_ms_max), (newton_all, e2e_newton_all, newton_any) = reduce_across_ranks(
        [ms, e2e_ms], [tot["newton_committed"], e2e["newton_committed"], tot["newton"]],
        world, "cuda")
    if rot is not None and world > 1:
        (rot_ms_max,), (rot_newton_all, same_all) = reduce_across_ranks(
            [rot["ms_per_step"] * args.steps], [rot["newton_committed"],
                                                float(rot["bit_identical_final_state"])],
            world, "cuda")
        rot["value"] = rot_newton_all / (rot_ms_max * 1e-3)
        rot["bit_identical_final_state"] = bool(same_all == world)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peak, peak_kind = peaks()
    spmv = durations.get("spmv", [])
    basm = durations.get("bond_assemble", [])
    easm = durations.get("element_assemble", [])
    spmv_ms = statistics.mean(spmv) if spmv else float("nan")
    basm_ms = statistics.mean(basm) if basm else float("nan")
    easm_ms = statistics.mean(easm) if easm else float("nan")
    asm_ms = basm_ms + easm_ms
    sb = spmv_bytes(dev)
    ab = assembly_bytes(dev)
    achieved = sb / (spmv_ms * 1e-3) / 1e9
    traffic = load_ncu_traffic()
    value = newton_all / (ms_max * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, paper_2308_10459_b200/configs.py)",
        "config": config_block(args),
        "value_counts": "Newton iterations of committed solves only; the timed region also "
                        "contains the split attempts (all_attempts_newton_per_s counts them)",
        "newton_iterations": tot["newton"],
        "newton_committed": tot["newton_committed"],
        "newton_in_split_attempts": tot["newton_split_off"],
        "all_attempts_newton_per_s": newton_any / (ms_max * 1e-3),
        "attempts": tot["attempts"], "split_attempts": tot["failed_attempts"],
        "every_step_committed": True,
        "pcg_per_newton": tot["pcg"] / max(tot["newton"], 1),
        "ls_trials_per_newton": tot["ls"] / max(tot["newton"], 1),
        "per_step": per_step, "broken_bonds": tot["broken"],
        "bonds_per_sec_assembled": dev.nb / (asm_ms * 1e-3),
        "assembly": {"ms": asm_ms, "bond_kernel_ms": basm_ms, "element_kernel_ms": easm_ms,
                     "launches": len(basm), "bytes": ab,
                     "bytes_rule": "SURVEY 8(d): n_b (161 + 288) + n_f (136+144+144+48+56)",
                     "achieved_gbs": ab / (asm_ms * 1e-3) / 1e9,
                     "frac": ab / (asm_ms * 1e-3) / 1e9 / peak,
                     "traffic": _sum_or_none(traffic.get(k, {}).get("dram_bytes_per_launch")
                                             for k in ("k_bond_rows", "k_element_assemble")),
                     "fp64_pipe_frac": {k: traffic.get(k, {}).get("fp64_pipe_frac")
                                        for k in ("k_bond_rows", "k_element_assemble")},
                     "traffic_source": "ncu dram__bytes_read+write per launch "
                                       "(profiles/ncu_traffic.json)"},
        "spmv": {"ms": spmv_ms, "launches": len(spmv), "bytes": sb, "achieved_gbs": achieved,
                 "timing": "CUDA events around every SpMV launch in a replay of the timed steps "
                           "(the timed region itself runs uninstrumented)",
                 "replay_newton_iterations": replay["newton"]},
        "pcg_iteration": pcg_it,
        "roofline": {"kernel": "bdem::k_spmv (PCG SpMV)", "bound": "hbm", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "peak_source": peak_kind,
                     "traffic": traffic.get("k_spmv", {}).get("dram_bytes_per_launch"),
                     "l2": l2_roofline(traffic.get("k_spmv", {}), spmv_ms, clocks)},
        "e2e": {"value": e2e_newton_all / (e2e_ms_max * 1e-3) if n_e2e else None, "unit": UNIT,
                "same_steps_as_value": n_e2e == args.steps,
                "newton_committed": e2e["newton_committed"],
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": n_e2e,
                "note": "h2d/d2h bytes per stable_step call (a step split in halves makes "
                        "several calls)"},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    if rot is not None:
        line["rot_zero_shortcut"] = rot
    if not args.no_c5:
        line["c5_block"] = c5_leg(args.c5_side, peak)
    if not args.no_cpu_baseline and world == 1:
        cores = os.cpu_count() or 1
        # a fresh copy of the inputs: the scene above mutated spec's arrays
        mid = gpu_mid_iterate(configs.plate(nx=args.nx, ny=args.ny, epsilon=args.epsilon),
                              args.epsilon)
        kind, runs, setup = reference_newton(args.nx, args.ny, args.epsilon, 1, ["mid-solve"],
                                             [cores], mid)
        r = runs[0]
        line["cpu_baseline"] = {
            "value": r["newton_per_s"], "unit": UNIT, "cores": cores, "kind": kind,
            "sample": (f"reference bdem (oracle/_ref bytecode) on {cpu_model()}: "
                       f"{r['newton_iterations']} Newton iteration of minimize_second_order on "
                       f"this 600K plate's step-1 problem from the GPU mid-solve iterate "
                       f"(iteration {mid[2]['start_iteration']} of {mid[2]['gpu_step1_newton']}), "
                       f"workers={cores}: {r['seconds']:.1f}s, PCG {r['pcg_per_iteration']}"),
            "setup": setup}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
