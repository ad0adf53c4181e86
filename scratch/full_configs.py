"""Every BASELINE config at full size and full step count through the GPU path
(stable_step, device-resident): committed steps, Newton/PCG counts, fracture
events, wall time, finiteness.  Writes one JSON per config to argv[1]."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2308_10459_b200 import SolverConfig, configs, stable_step
from paper_2308_10459_b200.scene import Scene

which = sys.argv[2:] or ["C1", "C2", "C3", "C4", "C5"]
out = {}
for name in which:
    spec = {"C1": lambda: configs.cantilever(), "C2": lambda: configs.cube(),
            "C3": lambda: configs.plate(epsilon=1e-3), "C4": lambda: configs.rope(),
            "C5": lambda: configs.block()}[name]()
    t0 = time.time()
    scene = Scene.from_spec(spec, host_sync=False)
    cfg = SolverConfig(epsilon=spec.epsilon, max_iterations=300)
    sched = spec.collider_schedule
    rec = {"spheres": int(spec.elements.n), "bonds": int(spec.bonds.n), "steps": spec.steps,
           "epsilon": spec.epsilon, "dt": spec.dt, "setup_s": time.time() - t0}
    torch.cuda.synchronize()
    t1 = time.time()
    newton = pcg = broken = committed = 0
    reasons = {}
    per_step = []
    for s in range(spec.steps):
        if sched is not None:
            scene.colliders = sched(scene.time + scene.dt)
        rep = stable_step(scene, cfg)
        newton += rep.solve.iterations
        pcg += rep.solve.pcg_total
        broken += len(rep.broken)
        committed += int(rep.committed)
        reasons[rep.solve.reason] = reasons.get(rep.solve.reason, 0) + 1
        per_step.append([rep.solve.iterations, rep.solve.pcg_total, len(rep.broken),
                         int(rep.committed)])
    torch.cuda.synchronize()
    wall = time.time() - t1
    dev = scene.device
    finite = bool(torch.isfinite(dev.p).all() and torch.isfinite(dev.q).all())
    rec.update({"committed_steps": committed, "newton_iterations": newton, "pcg_iterations": pcg,
                "broken_bonds": broken, "reasons": reasons, "wall_s": wall,
                "newton_per_s": newton / wall, "finite": finite, "per_step": per_step,
                "max_q_norm_dev": float((torch.linalg.vector_norm(dev.q, dim=1) - 1).abs().max())})
    out[name] = rec
    print(name, {k: v for k, v in rec.items() if k != "per_step"}, flush=True)
    del scene, dev
    torch.cuda.empty_cache()
json.dump(out, open(sys.argv[1], "w"), indent=1)
