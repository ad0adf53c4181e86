"""Every BASELINE config at full size and full step count on the round-2
library, advanced like the reference's runner (runner.advance: a step whose
solve does not commit is split in halves, 2 levels); a step that fails at
dt/4 ends that config's run (StepFailure), as in run_simulation.  One JSON
per config to argv[1]; a wall-clock guard per config (argv[2] seconds)."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2308_10459_b200 import SolverConfig, configs
from paper_2308_10459_b200.runner import StepFailure, advance
from paper_2308_10459_b200.scene import Scene
from paper_2308_10459_b200.state import DegenerateBondError, DegenerateShearError

guard = float(sys.argv[2]) if len(sys.argv) > 2 else 1200.0
which = sys.argv[3:] or ["C1", "C2", "C3", "C4", "C5"]
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
    newton = pcg = broken = committed = attempts_n = splits = 0
    stop = None
    per_step = []
    for s in range(spec.steps):
        if time.time() - t1 > guard:
            stop = f"wall-clock guard after {s} steps"
            break
        if sched is not None:
            scene.colliders = sched(scene.time + scene.dt)
        att = []
        try:
            done = advance(scene, cfg, attempts=att)
        except StepFailure as exc:
            stop = f"StepFailure at step {s}: {exc}"
            newton += sum(a.solve.iterations for a in att)
            pcg += sum(a.solve.pcg_total for a in att)
            break
        except (DegenerateBondError, DegenerateShearError) as exc:
            # the reference does not catch these either: a degenerate bond or an
            # antipodal pair at a line-search trial point ends the run
            stop = f"{type(exc).__name__} at step {s}: {exc}"
            newton += sum(a.solve.iterations for a in att)
            pcg += sum(a.solve.pcg_total for a in att)
            break
        newton += sum(a.solve.iterations for a in att)
        pcg += sum(a.solve.pcg_total for a in att)
        broken += sum(len(c.broken) for c in done)
        committed += 1
        attempts_n += len(att)
        splits += sum(1 for a in att if not a.committed)
        per_step.append([sum(a.solve.iterations for a in att), sum(a.solve.pcg_total for a in att),
                         len(att), sum(len(c.broken) for c in done)])
    torch.cuda.synchronize()
    wall = time.time() - t1
    dev = scene.device
    rec.update({"committed_steps": committed, "newton_iterations": newton, "pcg_iterations": pcg,
                "split_attempts": splits, "broken_bonds": broken, "stopped": stop,
                "wall_s": wall, "newton_per_s": newton / max(wall, 1e-9),
                "finite": bool(torch.isfinite(dev.p).all() and torch.isfinite(dev.q).all()),
                "sim_time": scene.time, "per_step": per_step})
    out[name] = rec
    print(name, {k: v for k, v in rec.items() if k != "per_step"}, flush=True)
    json.dump(out, open(sys.argv[1], "w"), indent=1)
    del scene, dev
    torch.cuda.empty_cache()
