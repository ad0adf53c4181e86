"""Full C3 plate through run_simulation (dt-halving retries, runner.py:47-71),
one step per frame: does the contact onset at step ~19 pass?"""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2308_10459_b200 import SolverConfig, configs
from paper_2308_10459_b200.runner import StepFailure, run_simulation
from paper_2308_10459_b200.scene import Scene
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 40
spec = configs.plate(epsilon=1e-3)
scene = Scene.from_spec(spec, host_sync=False)
cfg = SolverConfig(epsilon=1e-3, max_iterations=300)
t0 = time.time()
try:
    stats = run_simulation(scene, cfg, frames=frames, fps=1.0 / spec.dt, write_meshes=False)
    ok = True
except StepFailure as exc:
    print("StepFailure", exc, flush=True)
    ok = False
    stats = None
wall = time.time() - t0
rows = stats.rows if stats else []
res = {"frames": frames, "completed": ok, "wall_s": wall, "sim_time": scene.time,
       "newton": sum(r["newton_iterations"] for r in rows), "pcg": sum(r["pcg_iterations"] for r in rows),
       "broken": sum(r["bonds_broken"] for r in rows),
       "rows": [[r["frame"], r["newton_iterations"], r["pcg_iterations"], r["grad_norm"]] for r in rows]}
print(json.dumps({k: v for k, v in res.items() if k != "rows"}))
print([r[1] for r in res["rows"]])
json.dump(res, open(sys.argv[1], "w"), indent=1)
