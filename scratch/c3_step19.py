"""C3 plate: commit steps 0..17, then inspect the Newton records of step 18 (0-based)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2308_10459_b200 import SolverConfig, configs, stable_step
from paper_2308_10459_b200.scene import Scene
spec = configs.plate(epsilon=1e-3)
scene = Scene.from_spec(spec, host_sync=False)
cfg = SolverConfig(epsilon=1e-3, max_iterations=300)
for s in range(18):
    rep = stable_step(scene, cfg)
    r = rep.solve
    print(s, rep.committed, r.iterations, r.pcg_total, rep.contact_pairs, f"gn {r.grad_norm:.2e}", {k: f"{v:.3e}" for k, v in rep.energies.items()}, flush=True)
dev = scene.device
pz = dev.p[:, 2]
print("z min/max", float(pz.min()), float(pz.max()), "inside floor", int((pz < 0).sum()))
rep = stable_step(scene, cfg)
r = rep.solve
g = [x.grad_norm for x in r.records]
f = [x.f for x in r.records]
ls = [x.ls_trials for x in r.records]
print("step 18", rep.committed, r.reason, r.iterations, r.pcg_total)
print("gnorm first", [f"{v:.3e}" for v in g[:8]])
print("gnorm last", [f"{v:.3e}" for v in g[-8:]], "min", f"{min(g):.3e}")
print("f last", [f"{v:.10e}" for v in f[-6:]])
print("ls trials", ls[:10], ls[-10:])
print("pcg per it", [x.pcg_iterations for x in r.records][-10:] if hasattr(r.records[0], "pcg_iterations") else "")
