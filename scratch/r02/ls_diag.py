"""Diagnostic: GPU vs reference records on the random-q line-search cube."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from _fixtures import load
from paper_2308_10459_b200 import Scene, SolverConfig, configs as C, stable_step
f = load("failures.npz")
spec = C.cube(n_side=4, seed=2, random_q=True)
scene = Scene.from_spec(spec)
rep = stable_step(scene, SolverConfig(epsilon=1e-6, max_iterations=300))
print("gpu", rep.solve.reason, rep.solve.iterations)
for k, r in enumerate(rep.solve.records[:12]):
    ref = (f["ls_rec_f"][k], f["ls_rec_gnorm"][k], f["ls_rec_alpha"][k], f["ls_rec_pcg"][k]) if k < len(f["ls_rec_f"]) else None
    print(k, f"{r.f:.17e} {r.grad_norm:.17e} {r.alpha} {r.pcg_iterations}", "| ref", ref)
