"""A/B bit-identity: K steps of the plate (NX x NY) through stable_step; the
final element state and per-step counts go to OUT (npz).  Run once per tree."""
import os, sys, hashlib
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2308_10459_b200 import configs, SolverConfig, stable_step
from paper_2308_10459_b200.scene import Scene

nx, ny, K = int(os.environ.get("NX", 200)), int(os.environ.get("NY", 120)), int(os.environ.get("K", 4))
spec = configs.plate(nx=nx, ny=ny)
scene = Scene.from_spec(spec)
cfg = SolverConfig(epsilon=float(os.environ.get("EPS", 1e-3)), max_iterations=300)
counts = []
for _ in range(K):
    r = stable_step(scene, cfg)
    counts.append((r.solve.iterations, r.solve.pcg_total, int(r.committed)))
p, q = scene.elements.p, scene.elements.q
h = hashlib.sha256(p.tobytes() + q.tobytes()).hexdigest()[:16]
print("counts", counts, "hash", h)
np.save(os.environ["OUT"], np.concatenate([p.ravel(), q.ravel()]))   # scratch, compared on the box
