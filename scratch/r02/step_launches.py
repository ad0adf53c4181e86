"""Kernel launches of stable_step only (NVTX range 'step'), for the launch
list: a scene with contact pairs across fragments, fracture and a driver."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2308_10459_b200 import SolverConfig, configs as C, stable_step
from paper_2308_10459_b200.scene import Scene

spec = C.cube(n_side=6, random_q=False, seed=3, youngs=3e8, k_contact=1e9, speed=2.0, dt=1e-4)
scene = Scene.from_spec(spec, host_sync=False)
cfg = SolverConfig(epsilon=1e-6, max_iterations=300)
for s in range(6):
    scene.colliders = spec.collider_schedule(scene.time + scene.dt)
    if s >= 3:
        torch.cuda.nvtx.range_push("step")
    rep = stable_step(scene, cfg)
    if s >= 3:
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    print(s, rep.committed, rep.solve.iterations, len(rep.broken), rep.contact_pairs, flush=True)
rope = Scene.from_spec(C.rope(n=200), host_sync=False)
rope.device  # build the device system outside the measured range
for s in range(3):
    torch.cuda.nvtx.range_push("step")
    rep = stable_step(rope, SolverConfig(epsilon=1e-5, max_iterations=300))
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print("rope", s, rep.committed, rep.solve.iterations, flush=True)
