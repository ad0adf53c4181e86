import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2308_10459_b200 import configs, SolverConfig, stable_step
from paper_2308_10459_b200.scene import Scene
spec = configs.plate()
scene = Scene.from_spec(spec, host_sync=True)
cfg = SolverConfig(epsilon=1e-3, max_iterations=300)
dev = scene.device
def t(f, n=3):
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / n * 1e3
print("upload_elements ms", t(lambda: dev.upload_elements(scene.elements, scene.p_prev, scene.q_prev)))
print("upload_bond_state ms", t(lambda: dev.upload_bond_state(scene.bonds)))
print("download_state ms", t(lambda: dev.download_state(scene)))
for hs in (True, False):
    scene.host_sync = hs
    for k in range(2):
        torch.cuda.synchronize(); a = time.perf_counter()
        rep = stable_step(scene, cfg)
        torch.cuda.synchronize(); b = time.perf_counter()
        print("host_sync", hs, "step ms %.1f newton %d pcg %d" % ((b - a) * 1e3, rep.solve.iterations, rep.solve.pcg_total))
