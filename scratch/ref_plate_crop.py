"""Reference (pure Python bdem) stable_step on an nx x ny crop of the C3 plate:
per-step committed / Newton iterations / reason, to compare with the GPU path
on the same crop around the contact onset."""
import os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests", "golden"))
sys.path.insert(0, "/root/reference/pkg/src"); sys.dont_write_bytecode = True
import numpy as np
nx, ny, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
which = sys.argv[4]
from paper_2308_10459_b200 import configs as C
spec = C.plate(nx=nx, ny=ny, epsilon=1e-3)
t0 = time.time()
if which == "ref":
    import make_golden as MG
    from bdem import solver as rsv
    sc = MG.ref_scene(spec)
    cfg = rsv.SolverConfig(epsilon=1e-3, max_iterations=300)
    for s in range(steps):
        rep = rsv.stable_step(sc, cfg)
        print(s, rep.committed, rep.solve.iterations, rep.solve.pcg_total, rep.solve.reason,
              f"{rep.solve.grad_norm:.2e}", f"zmin {sc.elements.p[:,2].min():.3e}", f"{time.time()-t0:.0f}s", flush=True)
else:
    from paper_2308_10459_b200 import Scene, SolverConfig, stable_step
    sc = Scene.from_spec(spec)
    cfg = SolverConfig(epsilon=1e-3, max_iterations=300)
    for s in range(steps):
        rep = stable_step(sc, cfg)
        print(s, rep.committed, rep.solve.iterations, rep.solve.pcg_total, rep.solve.reason,
              f"{rep.solve.grad_norm:.2e}", f"zmin {sc.elements.p[:,2].min():.3e}", f"{time.time()-t0:.0f}s", flush=True)
