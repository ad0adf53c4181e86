"""Per-PCG-iteration cost on mid-size systems (C4 rope 100K, C2 cube 22^3
identity q): whole steps, and bdem_pcg_iterate chunks (CUDA events)."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2308_10459_b200 import SolverConfig, configs as C, stable_step
from paper_2308_10459_b200.scene import Scene
res = {}
for name, spec, eps in (("rope100k", C.rope(), 1e-5), ("cube22", C.cube(random_q=False), 1e-6)):
    scene = Scene.from_spec(spec, host_sync=False)
    cfg = SolverConfig(epsilon=eps, max_iterations=300)
    sched = getattr(spec, "collider_schedule", None)
    def step():
        if sched is not None:
            scene.colliders = sched(scene.time + scene.dt)
        return stable_step(scene, cfg)
    step()
    torch.cuda.synchronize()
    t = time.perf_counter()
    newton = pcg = 0
    for _ in range(3):
        r = step()
        newton += r.solve.iterations; pcg += r.solve.pcg_total
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
    dev = scene.device
    ptrs = (dev.y.data_ptr(), dev.r.data_ptr(), dev.zv.data_ptr(), dev.pv.data_ptr())
    best = 1e9
    for _ in range(3):
        dev.call("bdem_pcg_init", dev.sysp, dev.z.data_ptr(), -1.0, *ptrs, 1e-30, 100000, 0.0, dev.stream)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        dev.call("bdem_pcg_iterate", dev.sysp, *ptrs, dev.ap.data_ptr(), 32, dev.stream)
        b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / 32)
    res[name] = {"n": dev.n, "nb": dev.nb, "wall_s_3steps": wall, "newton": newton, "pcg": pcg,
                 "us_per_pcg_in_steps_upper": wall * 1e6 / max(pcg, 1), "pcg_chunk_us": best}
print(json.dumps(res, indent=1))
