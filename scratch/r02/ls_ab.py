"""Batched vs one-at-a-time line search on the 600K plate: the same steps
from the same start, CUDA-event time, Newton/LS counts, the distribution of
trials per Newton iteration, final-state identity."""
import collections, json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2308_10459_b200 import SolverConfig, configs, newton
from paper_2308_10459_b200.runner import advance
from paper_2308_10459_b200.scene import Scene

W, K = int(os.environ.get("W", 3)), int(os.environ.get("K", 8))
res = {}
finals = {}
modes = [("sequential", False, 1, 4), ("b1k4", True, 1, 4), ("b2k4", True, 2, 4),
         ("b1k2", True, 1, 2), ("b2k2", True, 2, 2), ("b2k3", True, 2, 3)]
for name, on, single, k in modes:
    newton.batched_line_search(on, single, k)
    scene = Scene.from_spec(configs.plate(epsilon=1e-3), host_sync=False)
    cfg = SolverConfig(epsilon=1e-3, max_iterations=300)
    for _ in range(W):
        advance(scene, cfg)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    newt = ls = 0
    hist = collections.Counter()
    a.record()
    for _ in range(K):
        att = []
        advance(scene, cfg, attempts=att)
        newt += sum(x.solve.iterations for x in att)
        for x in att:
            for r in x.solve.records:
                ls += r.ls_trials
                hist[r.ls_trials] += 1
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    scene.sync_to_host()
    finals[name] = (scene.elements.p.copy(), scene.elements.q.copy())
    res[name] = {"ms": ms, "newton": newt, "ls_trials": ls, "newton_per_s": newt / (ms * 1e-3),
                 "bit_identical": bool(np.array_equal(finals[name][0], finals["sequential"][0])
                                       and np.array_equal(finals[name][1], finals["sequential"][1]))}
    if name == "sequential":
        res["trials_hist"] = dict(sorted(hist.items()))
print(json.dumps(res))
