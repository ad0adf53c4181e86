import os, sys, json, collections
sys.path.insert(0, os.getcwd())
from paper_2308_10459_b200 import SolverConfig, configs, stable_step
from paper_2308_10459_b200.scene import Scene
spec = configs.plate(epsilon=1e-3)
scene = Scene.from_spec(spec, host_sync=False)
cfg = SolverConfig(epsilon=1e-3, max_iterations=300)
hist = collections.Counter(); pcg = collections.defaultdict(list)
for s in range(13):
    rep = stable_step(scene, cfg)
    if s >= 3:
        for r in rep.solve.records:
            hist[r.ls_trials] += 1
            pcg[r.ls_trials].append(r.pcg_iterations)
print(json.dumps({"ls_trials_hist": dict(sorted(hist.items())),
                  "mean_pcg_by_trials": {k: sum(v) / len(v) for k, v in sorted(pcg.items())}}))
