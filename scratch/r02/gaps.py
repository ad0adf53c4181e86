"""GPU idle gaps inside stable_step on the 600K plate: torch.profiler (CUPTI)
kernel timeline of 2 committed steps after warm-up; gaps between consecutive
kernels classified by the kernel that follows (host round trips show up as
gaps before the first kernel of each enqueued batch)."""
import collections, json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2308_10459_b200 import SolverConfig, configs
from paper_2308_10459_b200.runner import advance
from paper_2308_10459_b200.scene import Scene

scene = Scene.from_spec(configs.plate(epsilon=1e-3), host_sync=False)
cfg = SolverConfig(epsilon=1e-3, max_iterations=300)
for _ in range(3):
    advance(scene, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    att = []
    for _ in range(2):
        advance(scene, cfg, attempts=att)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev], key=lambda x: x[0])
busy = sum(b - a for a, b, _ in kern)
span = kern[-1][1] - kern[0][0]
gaps = collections.defaultdict(lambda: [0, 0.0])
hist = collections.Counter()
for (a0, b0, n0), (a1, b1, n1) in zip(kern, kern[1:]):
    g = a1 - b0
    if g <= 0:
        continue
    key = (n0.split("(")[0].replace("bdem::", "")[:30], n1.split("(")[0].replace("bdem::", "")[:30])
    gaps[key][0] += 1
    gaps[key][1] += g
    hist[min(int(g // 5) * 5, 200)] += 1
newton = sum(x.solve.iterations for x in att)
out = {"kernels": len(kern), "busy_us": busy, "span_us": span, "idle_us": span - busy,
       "newton": newton, "idle_per_newton_us": (span - busy) / max(newton, 1),
       "top_gaps": sorted(([k[0], k[1], v[0], round(v[1], 1)] for k, v in gaps.items()),
                          key=lambda x: -x[3])[:25],
       "gap_hist_5us": dict(sorted(hist.items()))}
print(json.dumps(out, indent=1))
