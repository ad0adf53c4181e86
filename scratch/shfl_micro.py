"""SpMV variant 4 (warp-shuffle hand-over) vs the default on the 600K plate:
time of bdem_spmv and of one PCG iteration, and agreement of y."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2308_10459_b200 import configs
from paper_2308_10459_b200.scene import Scene
from paper_2308_10459_b200.newton import GPUProblem
from paper_2308_10459_b200.step import contact_candidates

spec = configs.plate(nx=int(os.environ.get("NX", 1000)), ny=int(os.environ.get("NY", 600)))
scene = Scene.from_spec(spec, host_sync=False)
dev = scene.device
dev.set_pairs(contact_candidates(scene))
dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(),
         dev.qdot.data_ptr(), dev.p_prev.data_ptr(), dev.q_prev.data_ptr(), spec.dt,
         dev.p_hat.data_ptr(), dev.q_hat.data_ptr(), dev.mp_dt2.data_ptr(), dev.mq_dt2.data_ptr(),
         dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream)
GPUProblem(dev).assemble(dev.xp, dev.xq)
g = torch.Generator(device="cuda").manual_seed(3)
x = torch.randn(6 * dev.vstride, generator=g, dtype=torch.float64, device="cuda")
res = {"row_order": os.environ.get("BDEM_ROW_ORDER", "id"), "handed": dev.shfl_handed,
       "lib": os.environ.get("BDEM_LIB", "default")}
ptrs = (dev.y.data_ptr(), dev.r.data_ptr(), dev.zv.data_ptr(), dev.pv.data_ptr())

def tm(fn, reps):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps

ys = {}
for kern in (0, 4):
    dev.lib.bdem_spmv_set_kernel(kern)
    y = torch.zeros_like(x)
    res[f"spmv_us_k{kern}"] = tm(lambda: dev.call("bdem_spmv", dev.sysp, x.data_ptr(), y.data_ptr(), dev.stream), 50)
    ys[kern] = y.clone()
    ts = []
    for rep in range(3):
        dev.call("bdem_pcg_init", dev.sysp, dev.z.data_ptr(), -1.0, *ptrs, 1e-30, 100000, 0.0, dev.stream)
        ts.append(tm(lambda: dev.call("bdem_pcg_iterate", dev.sysp, *ptrs, dev.ap.data_ptr(), 8, dev.stream), 4) / 8)
    res[f"pcg_iter_us_k{kern}"] = min(ts)
d = (ys[4] - ys[0]).abs().max().item() / ys[0].abs().max().item()
res["rel_diff"] = d
print(json.dumps(res))
