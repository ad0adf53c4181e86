"""Per-PCG-iteration time on the 600K plate (one assembled system), CUDA events
around chunks of bdem_pcg_iterate; env BDEM_FUSED_UPD / BDEM_PDL select paths."""
import os, sys, json
sys.path.insert(0, os.getcwd())
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
prob = GPUProblem(dev)
prob.assemble(dev.xp, dev.xq)
ptrs = (dev.y.data_ptr(), dev.r.data_ptr(), dev.zv.data_ptr(), dev.pv.data_ptr())
res = {}
for chunk in (8, 32):
    ts = []
    for rep in range(4):
        dev.call("bdem_pcg_init", dev.sysp, dev.z.data_ptr(), -1.0, *ptrs, 1e-30, 100000, 0.0, dev.stream)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        dev.call("bdem_pcg_iterate", dev.sysp, *ptrs, dev.ap.data_ptr(), chunk, dev.stream)
        b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / chunk)
    res[f"pcg_iter_us_chunk{chunk}"] = min(ts)
h = dev.pcg_state.cpu().numpy()
res["k"] = float(h[11]); res["state"] = float(h[13]); res["rel"] = float(h[6])
res["y_sum"] = float(dev.y.abs().sum())
res["env"] = {k: os.environ.get(k) for k in ("BDEM_FUSED_UPD", "BDEM_PDL")}
print(json.dumps(res))
