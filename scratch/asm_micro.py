"""Time the assembly kernels on the 600K plate predictor state (and a perturbed state)."""
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
KC = int(os.environ.get("KC", "5"))
res = {}
def timeit(name, fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    res[name] = a.elapsed_time(b) / reps * 1e3
xq_rest = dev.xq.clone()
for tag, pert in (("rest", 0.0), ("pert", float(os.environ.get("PERT", "1e-3")))):
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    dev.xq.copy_(xq_rest + pert * torch.randn(xq_rest.shape, generator=g, device="cuda", dtype=torch.float64))
    dev.xq.div_(dev.xq.norm(dim=1, keepdim=True))
    timeit(f"bond_assemble_{tag}_us", lambda: dev.call("bdem_bond_assemble", dev.sysp, dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream))
    torch.cuda.synchronize()
    res[f"clamp_queue_{tag}"] = int(dev.counter[KC].item())
    st = dev.stage.double() if hasattr(dev, "stage") else None
    if st is not None:
        res[f"stage_sum_{tag}"] = float(st.abs().sum())
        res[f"scoef_sum_{tag}"] = float(dev.scoef.abs().sum())
res["lib"] = os.environ.get("BDEM_LIB", "default")
res["n_bond"] = int(dev.nb) if hasattr(dev, "nb") else None
print(json.dumps(res))
