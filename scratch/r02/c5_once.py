"""One assembly (bond rows + eigen-clamp + element) of the C5 2M block, random q,
at its step-1 predictor (ncu target for the FP64 counters)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2308_10459_b200 import configs
from paper_2308_10459_b200.newton import GPUProblem
from paper_2308_10459_b200.scene import Scene

spec = configs.block(n_side=int(os.environ.get("SIDE", 126)), random_q=True)
scene = Scene.from_spec(spec, host_sync=False)
dev = scene.device
dev.set_physics(spec.gravity, spec.k_contact, 0.0, [])
dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(),
         dev.qdot.data_ptr(), dev.p_prev.data_ptr(), dev.q_prev.data_ptr(), spec.dt,
         dev.p_hat.data_ptr(), dev.q_hat.data_ptr(), dev.mp_dt2.data_ptr(),
         dev.mq_dt2.data_ptr(), dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream)
prob = GPUProblem(dev)
for _ in range(2):
    prob.assemble(dev.xp, dev.xq)
torch.cuda.synchronize()
print("ok queued", int(dev.counter[5]), "bonds", dev.nb)
