"""Phase breakdown (clock64, thread 0 of every CTA) of the tiled SpMV."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2308_10459_b200 import configs
from paper_2308_10459_b200.scene import Scene
from paper_2308_10459_b200.newton import GPUProblem
from paper_2308_10459_b200.step import contact_candidates
spec = configs.plate(epsilon=1e-3)
scene = Scene.from_spec(spec, host_sync=False)
dev = scene.device
dev.set_physics(scene.gravity, scene.k_contact, scene.k_element, scene.colliders)
dev.set_pairs(contact_candidates(scene))
dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(),
         dev.qdot.data_ptr(), dev.p_prev.data_ptr(), dev.q_prev.data_ptr(), spec.dt,
         dev.p_hat.data_ptr(), dev.q_hat.data_ptr(), dev.mp_dt2.data_ptr(), dev.mq_dt2.data_ptr(),
         dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream)
GPUProblem(dev).assemble(dev.xp, dev.xq)
x = torch.randn(6 * dev.vstride, dtype=torch.float64, device="cuda"); y = torch.zeros_like(x)
out = (ctypes.c_ulonglong * 8)()
for _ in range(3): dev.call("bdem_spmv", dev.sysp, x.data_ptr(), y.data_ptr(), dev.stream)
torch.cuda.synchronize(); dev.lib.bdem_tile_prof(out)
R = 20
for _ in range(R): dev.call("bdem_spmv", dev.sysp, x.data_ptr(), y.data_ptr(), dev.stream)
torch.cuda.synchronize(); dev.lib.bdem_tile_prof(out)
names = ["wait", "slots", "sync1", "tail", "sync2", "issue"]
tot = sum(out[k] for k in range(6))
print({n: f"{out[k] / tot:.3f}" for k, n in enumerate(names)}, "cycles/launch/CTA-sum", tot / R)
