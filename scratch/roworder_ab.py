"""Plate 600K: SpMV / assembly / element kernel times with BDEM_ROW_ORDER=z vs id."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2308_10459_b200 import configs
from paper_2308_10459_b200.scene import Scene
from paper_2308_10459_b200.newton import GPUProblem
from paper_2308_10459_b200.step import contact_candidates

def ev(): return torch.cuda.Event(enable_timing=True)
def timeit(fn, reps=30):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a, b = ev(), ev(); a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / reps * 1e3

mode = sys.argv[1] if len(sys.argv) > 1 else "z"
os.environ["BDEM_ROW_ORDER"] = mode
spec = configs.plate(epsilon=1e-3)
scene = Scene.from_spec(spec, host_sync=False)
dev = scene.device
dev.set_physics(scene.gravity, scene.k_contact, scene.k_element, scene.colliders)
dev.set_pairs(contact_candidates(scene))
dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(),
         dev.qdot.data_ptr(), dev.p_prev.data_ptr(), dev.q_prev.data_ptr(), spec.dt,
         dev.p_hat.data_ptr(), dev.q_hat.data_ptr(), dev.mp_dt2.data_ptr(), dev.mq_dt2.data_ptr(),
         dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream)
prob = GPUProblem(dev)
prob.assemble(dev.xp, dev.xq)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(6 * dev.vstride, generator=g, dtype=torch.float64, device="cuda"); y = torch.zeros_like(x)
res = {"mode": mode, "n_pos/nb": dev.sell.n_pos / dev.nb, "kmax": dev.sell.kmax}
res["spmv_us"] = timeit(lambda: dev.call("bdem_spmv", dev.sysp, x.data_ptr(), y.data_ptr(), dev.stream))
res["bond_asm_us"] = timeit(lambda: dev.call("bdem_bond_assemble", dev.sysp, dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream), 10)
res["elem_asm_us"] = timeit(lambda: dev.call("bdem_element_assemble", dev.sysp, dev.xp.data_ptr(), dev.xq.data_ptr(), dev.z.data_ptr(), dev.stream), 10)
# x.Ax (row-order independent up to round-off) as a sanity value
dev.call("bdem_spmv", dev.sysp, x.data_ptr(), y.data_ptr(), dev.stream)
res["xAx"] = float(torch.dot(x, y))
print(json.dumps(res))
