"""Time the PCG SpMV / update kernels on the 600K plate (one assembled system)."""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import torch
from paper_2308_10459_b200 import configs, SolverConfig
from paper_2308_10459_b200.scene import Scene
from paper_2308_10459_b200.newton import GPUProblem
from paper_2308_10459_b200.step import contact_candidates
from paper_2308_10459_b200 import _lib as L

spec = configs.plate(nx=int(os.environ.get("NX", 1000)), ny=int(os.environ.get("NY", 600)))
scene = Scene.from_spec(spec, host_sync=False)
dev = scene.device
dev.set_pairs(contact_candidates(scene))
dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(),
         dev.qdot.data_ptr(), dev.p_prev.data_ptr(), dev.q_prev.data_ptr(), spec.dt,
         dev.p_hat.data_ptr(), dev.q_hat.data_ptr(), dev.mp_dt2.data_ptr(), dev.mq_dt2.data_ptr(),
         dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream)
prob = GPUProblem(dev)
f, g, c, _ = prob.assemble(dev.xp, dev.xq)
x = torch.randn(6 * dev.nf, dtype=torch.float64, device="cuda")
y = torch.zeros_like(x)
res = {}
def timeit(name, fn, reps=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    res[name] = a.elapsed_time(b) / reps * 1e3
timeit("spmv_us", lambda: dev.call("bdem_spmv", dev.sysp, x.data_ptr(), y.data_ptr(), dev.stream))
ref = y.clone()
# PCG pieces
ptrs = (dev.y.data_ptr(), dev.r.data_ptr(), dev.zv.data_ptr(), dev.pv.data_ptr())
dev.call("bdem_pcg_init", dev.sysp, dev.z.data_ptr(), -1.0, *ptrs, 1e-30, 100000, 0.0, dev.stream)
timeit("pcg_spmv_us", lambda: dev.call("bdem_pcg_spmv", dev.sysp, ptrs[3], dev.ap.data_ptr(), dev.stream))
timeit("pcg_update_us", lambda: dev.call("bdem_pcg_update", dev.sysp, *ptrs, dev.ap.data_ptr(), dev.stream))
timeit("pcg_iter_us", lambda: dev.call("bdem_pcg_iterate", dev.sysp, *ptrs, dev.ap.data_ptr(), 1, dev.stream))
timeit("bond_assemble_us", lambda: dev.call("bdem_bond_assemble", dev.sysp, dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream), 10)
timeit("element_assemble_us", lambda: dev.call("bdem_element_assemble", dev.sysp, dev.xp.data_ptr(), dev.xq.data_ptr(), dev.z.data_ptr(), dev.stream), 10)
timeit("bond_energy_us", lambda: dev.call("bdem_bond_energy", dev.sysp, dev.xp.data_ptr(), dev.xq.data_ptr(), 7, dev.stream), 10)
res["lib"] = os.environ.get("BDEM_LIB", "default")
res["y_checksum"] = float(ref.abs().sum())
print(json.dumps(res))
