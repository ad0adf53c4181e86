"""C5 scale block: time the fused bond kernel (random q: every rotation block
indefinite -> Jacobi eigen-clamp) and the SpMV at 2M spheres / ~12M bonds."""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2308_10459_b200 import configs
from paper_2308_10459_b200.scene import Scene
from paper_2308_10459_b200.newton import GPUProblem
t0 = time.time()
m = int(os.environ.get("NSIDE", 126))
spec = configs.block(n_side=m, random_q=os.environ.get("RANDQ", "1") == "1")
t1 = time.time()
scene = Scene.from_spec(spec, host_sync=False)
dev = scene.device
dev.set_physics(spec.gravity, spec.k_contact, 0.0, [])
dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(),
         dev.qdot.data_ptr(), dev.p_prev.data_ptr(), dev.q_prev.data_ptr(), spec.dt,
         dev.p_hat.data_ptr(), dev.q_hat.data_ptr(), dev.mp_dt2.data_ptr(), dev.mq_dt2.data_ptr(),
         dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream)
torch.cuda.synchronize(); t2 = time.time()
prob = GPUProblem(dev)
f, g, c, _ = prob.assemble(dev.xp, dev.xq)
res = {"n": dev.n, "n_bond": dev.nb, "gen_s": t1 - t0, "upload_s": t2 - t1, "f": f, "gnorm": g}
def timeit(name, fn, reps=5):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    res[name] = a.elapsed_time(b) / reps * 1e3
timeit("bond_assemble_us", lambda: dev.call("bdem_bond_assemble", dev.sysp, dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream))
timeit("element_assemble_us", lambda: dev.call("bdem_element_assemble", dev.sysp, dev.xp.data_ptr(), dev.xq.data_ptr(), dev.z.data_ptr(), dev.stream))
x = torch.randn(6 * dev.vstride, dtype=torch.float64, device="cuda")
y = torch.zeros_like(x)
timeit("spmv_us", lambda: dev.call("bdem_spmv", dev.sysp, x.data_ptr(), y.data_ptr(), dev.stream), 20)
timeit("bond_energy_us", lambda: dev.call("bdem_bond_energy", dev.sysp, dev.xp.data_ptr(), dev.xq.data_ptr(), 7, dev.stream))
res["bonds_per_s"] = dev.nb / (res["bond_assemble_us"] * 1e-6)
res["mem_gb"] = torch.cuda.max_memory_allocated() / 1e9
print(json.dumps(res))
