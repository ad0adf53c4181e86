"""Dump assembly + SpMV outputs of the golden cube's first predicted state."""
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from _fixtures import load, elements_from, bonds_from
from paper_2308_10459_b200 import configs as C
from paper_2308_10459_b200.scene import Scene
from paper_2308_10459_b200.newton import GPUProblem
from paper_2308_10459_b200.step import contact_candidates
d = load("traj_cube.npz")
spec = C.cube(n_side=5, random_q=False, seed=3, youngs=3e8, k_contact=1e9, speed=2.0, dt=1e-4)
el = elements_from(d, "init_el_"); b = bonds_from(d, "init_b_")
scene = Scene("cube", None, el, b, colliders=spec.collider_schedule(spec.dt), gravity=d["gravity"], dt=float(d["dt"]),
              youngs=float(d["youngs"]), k_contact=float(d["k_contact"]), k_element=float(d["k_element"]), host_sync=False)
dev = scene.device
dev.set_physics(scene.gravity, scene.k_contact, scene.k_element, scene.colliders)
dev.set_pairs(contact_candidates(scene))
dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(), dev.qdot.data_ptr(),
         dev.p_prev.data_ptr(), dev.q_prev.data_ptr(), scene.dt, dev.p_hat.data_ptr(), dev.q_hat.data_ptr(),
         dev.mp_dt2.data_ptr(), dev.mq_dt2.data_ptr(), dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream)
prob = GPUProblem(dev)
f, gnorm, cnorm, _ = prob.assemble(dev.xp, dev.xq)
vs, nf = dev.vstride, dev.nf
cols = np.asarray(dev.slot_np[dev.free_ids_np], dtype=np.int64)
z = dev.z.view(6, vs)[:, cols].cpu().numpy()
diag = dev.diag[:, cols].cpu().numpy()
g = torch.Generator(device="cuda").manual_seed(3)
xa = torch.randn(6, nf, generator=g, dtype=torch.float64, device="cuda")
x = torch.zeros(6, vs, dtype=torch.float64, device="cuda"); x[:, torch.as_tensor(cols, device="cuda")] = xa
y = torch.zeros_like(x)
dev.call("bdem_spmv", dev.sysp, x.data_ptr(), y.data_ptr(), dev.stream)
torch.cuda.synchronize()
y = y[:, torch.as_tensor(cols, device="cuda")].cpu().numpy()
np.savez(sys.argv[1], f=f, gnorm=gnorm, z=z, diag=diag, y=y, npairs=dev.n_pair)
print(sys.argv[1], f, gnorm, dev.n_pair)
