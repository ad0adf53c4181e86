"""PCG kernel timeline on the 600K plate (diagnostic library built with
-DBDEM_TIMELINE=1, passed as BDEM_LIB): per iteration, each kernel's first-CTA
arrival, release from griddepcontrol.wait and last-CTA exit (globaltimer)."""
import os, sys, json, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2308_10459_b200 import configs
from paper_2308_10459_b200.scene import Scene
from paper_2308_10459_b200.newton import GPUProblem
from paper_2308_10459_b200.step import contact_candidates
spec = configs.plate()
scene = Scene.from_spec(spec, host_sync=False)
dev = scene.device
dev.set_pairs(contact_candidates(scene))
dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(),
         dev.qdot.data_ptr(), dev.p_prev.data_ptr(), dev.q_prev.data_ptr(), spec.dt,
         dev.p_hat.data_ptr(), dev.q_hat.data_ptr(), dev.mp_dt2.data_ptr(), dev.mq_dt2.data_ptr(),
         dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream)
GPUProblem(dev).assemble(dev.xp, dev.xq)
lib = dev.lib
ptrs = (dev.y.data_ptr(), dev.r.data_ptr(), dev.zv.data_ptr(), dev.pv.data_ptr())
for rep in range(2):
    dev.call("bdem_pcg_init", dev.sysp, dev.z.data_ptr(), -1.0, *ptrs, 1e-30, 100000, 0.0, dev.stream)
    torch.cuda.synchronize()
    lib.bdem_timeline_reset()
    dev.call("bdem_pcg_iterate", dev.sysp, *ptrs, dev.ap.data_ptr(), 40, dev.stream)
    torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (3 * 1024 * 3))()
lib.bdem_timeline_read(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(3, 1024, 3).astype(np.float64)
# kernel order per iteration: spmv(K=k), update(K=k), pupdate(K=k+1)
rows = []
for k in range(5, 35):
    sp = a[0, k]; up = a[1, k]; pu = a[2, k + 1]
    nsp = a[0, k + 1]
    rows.append([sp[2] - sp[1], up[2] - up[1], pu[2] - pu[1],      # busy spans (release -> exit)
                 up[1] - sp[2], pu[1] - up[2], nsp[1] - pu[2],      # gaps: exit -> next release
                 nsp[1] - sp[1]])                                   # iteration period
r = np.array(rows) / 1e3
names = ["spmv_span", "update_span", "pupdate_span", "gap_spmv_update", "gap_update_pupdate",
         "gap_pupdate_spmv", "period"]
print(json.dumps({n: [round(float(np.median(r[:, i])), 2), round(float(r[:, i].min()), 2),
                      round(float(r[:, i].max()), 2)] for i, n in enumerate(names)}))
print(json.dumps({"arrive_before_release_us": [round(float(np.median((a[0, 5:35, 1] - a[0, 5:35, 0]) / 1e3)), 2),
                                               round(float(np.median((a[1, 5:35, 1] - a[1, 5:35, 0]) / 1e3)), 2),
                                               round(float(np.median((a[2, 6:36, 1] - a[2, 6:36, 0]) / 1e3)), 2)]}))
