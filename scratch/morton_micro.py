"""SpMV on the 600K plate with row-major vs Morton-ordered element numbering."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2308_10459_b200 import configs
from paper_2308_10459_b200.state import BondSet, ElementSet
from paper_2308_10459_b200.scene import Scene
from paper_2308_10459_b200.newton import GPUProblem

def morton_perm(p):
    lo, hi = p.min(0), p.max(0)
    g = ((p - lo) / np.maximum(hi - lo, 1e-30) * (2**20 - 1)).astype(np.uint64)
    key = np.zeros(len(p), dtype=np.uint64)
    for bit in range(20):
        for ax in range(3):
            key |= ((g[:, ax] >> np.uint64(bit)) & np.uint64(1)) << np.uint64(3 * bit + ax)
    return np.argsort(key, kind="stable")

def renumber(spec, perm):
    inv = np.empty_like(perm); inv[perm] = np.arange(len(perm))
    el = spec.elements
    el2 = ElementSet(*(np.ascontiguousarray(getattr(el, f)[perm]) for f in ("p","q","v","qdot","mass","radius","pinned")))
    b = spec.bonds
    i2, j2 = inv[b.i], inv[b.j]
    lo, hi = np.minimum(i2, j2), np.maximum(i2, j2)
    order = np.lexsort((hi, lo))
    kw = {f: np.asarray(getattr(b, f))[order] for f in b.__dataclass_fields__}
    kw["i"], kw["j"] = i2[order], j2[order]
    swap = (i2 > j2)[order]
    # swapping endpoints flips d0; keep the original orientation by keeping (i,j) roles
    kw["i"], kw["j"] = i2[order], j2[order]
    spec.elements, spec.bonds = el2, BondSet(**kw)
    return spec

res = {}
for mode in ("rowmajor", "morton"):
    spec = configs.plate()
    if mode == "morton":
        spec = renumber(spec, morton_perm(spec.elements.p))
    scene = Scene.from_spec(spec, host_sync=False)
    dev = scene.device
    dev.call("bdem_predict", dev.sysp, dev.p.data_ptr(), dev.q.data_ptr(), dev.v.data_ptr(),
             dev.qdot.data_ptr(), dev.p_prev.data_ptr(), dev.q_prev.data_ptr(), spec.dt,
             dev.p_hat.data_ptr(), dev.q_hat.data_ptr(), dev.mp_dt2.data_ptr(), dev.mq_dt2.data_ptr(),
             dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream)
    GPUProblem(dev).assemble(dev.xp, dev.xq)
    x = torch.randn(6 * dev.vstride, dtype=torch.float64, device="cuda"); y = torch.zeros_like(x)
    def run(): dev.call("bdem_spmv", dev.sysp, x.data_ptr(), y.data_ptr(), dev.stream)
    for _ in range(3): run()
    torch.cuda.synchronize(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(30): run()
    b.record(); torch.cuda.synchronize()
    res[mode] = {"spmv_us": a.elapsed_time(b) / 30 * 1e3, "P_over_nb": dev.sell.n_pos / dev.nb, "PJ_over_nb": dev.sell.n_jpos / dev.nb}
    del scene, dev; torch.cuda.empty_cache()
print(json.dumps(res))
