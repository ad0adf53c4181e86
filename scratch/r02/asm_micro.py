"""Time the assembly kernels (bond rows + clamp, element) on the 600K plate
predictor state: CUDA events over repeated launches, plus a perturbed-q state
(every rotation block through the eigen-clamp)."""
import json, os, sys
sys.path.insert(0, os.getcwd())  # the tree under test (cwd)
import torch
from paper_2308_10459_b200 import configs
from paper_2308_10459_b200.scene import Scene
from paper_2308_10459_b200.step import prepare_step

spec = configs.plate(nx=int(os.environ.get("NX", 1000)), ny=int(os.environ.get("NY", 600)))
scene = Scene.from_spec(spec, host_sync=False)
prep = prepare_step(scene)
dev = scene.device
res = {}


def timeit(name, fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    res[name] = a.elapsed_time(b) / reps * 1e3


bond = lambda: dev.call("bdem_bond_assemble", dev.sysp, dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream)
elem = lambda: dev.call("bdem_element_assemble", dev.sysp, dev.xp.data_ptr(), dev.xq.data_ptr(), dev.z.data_ptr(), dev.stream)
xq_rest = dev.xq.clone()
for tag, pert in (("rest", 0.0), ("pert", float(os.environ.get("PERT", "1e-3")))):
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    dev.xq.copy_(xq_rest + pert * torch.randn(xq_rest.shape, generator=g, device="cuda", dtype=torch.float64))
    dev.xq.div_(dev.xq.norm(dim=1, keepdim=True))
    timeit(f"bond_us_{tag}", bond)
    timeit(f"element_us_{tag}", elem)
    timeit(f"both_us_{tag}", lambda: (bond(), elem()))
    if hasattr(dev.lib, "bdem_assemble_fused") and os.environ.get("NO_FUSED") is None:
        from paper_2308_10459_b200 import _lib as L
        fused = lambda: dev.call("bdem_assemble_fused", dev.sysp, dev.xp.data_ptr(), dev.xq.data_ptr(), dev.z.data_ptr(), dev.stream)
        bond(); elem(); torch.cuda.synchronize()
        zr, dr, mr = dev.z.clone(), dev.diag.clone(), dev.minv.clone()
        timeit(f"fused_us_{tag}", fused)
        torch.cuda.synchronize()
        res[f"fused_nclamp_{tag}"] = float(dev.scalars[L.SC["NCLAMP"]].item())
        res[f"fused_identical_{tag}"] = bool(torch.equal(zr, dev.z) and torch.equal(dr, dev.diag) and torch.equal(mr, dev.minv))
    torch.cuda.synchronize()
    res[f"clamp_queue_{tag}"] = int(dev.counter[5].item())
    res[f"z_sum_{tag}"] = float(dev.z.abs().sum())
    res[f"diag_sum_{tag}"] = float(dev.diag.abs().sum())
res["n_bond"] = dev.nb
res["bytes_rule_GB"] = (dev.nb * (161 + 288) + dev.nf * (136 + 144 + 144 + 48 + 56)) / 1e9
res["frac_rest"] = res["bytes_rule_GB"] * 1e9 / (res["both_us_rest"] * 1e-6) / 6547.5e9
print(json.dumps(res))
