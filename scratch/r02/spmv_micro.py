"""SpMV / PCG-iteration timing on the 600K plate step-1 system (CUDA events),
plus checksums to confirm bit-identical results across library variants."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2308_10459_b200 import configs
from paper_2308_10459_b200.scene import Scene
from paper_2308_10459_b200.step import prepare_step

spec = configs.plate(nx=int(os.environ.get("NX", 1000)), ny=int(os.environ.get("NY", 600)))
scene = Scene.from_spec(spec, host_sync=False)
prob = prepare_step(scene).problem
dev = scene.device
prob.assemble(dev.xp, dev.xq)
res = {}


def timeit(name, fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    res[name] = a.elapsed_time(b) / reps * 1e3


g = torch.Generator(device="cuda"); g.manual_seed(3)
x = torch.randn(6 * dev.vstride, generator=g, dtype=torch.float64, device="cuda")
y = torch.zeros_like(x)
timeit("spmv_us", lambda: dev.call("bdem_spmv", dev.sysp, x.data_ptr(), y.data_ptr(), dev.stream))
res["y_checksum"] = float(y.abs().sum())
ptrs = (dev.y.data_ptr(), dev.r.data_ptr(), dev.zv.data_ptr(), dev.pv.data_ptr())
for chunk in (32,):
    ts = []
    for rep in range(4):
        dev.call("bdem_pcg_init", dev.sysp, dev.z.data_ptr(), -1.0, *ptrs, 1e-30, 100000, 0.0, dev.stream)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        dev.call("bdem_pcg_iterate", dev.sysp, *ptrs, dev.ap.data_ptr(), chunk, dev.stream)
        b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / chunk)
    res[f"pcg_iter_us"] = min(ts)
res["pcg_state"] = [float(v) for v in dev.pcg_state.cpu().numpy()[:14]]
res["pcg_y_checksum"] = float(dev.y.abs().sum())
res["lib"] = os.environ.get("BDEM_LIB", "default")
print(json.dumps(res))
