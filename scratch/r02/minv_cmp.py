"""minv / diag / z of one plate assembly (predictor state and a perturbed-q
state) to compare library builds bit for bit."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2308_10459_b200 import configs, _lib as L
from paper_2308_10459_b200.scene import Scene
from paper_2308_10459_b200.step import prepare_step
scene = Scene.from_spec(configs.plate(nx=200, ny=120), host_sync=False)
prob = prepare_step(scene).problem
dev = scene.device
out = {}
for tag, pert in (("rest", 0.0), ("pert", 1e-3)):
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    xq = dev.xq.clone()
    dev.xq.add_(pert * torch.randn(xq.shape, generator=g, device="cuda", dtype=torch.float64))
    dev.xq.div_(dev.xq.norm(dim=1, keepdim=True))
    prob.assemble(dev.xp, dev.xq)
    out[f"{tag}_minv"] = dev.minv.cpu().numpy(); out[f"{tag}_diag"] = dev.diag.cpu().numpy()
    out[f"{tag}_z"] = dev.z.cpu().numpy(); out[f"{tag}_nsing"] = float(dev.scalars[L.SC["NSING"]])
    dev.xq.copy_(xq)
np.savez(os.environ["OUT"], **out)
print({k: v for k, v in out.items() if "nsing" in k})
