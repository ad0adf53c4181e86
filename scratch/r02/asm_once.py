"""Two bond + element assemblies on the 600K plate predictor state (ncu target)."""
import os, sys
sys.path.insert(0, os.getcwd())  # the tree under test (cwd)
import torch
from paper_2308_10459_b200 import configs
from paper_2308_10459_b200.scene import Scene
from paper_2308_10459_b200.step import prepare_step

scene = Scene.from_spec(configs.plate(), host_sync=False)
prepare_step(scene)
dev = scene.device
for _ in range(2):
    dev.call("bdem_bond_assemble", dev.sysp, dev.xp.data_ptr(), dev.xq.data_ptr(), dev.stream)
    dev.call("bdem_element_assemble", dev.sysp, dev.xp.data_ptr(), dev.xq.data_ptr(), dev.z.data_ptr(), dev.stream)
torch.cuda.synchronize()
print("ok")
