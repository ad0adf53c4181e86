"""Distribution of ikpre (first staged (i,i) quadrant slot per row) on the
assembly goldens and a perturbed plate: is the mixed case (kpre > 0) hit?"""
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import test_gpu_parity as T
from _fixtures import load
for tag in ("near", "rand"):
    d = load("newton_pieces.npz")
    dev, prob = T._gpu_problem(d, tag)
    prob.assemble(dev.xp, dev.xq)
    k = dev.ikpre[:dev.n].cpu().numpy()
    print(tag, "queued", int(dev.counter[5]), "rows kpre=-1/0/>0:", int((k < 0).sum()), int((k == 0).sum()), int((k > 0).sum()))
