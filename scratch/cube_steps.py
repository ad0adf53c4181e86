import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from _fixtures import load, elements_from, bonds_from
from paper_2308_10459_b200 import Scene, SolverConfig, stable_step
from paper_2308_10459_b200 import configs as C
d = load("traj_cube.npz")
spec = C.cube(n_side=5, random_q=False, seed=3, youngs=3e8, k_contact=1e9, speed=2.0, dt=1e-4)
el = elements_from(d, "init_el_"); b = bonds_from(d, "init_b_")
from paper_2308_10459_b200 import PlasticParams
scene = Scene("cube", None, el, b, colliders=[], gravity=d["gravity"], dt=float(d["dt"]), youngs=float(d["youngs"]), plastic=PlasticParams(*d["plastic"]),
              k_contact=float(d["k_contact"]), k_element=float(d["k_element"]))
for s in range(6):
    scene.colliders = spec.collider_schedule(scene.time + scene.dt)
    rep = stable_step(scene, SolverConfig(epsilon=float(d["epsilon"]), max_iterations=300))
    r = rep.solve
    print(s, len(rep.broken), rep.committed, r.iterations, r.pcg_total, rep.contact_pairs, f"{r.grad_norm:.6e}", [f"{x.grad_norm:.4e}" for x in r.records[:3]], "gold", d["newton"][s], d["pcg"][s])
