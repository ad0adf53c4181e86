import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from _fixtures import load, elements_from, bonds_from
from paper_2308_10459_b200 import Scene, SolverConfig, stable_step
from paper_2308_10459_b200 import configs as C
d = load("traj_stack.npz")
el = elements_from(d, "init_el_"); b = bonds_from(d, "init_b_")
for mu in (True, False):
    scene = Scene("stack", None, el.copy(), b.copy(), colliders=C.stack().colliders, gravity=d["gravity"], dt=float(d["dt"]),
                  youngs=float(d["youngs"]), k_contact=float(d["k_contact"]), k_element=float(d["k_element"]),
                  mu_s=float(d["mu_s"]) if mu else 0.0, mu_r=float(d["mu_r"]) if mu else 0.0)
    for s in range(8):
        rep = stable_step(scene, SolverConfig(epsilon=float(d["epsilon"]), max_iterations=300))
        r = rep.solve
        print(mu, s, rep.committed, r.reason, r.iterations, "golden its", d["newton"][s], "gn", [f"{x.grad_norm:.2e}" for x in r.records[-4:]],
              "gold gnorm", f"{d['gnorm'][s]:.2e}")
        if mu:
            print("   dp", np.abs(scene.elements.p - d["p"][s]).max(), "dv", np.abs(scene.elements.v - d["v"][s]).max())
        if not rep.committed:
            print("   ls trials", [ (x.alpha, x.f) for x in r.records[-2:]] if hasattr(r.records[-1], "alpha") else r.records[-1])
            break
