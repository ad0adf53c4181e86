"""Diagnostic: max |GPU - reference| per trajectory golden and quantity."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from _fixtures import bonds_from, elements_from, load
from paper_2308_10459_b200 import HalfSpace, PlasticParams, Scene, SolverConfig, stable_step
from paper_2308_10459_b200 import configs as C
from paper_2308_10459_b200.scene import TwistDriver

for name in ["cantilever", "rope", "plate", "cube", "stack"]:
    d = load(f"traj_{name}.npz")
    el = elements_from(d, "init_el_"); b = bonds_from(d, "init_b_")
    driver, sched, cols = None, None, []
    if name == "rope":
        spec = C.rope(n=30)
        driver = TwistDriver(spec.driver.ids, spec.driver.p0, spec.driver.axis_point, spec.driver.rate)
    if name == "cube":
        spec = C.cube(n_side=5, random_q=False, seed=3, youngs=3e8, k_contact=1e9, speed=2.0, dt=1e-4)
        sched = spec.collider_schedule
    if name == "plate":
        cols = [HalfSpace((0.0, 0.0, 1.0), 0.0)]
    if name == "stack":
        cols = C.stack().colliders
    plastic = PlasticParams(*d["plastic"]) if "plastic" in d else None
    scene = Scene(name, None, el, b, colliders=cols, gravity=d["gravity"], dt=float(d["dt"]),
                  youngs=float(d["youngs"]), k_contact=float(d["k_contact"]),
                  k_element=float(d["k_element"]), plastic=plastic, driver=driver,
                  mu_s=float(d.get("mu_s", 0.0)), mu_r=float(d.get("mu_r", 0.0)))
    cfg = SolverConfig(epsilon=float(d["epsilon"]), max_iterations=300)
    out = []
    for s in range(d["p"].shape[0]):
        if sched is not None:
            scene.colliders = sched(scene.time + scene.dt)
        rep = stable_step(scene, cfg)
        e = {k: float(np.abs(getattr(scene.elements, k) - d[k][s]).max()) for k in ("p", "q", "v", "qdot")}
        mv = {k: float(np.abs(d[k][s] - d["init_el_" + k]).max()) for k in ("p", "q")}
        out.append((s, rep.committed == bool(d["committed"][s]), rep.solve.iterations, int(d["newton"][s]),
                    rep.solve.pcg_total, int(d["pcg"][s]), e, mv))
    print(f"== {name} eps={float(d['epsilon'])}")
    for o in out:
        print("  step %d commit_ok=%s newton %d/%d pcg %d/%d err %s moved %s" % (
            o[0], o[1], o[2], o[3], o[4], o[5], {k: f"{v:.2e}" for k, v in o[6].items()},
            {k: f"{v:.2e}" for k, v in o[7].items()}), flush=True)
