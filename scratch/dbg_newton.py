import sys; sys.path.insert(0, "tests")
import numpy as np
from _fixtures import load
from test_gpu_parity import _gpu_problem
from paper_2308_10459_b200 import SolverConfig, minimize_second_order
d = load("newton_pieces.npz")
dev, prob = _gpu_problem(d, "near")
sol = minimize_second_order(prob, dev.xp.clone(), dev.xq.clone(), SolverConfig(epsilon=1e-7, max_iterations=30))
print("gpu ", sol.iterations, sol.converged, [("%.3e" % r.grad_norm, r.pcg_iterations, r.alpha) for r in sol.records])
print("gold", int(d["solve_iterations"]), [("%.3e" % g, int(k), a) for g, k, a in zip(d["solve_rec_gnorm"], d["solve_rec_pcg"], d["solve_rec_alpha"])])
print("f gpu", [r.f for r in sol.records][:6])
print("f ref", list(d["solve_rec_f"][:6]))
dp = np.abs(sol.p.cpu().numpy() - d["solve_p"]).max(axis=1)
print("rows differing", np.nonzero(dp > 1e-9)[0], dp.max())
