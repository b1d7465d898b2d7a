import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import binding as O
from paper_2206_03410_b200 import registration as R
from tests.helpers import strip_problem
p = strip_problem(24, 10, seed=4242, mult=5.0, amp_scale=2.5)
Xo, vo, ro = O.register(p, O.config())
q = R.Problem(p.source, p.target * (1 + 1e-13), p.graph, p.src_avg_edge_length, p.faces)
Xs, vs, rs = O.register(q, O.config())
print("oracle vs perturbed: vdiff", np.max(np.linalg.norm(vs - vo, axis=1)), "final E", ro["stages"][-1]["iterations"][-1]["E"], rs["stages"][-1]["iterations"][-1]["E"])
for rtol in (1e-12, 1e-11, 1e-10):
    ctx = R.Context(pcg_rtol=rtol)
    Xg, vg, rg = ctx.register(R.solver_config(), one_shot_problem=p)
    print("rtol", rtol, "vdiff", np.max(np.linalg.norm(vg - vo, axis=1)), "iters", rg["total_iterations"], ro["total_iterations"],
          "stages", [(len(s["iterations"]), s["reverts"], s["converged"]) for s in rg["stages"]],
          [(len(s["iterations"]), s["reverts"], s["converged"]) for s in ro["stages"]],
          "final E", rg["stages"][-1]["iterations"][-1]["E"])
