import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import binding as O
from paper_2206_03410_b200 import registration as R
from tests.helpers import strip_problem
p = strip_problem(24, 10, seed=4242, mult=5.0, amp_scale=2.5)
print("N", p.graph.node_count)
for rtol in (1e-12,):
    ctx = R.Context(pcg_rtol=rtol, record_passes=1)
    Xg, vg, rg = ctx.register(R.solver_config(aa_window=0), one_shot_problem=p)
    Xo, vo, ro = O.register(p, O.config(aa_window=0), pass_cap=5000)
    print("iters", rg["total_iterations"], ro["total_iterations"], "vdiff", np.max(np.linalg.norm(vg - vo, axis=1)),
          "Xdiff", np.max(np.abs(Xg - Xo)), "pcg", rg["linear_iterations"])
    for s, (sg, so) in enumerate(zip(rg["stages"], ro["stages"])):
        eg = np.array([it["E"] for it in sg["iterations"]]); eo = np.array([it["E"] for it in so["iterations"]])
        dg = np.array([it["max_disp"] for it in sg["iterations"]]); do = np.array([it["max_disp"] for it in so["iterations"]])
        n = min(len(eg), len(eo))
        print(s, len(eg), len(eo), "Erel", np.max(np.abs(eg[:n] - eo[:n]) / np.abs(eo[:n])), "last disp", dg[-3:], do[-3:])
