"""GPU vs oracle on a fixed-count single-stage run of a synthetic config (bench idiom)."""
import sys
import time
import numpy as np
sys.path.insert(0, ".")
from oracle import binding as O
from paper_2206_03410_b200 import registration as R
cfgid, scale, iters = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
p = R.make_problem(cfgid, scale=scale)
prm = O.init_parameters(p)
kw = dict(nu_a_init=prm["nu_a"], nu_a_min=prm["nu_a"], nu_r_init=prm["nu_r"], eps=1e-300, i_max=iters)
t = time.time()
Xo, vo, ro = O.register(p, O.config(**kw))
print("n", p.n, "N", p.graph.node_count, "oracle s", time.time() - t, flush=True)
eo = np.array([it["E"] for it in ro["stages"][0]["iterations"]])
fo = [it["aa_accepted"] for it in ro["stages"][0]["iterations"]]
diag = np.linalg.norm(p.source.max(0) - p.source.min(0))
for rtol in (1e-10, 1e-12, 1e-13):
    ctx = R.Context(pcg_rtol=rtol)
    Xg, vg, rg = ctx.register(R.solver_config(**kw), one_shot_problem=p)
    eg = np.array([it["E"] for it in rg["stages"][0]["iterations"]])
    fg = [it["aa_accepted"] for it in rg["stages"][0]["iterations"]]
    rel = np.abs(eg - eo) / np.abs(eo)
    flip = next((k for k in range(len(fg)) if fg[k] != fo[k]), None)
    print("rtol %g: max Erel %.2e (first 10: %.1e) first flag flip %s  vdiff/diag %.2e  reverts %d/%d pcg %d" % (
        rtol, rel.max(), rel[:10].max(), flip, np.max(np.linalg.norm(vg - vo, axis=1)) / diag,
        rg["stages"][0]["reverts"], ro["stages"][0]["reverts"], rg["linear_iterations"]), flush=True)
