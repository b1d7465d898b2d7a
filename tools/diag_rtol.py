"""PCG tolerance vs AA trajectory horizon (GPU vs oracle) and bench cost."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import binding as O
from paper_2206_03410_b200 import registration as R
from tests.test_gpu_parity import _trace, _horizon

cases = [(0, 0.4, 100), (2, 0.05, 40), (0, 1.0, 60)]
probs = []
for cfg, scale, iters in cases:
    p = R.make_problem(cfg, scale=scale)
    prm = O.init_parameters(p)
    kw = dict(nu_a_init=prm["nu_a"], nu_a_min=prm["nu_a"], nu_r_init=prm["nu_r"], eps=1e-300, i_max=iters)
    _, vo, ro = O.register(p, O.config(**kw))
    probs.append((p, kw, _trace(ro)))
for rtol in [float(x) for x in sys.argv[1].split(",")]:
    ctx = R.Context(pcg_rtol=rtol)
    hs = []
    for p, kw, eo in probs:
        Xg, vg, rg = ctx.register(R.solver_config(**kw), one_shot_problem=p)
        hs.append(_horizon(_trace(rg), eo))
    print("rtol", rtol, "factor", os.environ.get("NRR_PCG_TRUE_FACTOR", "100"), "horizons", hs, flush=True)
