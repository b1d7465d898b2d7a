"""Diagnostic: per-iteration energy trajectories of the GPU path vs the oracle."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import binding as O  # noqa: E402
from paper_2206_03410_b200 import registration as R  # noqa: E402
from tests.helpers import strip_problem  # noqa: E402


def run(p, aa, rtol, i_max=100):
    ctx = R.Context(pcg_rtol=rtol, record_passes=1)
    Xg, vg, rg = ctx.register(R.solver_config(aa_window=aa, i_max=i_max), one_shot_problem=p)
    Xo, vo, ro = O.register(p, O.config(aa_window=aa, i_max=i_max), pass_cap=5000)
    print("aa", aa, "rtol", rtol, "iters", rg["total_iterations"], ro["total_iterations"],
          "vdiff", np.max(np.linalg.norm(vg - vo, axis=1)), "pcg iters", rg["linear_iterations"])
    for s, (sg, so) in enumerate(zip(rg["stages"], ro["stages"])):
        eg = np.array([it["E"] for it in sg["iterations"]])
        eo = np.array([it["E"] for it in so["iterations"]])
        n = min(len(eg), len(eo))
        rel = np.abs(eg[:n] - eo[:n]) / np.abs(eo[:n])
        fa = [it["aa_accepted"] for it in sg["iterations"]]
        fo = [it["aa_accepted"] for it in so["iterations"]]
        first_flag = next((k for k in range(n) if fa[k] != fo[k]), None)
        print(f"  stage {s}: len {len(eg)}/{len(eo)} reverts {sg['reverts']}/{so['reverts']} "
              f"max rel {rel.max():.2e} at {rel.argmax()} first aa-flag diff {first_flag} "
              f"rel@10 {rel[min(10, n - 1)]:.1e}")


p = strip_problem(24, 10, seed=4242, mult=5.0, amp_scale=2.5)
for aa in (0, 5):
    for rtol in (1e-12, 1e-14):
        run(p, aa, rtol)
