"""Generates tests/golden/cfg2_full_<case>.npz: oracle trajectories at the
FULL headline size (BASELINE config 2: 99,856-vertex source, ~3,000 nodes).

The inputs are not stored (they are ~10 MB): `registration.make_problem(2)`
regenerates them bit for bit from the seeded generator, and the fixture keeps
checksums of the regenerated arrays so a test can tell if they drifted. The
fixture holds the oracle's per-iteration energies, stage lengths, revert
counts and final transforms X (the final vertices are deform(X)).

    python tests/golden/make_golden_full.py CASE [CASE ...]
      CASE: aa100      fixed nu (bench idiom), AA m=5, 100 iterations, RCM ordering
            aa100_nat  the same with the natural node ordering of the direct solve
                       (the reference's own reproducibility envelope)
            mm100      fixed nu, plain MM (aa_window = 0), 100 iterations
            mm_default plain MM, default schedule (annealing)
            aa_default default SolverConfig (annealing, AA m = 5)
"""
import dataclasses
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import binding as O  # noqa: E402
from paper_2206_03410_b200 import registration as R  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def checksums(p):
    """sha256 of every input array of the problem (source, target, graph)."""
    out = {"source": p.source, "target": p.target}
    for f in dataclasses.fields(p.graph):
        v = getattr(p.graph, f.name)
        if isinstance(v, np.ndarray):
            out["graph_" + f.name] = v
    return {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() for k, v in out.items()}


def case_config(case, prm):
    fixed = dict(nu_a_init=prm["nu_a"], nu_a_min=prm["nu_a"], nu_r_init=prm["nu_r"], eps=1e-300, i_max=100)
    return {"aa100": (fixed, 0), "aa100_nat": (fixed, 1), "mm100": (dict(fixed, aa_window=0), 0),
            "mm_default": (dict(aa_window=0), 0), "aa_default": ({}, 0)}[case]


def main(cases):
    p = R.make_problem(2)
    prm = O.init_parameters(p)
    sums = checksums(p)
    for case in cases:
        kw, ordering = case_config(case, prm)
        t0 = time.time()
        X, v, rep = O.register(p, O.config(**kw), ordering=ordering)
        E = np.array([it["E"] for st in rep["stages"] for it in st["iterations"]])
        np.savez_compressed(
            os.path.join(OUT, f"cfg2_full_{case}.npz"), E=E, X=X,
            E_parts=np.array([[it["E_align"], it["E_reg"], it["E_rot"]] for st in rep["stages"]
                              for it in st["iterations"]]),
            aa_accepted=np.array([it["aa_accepted"] for st in rep["stages"] for it in st["iterations"]]),
            stages=np.array([len(st["iterations"]) for st in rep["stages"]]),
            reverts=np.array([st["reverts"] for st in rep["stages"]]),
            stage_prm=np.array([[st["alpha"], st["beta"], st["nu_a"], st["nu_r"]] for st in rep["stages"]]),
            checksums=np.array(sorted(sums.items())))
        print(case, "iterations", len(E), "stages", len(rep["stages"]), "%.1fs" % (time.time() - t0), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["aa100", "aa100_nat", "mm100", "mm_default", "aa_default"])
