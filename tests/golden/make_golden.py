"""Generates tests/golden/*.npz from the pinned CPU oracle (oracle/, checked
against the reference's known-answer tests by tests/cpp/oracle_kats.cpp).
The fixtures hold the inputs and the oracle's answers, so the GPU tests have a
fixed expected result that travels to the GPU box without the oracle build.

    python tests/golden/make_golden.py
"""
import dataclasses
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import binding as O  # noqa: E402
from paper_2206_03410_b200 import registration as R  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def problem_arrays(p):
    d = {"source": p.source, "target": p.target, "src_avg_edge_length": p.src_avg_edge_length}
    for f in dataclasses.fields(p.graph):
        d["graph_" + f.name] = np.asarray(getattr(p.graph, f.name))
    return d


def main():
    for name, cfg, scale in [("cfg0_s02", 0, 0.2), ("cfg2_s002", 2, 0.02)]:
        p = R.make_problem(cfg, scale=scale)
        N = p.graph.node_count
        rp, cols = R.bsr_pattern(p.graph)
        prm = O.init_parameters(p)
        prm4 = np.array([prm["alpha"], prm["beta"], prm["nu_a"], prm["nu_r"]])
        X0 = R.identity_transforms(N)
        s0 = O.step(p, X0, prm4, len(cols))
        kw = dict(nu_a_init=prm["nu_a"], nu_a_min=prm["nu_a"], nu_r_init=prm["nu_r"], eps=1e-300, i_max=20)
        Xp, vp, rpm = O.register(p, O.config(aa_window=0, **kw))
        Xa, va, ra = O.register(p, O.config(**dict(kw, i_max=10)))
        Xd, vd, rd = O.register(p, O.config(aa_window=0))
        np.savez_compressed(
            os.path.join(OUT, name + ".npz"), **problem_arrays(p),
            prm4=prm4, step_index=s0["index"], step_energy=s0["energy"], step_K=s0["K"], step_B=s0["B"],
            step_Xmm=s0["Xmm"],
            plain_E=np.array([it["E"] for st in rpm["stages"] for it in st["iterations"]]), plain_X=Xp,
            plain_v=vp,
            aa_E=np.array([it["E"] for st in ra["stages"] for it in st["iterations"]]),
            default_E=np.array([it["E"] for st in rd["stages"] for it in st["iterations"]]),
            default_stages=np.array([len(st["iterations"]) for st in rd["stages"]]), default_v=vd)
        print(name, "n", len(p.source), "N", N, "default stages", len(rd["stages"]))


if __name__ == "__main__":
    main()
