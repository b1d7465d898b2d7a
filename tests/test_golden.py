"""Golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py
from the pinned oracle). CPU: the oracle still reproduces them (regression
pin of the checker). GPU: the product matches them without running the
oracle."""
import dataclasses
import os

import numpy as np
import pytest

from paper_2206_03410_b200 import registration as R

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["cfg0_s02", "cfg2_s002"]


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    gf = {f.name: z["graph_" + f.name] for f in dataclasses.fields(R.Graph)}
    gf["radius"] = float(gf["radius"])
    p = R.Problem(z["source"], z["target"], R.Graph(**gf), float(z["src_avg_edge_length"]), None)
    return p, z


def fixed_kw(z):
    a, b, nu_a, nu_r = z["prm4"]
    return dict(nu_a_init=nu_a, nu_a_min=nu_a, nu_r_init=nu_r, eps=1e-300)


def rel(a, b):
    return np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_golden(name):
    from oracle import binding as O

    p, z = load(name)
    nnzb = len(R.bsr_pattern(p.graph)[1])
    s = O.step(p, R.identity_transforms(p.graph.node_count), z["prm4"], nnzb)
    assert np.array_equal(s["index"], z["step_index"])
    assert np.array_equal(s["energy"], z["step_energy"])
    _, _, rep = O.register(p, O.config(aa_window=0, i_max=20, **fixed_kw(z)))
    E = np.array([it["E"] for st in rep["stages"] for it in st["iterations"]])
    assert np.array_equal(E, z["plain_E"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_product_matches_golden(name):
    p, z = load(name)
    N = p.graph.node_count
    nnzb = len(R.bsr_pattern(p.graph)[1])
    diag = np.linalg.norm(p.source.max(0) - p.source.min(0))
    ctx = R.Context()
    try:
        ctx.set_problem(p)
        s = ctx.step(R.identity_transforms(N), z["prm4"], nnzb=nnzb)
        assert np.array_equal(s["index"], z["step_index"])
        assert rel(s["energy"], z["step_energy"]) <= 1e-12
        assert np.max(np.abs(s["K"] - z["step_K"])) <= 1e-13 * np.max(np.abs(z["step_K"]))
        assert np.max(np.abs(s["B"] - z["step_B"])) <= 1e-13 * (1 + np.max(np.abs(z["step_B"])))
        assert np.max(np.abs(s["Xmm"] - z["step_Xmm"])) <= 1e-9
        # plain MM trajectory (north_star tolerances)
        X, v, rep = ctx.register(R.solver_config(aa_window=0, i_max=20, **fixed_kw(z)), one_shot_problem=p)
        E = np.array([it["E"] for st in rep["stages"] for it in st["iterations"]])
        assert len(E) == len(z["plain_E"]) and rel(E, z["plain_E"]) <= 1e-6
        assert np.max(np.linalg.norm(v - z["plain_v"], axis=1)) <= 1e-5 * diag
        # Anderson-accelerated start (10 iterations: inside the reproducibility horizon)
        X, v, rep = ctx.register(R.solver_config(i_max=10, **fixed_kw(z)), one_shot_problem=p)
        E = np.array([it["E"] for st in rep["stages"] for it in st["iterations"]])
        assert len(E) == len(z["aa_E"]) and rel(E, z["aa_E"]) <= 1e-6
        # default schedule, plain MM
        X, v, rep = ctx.register(R.solver_config(aa_window=0), one_shot_problem=p)
        E = np.array([it["E"] for st in rep["stages"] for it in st["iterations"]])
        assert [len(st["iterations"]) for st in rep["stages"]] == list(z["default_stages"])
        assert rel(E, z["default_E"]) <= 1e-6
        assert np.max(np.linalg.norm(v - z["default_v"], axis=1)) <= 1e-5 * diag
    finally:
        ctx.close()
