"""Landmark term on the B200 against the CPU oracle.

Landmarks are fixed (source vertex, target position) pairs with weight w = 1
point rows added to the alignment part of K and B in the first stage only
(reference energy.hpp:198-199,218-227; solver.hpp:203-208,217-218); their
energy sum_l |v_hat(l) - target_l|^2 is reported as E_landmark and weighted
into the accepted energy. Checked teacher-forced (same X: energies incl.
E_landmark, K, B, x_mm) and over whole registrations (plain MM: every
iteration; AA: the reference's own reproducibility horizon as in
test_gpu_parity.py), plus the reference's range checks.
"""
import numpy as np
import pytest

from oracle import binding as O
from paper_2206_03410_b200 import capi
from paper_2206_03410_b200 import registration as R
from tests.helpers import bbox_diag, random_transforms, strip_problem

pytestmark = pytest.mark.gpu


def _landmarks(p, k, seed):
    rng = np.random.default_rng(seed)
    idx = rng.choice(p.n, size=k, replace=False)
    return [(int(i), p.target[int(i)] + 0.01 * rng.standard_normal(3)) for i in idx]


@pytest.fixture(scope="module")
def prob():
    return strip_problem(20, 9, seed=77, mult=4.0, amp_scale=2.0)


@pytest.fixture(scope="module")
def ctx(prob):
    c = R.Context()
    c.set_problem(prob)
    yield c
    c.close()


@pytest.mark.parametrize("lw", [1.0, 37.5])
def test_landmark_step_parity(ctx, prob, lw):
    """energy.hpp:218-227: landmark rows in K/B; solver.hpp:203-208 energy."""
    N = prob.graph.node_count
    nnzb = int(R.bsr_pattern(prob.graph)[0][-1])
    lms = _landmarks(prob, 12, 5)
    X = random_transforms(N, 9, 0.1)
    prm = (0.7, 1.3, 0.08, 0.11)
    g = ctx.step(X, prm, landmark_weight=lw, cfg=R.solver_config(landmarks=lms), nnzb=nnzb)
    o = O.step(prob, X, prm, nnzb, landmark_weight=lw, cfg=O.config(landmarks=lms))
    assert np.array_equal(g["index"], o["index"])
    assert np.allclose(g["energy"], o["energy"], rtol=1e-12, atol=1e-300)
    assert np.max(np.abs(g["K"] - o["K"])) <= 1e-12 * np.max(np.abs(o["K"]))
    assert np.max(np.abs(g["B"] - o["B"])) <= 1e-12 * np.max(np.abs(o["B"]))
    assert np.max(np.abs(g["Xmm"] - o["Xmm"])) <= 1e-8 * (1 + np.max(np.abs(o["Xmm"])))
    # the landmark rows change the system (they are not silently dropped)
    g0 = ctx.step(X, prm, landmark_weight=0.0, cfg=R.solver_config(landmarks=lms), nnzb=nnzb)
    assert np.max(np.abs(g0["K"] - g["K"])) > 0


def _iters(rep):
    return [it for st in rep["stages"] for it in st["iterations"]]


def test_landmark_register_mm_parity(prob):
    """Plain MM with landmarks, default schedule: identical stage/iteration
    counts, every E and E_landmark within 1e-6, vertices within 1e-5 diag."""
    lms = _landmarks(prob, 8, 11)
    c = R.Context()
    try:
        Xg, vg, rg = c.register(R.solver_config(aa_window=0, landmarks=lms), one_shot_problem=prob)
    finally:
        c.close()
    Xo, vo, ro = O.register(prob, O.config(aa_window=0, landmarks=lms))
    ig, io = _iters(rg), _iters(ro)
    assert [len(s["iterations"]) for s in rg["stages"]] == [len(s["iterations"]) for s in ro["stages"]]
    for a, b in zip(ig, io):
        assert abs(a["E"] - b["E"]) <= 1e-6 * abs(b["E"])
        assert abs(a["E_landmark"] - b["E_landmark"]) <= 1e-6 * abs(b["E_landmark"]) + 1e-300
    # stage 0 carries the landmark energy, later stages do not (solver.hpp:217-218)
    assert rg["stages"][0]["iterations"][0]["E_landmark"] > 0
    for st in rg["stages"][1:]:
        assert all(it["E_landmark"] == 0.0 for it in st["iterations"])
    assert np.max(np.linalg.norm(vg - vo, axis=1)) <= 1e-5 * bbox_diag(prob.source)


def test_landmark_register_aa_parity(prob):
    """AA with landmarks: energies within 1e-6 over the leading iterations the
    reference reproduces itself (see test_gpu_parity._aa_parity)."""
    lms = _landmarks(prob, 8, 13)
    kw = dict(landmarks=lms, i_max=40)
    c = R.Context()
    try:
        _, vg, rg = c.register(R.solver_config(**kw), one_shot_problem=prob)
    finally:
        c.close()
    _, vo, ro = O.register(prob, O.config(**kw))
    eg = np.array([it["E"] for it in _iters(rg)])
    eo = np.array([it["E"] for it in _iters(ro)])
    n = min(len(eg), len(eo))
    bad = np.nonzero(np.abs(eg[:n] - eo[:n]) > 1e-6 * np.abs(eo[:n]))[0]
    horizon = int(bad[0]) if len(bad) else n
    assert horizon >= min(10, n), (horizon, n)


def test_landmark_errors(prob):
    """Out-of-range landmark source indices are ConfigErrors (energy.hpp
    SystemAssembler constructor), on both the register and the step entry."""
    c = R.Context()
    try:
        with pytest.raises(capi.ConfigError):
            c.register(R.solver_config(landmarks=[(prob.n + 3, np.zeros(3))]), one_shot_problem=prob)
        c.set_problem(prob)
        nnzb = int(R.bsr_pattern(prob.graph)[0][-1])
        with pytest.raises(capi.ConfigError):
            c.step(R.identity_transforms(prob.graph.node_count), (1, 1, 0.1, 0.1), landmark_weight=1.0,
                   cfg=R.solver_config(landmarks=[(-1, np.zeros(3))]), nnzb=nnzb)
    finally:
        c.close()
