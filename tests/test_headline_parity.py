"""Parity at the HEADLINE size (BASELINE config 2: 99,856-vertex source,
~3,000-node graph — the workload bench.py measures) and at full size for the
batched (config 3) and 1M-vertex (config 4) configs.

Two levels:

1. Teacher-forced, at EVERY pass of the device trajectory
   (tests/trace_check.py): at each iterate X_k the device evaluated, the CPU
   oracle recomputes correspondences, energies, the normal equations, the
   Anderson combine and the safeguard decision; the device's x_mm must meet
   the reference's own solve bar on the oracle's system. This is the
   north_star bar (NN identical up to ties, energies within 1e-6) applied at
   every iterate, independent of trajectory chaos.
2. Trajectory: plain MM (aa_window = 0) is contractive, so the whole device
   run must match the oracle's run (committed fixtures,
   tests/golden/make_golden_full.py): every per-iteration energy within 1e-6
   relative, identical stage lengths, final vertices within 1e-5 of the bbox
   diagonal. Anderson-accelerated runs with the strict safeguard are chaotic
   in floating point: at this size the reference algorithm run with a
   different (equally valid) direct-solver node ordering leaves the 1e-6 band
   after h_ref = 13 iterations and ends 4.4e-4 x diag away from itself. The
   device must stay within 1e-6 for >= h_ref / 2 iterations and end within
   10x that self-spread of the reference.
"""
import dataclasses
import hashlib
import os
import time

import numpy as np
import pytest

from oracle import binding as O
from paper_2206_03410_b200 import registration as R
from tests.helpers import bbox_diag
from tests.trace_check import check_trace, pattern, bsr_matvec

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
E_REL = 1e-6
V_REL = 1e-5


def golden(case):
    return np.load(os.path.join(GOLDEN, f"cfg2_full_{case}.npz"))


@pytest.fixture(scope="module")
def cfg2():
    p = R.make_problem(2)
    z = golden("aa100")
    # the fixtures were made from exactly these inputs
    sums = dict(z["checksums"])
    arrays = {"source": p.source, "target": p.target}
    for f in dataclasses.fields(p.graph):
        v = getattr(p.graph, f.name)
        if isinstance(v, np.ndarray):
            arrays["graph_" + f.name] = v
    for k, v in arrays.items():
        assert hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() == sums[k], k
    assert p.n == 99856
    return p


def fixed_kw(p, **kw):
    prm = O.init_parameters(p)
    return dict(dict(nu_a_init=prm["nu_a"], nu_a_min=prm["nu_a"], nu_r_init=prm["nu_r"], eps=1e-300, i_max=100), **kw)


def run_traced(p, kw, **ctx_kw):
    ctx = R.Context(record_passes=3, **ctx_kw)
    try:
        t0 = time.time()
        X, v, rep = ctx.register(R.solver_config(**kw), one_shot_problem=p)
        tr = ctx.trace()
        print("device run %.2fs, %d passes" % (time.time() - t0, len(tr)))
    finally:
        ctx.close()
    return X, v, rep, tr


def energies(rep):
    return np.array([it["E"] for st in rep["stages"] for it in st["iterations"]])


def horizon(ea, eb):
    n = min(len(ea), len(eb))
    bad = np.nonzero(np.abs(ea[:n] - eb[:n]) > E_REL * np.abs(eb[:n]))[0]
    return int(bad[0]) if len(bad) else n


def test_cfg2_full_aa_fixed_count_teacher_forced(cfg2):
    """The bench workload itself: fixed nu, AA m = 5, 100 accepted iterations
    (acceptance_main.cpp:207-215), checked at every pass."""
    p = cfg2
    kw = fixed_kw(p)
    X, v, rep, tr = run_traced(p, kw)
    assert rep["total_iterations"] == 100
    t0 = time.time()
    w = check_trace(p, tr, rep, kw)
    print("oracle check %.1fs" % (time.time() - t0))
    assert w["accepted"] == 100
    # trajectory envelope (chaotic: see the module docstring)
    za, zn = golden("aa100"), golden("aa100_nat")
    h_ref = horizon(zn["E"], za["E"])
    h_gpu = horizon(energies(rep), za["E"])
    diag = bbox_diag(p.source)
    spread = np.max(np.linalg.norm(O.deform(p, zn["X"]) - O.deform(p, za["X"]), axis=1))
    dev = np.max(np.linalg.norm(v - O.deform(p, za["X"]), axis=1))
    print(f"h_gpu {h_gpu} h_ref {h_ref}; final vertices {dev / diag:.2e} x diag (reference self-spread "
          f"{spread / diag:.2e})")
    assert h_gpu >= max(1, h_ref // 2)
    assert dev <= max(V_REL * diag, 10 * spread)


def test_cfg2_full_plain_mm_trajectory(cfg2):
    """aa_window = 0, fixed nu, 100 iterations: the whole trajectory within the
    north_star tolerances, and teacher-forced at every pass."""
    p = cfg2
    kw = fixed_kw(p, aa_window=0)
    X, v, rep, tr = run_traced(p, kw)
    z = golden("mm100")
    E = energies(rep)
    assert len(E) == len(z["E"]) == 100
    r = np.max(np.abs(E - z["E"]) / np.abs(z["E"]))
    vo = O.deform(p, z["X"])
    dv = np.max(np.linalg.norm(v - vo, axis=1)) / bbox_diag(p.source)
    print(f"plain MM: energies within {r:.2e}, final vertices within {dv:.2e} x diag")
    assert r <= E_REL
    assert dv <= V_REL
    check_trace(p, tr, rep, kw)


def test_cfg2_full_default_schedule_plain_mm(cfg2):
    """SolverConfig defaults with aa_window = 0: annealing stages, convergence
    test, stage lengths identical to the oracle's."""
    p = cfg2
    X, v, rep, tr = run_traced(p, dict(aa_window=0))
    z = golden("mm_default")
    assert [len(s["iterations"]) for s in rep["stages"]] == list(z["stages"])
    got = np.array([[s["alpha"], s["beta"], s["nu_a"], s["nu_r"]] for s in rep["stages"]])
    assert np.allclose(got, z["stage_prm"], rtol=1e-12, atol=0)
    E = energies(rep)
    r = np.max(np.abs(E - z["E"]) / np.abs(z["E"]))
    dv = np.max(np.linalg.norm(v - O.deform(p, z["X"]), axis=1)) / bbox_diag(p.source)
    print(f"default plain MM: {list(z['stages'])} iterations, energies within {r:.2e}, vertices {dv:.2e} x diag")
    assert r <= E_REL
    assert dv <= V_REL


def test_cfg2_full_default_schedule_aa_teacher_forced(cfg2):
    """Full SolverConfig defaults (annealing, AA m = 5, eps = 1e-5): every pass
    teacher-forced, and the trajectory within the reference's own envelope."""
    p = cfg2
    X, v, rep, tr = run_traced(p, {})
    w = check_trace(p, tr, rep, {})
    z = golden("aa_default")
    E = energies(rep)
    h_gpu = horizon(E, z["E"])
    print(f"default AA: device stages {[len(s['iterations']) for s in rep['stages']]} vs oracle {list(z['stages'])}, "
          f"horizon {h_gpu}, reverts {w['reverted']}")
    assert len(rep["stages"]) == len(z["stages"])
    assert h_gpu >= 6


@pytest.mark.parametrize("pair", [0, 37, 101, 255])
def test_cfg3_full_size_pairs_teacher_forced(pair):
    """Config 3 pairs at full size (20K vertices, ~600 nodes), the bench's
    50-iteration fixed-count idiom, every pass teacher-forced."""
    p = R.make_problem(3, seed=4000 + pair)
    kw = fixed_kw(p, i_max=50)
    X, v, rep, tr = run_traced(p, kw)
    assert rep["total_iterations"] == 50
    check_trace(p, tr, rep, kw)


def test_cfg3_side_by_side_contexts_teacher_forced():
    """Four config-3 pairs run side by side on one GPU (capped PCG grids, one
    host thread each, as bench.py --config 3 runs them); each pair's
    trajectory is teacher-forced against the oracle."""
    import threading

    probs = [R.make_problem(3, seed=4000 + q) for q in (3, 4, 5, 6)]
    out = [None] * len(probs)
    errs = []

    def work(k):
        try:
            kw = fixed_kw(probs[k], i_max=50)
            out[k] = (kw,) + run_traced(probs[k], kw, max_ctas=36)
        except Exception as e:  # surfaced after the join
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(len(probs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    for p, (kw, X, v, rep, tr) in zip(probs, out):
        assert rep["total_iterations"] == 50
        check_trace(p, tr, rep, kw)


@pytest.fixture(scope="module")
def cfg4():
    return R.make_problem(4)


def test_cfg4_full_size_teacher_forced_passes(cfg4):
    """Config 4 (1M source vertices, ~18K nodes): the first registration
    passes of the bench workload, teacher-forced (NN, energies, the solve on
    the oracle's 70K-unknown system, the Anderson combine)."""
    p = cfg4
    assert p.n == 1000000
    kw = fixed_kw(p, i_max=4)
    X, v, rep, tr = run_traced(p, kw)
    assert rep["total_iterations"] == 4
    check_trace(p, tr, rep, kw, threads=4)


def test_cfg4_full_size_step_parity(cfg4):
    """One teacher-forced step at a perturbed iterate: K and B against the
    oracle's fill, x_mm against the oracle's direct solve."""
    p = cfg4
    N = p.graph.node_count
    rows, cols = pattern(p.graph)
    nnzb = len(cols)
    rng = np.random.default_rng(44)
    X = R.identity_transforms(N) + 1e-3 * rng.standard_normal(12 * N)
    prm = O.init_parameters(p)
    prm4 = (prm["alpha"], prm["beta"], prm["nu_a"], prm["nu_r"])
    ctx = R.Context()
    try:
        ctx.set_problem(p)
        g = ctx.step(X, prm4, nnzb=nnzb)
    finally:
        ctx.close()
    o = O.step(p, X, prm4, nnzb)
    bad = np.nonzero(g["index"] != o["index"])[0]
    assert np.all(np.abs(g["sqdist"][bad] - o["sqdist"][bad]) <= 1e-6 * o["sqdist"][bad])
    assert np.max(np.abs(g["energy"] - o["energy"]) / np.abs(o["energy"])) <= 1e-10
    assert np.max(np.abs(g["K"] - o["K"])) <= 1e-12 * np.max(np.abs(o["K"]))
    assert np.max(np.abs(g["B"] - o["B"])) <= 1e-12 * (1 + np.max(np.abs(o["B"])))
    res = np.max(np.abs(o["B"] - bsr_matvec(rows, cols, o["K"], g["Xmm"], N)))
    assert res <= 1e-8 * (1 + np.max(np.abs(o["B"])))
    assert np.max(np.abs(g["Xmm"] - o["Xmm"])) <= 1e-6 * (1 + np.max(np.abs(o["Xmm"])))
