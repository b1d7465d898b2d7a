"""Teacher-forced parity of a whole device trajectory (test infrastructure).

The device run records every evaluated pass (Context(record_passes=3),
nrr_ctx_trace): the iterate X_k it was evaluated at, its correspondences,
energies, the accept/revert decision and, on accepted passes, the solve's
x_mm. At EVERY X_k the CPU oracle re-runs the reference step
(find_correspondences + evaluate_energy + fill + solve, energy.hpp:28-254)
and the Anderson combine (anderson.hpp:22-46) on the device's own history, so
each stage of the map X_k -> X_{k+1} is compared against the reference at the
same input, independent of floating-point trajectory chaos:

  NN       indices identical except distance ties within 1e-6 relative
  energy   align / reg / rot / total within 1e-6 relative (north_star)
  solve    the device x_mm meets the reference's own acceptance bar on the
           ORACLE's system: ||B - K x_mm||_inf <= 1e-8 (1 + ||B||_inf)
           (energy.hpp:245)
  AA       the device's next iterate equals the oracle's anderson_combine of
           the device history (window per anderson.hpp:50-73, solver.hpp:267-270)
  revert   the device's safeguard decision equals the reference rule
           (solver.hpp:239) applied to the oracle energies, except inside the
           1e-6 tolerance band around a tie
  revert   after a revert the next iterate is x_mm of the last accepted pass
           (solver.hpp:244-248), bit for bit
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from oracle import binding as O
from paper_2206_03410_b200 import registration as R

NN_TIE_REL = 1e-6
E_REL = 1e-6
SOLVE_BAR = 1e-8


def bsr_matvec(rows, cols, Kvals, X, N):
    """K x for the 3 coordinate columns (X 12N reference layout, K BSR values
    16 row-major doubles per block in pattern order)."""
    Kb = Kvals.reshape(-1, 4, 4)
    x = X.reshape(3, N, 4)
    y = np.zeros((3, N, 4))
    for c in range(3):
        contrib = np.einsum("kij,kj->ki", Kb, x[c, cols, :])
        np.add.at(y[c], rows, contrib)
    return y.reshape(-1)


def pattern(graph):
    row_ptr, cols = R.bsr_pattern(graph)
    rows = np.repeat(np.arange(graph.node_count), np.diff(row_ptr))
    return rows, cols


def check_trace(p, trace, report, cfg_kw, threads=16, landmarks=None, log=print):
    """Checks a device trace (Context.trace()) against the oracle at every
    pass; returns a dict of the worst deviations seen."""
    N = p.graph.node_count
    rows, cols = pattern(p.graph)
    nnzb = len(cols)
    stages = report["stages"]
    aa_m = cfg_kw.get("aa_window", 5)
    ocfg = O.config(**cfg_kw) if landmarks else None

    def prm_of(k):
        s = stages[trace[k]["stage"]]
        return (s["alpha"], s["beta"], s["nu_a"], s["nu_r"])

    def lm_w(k):
        return 1.0 if (landmarks and trace[k]["stage"] == 0) else 0.0

    def oracle_pass(k):
        t = trace[k]
        o = O.step(p, t["X"], prm_of(k), nnzb, landmark_weight=lm_w(k), cfg=ocfg, want_solve=False)
        v = O.deform(p, t["X"])
        return o, v

    with ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(oracle_pass, range(len(trace))))

    worst = {"nn_ties": 0, "e_rel": 0.0, "solve_res": 0.0, "aa_rel": 0.0,
             "passes": len(trace), "accepted": 0, "reverted": 0, "decisions_in_tie_band": 0}
    # --- per-pass step parity
    for k, (t, (o, v)) in enumerate(zip(trace, res)):
        # correspondences
        gi, oi = t["index"], o["index"]
        bad = np.nonzero(gi != oi)[0]
        if len(bad):
            dg = np.sum((v[bad] - p.target[gi[bad]]) ** 2, axis=1)
            do = np.sum((v[bad] - p.target[oi[bad]]) ** 2, axis=1)
            assert np.all(np.abs(dg - do) <= NN_TIE_REL * np.maximum(do, 1e-300)), \
                f"pass {k}: {len(bad)} correspondences differ beyond a tie"
            worst["nn_ties"] = max(worst["nn_ties"], len(bad))
        # energies (align, reg, rot, total)
        eo, eg = o["energy"], t["energy"]
        scale = np.maximum(np.abs(eo), 1e-12 * abs(eo[3]))
        r = np.max(np.abs(eg - eo) / np.maximum(scale, 1e-300))
        assert r <= E_REL, f"pass {k}: energies {eg} vs oracle {eo} (rel {r:.2e})"
        worst["e_rel"] = max(worst["e_rel"], float(r))
        # the solve: device x_mm against the oracle's own system
        if t["Xmm"] is not None:
            worst["accepted"] += 1
            Bo = o["B"]
            res_inf = np.max(np.abs(Bo - bsr_matvec(rows, cols, o["K"], t["Xmm"], N)))
            bar = SOLVE_BAR * (1.0 + np.max(np.abs(Bo)))
            assert res_inf <= bar, f"pass {k}: ||B - K x_mm|| = {res_inf:.3e} > {bar:.3e}"
            worst["solve_res"] = max(worst["solve_res"], float(res_inf / (1.0 + np.max(np.abs(Bo)))))
        else:
            worst["reverted"] += 1

    # --- decisions, Anderson combine and the revert path (solver.hpp:219-289)
    stage = -1
    hist_g, hist_f = [], []
    e_prev = np.inf
    current_is_aa = False
    last_xmm = None
    for k, t in enumerate(trace):
        if t["stage"] != stage:  # window.reset(); e_prev = inf (solver.hpp:219-220)
            stage = t["stage"]
            hist_g, hist_f = [], []
            e_prev = np.inf
            current_is_aa = False
        e_acc = res[k][0]["energy"][3] + (lm_w(k) * t["E_landmark"] if lm_w(k) else 0.0)
        want_revert = e_acc > e_prev and current_is_aa
        if want_revert != t["reverted"]:
            assert abs(e_acc - e_prev) <= E_REL * abs(e_prev), \
                f"pass {k}: device {'reverted' if t['reverted'] else 'accepted'}, reference rule says otherwise " \
                f"(E {e_acc!r} vs E_prev {e_prev!r})"
            worst["decisions_in_tie_band"] += 1
        if t["reverted"]:
            current_is_aa = False
            assert k + 1 < len(trace), "a revert must be followed by a re-evaluation"
            assert np.array_equal(trace[k + 1]["X"], last_xmm), f"pass {k + 1}: not re-evaluated at x_mm"
            continue
        e_prev = e_acc
        g = t["Xmm"]
        last_xmm = g
        hist_g.append(g)
        hist_f.append(g - t["X"])
        if len(hist_g) > aa_m + 1:
            hist_g.pop(0)
            hist_f.pop(0)
        extrap = aa_m > 0 and len(hist_g) > 1
        current_is_aa = extrap
        if k + 1 < len(trace):
            if extrap:
                want, _ = O.anderson_combine(np.array(hist_g), np.array(hist_f), aa_m)
            else:
                want = g
            got = trace[k + 1]["X"]
            d = np.max(np.abs(got - want)) / (1.0 + np.max(np.abs(want)))
            worst["aa_rel"] = max(worst["aa_rel"], float(d))
            assert d <= 1e-8, f"pass {k + 1}: next iterate differs from the reference combine by {d:.3e}"
    log("trace check: %s" % worst)
    return worst
