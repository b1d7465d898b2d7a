"""Offline study (CPU, scipy): the A-DEF2 two-level preconditioner (Tang et al.
2009: (I - Q K) M^-1 + Q, Q = Psi E^-1 Psi^T, E = Psi^T K Psi) with parts of it
computed from an OLDER system, as the device reuses its preconditioner within
a stage. K_old from the oracle step `iters_before` iterations into a
fixed-count AA run, K_new `lag` iterations later; PCG on K_new.

    python tools/adef_study.py [iters_before] [lag] [rtol]
"""
import os
import sys

import numpy as np
import scipy.linalg as sl

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from precond_study import affine_space, block_jacobi, pcg, rcb, system  # noqa: E402
from paper_2206_03410_b200 import registration as R  # noqa: E402


def adef2(K_e, K_d, Mf, Z):
    """E from K_e, the (I - Q K) factor with K_d"""
    E = (Z.T @ K_e @ Z).toarray()
    Ei = sl.pinvh(E)
    ZtK = (K_d @ Z).T.tocsr()

    def apply(r):
        m = Mf(r)
        return m + Z @ (Ei @ (Z.T @ r - ZtK @ m))
    return apply


def additive(K_e, Mf, Z):
    Ei = sl.pinvh((Z.T @ K_e @ Z).toarray())
    return lambda r: Mf(r) + Z @ (Ei @ (Z.T @ r))


def main():
    kb = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    lag = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    rtol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-13
    p = R.make_problem(2)
    K0, _, _, _ = system(p, kb)
    K1, B, x0, _ = system(p, kb + lag)
    N = p.graph.node_count
    pos = p.graph.node_positions
    subs = rcb(pos, np.arange(N), 148)
    M_old, M_new = block_jacobi(K0, subs), block_jacobi(K1, subs)
    print("K change |K1-K0|/|K1| = %.3e (lag %d)" % (abs(K1 - K0).max() / abs(K1).max(), lag))
    for nagg in (19, 37, 74):
        per = 148 // nagg
        aggs = [np.concatenate(subs[a * per:(a + 1) * per]) for a in range(nagg)]
        Z = affine_space(pos, aggs, N)
        res = {
            "additive, all old": additive(K0, M_old, Z),
            "additive, all fresh": additive(K1, M_new, Z),
            "ADEF2 all fresh": adef2(K1, K1, M_new, Z),
            "ADEF2 M old": adef2(K1, K1, M_old, Z),
            "ADEF2 M,E old": adef2(K0, K1, M_old, Z),
            "ADEF2 M,E,D old": adef2(K0, K0, M_old, Z),
        }
        for k, f in res.items():
            print("x%-3d %-24s %5d iterations" % (nagg, k, pcg(K1, B, x0, f, rtol)[0]))


if __name__ == "__main__":
    main()
