"""Offline study (CPU, scipy): PCG iterations per MM pass with the warm start
the device uses (x0 = current iterate) versus a Galerkin-projected initial
guess over the previous passes' solutions (Fischer's method for successive
right-hand sides: x0 = x + W (W^T K W)^-1 W^T (B - K x), W = differences of
the last m solutions). Plain-MM sequence on config 2 from the oracle, the
additive two-level preconditioner (subdomain block Jacobi over 148 RCB
subdomains + affine coarse space over 19 aggregates), stop at
max|r| <= rtol (1 + max|B|).

    python tools/recycle_study.py [passes] [m]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import binding as O  # noqa: E402
from paper_2206_03410_b200 import registration as R  # noqa: E402
from tools.precond_study import affine_space, block_jacobi, pcg, rcb, two_level  # noqa: E402

import scipy.sparse as sp  # noqa: E402


def kmat(p, Kflat):
    row_ptr, cols = R.bsr_pattern(p.graph)
    N = p.graph.node_count
    Kb = Kflat.reshape(-1, 4, 4)
    rows = np.repeat(np.arange(N), np.diff(row_ptr))
    I = (4 * rows[:, None, None] + np.arange(4)[None, :, None]).repeat(4, 2)
    J = (4 * cols[:, None, None] + np.arange(4)[None, None, :]).repeat(4, 1)
    return sp.csr_matrix((Kb.ravel(), (I.ravel(), J.ravel())), shape=(4 * N, 4 * N))


def main():
    passes = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    rtol = 1e-13
    p = R.make_problem(2)
    N = p.graph.node_count
    pos = p.graph.node_positions
    prm0 = O.init_parameters(p)
    cfg = O.config(nu_a_init=prm0["nu_a"], nu_a_min=prm0["nu_a"], nu_r_init=prm0["nu_r"], eps=1e-300, i_max=1)
    _, _, rep = O.register(p, cfg)
    st = rep["stages"][0]
    prm = (st["alpha"], st["beta"], st["nu_a"], st["nu_r"])
    nnzb = int(R.bsr_pattern(p.graph)[0][-1])
    X = R.identity_transforms(N)
    subs = rcb(pos, np.arange(N), 148)
    aggs = [np.concatenate(subs[a * 8:(a + 1) * 8]) for a in range(18)] + [np.concatenate(subs[144:])]
    Z = affine_space(pos, aggs, N)
    hist = []  # previous solutions (4N x 3)
    print("pass  warm  galerkin(m=%d)  |r0| warm  |r0| galerkin" % m)
    for k in range(passes):
        o = O.step(p, X, prm, nnzb)
        K = kmat(p, o["K"])
        B = o["B"].reshape(3, 4 * N).T
        x0 = X.reshape(3, 4 * N).T.copy()
        M = two_level(K, block_jacobi(K, subs), Z)
        it_w, xs = pcg(K, B, x0, M, rtol)
        r_w = np.abs(B - K @ x0).max()
        it_g, r_g = it_w, r_w
        if len(hist) >= 2:
            W = np.stack([hist[-1 - j] - hist[-2 - j] for j in range(min(m, len(hist) - 1))], axis=-1)  # 4N x 3 x q
            xg = x0.copy()
            for c in range(3):  # per column (the three RHS share K)
                Wc = W[:, c, :]
                r = B[:, c] - K @ x0[:, c]
                KW = K @ Wc
                G = Wc.T @ KW
                coef = np.linalg.lstsq(G, Wc.T @ r, rcond=1e-14)[0]
                xg[:, c] = x0[:, c] + Wc @ coef
            r_g = np.abs(B - K @ xg).max()
            it_g, _ = pcg(K, B, xg, M, rtol)
        print("%4d  %4d  %4d           %.2e  %.2e" % (k, it_w, it_g, r_w, r_g))
        hist.append(xs.copy())
        X = xs.T.reshape(-1).copy()  # plain MM: the next iterate is the solve


if __name__ == "__main__":
    main()
