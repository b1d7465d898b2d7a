"""Offline study (CPU, scipy): PCG iteration counts on a real config-2 system
for preconditioner variants, to decide where the device PCG's iteration count
can go. K, B come from the oracle's step at an iterate of a fixed-count AA run
(10 iterations in), warm start x0 = that iterate (the device solve's warm
start), stop at max|r| <= rtol * (1 + max|B|) as pcg.cu does.

    python tools/precond_study.py [iters_before] [rtol]
"""
import os
import sys
import time

import numpy as np
import scipy.linalg as sl
import scipy.sparse as sp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import binding as O  # noqa: E402
from paper_2206_03410_b200 import registration as R  # noqa: E402


def rcb(pos, ids, parts):
    """recursive coordinate bisection into `parts` groups (sizes proportional)"""
    if parts == 1:
        return [ids]
    lo = parts // 2
    ext = pos[ids].max(0) - pos[ids].min(0)
    ax = int(np.argmax(ext))
    order = ids[np.argsort(pos[ids, ax], kind="stable")]
    cut = len(order) * lo // parts
    return rcb(pos, order[:cut], lo) + rcb(pos, order[cut:], parts - lo)


def system(p, k_before):
    prm = O.init_parameters(p)
    cfg = O.config(nu_a_init=prm["nu_a"], nu_a_min=prm["nu_a"], nu_r_init=prm["nu_r"], eps=1e-300, i_max=k_before)
    X, _, rep = O.register(p, cfg)
    st = rep["stages"][0]
    row_ptr, cols = R.bsr_pattern(p.graph)
    nnzb = int(row_ptr[-1])
    o = O.step(p, X, (st["alpha"], st["beta"], st["nu_a"], st["nu_r"]), nnzb)
    N = p.graph.node_count
    Kb = o["K"].reshape(-1, 4, 4)
    rows = np.repeat(np.arange(N), np.diff(row_ptr))
    I = (4 * rows[:, None, None] + np.arange(4)[None, :, None]).repeat(4, 2)
    J = (4 * cols[:, None, None] + np.arange(4)[None, None, :]).repeat(4, 1)
    K = sp.csr_matrix((Kb.ravel(), (I.ravel(), J.ravel())), shape=(4 * N, 4 * N))
    B = o["B"].reshape(3, 4 * N).T  # column-major 4N x 3
    x0 = X.reshape(3, 4 * N).T
    xs = o["Xmm"].reshape(3, 4 * N).T
    return K, B, x0, xs


def pcg(K, B, x0, apply_M, rtol, maxit=5000):
    x = x0.copy()
    r = B - K @ x
    bar = rtol * (1 + np.abs(B).max())
    z = apply_M(r)
    pdir = z.copy()
    rz = np.sum(r * z, axis=0)
    for it in range(1, maxit + 1):
        q = K @ pdir
        alpha = rz / np.sum(pdir * q, axis=0)
        x += alpha * pdir
        r -= alpha * q
        if np.abs(r).max() <= bar:
            return it, x
        z = apply_M(r)
        rz_new = np.sum(r * z, axis=0)
        pdir = z + (rz_new / rz) * pdir
        rz = rz_new
    return maxit, x


def block_jacobi(K, groups):
    invs = []
    for g in groups:
        idx = (4 * g[:, None] + np.arange(4)).ravel()
        invs.append((idx, np.linalg.inv(K[idx][:, idx].toarray())))

    def apply(r):
        z = np.zeros_like(r)
        for idx, Ai in invs:
            z[idx] = Ai @ r[idx]
        return z
    return apply


def affine_space(pos, aggs, n):
    """4 modes per aggregate: [e_k; p - c] (k < 3) and e_3 (pcg.cu:62-68)"""
    cols = []
    for g in aggs:
        c = pos[g].mean(0)
        for k in range(4):
            v = np.zeros(4 * n)
            for j in g:
                if k < 3:
                    v[4 * j + k] = 1.0
                    v[4 * j + 3] = pos[j][k] - c[k]
                else:
                    v[4 * j + 3] = 1.0
            cols.append(v)
    return sp.csc_matrix(np.array(cols).T)


def two_level(K, Mf, Z, mode="additive"):
    E = (Z.T @ K @ Z).toarray()
    Ei = sl.pinvh(E)
    KZ = K @ Z

    if mode == "additive":
        return lambda r: Mf(r) + Z @ (Ei @ (Z.T @ r))

    def adef1(r):  # M^-1 (I - K Q) r + Q r  (Tang et al. A-DEF1)
        y = Ei @ (Z.T @ r)
        return Mf(r - KZ @ y) + Z @ y

    def adef2(r):  # (I - Q K) M^-1 r + Q r  (Tang et al. A-DEF2): M^-1 r + Z E^-1 Z^T (r - K M^-1 r)
        m = Mf(r)
        return m + Z @ (Ei @ (Z.T @ (r - K @ m)))
    return adef1 if mode == "adef1" else adef2


def coarse_start(K, B, x0, Z):
    """x0 + Q r0: the initial residual orthogonal to the coarse space (A-DEF2's start)"""
    E = (Z.T @ K @ Z).toarray()
    return x0 + Z @ sl.solve(E, Z.T @ (B - K @ x0), assume_a="pos")


def main():
    kb = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    rtol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-13
    p = R.make_problem(2)
    t0 = time.time()
    K, B, x0, xs = system(p, kb)
    N = p.graph.node_count
    pos = p.graph.node_positions
    print("N=%d nnz=%d system in %.1fs" % (N, K.nnz, time.time() - t0))
    subs = rcb(pos, np.arange(N), 148)
    Mf = block_jacobi(K, subs)
    Mnode = block_jacobi(K, [np.array([j]) for j in range(N)])
    res = {}
    res["node block Jacobi"] = pcg(K, B, x0, Mnode, rtol)[0]
    res["subdomain BJ (148)"] = pcg(K, B, x0, Mf, rtol)[0]
    for nagg in (19, 37, 74, 148):
        per = 148 // nagg
        aggs = [np.concatenate(subs[a * per:(a + 1) * per]) for a in range(nagg)]
        Z = affine_space(pos, aggs, N)
        res["BJ + additive affine x%d" % nagg] = pcg(K, B, x0, two_level(K, Mf, Z), rtol)[0]
        res["BJ + ADEF1 affine x%d" % nagg] = pcg(K, B, x0, two_level(K, Mf, Z, "adef1"), rtol)[0]
        res["BJ + ADEF2 affine x%d" % nagg] = pcg(K, B, x0, two_level(K, Mf, Z, "adef2"), rtol)[0]
        res["BJ + ADEF2 affine x%d, Q start" % nagg] = pcg(K, B, coarse_start(K, B, x0, Z), two_level(K, Mf, Z, "adef2"), rtol)[0]
    # overlapping subdomains (one ring of neighbours), additive Schwarz + affine x19
    nb = [set() for _ in range(N)]
    for a, b in p.graph.edges:
        nb[a].add(b)
        nb[b].add(a)
    over = [np.array(sorted(set(g) | set().union(*[nb[j] for j in g]))) for g in subs]
    Mo = block_jacobi(K, over)
    aggs = [np.concatenate(subs[a * 8:(a + 1) * 8]) for a in range(18)] + [np.concatenate(subs[144:])]
    Z19 = affine_space(pos, aggs, N)
    res["overlap-1 AS + additive affine x19"] = pcg(K, B, x0, two_level(K, Mo, Z19), rtol)[0]
    for k, v in res.items():
        print("%-40s %5d iterations" % (k, v))


if __name__ == "__main__":
    main()
