"""Offline study (CPU, scipy): PCG iteration counts on the real config-2
normal equations for candidate preconditioners. Drives the choice of the
device preconditioner; not part of the product."""
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.linalg as sl

sys.path.insert(0, ".")
from oracle import binding as O
from paper_2206_03410_b200 import registration as R

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
p = R.make_problem(cfg, scale=scale)
g = p.graph
N = g.node_count
rp, cols = R.bsr_pattern(g)
nnzb = len(cols)
prm0 = O.init_parameters(p)
prm = np.array([prm0["alpha"], prm0["beta"], prm0["nu_a"], prm0["nu_r"]])
X = R.identity_transforms(N) if hasattr(R, "identity_transforms") else None
X = np.asarray(X, dtype=np.float64).ravel()
for it in range(6):
    s = O.step(p, X, prm, nnzb)
    Xprev, X = X, s["Xmm"]
s = O.step(p, X, prm, nnzb)
Kv, B = s["K"], s["B"]
# scalar 4N CSR
rows, cc, vals = [], [], []
for a in range(N):
    for k in range(rp[a], rp[a + 1]):
        b = cols[k]
        blk = Kv[16 * k:16 * k + 16].reshape(4, 4)
        for r in range(4):
            for c in range(4):
                rows.append(4 * a + r)
                cc.append(4 * b + c)
                vals.append(blk[r, c])
K = sp.csr_matrix((vals, (rows, cc)), shape=(4 * N, 4 * N))
Bm = B.reshape(3, 4 * N).T  # column-major 4N x 3
X0 = X.reshape(3, 4 * N).T  # warm start = current iterate
xs = sp.linalg.spsolve(K.tocsc(), Bm)
print(f"config {cfg}: N={N} nnzb={nnzb} |B|max={np.abs(Bm).max():.3e}")

pos = g.node_positions


def rcb(idx, parts):
    if parts == 1:
        return [idx]
    pts = pos[idx]
    ax = np.argmax(pts.max(0) - pts.min(0))
    o = idx[np.argsort(pts[:, ax], kind="stable")]
    left = parts // 2
    cut = int(round(len(o) * left / parts))
    return rcb(o[:cut], left) + rcb(o[cut:], parts - left)


def pcg(apply_m, x0, rtol=1e-13, maxit=5000):
    x = x0.copy()
    r = Bm - K @ x
    tol = rtol * (1 + np.abs(Bm).max())
    z = apply_m(r)
    pv = z.copy()
    rz = np.sum(r * z, 0)
    for it in range(maxit):
        if np.abs(r).max() <= tol:
            return it, x
        q = K @ pv
        al = rz / np.sum(pv * q, 0)
        x += al * pv
        r -= al * q
        z = apply_m(r)
        rzn = np.sum(r * z, 0)
        pv = z + (rzn / rz) * pv
        rz = rzn
    return maxit, x


# block Jacobi 4x4
Minv = np.zeros((N, 4, 4))
Kd = K.todia() if False else None
Kc = K.tocsr()
for a in range(N):
    Minv[a] = np.linalg.inv(Kc[4 * a:4 * a + 4, 4 * a:4 * a + 4].toarray())


def bj(r):
    return np.einsum("nij,njc->nic", Minv, r.reshape(N, 4, 3)).reshape(4 * N, 3)


def coarse_space(groups):
    cols_, rr, vv = [], [], []
    for gi, nodes in enumerate(groups):
        ctr = pos[nodes].mean(0)
        for k in range(4):
            col = 4 * gi + k
            for j in nodes:
                if k < 3:
                    rr += [4 * j + k, 4 * j + 3]
                    vv += [1.0, pos[j, k] - ctr[k]]
                    cols_ += [col, col]
                else:
                    rr.append(4 * j + 3)
                    vv.append(1.0)
                    cols_.append(col)
    Psi = sp.csr_matrix((vv, (rr, cols_)), shape=(4 * N, 4 * len(groups)))
    K0 = (Psi.T @ K @ Psi).toarray()
    K0i = np.linalg.pinv(K0, rcond=1e-12)
    return Psi, K0i


def two_level(base, Psi, K0i):
    return lambda r: base(r) + Psi @ (K0i @ (Psi.T @ r))


def subdomain_exact(parts):
    inv = []
    for nodes in parts:
        ix = np.concatenate([4 * nodes[:, None] + np.arange(4)[None, :]]).ravel()
        inv.append((ix, np.linalg.inv(Kc[ix][:, ix].toarray())))

    def f(r):
        z = np.zeros_like(r)
        for ix, Ai in inv:
            z[ix] = Ai @ r[ix]
        return z
    return f


res = []
it, x = pcg(bj, X0)
print("block-Jacobi 4x4:", it, "err", np.abs(x - xs).max())
for nparts, per_agg in [(148, 8), (148, 4), (148, 2), (148, 1), (296, 1), (592, 1)]:
    parts = rcb(np.arange(N), nparts)
    groups = [np.concatenate(parts[i:i + per_agg]) for i in range(0, nparts, per_agg)]
    Psi, K0i = coarse_space(groups)
    it, x = pcg(two_level(bj, Psi, K0i), X0)
    it2, _ = pcg(two_level(subdomain_exact(parts), Psi, K0i), X0)
    print(f"parts {nparts} aggregates {len(groups)} (nc={4 * len(groups)}): BJ4+coarse {it}  subdomain-exact+coarse {it2}")
