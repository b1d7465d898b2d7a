"""Offline study: geometric nested dissection of the node graph and the
symbolic Cholesky cost (fill, flops, front sizes, tree depth)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2206_03410_b200 import registration as R

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 32
p = R.make_problem(cfg)
g = p.graph
N = g.node_count
pos = g.node_positions
adj = [set() for _ in range(N)]
for a, b in g.edges:
    adj[a].add(b)
    adj[b].add(a)

order = []
levels = []


def nd(idx, depth):
    if len(idx) <= leaf:
        order.extend(idx.tolist())
        levels.append((depth, len(idx), "leaf"))
        return
    pts = pos[idx]
    ax = np.argmax(pts.max(0) - pts.min(0))
    o = idx[np.argsort(pts[:, ax], kind="stable")]
    half = len(o) // 2
    L, Rr = set(o[:half].tolist()), set(o[half:].tolist())
    # separator: nodes of the smaller side with a neighbour on the other side (greedy vertex cover)
    sep = set()
    for a in L:
        if any(b in Rr for b in adj[a]):
            sep.add(a)
    L -= sep
    nd(np.array(sorted(L), dtype=int), depth + 1)
    nd(np.array(sorted(Rr), dtype=int), depth + 1)
    order.extend(sorted(sep))
    levels.append((depth, len(sep), "sep"))


nd(np.arange(N), 0)
perm = np.array(order)
inv = np.empty(N, int)
inv[perm] = np.arange(N)
# symbolic elimination on the node graph (quotient not needed: exact fill via row structure)
struct = [set(inv[b] for b in adj[perm[i]] if inv[b] > i) for i in range(N)]
parent = np.full(N, -1)
nnz = 0
flops = 0.0
colcount = np.zeros(N, int)
for i in range(N):
    s = struct[i]
    colcount[i] = len(s)
    if s:
        par = min(s)
        parent[i] = par
        struct[par] |= (s - {par})
    c = 4 * len(s) + 4  # scalar column count of the 4 columns of node i (approx)
    nnz += 4 * c
    flops += 4 * c * c
# depth of etree
depth = np.zeros(N, int)
for i in range(N - 1, -1, -1):
    if parent[i] >= 0:
        depth[i] = depth[parent[i]] + 1
print(f"config {cfg}: N={N} edges={len(g.edges)} leaf={leaf}")
print(f"scalar nnz(L) ~ {nnz/1e6:.2f} M ({nnz*8/1e6:.1f} MB), factor flops ~ {flops/1e6:.1f} MFLOP, etree height {depth.max()}")
seps = sorted([l for l in levels if l[2] == "sep"])
by = {}
for d, n, _ in levels:
    by.setdefault(d, []).append(n)
for d in sorted(by):
    print(d, len(by[d]), "max", max(by[d]), "sum", sum(by[d]))
print("max front (nodes):", colcount.max() + 1)
