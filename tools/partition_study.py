"""Offline study (CPU, scipy): does the shape of the 148 subdomains change the
PCG iteration count? Same system and stopping rule as tools/precond_study.py
(block Jacobi on the subdomains + additive affine coarse space x19);
partitions: recursive coordinate bisection (the device plan's), RCB followed
by Lloyd relaxation with a size cap (rounder subdomains, same aggregate
numbering), recursive inertial bisection.

    python tools/partition_study.py [iters_before]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.precond_study import affine_space, block_jacobi, pcg, rcb, system, two_level  # noqa: E402
from paper_2206_03410_b200 import registration as R  # noqa: E402


def inertial(pos, ids, parts):
    if parts == 1:
        return [ids]
    lo = parts // 2
    c = pos[ids] - pos[ids].mean(0)
    w, v = np.linalg.eigh(c.T @ c)
    order = ids[np.argsort(c @ v[:, -1], kind="stable")]
    cut = len(order) * lo // parts
    return inertial(pos, order[:cut], lo) + inertial(pos, order[cut:], parts - lo)


def lloyd(pos, subs, cap, rounds):
    """move every node to the nearest subdomain centroid that still has room (greedy by distance gap)"""
    G = len(subs)
    label = np.empty(len(pos), int)
    for g, s in enumerate(subs):
        label[s] = g
    for _ in range(rounds):
        cen = np.array([pos[label == g].mean(0) for g in range(G)])
        d = ((pos[:, None, :] - cen[None, :, :]) ** 2).sum(2)
        order = np.argsort(d.min(1) - np.partition(d, 1, axis=1)[:, 1])  # most decided first
        count = np.zeros(G, int)
        new = np.empty_like(label)
        for j in order:
            for g in np.argsort(d[j]):
                if count[g] < cap:
                    new[j] = g
                    count[g] += 1
                    break
        label = new
    return [np.where(label == g)[0] for g in range(G)]


def count(K, B, x0, pos, subs, N, rtol=1e-13):
    Mf = block_jacobi(K, subs)
    aggs = [np.concatenate(subs[a * 8:(a + 1) * 8]) for a in range(18)] + [np.concatenate(subs[144:])]
    Z = affine_space(pos, aggs, N)
    return pcg(K, B, x0, two_level(K, Mf, Z), rtol)[0]


def main():
    kb = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    p = R.make_problem(2)
    K, B, x0, _ = system(p, kb)
    N = p.graph.node_count
    pos = p.graph.node_positions
    base = rcb(pos, np.arange(N), 148)
    print("RCB                      max rows %2d  %4d iterations" % (max(map(len, base)), count(K, B, x0, pos, base, N)))
    for cap in (22, 24):
        for rounds in (1, 3, 8):
            s = lloyd(pos, base, cap, rounds)
            print("RCB + Lloyd x%d cap %d     max rows %2d  %4d iterations" %
                  (rounds, cap, max(map(len, s)), count(K, B, x0, pos, s, N)))
    s = inertial(pos, np.arange(N), 148)
    print("inertial bisection       max rows %2d  %4d iterations" % (max(map(len, s)), count(K, B, x0, pos, s, N)))


if __name__ == "__main__":
    main()
