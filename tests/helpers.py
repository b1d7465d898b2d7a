"""Shared fixtures for the parity tests: seeded instances re-derived from the
reference tests (proj/tests/helpers.hpp:89-135, robust_energy_tests.cpp:22-57)
with numpy's PCG64 generators (the reference's libstdc++ distributions are
reproduced bit-exactly only in the C++ KAT programs)."""
import numpy as np

from paper_2206_03410_b200 import registration as R


def make_strip(nx, ny, len_x=1.0, len_y=0.5):
    """helpers.hpp:89-105 triangulated rectangle."""
    pts = np.array([(len_x * i / (nx - 1), len_y * j / (ny - 1), 0.0) for j in range(ny) for i in range(nx)])
    faces = []
    for j in range(ny - 1):
        for i in range(nx - 1):
            a, b, c, d = j * nx + i, j * nx + i + 1, (j + 1) * nx + i, (j + 1) * nx + i + 1
            faces += [(a, b, d), (a, d, c)]
    return pts, np.array(faces, np.int32)


def warp(pts, amplitude=0.05, frequency=1.0, phase=0.0, tilt=0.0):
    """helpers.hpp:124-128"""
    out = pts.copy()
    out[:, 2] += amplitude * np.sin(2 * np.pi * (frequency * pts[:, 0] + phase)) + \
        tilt * amplitude * np.sin(2 * np.pi * pts[:, 1])
    return out


def random_warp(rng, scale=1.0):
    """helpers.hpp:114-122"""
    u = rng.random(4)
    return dict(amplitude=scale * (0.03 + 0.05 * u[0]), frequency=0.6 + 0.9 * u[1], phase=u[2], tilt=0.3 * u[3])


def strip_problem(nx, ny, seed, mult=5.0, amp_scale=1.0, normalize=True):
    rng = np.random.default_rng(seed)
    src, faces = make_strip(nx, ny)
    tgt = warp(src, **random_warp(rng, amp_scale))
    if normalize:
        src, tgt, _, _ = R.normalize_pair(src, tgt)
    edges = R.edges_from_faces(faces, len(src))
    lbar = R.avg_edge_length(src, edges)
    g = R.build_graph(src, edges, mult * lbar)
    return R.Problem(src, tgt, g, lbar, faces)


def random_transforms(N, seed, scale=0.3):
    """robust_energy_tests.cpp:47-57 (A = I + scale U(-1,1), t = scale U(-1,1))."""
    rng = np.random.default_rng(seed)
    X = R.identity_transforms(N).reshape(3, 4 * N)
    for j in range(N):
        A = np.eye(3) + scale * rng.uniform(-1, 1, (3, 3))
        t = scale * rng.uniform(-1, 1, 3)
        for c in range(3):
            for r in range(3):
                X[c, 4 * j + r] = A[c, r]
            X[c, 4 * j + 3] = t[c]
    return X.reshape(-1)


def bbox_diag(p):
    return float(np.linalg.norm(p.max(0) - p.min(0)))
