"""CPU-only checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/nrr_cuda.h declares (no compute calls without a GPU),
the product's setup code reproduces the oracle's graph construction bit for
bit, and the synthetic configs are deterministic."""
import os
import re

import numpy as np
import pytest

from oracle import binding as O
from paper_2206_03410_b200 import capi
from paper_2206_03410_b200 import registration as R
from tests.helpers import make_strip, strip_problem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "nrr_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nrr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = capi.load()
    names = _declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    # and the Python binding covers the same set
    assert set(names) == set(capi.EXPORTED)


def test_no_device_fails_loudly():
    """Without a GPU the device entry points raise instead of falling back."""
    if R.has_device():
        pytest.skip("a device is present")
    with pytest.raises(capi.CudaError):
        R.Context()


@pytest.mark.parametrize("nx,ny,mult", [(12, 6, 5.0), (24, 10, 4.0), (40, 16, 3.0), (60, 24, 5.0)])
def test_build_graph_matches_oracle_strips(nx, ny, mult):
    src, faces = make_strip(nx, ny)
    rng = np.random.default_rng(nx)
    src = src + rng.uniform(-0.004, 0.004, src.shape)
    e = R.edges_from_faces(faces, len(src))
    assert np.array_equal(e, O.edges_from_faces(faces, len(src)))
    lbar = R.avg_edge_length(src, e)
    g = R.build_graph(src, e, mult * lbar)
    go = O.build_graph(src, e, mult * lbar)
    for k, v in go.items():
        assert np.array_equal(getattr(g, k), v), k


@pytest.mark.parametrize("config,scale", [(0, 0.5), (2, 0.05), (1, 0.02), (3, 0.05), (4, 0.004)])
def test_synthetic_configs_graph_parity(config, scale):
    src, faces, tgt = R.synth(config, scale=scale)
    src2, faces2, tgt2 = R.synth(config, scale=scale)
    assert np.array_equal(src, src2) and np.array_equal(tgt, tgt2)  # deterministic
    s, t, sc, ctr = R.normalize_pair(src, tgt)
    allp = np.vstack([s, t])
    assert abs(np.linalg.norm(allp.max(0) - allp.min(0)) - 1.0) < 1e-12
    if faces is not None:
        e = R.edges_from_faces(faces, len(s))
        eo = O.edges_from_faces(faces, len(s))
    else:
        e = R.knn_edges(s, 6)
        eo = O.knn_edges(s, 6)
    assert np.array_equal(e, eo)
    lbar = R.avg_edge_length(s, e)
    g = R.build_graph(s, e, R.GRAPH_MULT[config] * lbar)
    go = O.build_graph(s, e, R.GRAPH_MULT[config] * lbar)
    for k, v in go.items():
        assert np.array_equal(getattr(g, k), v), k


def test_graph_invariants():
    """helpers.hpp:172-206: weights positive and normalised, distances < R,
    every edge shared by an influenced point, mean reg weight 1."""
    p = strip_problem(30, 14, seed=606, mult=3.5)
    g = p.graph
    off = g.infl_offsets
    for i in range(p.n):
        w = g.infl_weights[off[i]:off[i + 1]]
        assert len(w) > 0 and np.all(w > 0) and abs(w.sum() - 1) < 1e-10
        assert np.all(g.infl_dist[off[i]:off[i + 1]] < g.radius)
    shared = set()
    for i in range(p.n):
        nodes = sorted(g.infl_nodes[off[i]:off[i + 1]])
        for a in range(len(nodes)):
            for b in range(a + 1, len(nodes)):
                shared.add((nodes[a], nodes[b]))
    assert {tuple(e) for e in g.edges} == shared
    assert abs(g.reg_weights.mean() - 1.0) < 1e-10


def test_setup_errors_map_to_reference_classes():
    with pytest.raises(capi.ConfigError):
        R.build_graph(np.zeros((0, 3)), np.zeros((0, 2), np.int32), 1.0)  # deformation_graph.hpp:159
    with pytest.raises(capi.ConfigError):
        R.build_graph(np.zeros((2, 3)), np.array([[0, 1]], np.int32), -1.0)  # :160
    with pytest.raises(capi.NumericalError):
        R.edges_from_faces(np.array([[0, 1, 5]], np.int32), 3)  # surface.hpp:56-57
    with pytest.raises(capi.ConfigError):
        R.knn_edges(np.zeros((3, 3)), 3)  # surface.hpp:73
    with pytest.raises(capi.NumericalError):
        R.normalize_pair(np.zeros((2, 3)), np.zeros((2, 3)))  # surface.hpp:138-139


def test_knn_edges_ties_match_exhaustive():
    """Lattice points: many equal distances; (distance, index) order wins."""
    g = np.arange(5, dtype=np.float64)
    pts = np.array(np.meshgrid(g, g, g, indexing="ij")).reshape(3, -1).T.copy()
    pts = pts[np.random.default_rng(1).permutation(len(pts))]
    assert np.array_equal(R.knn_edges(pts, 6), O.knn_edges(pts, 6))


def test_limited_geodesic_matches_dijkstra():
    """limited_geodesic (geodesic.hpp:22-84): the vertices whose edge-graph
    distance from the source is < R, ascending, with their distances; checked
    against scipy's Dijkstra restricted to the Euclidean ball's connected
    component (the reference's BFS-then-Dijkstra construction)."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import dijkstra
    from tests.helpers import make_strip

    pts, faces = make_strip(20, 9)
    pts = pts + np.random.default_rng(3).normal(0, 0.01, pts.shape)
    e = R.edges_from_faces(faces, len(pts))
    lbar = R.avg_edge_length(pts, e)
    for src, mult in ((0, 3.0), (97, 4.5), (150, 2.0)):
        radius = mult * lbar
        idx, dist = R.limited_geodesic(pts, e, src, radius)
        ball = np.linalg.norm(pts - pts[src], axis=1) < radius
        w = np.linalg.norm(pts[e[:, 0]] - pts[e[:, 1]], axis=1)
        keep = ball[e[:, 0]] & ball[e[:, 1]]
        A = sp.coo_matrix((w[keep], (e[keep, 0], e[keep, 1])), shape=(len(pts), len(pts)))
        d = dijkstra(A, directed=False, indices=src)
        expect = np.nonzero(d < radius)[0]
        assert np.array_equal(idx, expect)
        assert np.allclose(dist, d[expect], rtol=1e-14, atol=1e-15)
        assert idx[0] <= src <= idx[-1] and dist[np.searchsorted(idx, src)] == 0.0
    with pytest.raises(capi.ConfigError):
        R.limited_geodesic(pts, e, len(pts), 1.0)
    with pytest.raises(capi.ConfigError):
        R.limited_geodesic(pts, e, 0, -1.0)
