"""Device graph setup against the host build and the oracle.

The device kNN connectivity (knn_edges, surface.hpp:70-94) and the device
deformation-graph build (build_graph, deformation_graph.hpp:157-210: PCA
order, limited geodesic balls, the node sweep, influence weights, edges and
the regularization table) must equal the host restatement bit for bit; the
host restatement is itself bitwise equal to the oracle (test_cpu_boundary.py),
which the smaller cases here re-check directly. Sizes reach the headline
(config 2, 99,856 vertices) and config 4 (1M vertices).
"""
import time

import numpy as np
import pytest

from oracle import binding as O
from paper_2206_03410_b200 import capi
from paper_2206_03410_b200 import registration as R
from tests.helpers import make_strip

pytestmark = pytest.mark.gpu


def _graph_equal(a, b):
    for f in ("node_indices", "node_positions", "edges", "infl_offsets", "infl_nodes", "infl_weights", "infl_dist",
              "reg_pairs", "reg_weights"):
        x, y = [o[f] if isinstance(o, dict) else getattr(o, f) for o in (a, b)]
        assert x.shape == y.shape, (f, x.shape, y.shape)
        assert np.array_equal(x.view(np.uint8) if x.dtype == np.float64 else x,
                              y.view(np.uint8) if y.dtype == np.float64 else y), f  # bitwise
    return True


@pytest.mark.parametrize("n,k,kind", [(200, 1, "cloud"), (1000, 6, "cloud"), (5000, 6, "cloud"), (3000, 16, "cloud"),
                                      (2000, 32, "cloud"), (1331, 6, "lattice"), (800, 6, "duplicates"),
                                      (4000, 6, "flat")])
def test_knn_edges_device_matches_oracle(n, k, kind):
    rng = np.random.default_rng(n + k)
    if kind == "cloud":
        pts = rng.uniform(-1, 1, (n, 3))
    elif kind == "lattice":  # every distance tied many times: ties resolve to the smaller index
        g = np.arange(11, dtype=float)
        pts = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
        pts = pts[rng.permutation(len(pts))]
    elif kind == "duplicates":
        base = rng.uniform(-1, 1, (n // 4, 3))
        pts = np.repeat(base, 4, axis=0)[rng.permutation(n)]
    else:
        pts = np.column_stack([rng.uniform(0, 2, n), rng.uniform(0, 1, n), np.zeros(n)])
    eg = R.knn_edges(pts, k, device=0)
    eo = O.knn_edges(pts, k)
    assert np.array_equal(eg, eo)


@pytest.mark.parametrize("config", [0, 1, 3])
def test_knn_edges_device_synthetic_configs(config):
    """The point-cloud configs' connectivity (kNN k=6) at full size."""
    src, faces, tgt = R.synth(config, 4000 if config == 3 else None)
    src, tgt, _, _ = R.normalize_pair(src, tgt)
    eg = R.knn_edges(src, 6, device=0)
    eh = R.knn_edges(src, 6, device=False)
    assert np.array_equal(eg, eh)
    if len(src) <= 20000:
        assert np.array_equal(eg, O.knn_edges(src, 6))


def test_knn_edges_device_errors():
    with pytest.raises(capi.ConfigError):
        R.knn_edges(np.zeros((3, 3)), 3, device=0)  # surface.hpp:73
    with pytest.raises(capi.ConfigError):
        R.knn_edges(np.zeros((100, 3)), 0, device=0)
    with pytest.raises(capi.ConfigError):
        R.knn_edges(np.random.default_rng(1).uniform(size=(100, 3)), 33, device=0)  # device k cap


@pytest.mark.parametrize("slow", [False, True])
@pytest.mark.parametrize("nx,ny,mult", [(8, 5, 2.0), (24, 10, 4.0), (40, 17, 5.7), (30, 30, 9.0), (60, 7, 1.5),
                                        (70, 70, 32.0)])
def test_build_graph_device_strips(nx, ny, mult, slow, monkeypatch):
    """(70, 70, 32): balls of ~3000 vertices overflow the shared-memory ball
    path, so the build reruns on the global-memory path; slow=True forces
    the host-stepped sweep (NRR_GRAPH_SLOW_SWEEP)."""
    if slow:
        monkeypatch.setenv("NRR_GRAPH_SLOW_SWEEP", "1")
    src, faces = make_strip(nx, ny)
    src = src + np.random.default_rng(nx).normal(0, 0.01, src.shape)
    e = R.edges_from_faces(faces, len(src))
    lbar = R.avg_edge_length(src, e)
    gd = R.build_graph(src, e, mult * lbar, device=0)
    gh = R.build_graph(src, e, mult * lbar, device=False)
    go = O.build_graph(src, e, mult * lbar)
    _graph_equal(gd, gh)
    _graph_equal(gd, go)


@pytest.mark.parametrize("config", [0, 1, 2, 3, 4])
def test_build_graph_device_synthetic_configs(config, capsys):
    """Full-size configs (config 4: 1M vertices): device == host, bitwise."""
    src, faces, tgt = R.synth(config, 4000 if config == 3 else None)
    src, tgt, _, _ = R.normalize_pair(src, tgt)
    e = R.edges_from_faces(faces, len(src)) if faces is not None else R.knn_edges(src, 6, device=0)
    lbar = R.avg_edge_length(src, e)
    radius = R.GRAPH_MULT[config] * lbar
    st = {}
    R.build_graph(src, e, radius, device=0)  # warm (context, modules)
    t0 = time.perf_counter()
    gd = R.build_graph(src, e, radius, device=0, stats=st)
    t1 = time.perf_counter()
    gh = R.build_graph(src, e, radius, device=False)
    t2 = time.perf_counter()
    _graph_equal(gd, gh)
    with capsys.disabled():
        print("\nconfig %d: n=%d N=%d rounds=%d device %.1f ms host %.1f ms" %
              (config, len(src), gd.node_count, st["rounds"], 1e3 * (t1 - t0), 1e3 * (t2 - t1)))


def test_build_graph_device_point_cloud_and_errors():
    rng = np.random.default_rng(5)
    pts = rng.uniform(-1, 1, (3000, 3))
    e = R.knn_edges(pts, 6, device=0)
    lbar = R.avg_edge_length(pts, e)
    _graph_equal(R.build_graph(pts, e, 3.0 * lbar, device=0), O.build_graph(pts, e, 3.0 * lbar))
    # isolated points (no edges): every point its own node
    iso = rng.uniform(size=(50, 3))
    _graph_equal(R.build_graph(iso, np.zeros((0, 2), np.int32), 0.05, device=0),
                 R.build_graph(iso, np.zeros((0, 2), np.int32), 0.05, device=False))
    with pytest.raises(capi.ConfigError):
        R.build_graph(np.zeros((0, 3)), np.zeros((0, 2), np.int32), 1.0, device=0)
    with pytest.raises(capi.ConfigError):
        R.build_graph(pts, e, -1.0, device=0)
    with pytest.raises(capi.NumericalError):
        R.build_graph(pts, np.array([[0, 5000]], np.int32), 0.1, device=0)
