"""B200 (sm_100a) implementation of the per-iteration hot path of Welsch
majorization-minimization non-rigid registration (arXiv 2206.03410).

The product is libnrr_b200.so (C ABI in include/nrr_cuda.h); this package is
the Python binding used by the tests and the bench.
"""
from .capi import ConfigError, CudaError, IoError, NumericalError, load  # noqa: F401
from .registration import (  # noqa: F401
    Context, Graph, Problem, avg_edge_length, build_graph, edges_from_faces, knn_edges, make_problem,
    normalize_pair, solver_config, synth)
