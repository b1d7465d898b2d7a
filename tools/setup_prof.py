"""Device graph build of config 2 once (for an ncu launch list) + wall time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time

from paper_2206_03410_b200 import registration as R

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
src, faces, tgt = R.synth(cfg, 4000 if cfg == 3 else None)
src, tgt, _, _ = R.normalize_pair(src, tgt)
e = R.edges_from_faces(faces, len(src)) if faces is not None else R.knn_edges(src, 6, device=0)
lbar = R.avg_edge_length(src, e)
R.build_graph(src[:2000], e[:0], 0.1, device=0)
for _ in range(2):
    st = {}
    t0 = time.perf_counter()
    g = R.build_graph(src, e, R.GRAPH_MULT[cfg] * lbar, device=0, stats=st)
    print("config %d device build %.1f ms rounds %d" % (cfg, 1e3 * (time.perf_counter() - t0), st["rounds"]))
