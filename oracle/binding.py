"""ORACLE — TEST INFRASTRUCTURE ONLY. ctypes binding of oracle/_build/liboracle.so
(the CPU restatement of the reference hot path). Imported only by tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs, as the checker.
"""
import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class ProblemView(C.Structure):  # same layout as nrr_problem_view
    _fields_ = [
        ("n", C.c_int32), ("source", f64p), ("src_avg_edge_length", C.c_double),
        ("m", C.c_int32), ("target", f64p),
        ("node_count", C.c_int32), ("node_positions", f64p),
        ("edge_count", C.c_int32), ("edges", i32p),
        ("infl_offsets", i32p), ("infl_nodes", i32p), ("infl_weights", f64p),
        ("pair_count", C.c_int32), ("reg_pairs", i32p), ("reg_weights", f64p),
    ]


class SolverConfig(C.Structure):
    _fields_ = [
        ("k_alpha", C.c_double), ("k_beta", C.c_double), ("eps", C.c_double),
        ("i_max", C.c_int32), ("aa_window", C.c_int32),
        ("nu_a_init", C.c_double), ("nu_a_min", C.c_double), ("nu_r_init", C.c_double),
        ("nu_r_floor", C.c_double),
        ("landmark_count", C.c_int32), ("landmark_index", i32p), ("landmark_pos", f64p),
    ]


class IterationRecord(C.Structure):
    _fields_ = [("e_total", C.c_double), ("e_align", C.c_double), ("e_reg", C.c_double),
                ("e_rot", C.c_double), ("e_landmark", C.c_double), ("max_disp", C.c_double),
                ("aa_accepted", C.c_int32), ("stage", C.c_int32)]


class StageRecord(C.Structure):
    _fields_ = [("nu_a", C.c_double), ("nu_r", C.c_double), ("alpha", C.c_double), ("beta", C.c_double),
                ("reverts", C.c_int32), ("converged", C.c_int32), ("first_iteration", C.c_int32),
                ("iteration_count", C.c_int32)]


class PassRecord(C.Structure):
    _fields_ = [("e_total", C.c_double), ("stage", C.c_int32), ("reverted", C.c_int32)]


class ReportSummary(C.Structure):
    _fields_ = [("stage_count", C.c_int32), ("total_iterations", C.c_int32),
                ("degenerate_rotations", C.c_int32), ("alpha_forced_zero", C.c_int32),
                ("total_passes", C.c_int32), ("linear_iterations", C.c_int32),
                ("solve_seconds", C.c_double), ("setup_seconds", C.c_double), ("loop_seconds", C.c_double)]


_lib = None


def build():
    r = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stdout + r.stderr)


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        lib = C.CDLL(LIB_PATH)
        lib.oracle_last_error.restype = C.c_char_p
        lib.oracle_graph_counts.restype = None
        lib.oracle_graph_export.restype = None
        lib.oracle_graph_free.restype = None
        _lib = lib
    return _lib


def _check(rc):
    if rc != 0:
        raise OracleError(rc, load().oracle_last_error().decode())


def _d(a):
    return None if a is None else a.ctypes.data_as(f64p)


def _i(a):
    return None if a is None else a.ctypes.data_as(i32p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def view(problem):
    """ProblemView over a paper_2206_03410_b200.registration.Problem-like object."""
    g = problem.graph
    arrs = [_f64(problem.source), _f64(problem.target), _f64(g.node_positions), _i32(g.edges),
            _i32(g.infl_offsets), _i32(g.infl_nodes), _f64(g.infl_weights), _i32(g.reg_pairs),
            _f64(g.reg_weights)]
    v = ProblemView()
    v._keep = arrs
    v.n, v.source, v.src_avg_edge_length = len(arrs[0]), _d(arrs[0]), float(problem.src_avg_edge_length)
    v.m, v.target = len(arrs[1]), _d(arrs[1])
    v.node_count, v.node_positions = len(arrs[2]), _d(arrs[2])
    v.edge_count, v.edges = len(arrs[3]), _i(arrs[3])
    v.infl_offsets, v.infl_nodes, v.infl_weights = _i(arrs[4]), _i(arrs[5]), _d(arrs[6])
    v.pair_count, v.reg_pairs, v.reg_weights = len(arrs[8]), _i(arrs[7]), _d(arrs[8])
    return v


def config(k_alpha=100.0, k_beta=1.0, eps=1e-5, i_max=100, aa_window=5, nu_a_init=float("nan"),
           nu_a_min=float("nan"), nu_r_init=float("nan"), nu_r_floor=1e-8, landmarks=None):
    c = SolverConfig()
    c.k_alpha, c.k_beta, c.eps, c.i_max, c.aa_window = k_alpha, k_beta, eps, i_max, aa_window
    c.nu_a_init, c.nu_a_min, c.nu_r_init, c.nu_r_floor = nu_a_init, nu_a_min, nu_r_init, nu_r_floor
    c._keep = []
    if landmarks:
        idx = _i32([l[0] for l in landmarks])
        pos = _f64([l[1] for l in landmarks]).reshape(-1, 3)
        c._keep = [idx, pos]
        c.landmark_count, c.landmark_index, c.landmark_pos = len(idx), _i(idx), _d(pos)
    return c


def build_graph(points, edges, radius):
    lib = load()
    p, e = _f64(points).reshape(-1, 3), _i32(edges).reshape(-1, 2)
    h = C.c_void_p()
    _check(lib.oracle_build_graph(_d(p), len(p), _i(e), len(e), C.c_double(radius), C.byref(h)))
    N, E, S, P = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    lib.oracle_graph_counts(h, C.byref(N), C.byref(E), C.byref(S), C.byref(P))
    N, E, S, P = N.value, E.value, S.value, P.value
    out = dict(node_indices=np.zeros(N, np.int32), node_positions=np.zeros((N, 3)), edges=np.zeros((E, 2), np.int32),
               infl_offsets=np.zeros(len(p) + 1, np.int32), infl_nodes=np.zeros(S, np.int32),
               infl_weights=np.zeros(S), infl_dist=np.zeros(S), reg_pairs=np.zeros((P, 2), np.int32),
               reg_weights=np.zeros(P))
    lib.oracle_graph_export(h, _i(out["node_indices"]), _d(out["node_positions"]), _i(out["edges"]),
                            _i(out["infl_offsets"]), _i(out["infl_nodes"]), _d(out["infl_weights"]),
                            _d(out["infl_dist"]), _i(out["reg_pairs"]), _d(out["reg_weights"]))
    lib.oracle_graph_free(h)
    return out


def edges_from_faces(faces, n):
    lib = load()
    f = _i32(faces).reshape(-1, 3)
    out = np.zeros((3 * len(f), 2), np.int32)
    cnt = C.c_int32()
    _check(lib.oracle_edges_from_faces(_i(f), len(f), n, _i(out), len(out), C.byref(cnt)))
    return out[: cnt.value].copy()


def knn_edges(points, k):
    lib = load()
    p = _f64(points).reshape(-1, 3)
    out = np.zeros((len(p) * k, 2), np.int32)
    cnt = C.c_int32()
    _check(lib.oracle_knn_edges(_d(p), len(p), k, _i(out), len(out), C.byref(cnt)))
    return out[: cnt.value].copy()


def nearest(target, queries):
    lib = load()
    t, q = _f64(target).reshape(-1, 3), _f64(queries).reshape(-1, 3)
    idx = np.zeros(len(q), np.int32)
    dist = np.zeros(len(q))
    _check(lib.oracle_nearest(_d(t), len(t), _d(q), len(q), _i(idx), _d(dist)))
    return idx, dist


def deform(problem, X):
    lib = load()
    v = view(problem)
    out = np.zeros((problem.n if hasattr(problem, "n") else len(problem.source), 3))
    _check(lib.oracle_deform(C.byref(v), _d(_f64(X)), _d(out)))
    return out


def project_rotations(X, N):
    lib = load()
    R = np.zeros((N, 3, 3))
    deg = C.c_int32()
    _check(lib.oracle_project_rotations(_d(_f64(X)), N, _d(R), C.byref(deg)))
    return R, deg.value


def project_to_rotation(A):
    lib = load()
    R = np.zeros((3, 3))
    smin = C.c_double()
    _check(lib.oracle_project_to_rotation(_d(_f64(A)), _d(R), C.byref(smin)))
    return R, smin.value


def step(problem, X, prm, nnzb, landmark_weight=0.0, cfg=None, want_solve=True):
    lib = load()
    v = view(problem)
    n, N = len(problem.source), problem.graph.node_count
    idx = np.zeros(n, np.int32)
    sq = np.zeros(n)
    e4 = np.zeros(4)
    K = np.zeros(16 * nnzb)
    B = np.zeros(12 * N)
    Xmm = np.zeros(12 * N) if want_solve else None
    _check(lib.oracle_step(C.byref(v), _d(_f64(X)), _d(_f64(prm)), C.c_double(landmark_weight),
                           C.byref(cfg) if cfg else None, _i(idx), _d(sq), _d(e4), _d(K), _d(B), _d(Xmm)))
    return {"index": idx, "sqdist": sq, "energy": e4, "K": K, "B": B, "Xmm": Xmm}


def anderson_combine(G, F, m):
    lib = load()
    G, F = _f64(G), _f64(F)
    h, dim = G.shape
    out = np.zeros(dim)
    rank = C.c_int32()
    _check(lib.oracle_anderson_combine(_d(G), _d(F), h, dim, m, _d(out), C.byref(rank)))
    return out, rank.value


def init_parameters(problem, cfg=None):
    lib = load()
    v = view(problem)
    out = np.zeros(6)
    _check(lib.oracle_init_parameters(C.byref(v), C.byref(cfg or config()), _d(out)))
    return {"nu_a": out[0], "nu_r": out[1], "nu_a_min": out[2], "alpha": out[3], "beta": out[4],
            "alpha_forced_zero": bool(out[5])}


def register(problem, cfg=None, pass_cap=0, with_nn=False, ordering=0):
    """register_surfaces on the oracle; returns (X, deformed, report dict).
    ordering: node order of the direct solve, 0 = RCM, 1 = natural."""
    lib = load()
    lib.oracle_set_ldlt_ordering(int(ordering))
    cfg = cfg or config()
    v = view(problem)
    n, N = len(problem.source), problem.graph.node_count
    cap_it = 100000
    X = np.zeros(12 * N)
    out = np.zeros((n, 3))
    its = (IterationRecord * cap_it)()
    sts = (StageRecord * 1000)()
    pc = max(pass_cap, 1)
    ps = (PassRecord * pc)()
    nn = np.zeros((pc, n), np.int32) if with_nn else None
    s = ReportSummary()
    _check(lib.oracle_register(C.byref(v), C.byref(cfg), _d(X), _d(out), its, cap_it, sts, 1000, ps, pc,
                               _i(nn) if with_nn else None, C.byref(s)))
    stages = []
    for k in range(s.stage_count):
        st = sts[k]
        stages.append({"nu_a": st.nu_a, "nu_r": st.nu_r, "alpha": st.alpha, "beta": st.beta,
                       "reverts": st.reverts, "converged": bool(st.converged),
                       "iterations": [{"E": it.e_total, "E_align": it.e_align, "E_reg": it.e_reg,
                                       "E_rot": it.e_rot, "E_landmark": it.e_landmark,
                                       "aa_accepted": bool(it.aa_accepted), "max_disp": it.max_disp}
                                      for it in its[st.first_iteration: st.first_iteration + st.iteration_count]]})
    rep = {"stages": stages, "degenerate_rotations": s.degenerate_rotations,
           "alpha_forced_zero": bool(s.alpha_forced_zero), "total_iterations": s.total_iterations,
           "total_passes": s.total_passes, "solve_seconds": s.solve_seconds,
           "setup_seconds": s.setup_seconds, "loop_seconds": s.loop_seconds,
           "passes": [{"E": p.e_total, "stage": p.stage, "reverted": bool(p.reverted)}
                      for p in list(ps)[: min(pc, s.total_passes)]]}
    if with_nn:
        rep["pass_nn"] = nn[: min(pc, s.total_passes)]
    return X, out, rep


def time_iterations(problem, cfg, warmup, steps):
    """Seconds for `steps` accepted iterations after `warmup` (single thread)."""
    lib = load()
    v = view(problem)
    s = C.c_double()
    _check(lib.oracle_time_iterations(C.byref(v), C.byref(cfg), warmup, steps, C.byref(s)))
    return s.value


# ---------------------------------------------------------------- inputs
# Radius multipliers of the synthetic configs (R = mult * mean edge length),
# the same table as paper_2206_03410_b200.registration.GRAPH_MULT (a CPU test
# keeps them equal): the reference arm builds its inputs from the oracle
# alone, without loading the product library.
GRAPH_MULT = {0: 5.0, 1: 5.5, 2: 5.0, 3: 5.9, 4: 7.2}


@dataclass
class Graph:
    """DeformationGraph (deformation_graph.hpp:50-67) as flat arrays."""
    node_indices: np.ndarray
    node_positions: np.ndarray
    edges: np.ndarray
    infl_offsets: np.ndarray
    infl_nodes: np.ndarray
    infl_weights: np.ndarray
    infl_dist: np.ndarray
    reg_pairs: np.ndarray
    reg_weights: np.ndarray
    radius: float = 0.0

    @property
    def node_count(self):
        return len(self.node_indices)

    @property
    def pair_count(self):
        return len(self.reg_weights)


@dataclass
class Problem:
    source: np.ndarray
    target: np.ndarray
    graph: Graph
    src_avg_edge_length: float
    faces: object = None

    @property
    def n(self):
        return len(self.source)


def synth(config, seed=None, scale=1.0):
    lib = load()
    if seed is None:
        seed = 1000 * (config + 1)
    n, nf, m = C.c_int32(), C.c_int32(), C.c_int32()
    _check(lib.oracle_synth_config(config, C.c_uint64(seed), C.c_double(scale), C.byref(n), C.byref(nf), C.byref(m),
                                   None, None, None))
    src, faces, tgt = np.zeros((n.value, 3)), np.zeros((nf.value, 3), np.int32), np.zeros((m.value, 3))
    _check(lib.oracle_synth_config(config, C.c_uint64(seed), C.c_double(scale), C.byref(n), C.byref(nf), C.byref(m),
                                   _d(src), _i(faces), _d(tgt)))
    return src, (faces if nf.value else None), tgt


def normalize_pair(source, target):
    lib = load()
    s, t = _f64(source).reshape(-1, 3).copy(), _f64(target).reshape(-1, 3).copy()
    out = np.zeros(4)
    _check(lib.oracle_normalize_pair(_d(s), len(s), _d(t), len(t), _d(out)))
    return s, t, out[0], out[1:4].copy()


def avg_edge_length(points, edges):
    lib = load()
    p, e = _f64(points).reshape(-1, 3), _i32(edges).reshape(-1, 2)
    out = C.c_double()
    _check(lib.oracle_avg_edge_length(_d(p), len(p), _i(e), len(e), C.byref(out)))
    return out.value


def make_problem(config, seed=None, scale=1.0, mult=None):
    """The synthetic pair of BASELINE config `config` built by the oracle alone
    (synth -> normalize_pair -> edges -> build_graph, surface.hpp /
    deformation_graph.hpp restated): the same arrays as
    paper_2206_03410_b200.registration.make_problem (tests/test_oracle_kats.py
    checks bitwise equality)."""
    src, faces, tgt = synth(config, seed, scale)
    src, tgt, _, _ = normalize_pair(src, tgt)
    edges = edges_from_faces(faces, len(src)) if faces is not None else knn_edges(src, 6)
    lbar = avg_edge_length(src, edges)
    radius = (GRAPH_MULT[config] if mult is None else mult) * lbar
    g = build_graph(src, edges, radius)
    return Problem(src, tgt, Graph(radius=radius, **g), lbar, faces)
