"""Python mirror of the reference's registration API (proj/include/nrr) over
the C ABI: the names follow the reference (register_surfaces,
find_correspondences, deform_points, project_rotations, anderson_combine,
init_parameters, build_graph ...), every call runs the sm_100a path.

Arrays are numpy, float64 AoS (n, 3) for points; NodeTransforms X is the
reference's 4N x 3 column-major stacking flattened to 12N (solver.hpp:146).
"""
import ctypes as C
import os
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import capi
from .capi import check, d, f64, i, i32

NAN = float("nan")

# Radius multipliers (R = mult * mean source edge length) tuned once so the
# reference graph rule (deformation_graph.hpp:157-210) yields the node counts
# BASELINE.json states for each synthetic config.
GRAPH_MULT = {0: 5.0, 1: 5.5, 2: 5.0, 3: 5.9, 4: 7.2}


@dataclass
class Graph:
    """DeformationGraph (deformation_graph.hpp:50-67) as flat arrays."""
    node_indices: np.ndarray
    node_positions: np.ndarray  # (N, 3)
    edges: np.ndarray           # (E, 2)
    infl_offsets: np.ndarray    # (n+1,)
    infl_nodes: np.ndarray
    infl_weights: np.ndarray
    infl_dist: np.ndarray
    reg_pairs: np.ndarray       # (P, 2)
    reg_weights: np.ndarray
    radius: float = 0.0

    @property
    def node_count(self):
        return len(self.node_indices)

    @property
    def edge_count(self):
        return len(self.edges)

    @property
    def pair_count(self):
        return len(self.reg_weights)


@dataclass
class Problem:
    source: np.ndarray
    target: np.ndarray
    graph: Graph
    src_avg_edge_length: float
    faces: Optional[np.ndarray] = None
    _keep: list = field(default_factory=list, repr=False)

    @property
    def n(self):
        return len(self.source)

    def view(self):
        g = self.graph
        arrs = [f64(self.source), f64(self.target), f64(g.node_positions), i32(g.edges), i32(g.infl_offsets),
                i32(g.infl_nodes), f64(g.infl_weights), i32(g.reg_pairs), f64(g.reg_weights)]
        self._keep = arrs
        v = capi.ProblemView()
        v.n = len(self.source)
        v.source = d(arrs[0])
        v.src_avg_edge_length = float(self.src_avg_edge_length)
        v.m = len(self.target)
        v.target = d(arrs[1])
        v.node_count = g.node_count
        v.node_positions = d(arrs[2])
        v.edge_count = g.edge_count
        v.edges = i(arrs[3])
        v.infl_offsets = i(arrs[4])
        v.infl_nodes = i(arrs[5])
        v.infl_weights = d(arrs[6])
        v.pair_count = g.pair_count
        v.reg_pairs = i(arrs[7])
        v.reg_weights = d(arrs[8])
        return v


def solver_config(k_alpha=100.0, k_beta=1.0, eps=1e-5, i_max=100, aa_window=5, nu_a_init=NAN, nu_a_min=NAN,
                  nu_r_init=NAN, nu_r_floor=1e-8, landmarks=None):
    """SolverConfig (solver.hpp:16-39) with the reference defaults."""
    c = capi.SolverConfig()
    c.k_alpha, c.k_beta, c.eps = k_alpha, k_beta, eps
    c.i_max, c.aa_window = i_max, aa_window
    c.nu_a_init, c.nu_a_min, c.nu_r_init, c.nu_r_floor = nu_a_init, nu_a_min, nu_r_init, nu_r_floor
    c.landmark_count = 0
    c._keep = []
    if landmarks:
        idx = i32([l[0] for l in landmarks])
        pos = f64([l[1] for l in landmarks]).reshape(-1, 3)
        c._keep = [idx, pos]
        c.landmark_count = len(idx)
        c.landmark_index = i(idx)
        c.landmark_pos = d(pos)
    return c


# ------------------------------------------------------------------ setup (CPU)
def edges_from_faces(faces, n):
    lib = capi.load()
    faces = i32(faces).reshape(-1, 3)
    cnt = C.c_int32()
    out = np.zeros((3 * len(faces), 2), np.int32)
    check(lib.nrr_edges_from_faces(i(faces), len(faces), n, i(out), len(out), C.byref(cnt)))
    return out[: cnt.value].copy()


def _setup_device(device):
    """Where a setup entry runs: None = the B200 when one is visible (the
    C++ headers' rule, NRR_SETUP_HOST=1 forces the host), False = host, an
    int = that device."""
    if device is None:
        if os.environ.get("NRR_SETUP_HOST") == "1":
            return None
        cnt = C.c_int32()
        capi.load().nrr_device_count(C.byref(cnt))
        return 0 if cnt.value > 0 else None
    if device is False:
        return None
    return int(device)


def knn_edges(points, k=6, device=None):
    """knn_edges (surface.hpp:70-94); device: see _setup_device."""
    lib = capi.load()
    p = f64(points).reshape(-1, 3)
    cnt = C.c_int32()
    out = np.zeros((len(p) * k, 2), np.int32)
    dev = _setup_device(device)
    if dev is not None:
        check(lib.nrr_knn_edges_gpu(dev, d(p), len(p), k, i(out), len(out), C.byref(cnt)))
    else:
        check(lib.nrr_knn_edges(d(p), len(p), k, i(out), len(out), C.byref(cnt)))
    return out[: cnt.value].copy()


def limited_geodesic(points, edges, source, radius):
    """limited_geodesic (geodesic.hpp:22-84): (vertex ids, distances)."""
    lib = capi.load()
    p, e = f64(points).reshape(-1, 3), i32(edges).reshape(-1, 2)
    cnt = C.c_int32()
    check(lib.nrr_limited_geodesic(d(p), len(p), i(e), len(e), source, float(radius), None, None, 0, C.byref(cnt)))
    idx, dist = np.zeros(cnt.value, np.int32), np.zeros(cnt.value)
    check(lib.nrr_limited_geodesic(d(p), len(p), i(e), len(e), source, float(radius), i(idx), d(dist), len(idx),
                                   C.byref(cnt)))
    return idx, dist


def avg_edge_length(points, edges):
    lib = capi.load()
    p, e = f64(points).reshape(-1, 3), i32(edges).reshape(-1, 2)
    out = C.c_double()
    check(lib.nrr_avg_edge_length(d(p), len(p), i(e), len(e), C.byref(out)))
    return out.value


def normalize_pair(source, target):
    """normalize_pair (surface.hpp:125-149); returns (src, tgt, scale, center)."""
    lib = capi.load()
    s, t = f64(source).reshape(-1, 3).copy(), f64(target).reshape(-1, 3).copy()
    out = np.zeros(4)
    check(lib.nrr_normalize_pair(d(s), len(s), d(t), len(t), d(out)))
    return s, t, out[0], out[1:4].copy()


def build_graph(points, edges, radius, device=None, stats=None):
    """build_graph (deformation_graph.hpp:157-210); device: see _setup_device.
    `stats` (dict) receives the device sweep's round count."""
    lib = capi.load()
    p, e = f64(points).reshape(-1, 3), i32(edges).reshape(-1, 2)
    h = C.c_void_p()
    dev = _setup_device(device)
    if dev is not None:
        rounds = C.c_int32()
        check(lib.nrr_build_graph_gpu(dev, d(p), len(p), i(e), len(e), float(radius), C.byref(h), C.byref(rounds)))
        if stats is not None:
            stats["rounds"] = rounds.value
    else:
        check(lib.nrr_build_graph(d(p), len(p), i(e), len(e), float(radius), C.byref(h)))
    try:
        N, E, S, P = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        lib.nrr_graph_counts(h, C.byref(N), C.byref(E), C.byref(S), C.byref(P))
        N, E, S, P = N.value, E.value, S.value, P.value
        g = Graph(np.zeros(N, np.int32), np.zeros((N, 3)), np.zeros((E, 2), np.int32), np.zeros(len(p) + 1, np.int32),
                  np.zeros(S, np.int32), np.zeros(S), np.zeros(S), np.zeros((P, 2), np.int32), np.zeros(P), radius)
        lib.nrr_graph_export(h, i(g.node_indices), d(g.node_positions), i(g.edges), i(g.infl_offsets),
                             i(g.infl_nodes), d(g.infl_weights), d(g.infl_dist), i(g.reg_pairs), d(g.reg_weights))
    finally:
        lib.nrr_graph_free(h)
    return g


def synth(config, seed=None, scale=1.0):
    """Seeded synthetic pair standing in for BASELINE.json config `config`
    (SURVEY.md 8(d)); returns (source, faces or None, target)."""
    lib = capi.load()
    if seed is None:
        seed = 1000 * (config + 1)
    n, nf, m = C.c_int32(), C.c_int32(), C.c_int32()
    check(lib.nrr_synth_config(config, seed, scale, C.byref(n), C.byref(nf), C.byref(m), None, None, None))
    src = np.zeros((n.value, 3))
    faces = np.zeros((nf.value, 3), np.int32)
    tgt = np.zeros((m.value, 3))
    check(lib.nrr_synth_config(config, seed, scale, C.byref(n), C.byref(nf), C.byref(m), d(src), i(faces), d(tgt)))
    return src, (faces if nf.value else None), tgt


def shard_bounds(n, world, rank):
    """Contiguous vertex slice [v0, v1) of `rank`."""
    return n * rank // world, n * (rank + 1) // world


def shard_problem(p: Problem, v0, v1) -> Problem:
    """The problem view of one vertex shard: source slice with its influence
    CSR rebased; the target and the deformation graph stay whole (replicated)."""
    g = p.graph
    off = np.asarray(g.infl_offsets)
    k0, k1 = int(off[v0]), int(off[v1])
    g2 = Graph(g.node_indices, g.node_positions, g.edges, (off[v0:v1 + 1] - k0).astype(np.int32),
               g.infl_nodes[k0:k1], g.infl_weights[k0:k1], g.infl_dist[k0:k1], g.reg_pairs, g.reg_weights,
               g.radius)
    return Problem(p.source[v0:v1], p.target, g2, p.src_avg_edge_length, None)


def comm_unique_id() -> bytes:
    """NCCL unique id for Context.set_comm (call on rank 0, broadcast the bytes)."""
    lib = capi.load()
    buf = (C.c_char * 128)()
    check(lib.nrr_comm_unique_id(buf))
    return bytes(buf)


class LocalGroup:
    """In-process group of `world` contexts for the vertex-sharded path
    (nrr_local_group_*): each member context is driven by its own host
    thread; the collectives rendezvous on the host (tests on one GPU)."""

    def __init__(self, world: int):
        self.lib = capi.load()
        self.h = C.c_void_p()
        check(self.lib.nrr_local_group_create(world, C.byref(self.h)))
        self.world = world

    def close(self):
        if self.h:
            self.lib.nrr_local_group_destroy(self.h)
            self.h = C.c_void_p()


def make_problem(config, seed=None, scale=1.0, mult=None):
    """Synthetic pair -> normalize -> connectivity -> reference graph."""
    src, faces, tgt = synth(config, seed, scale)
    src, tgt, _, _ = normalize_pair(src, tgt)
    edges = edges_from_faces(faces, len(src)) if faces is not None else knn_edges(src, 6)
    lbar = avg_edge_length(src, edges)
    mult = GRAPH_MULT[config] if mult is None else mult
    g = build_graph(src, edges, mult * lbar)
    return Problem(src, tgt, g, lbar, faces)


# ------------------------------------------------------------------ device context
def report_dict(summary, stages, iters, passes=None):
    return {
        "stages": [{"nu_a": s.nu_a, "nu_r": s.nu_r, "alpha": s.alpha, "beta": s.beta, "reverts": s.reverts,
                    "converged": bool(s.converged),
                    "iterations": [{"E": it.e_total, "E_align": it.e_align, "E_reg": it.e_reg, "E_rot": it.e_rot,
                                    "E_landmark": it.e_landmark, "aa_accepted": bool(it.aa_accepted),
                                    "max_disp": it.max_disp}
                                   for it in iters[s.first_iteration: s.first_iteration + s.iteration_count]]}
                   for s in stages],
        "degenerate_rotations": summary.degenerate_rotations,
        "alpha_forced_zero": bool(summary.alpha_forced_zero),
        "total_iterations": summary.total_iterations,
        "total_passes": summary.total_passes,
        "linear_iterations": summary.linear_iterations,
        "solve_seconds": summary.solve_seconds,
        "setup_seconds": summary.setup_seconds,
        "loop_seconds": summary.loop_seconds,
        "passes": [{"E": p.e_total, "stage": p.stage, "reverted": bool(p.reverted)} for p in (passes or [])],
    }


class Context:
    """One nrr_ctx: all device buffers of one registration on one stream."""

    def __init__(self, device=0, pcg_rtol=None, pcg_max_iter=None, record_passes=0, max_ctas=0):
        self.lib = capi.load()
        h = C.c_void_p()
        check(self.lib.nrr_ctx_create(device, C.byref(h)))
        self.h = h
        self.n = 0
        self.N = 0
        if pcg_rtol is not None or pcg_max_iter is not None or record_passes or max_ctas:
            self.set_options(pcg_rtol or 1e-13, pcg_max_iter or 20000, record_passes, max_ctas)

    def close(self):
        if self.h:
            self.lib.nrr_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_options(self, pcg_rtol=1e-13, pcg_max_iter=20000, record_passes=0, max_ctas=0):
        o = capi.SolveOptions(pcg_rtol, pcg_max_iter, record_passes, max_ctas)
        check(self.lib.nrr_ctx_set_options(self.h, C.byref(o)))

    def set_comm(self, unique_id: bytes, world: int, rank: int):
        """Join the vertex-sharded run (NCCL communicator of this context)."""
        buf = (C.c_char * 128).from_buffer_copy(unique_id)
        check(self.lib.nrr_ctx_set_comm(self.h, buf, world, rank))

    def set_local_comm(self, group: "LocalGroup", rank: int):
        """Join an in-process group as `rank` (the sharded path on one GPU)."""
        check(self.lib.nrr_ctx_set_local_comm(self.h, group.h, rank))

    def set_shard(self, n_global: int):
        """This context's problem view is one vertex slice of n_global vertices."""
        check(self.lib.nrr_ctx_set_shard(self.h, n_global))

    def enable_timing(self, on=True):
        self.lib.nrr_ctx_enable_timing(self.h, 1 if on else 0)

    def set_target(self, target):
        t = f64(target).reshape(-1, 3)
        check(self.lib.nrr_ctx_set_target(self.h, d(t), len(t)))

    def set_problem(self, problem: Problem):
        v = problem.view()
        check(self.lib.nrr_ctx_set_problem(self.h, C.byref(v)))
        self.n, self.N = problem.n, problem.graph.node_count

    def register(self, cfg=None, one_shot_problem=None):
        """register_surfaces (solver.hpp:180-304): returns (X, deformed, report)."""
        cfg = cfg or solver_config()
        if one_shot_problem is not None:
            v = one_shot_problem.view()
            self.n, self.N = one_shot_problem.n, one_shot_problem.graph.node_count
            X = np.zeros(12 * self.N)
            out = np.zeros((self.n, 3))
            check(self.lib.nrr_register(self.h, C.byref(v), C.byref(cfg), d(X), d(out)))
        else:
            X = np.zeros(12 * self.N)
            out = np.zeros((self.n, 3))
            check(self.lib.nrr_ctx_register(self.h, C.byref(cfg), d(X), d(out)))
        return X, out, self.report()

    def begin(self, cfg):
        self._cfg = cfg
        check(self.lib.nrr_ctx_begin(self.h, C.byref(cfg)))

    def iterate(self, max_accepted, flush_l2=False):
        """Returns (accepted, done, device_ms)."""
        acc, done, ms = C.c_int32(), C.c_int32(), C.c_double()
        check(self.lib.nrr_ctx_iterate(self.h, max_accepted, 1 if flush_l2 else 0, C.byref(acc), C.byref(done),
                                       C.byref(ms)))
        return acc.value, bool(done.value), ms.value

    def finish(self):
        X = np.zeros(12 * self.N)
        out = np.zeros((self.n, 3))
        check(self.lib.nrr_ctx_finish(self.h, d(X), d(out)))
        return X, out, self.report()

    def report(self, with_nn=False):
        s = capi.ReportSummary()
        check(self.lib.nrr_ctx_report(self.h, C.byref(s), None, 0, None, 0, None, 0, None))
        st = (capi.StageRecord * max(1, s.stage_count))()
        it = (capi.IterationRecord * max(1, s.total_iterations))()
        npass = max(1, s.total_passes)
        ps = (capi.PassRecord * npass)()
        nn = np.zeros((npass, self.n), np.int32) if with_nn else None
        check(self.lib.nrr_ctx_report(self.h, C.byref(s), st, s.stage_count, it, s.total_iterations, ps, npass,
                                      i(nn) if with_nn else None))
        rep = report_dict(s, list(st)[: s.stage_count], list(it)[: s.total_iterations], list(ps))
        if with_nn:
            rep["pass_nn"] = nn
        return rep

    def trace(self):
        """Pass trace of the last run (record_passes=3): a list of dicts, one per
        evaluated pass, with the iterate X (12N, reference layout), the NN
        indices, the energies and, on accepted passes, x_mm."""
        cnt = C.c_int32()
        check(self.lib.nrr_ctx_trace_count(self.h, C.byref(cnt)))
        out = []
        for k in range(cnt.value):
            t = capi.PassTrace()
            X = np.zeros(12 * self.N)
            Xmm = np.zeros(12 * self.N)
            nn = np.zeros(self.n, np.int32)
            check(self.lib.nrr_ctx_trace(self.h, k, C.byref(t), d(X), d(Xmm), i(nn)))
            out.append({"X": X, "Xmm": Xmm if t.accepted_index >= 0 else None, "index": nn,
                        "energy": np.array([t.e_align, t.e_reg, t.e_rot, t.e_total]), "E_landmark": t.e_landmark,
                        "max_disp": t.max_disp, "stage": t.stage, "reverted": bool(t.reverted),
                        "pcg_iterations": t.pcg_iterations, "accepted_index": t.accepted_index})
        return out

    def nearest(self, queries, prev=None):
        """Exact nearest target (smallest index on ties); `prev` (target
        indices) warm-starts the bound as the registration passes do."""
        q = f64(queries).reshape(-1, 3)
        idx = np.zeros(len(q), np.int32)
        dist = np.zeros(len(q))
        if prev is None:
            check(self.lib.nrr_nearest(self.h, d(q), len(q), i(idx), d(dist)))
        else:
            pv = np.ascontiguousarray(prev, dtype=np.int32)
            check(self.lib.nrr_nearest_from(self.h, d(q), len(q), i(pv), i(idx), d(dist)))
        return idx, dist

    def deform(self, X):
        out = np.zeros((self.n, 3))
        check(self.lib.nrr_deform(self.h, d(f64(X)), d(out)))
        return out

    def project_rotations(self, X, N=None):
        X = f64(X)
        N = len(X) // 12 if N is None else N
        R = np.zeros((N, 3, 3))
        deg = C.c_int32()
        check(self.lib.nrr_project_rotations(self.h, d(X), N, d(R), C.byref(deg)))
        return R, deg.value

    def step(self, X, prm, landmark_weight=0.0, cfg=None, nnzb=None, want_solve=True):
        """One teacher-forced pass at X; prm = (alpha, beta, nu_a, nu_r)."""
        n, N = self.n, self.N
        idx = np.zeros(n, np.int32)
        sq = np.zeros(n)
        e4 = np.zeros(4)
        K = np.zeros(16 * nnzb) if nnzb else None
        B = np.zeros(12 * N)
        Xmm = np.zeros(12 * N) if want_solve else None
        p = f64(prm)
        check(self.lib.nrr_step(self.h, d(f64(X)), d(p), landmark_weight, C.byref(cfg) if cfg else None, i(idx),
                                d(sq), d(e4), d(K) if K is not None else None, d(B),
                                d(Xmm) if Xmm is not None else None))
        return {"index": idx, "sqdist": sq, "energy": e4, "K": K, "B": B, "Xmm": Xmm}

    def assemble(self, corr_points, w_align, w_reg, rotations, beta, landmark_weight=0.0, cfg=None, nnzb=None):
        """SystemAssembler::fill (energy.hpp:182-228) from caller correspondences,
        weights and rotations (N x 3 x 3); returns (K in pattern order, B 4N x 3
        column-major flat). The system stays resident for solve()."""
        N = self.N
        q, wa = f64(np.asarray(corr_points).reshape(-1, 3)), f64(w_align)
        wr = f64(w_reg) if len(w_reg) else np.zeros(1)
        R = f64(np.asarray(rotations).reshape(N, 9))
        K = np.zeros(16 * nnzb) if nnzb else None
        B = np.zeros(12 * N)
        check(self.lib.nrr_assemble(self.h, d(q), d(wa), d(wr), d(R), beta, landmark_weight,
                                    C.byref(cfg) if cfg else None, d(K) if K is not None else None, d(B)))
        return K, B

    def solve(self, K=None, B=None, X0=None):
        """SystemAssembler::solve (energy.hpp:233-254) on the device PCG."""
        out = np.zeros(12 * self.N)
        check(self.lib.nrr_solve(self.h, d(f64(K)) if K is not None else None, d(f64(B)) if B is not None else None,
                                 d(f64(X0)) if X0 is not None else None, d(out)))
        return out

    def anderson_combine(self, G, F, m):
        G, F = f64(G), f64(F)
        h, dim = G.shape
        out = np.zeros(dim)
        rank = C.c_int32()
        check(self.lib.nrr_anderson_combine(self.h, d(G), d(F), h, dim, m, d(out), C.byref(rank)))
        return out, rank.value

    def init_parameters(self, cfg=None):
        out = np.zeros(6)
        check(self.lib.nrr_init_parameters(self.h, C.byref(cfg or solver_config()), d(out)))
        return {"nu_a": out[0], "nu_r": out[1], "nu_a_min": out[2], "alpha": out[3], "beta": out[4],
                "alpha_forced_zero": bool(out[5])}

    def stats(self):
        n = C.c_int64()
        ms = np.zeros(6)
        it = C.c_int32()
        self.lib.nrr_ctx_stats(self.h, C.byref(n), d(ms), C.byref(it))
        comm = np.zeros(1)
        self.lib.nrr_ctx_comm_ms(self.h, d(comm))
        return {"launches": n.value, "kernel_ms": {"nn": ms[0], "terms": ms[1], "assemble": ms[2], "pcg": ms[3],
                                                    "aa": ms[4], "deform": ms[5]}, "pcg_iterations": it.value,
                "comm_ms": comm[0]}


def bsr_pattern(graph: Graph):
    """The fixed block pattern (energy.hpp:264-279): per node the sorted
    column list {j} U neighbours(j); returns (row_ptr, cols)."""
    N = graph.node_count
    cols = [[j] for j in range(N)]
    for a, b in graph.edges:
        cols[a].append(b)
        cols[b].append(a)
    row_ptr = [0]
    out = []
    for j in range(N):
        c = sorted(set(cols[j]))
        out.extend(c)
        row_ptr.append(len(out))
    return np.array(row_ptr, np.int32), np.array(out, np.int32)


def identity_transforms(N):
    X = np.zeros((3, 4 * N))
    for j in range(N):
        for c in range(3):
            X[c, 4 * j + c] = 1.0
    return X.reshape(-1)


def has_device():
    try:
        lib = capi.load()
        sm = C.c_int32()
        name = C.create_string_buffer(128)
        return lib.nrr_device_info(0, name, 128, C.byref(sm)) == 0
    except Exception:
        return False
