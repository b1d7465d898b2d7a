// ORACLE — TEST INFRASTRUCTURE ONLY. extern "C" layer over nrr_oracle.hpp.
#include "oracle_capi.h"
#include "nrr_synth.hpp"

#include <cstring>
#include <exception>
#include <string>

#include "nrr_oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const IoError& e) {
        g_err = e.what();
        return 2;
    } catch (const NumericalError& e) {
        g_err = e.what();
        return 3;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

std::vector<Vec3> to_vec3(const double* p, int n) {
    std::vector<Vec3> v(n);
    for (int i = 0; i < n; ++i) v[i] = Vec3(p[3 * i], p[3 * i + 1], p[3 * i + 2]);
    return v;
}

DeformationGraph graph_from_view(const oracle_problem_view* p) {
    DeformationGraph g;
    const int N = p->node_count;
    g.node_positions = to_vec3(p->node_positions, N);
    g.node_indices.assign(N, -1);
    g.graph_edges.resize(p->edge_count);
    g.node_neighbors.assign(N, {});
    for (int e = 0; e < p->edge_count; ++e) {
        const int a = p->edges[2 * e], b = p->edges[2 * e + 1];
        g.graph_edges[e] = {a, b};
        g.node_neighbors[a].push_back(b);
        g.node_neighbors[b].push_back(a);
    }
    for (auto& nb : g.node_neighbors) std::sort(nb.begin(), nb.end());
    g.influence.assign(p->n, {});
    for (int i = 0; i < p->n; ++i)
        for (int k = p->infl_offsets[i]; k < p->infl_offsets[i + 1]; ++k)
            g.influence[i].push_back({p->infl_nodes[k], p->infl_weights[k], 0.0});
    g.reg_pairs.resize(p->pair_count);
    g.reg_weights.resize(p->pair_count);
    for (int e = 0; e < p->pair_count; ++e) {
        g.reg_pairs[e] = {p->reg_pairs[2 * e], p->reg_pairs[2 * e + 1]};
        g.reg_weights[e] = p->reg_weights[e];
    }
    return g;
}

SolverConfig config_from(const oracle_solver_config* c) {
    SolverConfig s;
    s.k_alpha = c->k_alpha;
    s.k_beta = c->k_beta;
    s.eps = c->eps;
    s.i_max = c->i_max;
    s.aa_window = c->aa_window;
    s.nu_a_init = c->nu_a_init;
    s.nu_a_min = c->nu_a_min;
    s.nu_r_init = c->nu_r_init;
    s.nu_r_floor = c->nu_r_floor;
    for (int l = 0; l < c->landmark_count; ++l)
        s.landmarks.push_back({c->landmark_index[l],
                               Vec3(c->landmark_pos[3 * l], c->landmark_pos[3 * l + 1],
                                    c->landmark_pos[3 * l + 2])});
    return s;
}

NodeTransforms x_from(const double* X, int N) {
    NodeTransforms x = NodeTransforms::zeros(N);
    std::memcpy(x.stacked.data(), X, sizeof(double) * 12 * N);
    return x;
}
}  // namespace

struct oracle_graph {
    DeformationGraph g;
};

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

int oracle_edges_from_faces(const int32_t* faces, int32_t nf, int32_t n, int32_t* out_edges,
                            int32_t cap, int32_t* out_count) {
    return guard([&] {
        std::vector<std::array<int, 3>> f(nf);
        for (int i = 0; i < nf; ++i) f[i] = {faces[3 * i], faces[3 * i + 1], faces[3 * i + 2]};
        const auto e = edges_from_faces(f, n);
        *out_count = static_cast<int32_t>(e.size());
        if (static_cast<int>(e.size()) > cap) throw ConfigError("edge buffer too small");
        for (size_t i = 0; i < e.size(); ++i) {
            out_edges[2 * i] = e[i].first;
            out_edges[2 * i + 1] = e[i].second;
        }
    });
}

int oracle_knn_edges(const double* pts, int32_t n, int32_t k, int32_t* out_edges, int32_t cap,
                     int32_t* out_count) {
    return guard([&] {
        const auto e = knn_edges(to_vec3(pts, n), k);
        *out_count = static_cast<int32_t>(e.size());
        if (static_cast<int>(e.size()) > cap) throw ConfigError("edge buffer too small");
        for (size_t i = 0; i < e.size(); ++i) {
            out_edges[2 * i] = e[i].first;
            out_edges[2 * i + 1] = e[i].second;
        }
    });
}

int oracle_avg_edge_length(const double* pts, int32_t n, const int32_t* edges, int32_t ne,
                           double* out) {
    return guard([&] {
        Surface s;
        s.points = to_vec3(pts, n);
        for (int e = 0; e < ne; ++e) s.edges.emplace_back(edges[2 * e], edges[2 * e + 1]);
        s.finalize_edges();
        *out = s.avg_edge_length;
    });
}

int oracle_normalize_pair(double* src, int32_t n, double* tgt, int32_t m, double* out4) {
    return guard([&] {
        Surface s, t;
        s.points = to_vec3(src, n);
        t.points = to_vec3(tgt, m);
        const Normalization nm = normalize_pair(s, t);
        for (int i = 0; i < n; ++i)
            for (int c = 0; c < 3; ++c) src[3 * i + c] = s.points[i][c];
        for (int i = 0; i < m; ++i)
            for (int c = 0; c < 3; ++c) tgt[3 * i + c] = t.points[i][c];
        out4[0] = nm.scale;
        for (int c = 0; c < 3; ++c) out4[1 + c] = nm.center[c];
    });
}

int oracle_synth_config(int32_t which, uint64_t seed, double scale, int32_t* n, int32_t* nf_src, int32_t* m,
                        double* src, int32_t* src_faces, double* tgt) {
    return guard([&] {
        std::vector<double> s, t;
        std::vector<int32_t> f;
        try {
            nrr_synth::synth_config(which, seed, scale, s, f, t);
        } catch (const std::invalid_argument& e) {
            throw ConfigError(e.what());
        }
        *n = static_cast<int32_t>(s.size() / 3);
        *nf_src = static_cast<int32_t>(f.size() / 3);
        *m = static_cast<int32_t>(t.size() / 3);
        if (src) std::copy(s.begin(), s.end(), src);
        if (src_faces) std::copy(f.begin(), f.end(), src_faces);
        if (tgt) std::copy(t.begin(), t.end(), tgt);
    });
}

int oracle_build_graph(const double* pts, int32_t n, const int32_t* edges, int32_t ne,
                       double radius, oracle_graph** out) {
    return guard([&] {
        Surface s;
        s.points = to_vec3(pts, n);
        for (int e = 0; e < ne; ++e) s.edges.emplace_back(edges[2 * e], edges[2 * e + 1]);
        s.finalize_edges();
        auto* h = new oracle_graph;
        try {
            h->g = build_graph(s, radius);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void oracle_graph_counts(const oracle_graph* h, int32_t* N, int32_t* E, int32_t* sumk, int32_t* P) {
    *N = h->g.node_count();
    *E = h->g.edge_count();
    int s = 0;
    for (const auto& l : h->g.influence) s += static_cast<int>(l.size());
    *sumk = s;
    *P = h->g.directed_pair_count();
}

void oracle_graph_export(const oracle_graph* h, int32_t* node_indices, double* node_positions,
                         int32_t* edges, int32_t* infl_offsets, int32_t* infl_nodes,
                         double* infl_weights, double* infl_dist, int32_t* reg_pairs,
                         double* reg_weights) {
    const DeformationGraph& g = h->g;
    for (int j = 0; j < g.node_count(); ++j) {
        node_indices[j] = g.node_indices[j];
        for (int c = 0; c < 3; ++c) node_positions[3 * j + c] = g.node_positions[j][c];
    }
    for (int e = 0; e < g.edge_count(); ++e) {
        edges[2 * e] = g.graph_edges[e].first;
        edges[2 * e + 1] = g.graph_edges[e].second;
    }
    int k = 0;
    infl_offsets[0] = 0;
    for (size_t i = 0; i < g.influence.size(); ++i) {
        for (const auto& en : g.influence[i]) {
            infl_nodes[k] = en.node;
            infl_weights[k] = en.weight;
            infl_dist[k] = en.distance;
            ++k;
        }
        infl_offsets[i + 1] = k;
    }
    for (int e = 0; e < g.directed_pair_count(); ++e) {
        reg_pairs[2 * e] = g.reg_pairs[e].first;
        reg_pairs[2 * e + 1] = g.reg_pairs[e].second;
        reg_weights[e] = g.reg_weights[e];
    }
}

void oracle_graph_free(oracle_graph* g) { delete g; }

int oracle_nearest(const double* target, int32_t m, const double* queries, int32_t q,
                   int32_t* out_index, double* out_distance) {
    return guard([&] {
        const SpatialIndex idx(to_vec3(target, m));
        for (int i = 0; i < q; ++i) {
            const auto hit = idx.nearest(Vec3(queries[3 * i], queries[3 * i + 1], queries[3 * i + 2]));
            out_index[i] = hit.index;
            out_distance[i] = hit.distance;
        }
    });
}

int oracle_deform(const oracle_problem_view* p, const double* X, double* out_points) {
    return guard([&] {
        const DeformationGraph g = graph_from_view(p);
        const auto v = deform_points(to_vec3(p->source, p->n), g, x_from(X, p->node_count));
        for (int i = 0; i < p->n; ++i)
            for (int c = 0; c < 3; ++c) out_points[3 * i + c] = v[i][c];
    });
}

int oracle_project_rotations(const double* X, int32_t N, double* out_R, int32_t* out_degenerate) {
    return guard([&] {
        int deg = 0;
        const auto r = project_rotations(x_from(X, N), &deg);
        for (int j = 0; j < N; ++j)
            for (int k = 0; k < 9; ++k) out_R[9 * j + k] = r[j].m[k];
        *out_degenerate = deg;
    });
}

int oracle_project_to_rotation(const double* A, double* out_R, double* out_sigma_min) {
    return guard([&] {
        Mat3 a;
        for (int k = 0; k < 9; ++k) a.m[k] = A[k];
        const Mat3 r = project_to_rotation(a, out_sigma_min);
        for (int k = 0; k < 9; ++k) out_R[k] = r.m[k];
    });
}

int oracle_step(const oracle_problem_view* p, const double* X, const double* prm,
                double landmark_weight, const oracle_solver_config* cfg, int32_t* out_index,
                double* out_sqdist, double* out_energy4, double* out_K, double* out_B,
                double* out_Xmm) {
    return guard([&] {
        const DeformationGraph g = graph_from_view(p);
        const auto src = to_vec3(p->source, p->n);
        const NodeTransforms x = x_from(X, p->node_count);
        const SpatialIndex tindex(to_vec3(p->target, p->m));
        const auto v_hat = deform_points(src, g, x);
        const Correspondences corr = find_correspondences(v_hat, tindex);
        const auto rot = project_rotations(x);
        const EnergyParams ep{prm[0], prm[1], prm[2], prm[3]};
        const EnergyBreakdown e = evaluate_energy(v_hat, x, g, corr, rot, ep);
        if (out_index)
            for (int i = 0; i < p->n; ++i) out_index[i] = corr.target_index[i];
        if (out_sqdist)
            for (int i = 0; i < p->n; ++i) out_sqdist[i] = corr.squared_distance[i];
        if (out_energy4) {
            out_energy4[0] = e.align;
            out_energy4[1] = e.reg;
            out_energy4[2] = e.rot;
            out_energy4[3] = e.total;
        }
        std::vector<Landmark> lms;
        if (cfg) lms = config_from(cfg).landmarks;
        SystemAssembler as(src, g, lms);
        as.fill(corr, rot, alignment_weights(corr, ep.nu_a),
                regularization_weights(g, x, ep.nu_r, ep.alpha), ep.beta, landmark_weight);
        const LinearSystem& sys = as.system();
        if (out_K) std::memcpy(out_K, sys.K.val.data(), sizeof(double) * sys.K.val.size());
        if (out_B) std::memcpy(out_B, sys.B.data(), sizeof(double) * sys.B.size());
        if (out_Xmm) {
            const NodeTransforms xm = as.solve();
            std::memcpy(out_Xmm, xm.stacked.data(), sizeof(double) * xm.stacked.size());
        }
    });
}

int oracle_anderson_combine(const double* G, const double* F, int32_t h, int32_t dim, int32_t m,
                            double* out, int32_t* out_rank) {
    return guard([&] {
        std::deque<AndersonEntry> hist;
        for (int k = 0; k < h; ++k) {
            AndersonEntry e;
            e.g.assign(G + static_cast<size_t>(k) * dim, G + static_cast<size_t>(k + 1) * dim);
            e.f.assign(F + static_cast<size_t>(k) * dim, F + static_cast<size_t>(k + 1) * dim);
            hist.push_back(std::move(e));
        }
        int rank = -1;
        const auto x = anderson_combine(hist, m, &rank);
        std::memcpy(out, x.data(), sizeof(double) * dim);
        if (out_rank) *out_rank = rank;
    });
}

namespace {
struct Recorder : PassObserver {
    oracle_pass_record* passes;
    int32_t cap;
    int32_t* nn;
    int n;
    int count = 0;
    void on_pass(int stage, int pass, const Correspondences& corr, const EnergyBreakdown& e,
                 bool reverted) override {
        (void)pass;
        if (count < cap) {
            if (passes) passes[count] = {e.total, stage, reverted ? 1 : 0};
            if (nn)
                for (int i = 0; i < n; ++i) nn[static_cast<size_t>(count) * n + i] = corr.target_index[i];
        }
        ++count;
    }
};
}  // namespace

void oracle_set_ldlt_ordering(int mode) { oracle::ldlt_ordering() = mode; }

int oracle_register(const oracle_problem_view* p, const oracle_solver_config* c, double* out_X,
                    double* out_deformed, oracle_iteration_record* iters, int32_t iter_cap,
                    oracle_stage_record* stages, int32_t stage_cap, oracle_pass_record* passes,
                    int32_t pass_cap, int32_t* pass_nn_index, oracle_report_summary* summary) {
    return guard([&] {
        const auto t0 = std::chrono::steady_clock::now();
        const DeformationGraph g = graph_from_view(p);
        const auto src = to_vec3(p->source, p->n);
        const auto tgt = to_vec3(p->target, p->m);
        const SolverConfig cfg = config_from(c);
        Recorder rec;
        rec.passes = passes;
        rec.cap = pass_cap;
        rec.nn = pass_nn_index;
        rec.n = p->n;
        const auto t1 = std::chrono::steady_clock::now();
        const RegistrationResult r = register_surfaces(src, p->src_avg_edge_length, tgt, g, cfg, &rec);
        const auto t2 = std::chrono::steady_clock::now();
        if (out_X) std::memcpy(out_X, r.transforms.stacked.data(), sizeof(double) * 12 * g.node_count());
        if (out_deformed)
            for (int i = 0; i < p->n; ++i)
                for (int k = 0; k < 3; ++k) out_deformed[3 * i + k] = r.deformed_points[i][k];
        int it = 0;
        for (size_t s = 0; s < r.report.stages.size(); ++s) {
            const auto& st = r.report.stages[s];
            if (static_cast<int>(s) < stage_cap && stages)
                stages[s] = {st.nu_a, st.nu_r, st.alpha, st.beta, st.reverts, st.converged ? 1 : 0, it,
                             static_cast<int32_t>(st.iterations.size())};
            for (const auto& ir : st.iterations) {
                if (it < iter_cap && iters)
                    iters[it] = {ir.e_total, ir.e_align, ir.e_reg, ir.e_rot, ir.e_landmark, ir.max_disp,
                                 ir.aa_accepted ? 1 : 0, static_cast<int32_t>(s)};
                ++it;
            }
        }
        if (summary) {
            summary->stage_count = static_cast<int32_t>(r.report.stages.size());
            summary->total_iterations = r.report.total_iterations();
            summary->degenerate_rotations = r.report.degenerate_rotations;
            summary->alpha_forced_zero = r.report.alpha_forced_zero ? 1 : 0;
            summary->total_passes = rec.count;
            summary->linear_iterations = 0;
            summary->solve_seconds = r.report.solve_seconds;
            summary->setup_seconds = std::chrono::duration<double>(t1 - t0).count();
            summary->loop_seconds = std::chrono::duration<double>(t2 - t1).count();
        }
    });
}

namespace {
struct Stopwatch : PassObserver {
    int accepted = 0, warmup = 0, steps = 0;
    std::chrono::steady_clock::time_point t_begin, t_end;
    bool started = false, stopped = false;
    void on_pass(int, int, const Correspondences&, const EnergyBreakdown&, bool reverted) override {
        // a pass is observed before it is solved: the interval from the pass
        // that starts iteration `warmup` to the pass that starts iteration
        // `warmup + steps` covers exactly `steps` accepted iterations
        if (reverted) return;
        if (accepted == warmup && !started) {
            started = true;
            t_begin = std::chrono::steady_clock::now();
        }
        if (accepted == warmup + steps && !stopped) {
            stopped = true;
            t_end = std::chrono::steady_clock::now();
        }
        ++accepted;
    }
};
}  // namespace

int oracle_time_iterations(const oracle_problem_view* p, const oracle_solver_config* c, int32_t warmup,
                           int32_t steps, double* seconds) {
    return guard([&] {
        const DeformationGraph g = graph_from_view(p);
        const auto src = to_vec3(p->source, p->n);
        const auto tgt = to_vec3(p->target, p->m);
        SolverConfig cfg = config_from(c);
        cfg.i_max = warmup + steps + 1;  // one extra pass closes the timed interval
        Stopwatch sw;
        sw.warmup = warmup;
        sw.steps = steps;
        register_surfaces(src, p->src_avg_edge_length, tgt, g, cfg, &sw);
        if (!sw.stopped) throw NumericalError("oracle_time_iterations: run ended before the timed iterations");
        *seconds = std::chrono::duration<double>(sw.t_end - sw.t_begin).count();
    });
}

int oracle_init_parameters(const oracle_problem_view* p, const oracle_solver_config* c, double* out6) {
    return guard([&] {
        const DeformationGraph g = graph_from_view(p);
        const SpatialIndex tindex(to_vec3(p->target, p->m));
        const SolverParams s =
            init_parameters(to_vec3(p->source, p->n), p->src_avg_edge_length, tindex, g, config_from(c));
        out6[0] = s.nu_a;
        out6[1] = s.nu_r;
        out6[2] = s.nu_a_min;
        out6[3] = s.alpha;
        out6[4] = s.beta;
        out6[5] = s.alpha_forced_zero ? 1.0 : 0.0;
    });
}

}  // extern "C"
