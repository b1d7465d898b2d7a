// Deformation model (reference deformation_graph.hpp:17-245): node
// transforms, the graph, its construction (host, C ABI setup entry points) and
// deform_points on the device.
#pragma once

#include <utility>
#include <vector>

#include "nrr/common.hpp"
#include "nrr/surface.hpp"

namespace nrr {

/// deformation_graph.hpp:17-38: 4N x 3 column-major, node j = rows 4j..4j+3 = [A_j^T; t_j^T]
struct NodeTransforms {
    MatrixX stacked;

    static NodeTransforms identity(int node_count) {
        NodeTransforms x;
        x.stacked.setZero(4 * node_count, 3);
        for (int j = 0; j < node_count; ++j)
            for (int c = 0; c < 3; ++c) x.stacked(4 * j + c, c) = 1.0;
        return x;
    }
    int node_count() const { return stacked.rows() / 4; }
    Mat3 affine(int j) const {
        Mat3 a;
        for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r) a(c, r) = stacked(4 * j + r, c);
        return a;
    }
    Vec3 translation(int j) const { return {stacked(4 * j + 3, 0), stacked(4 * j + 3, 1), stacked(4 * j + 3, 2)}; }
    void set(int j, const Mat3& a, const Vec3& t) {
        for (int c = 0; c < 3; ++c) {
            for (int r = 0; r < 3; ++r) stacked(4 * j + r, c) = a(c, r);
            stacked(4 * j + 3, c) = t[c];
        }
    }
    bool all_finite() const { return stacked.allFinite(); }
};

struct InfluenceEntry {  // deformation_graph.hpp:40-44
    int node = -1;
    double weight = 0;
    double distance = 0;
};

struct DeformationGraph {  // deformation_graph.hpp:50-67
    std::vector<int> node_indices;
    std::vector<Vec3> node_positions;
    std::vector<std::pair<int, int>> graph_edges;
    std::vector<std::vector<InfluenceEntry>> influence;
    std::vector<std::vector<int>> node_neighbors;
    std::vector<std::pair<int, int>> reg_pairs;
    std::vector<double> reg_weights;
    double radius = 0.0;

    int node_count() const { return static_cast<int>(node_indices.size()); }
    int directed_pair_count() const { return static_cast<int>(reg_pairs.size()); }
    int edge_count() const { return static_cast<int>(graph_edges.size()); }
};

/// deformation_graph.hpp:157-210: on the B200 when one is visible (setup_graph.cu,
/// bitwise equal to the host sweep), else the host build
inline DeformationGraph build_graph(const Surface& source, double radius) {
    const auto pts = detail::flat(source.points);
    std::vector<int32_t> e(2 * source.edges.size());
    for (size_t i = 0; i < source.edges.size(); ++i) {
        e[2 * i] = source.edges[i].first;
        e[2 * i + 1] = source.edges[i].second;
    }
    nrr_graph* h = nullptr;
    if (detail::setup_on_device() && source.point_count() > 0)
        detail::check(nrr_build_graph_gpu(0, pts.data(), source.point_count(), e.data(),
                                          static_cast<int32_t>(source.edges.size()), radius, &h, nullptr));
    else
        detail::check(nrr_build_graph(pts.data(), source.point_count(), e.data(),
                                      static_cast<int32_t>(source.edges.size()), radius, &h));
    int32_t N, E, S, P;
    nrr_graph_counts(h, &N, &E, &S, &P);
    const int n = source.point_count();
    std::vector<int32_t> ni(N), ed(2 * E), off(n + 1), inn(S), pr(2 * P);
    std::vector<double> np(3 * N), iw(S), idist(S), pw(P);
    nrr_graph_export(h, ni.data(), np.data(), ed.data(), off.data(), inn.data(), iw.data(), idist.data(), pr.data(),
                     pw.data());
    nrr_graph_free(h);
    DeformationGraph g;
    g.radius = radius;
    g.node_indices.assign(ni.begin(), ni.end());
    g.node_positions = detail::unflat(np.data(), N);
    for (int k = 0; k < E; ++k) g.graph_edges.emplace_back(ed[2 * k], ed[2 * k + 1]);
    g.influence.resize(n);
    for (int i = 0; i < n; ++i)
        for (int k = off[i]; k < off[i + 1]; ++k) g.influence[i].push_back({inn[k], iw[k], idist[k]});
    g.node_neighbors.assign(N, {});
    for (const auto& [a, b] : g.graph_edges) {
        g.node_neighbors[a].push_back(b);
        g.node_neighbors[b].push_back(a);
    }
    for (auto& nb : g.node_neighbors) std::sort(nb.begin(), nb.end());
    for (int k = 0; k < P; ++k) g.reg_pairs.emplace_back(pr[2 * k], pr[2 * k + 1]);
    g.reg_weights.assign(pw.begin(), pw.end());
    return g;
}

/// deformation_graph.hpp:214-222 (single point, host)
inline Vec3 deformed_position(const Vec3& v, const std::vector<InfluenceEntry>& inf, const DeformationGraph& graph,
                              const NodeTransforms& x) {
    Vec3 out = Vec3::Zero();
    for (const auto& e : inf) {
        const Vec3& p = graph.node_positions[e.node];
        out += e.weight * (x.affine(e.node) * (v - p) + p + x.translation(e.node));
    }
    return out;
}

namespace detail {
// flat arrays of (source, target, graph) kept alive for one C-ABI call
struct ProblemArrays {
    std::vector<double> src, tgt, node_pos, infl_w, reg_w;
    std::vector<int32_t> edges, infl_off, infl_node, pairs;
    nrr_problem_view view{};
    ProblemArrays(const Surface& source, const std::vector<Vec3>* target, const DeformationGraph& g) {
        src = flat(source.points);
        if (target) tgt = flat(*target);
        node_pos = flat(g.node_positions);
        for (const auto& [a, b] : g.graph_edges) {
            edges.push_back(a);
            edges.push_back(b);
        }
        infl_off.push_back(0);
        for (const auto& list : g.influence) {
            for (const auto& e : list) {
                infl_node.push_back(e.node);
                infl_w.push_back(e.weight);
            }
            infl_off.push_back(static_cast<int32_t>(infl_node.size()));
        }
        for (const auto& [i, j] : g.reg_pairs) {
            pairs.push_back(i);
            pairs.push_back(j);
        }
        reg_w = g.reg_weights;
        view.n = source.point_count();
        view.source = src.data();
        view.src_avg_edge_length = source.avg_edge_length;
        view.m = target ? static_cast<int32_t>(target->size()) : 0;
        view.target = target ? tgt.data() : nullptr;
        view.node_count = g.node_count();
        view.node_positions = node_pos.data();
        view.edge_count = g.edge_count();
        view.edges = edges.data();
        view.infl_offsets = infl_off.data();
        view.infl_nodes = infl_node.data();
        view.infl_weights = infl_w.data();
        view.pair_count = g.directed_pair_count();
        view.reg_pairs = pairs.data();
        view.reg_weights = reg_w.data();
    }
};

// The default context keeps the last problem it was given (plan, BSR
// pattern, assembly lists, target index): deform_points / mm_step called
// again with the same source and graph (and target) reuse it instead of
// rebuilding the plan (~5 ms at 100K vertices). Content is compared, not
// addresses, so a caller that edits its arrays in place gets a fresh plan.
inline void use_problem(nrr_ctx* c, const ProblemArrays& pa) {
    struct Kept {
        std::vector<double> src, tgt, node_pos, infl_w, reg_w;
        std::vector<int32_t> edges, infl_off, infl_node, pairs;
        double avg = 0.0;
        bool valid = false, has_target = false;
    };
    thread_local Kept k;
    const bool same = k.valid && k.avg == pa.view.src_avg_edge_length && k.src == pa.src && k.node_pos == pa.node_pos &&
                      k.edges == pa.edges && k.infl_off == pa.infl_off && k.infl_node == pa.infl_node &&
                      k.infl_w == pa.infl_w && k.pairs == pa.pairs && k.reg_w == pa.reg_w;
    if (!same) {
        k.valid = false;
        check(nrr_ctx_set_problem(c, &pa.view));
        k.src = pa.src;
        k.node_pos = pa.node_pos;
        k.edges = pa.edges;
        k.infl_off = pa.infl_off;
        k.infl_node = pa.infl_node;
        k.infl_w = pa.infl_w;
        k.pairs = pa.pairs;
        k.reg_w = pa.reg_w;
        k.avg = pa.view.src_avg_edge_length;
        k.has_target = pa.view.target != nullptr;
        k.tgt = pa.tgt;
        k.valid = true;
    } else if (pa.view.target && (!k.has_target || k.tgt != pa.tgt)) {
        check(nrr_ctx_set_target(c, pa.tgt.data(), pa.view.m));
        k.tgt = pa.tgt;
        k.has_target = true;
    }
}
}  // namespace detail

/// deformation_graph.hpp:225-245 on the device (csrc/kernels.cu deform_kernel)
inline std::vector<Vec3> deform_points(const Surface& source, const DeformationGraph& graph, const NodeTransforms& x) {
    detail::ProblemArrays pa(source, nullptr, graph);
    nrr_ctx* c = detail::default_context();
    detail::use_problem(c, pa);
    std::vector<double> out(3 * source.points.size());
    detail::check(nrr_deform(c, x.stacked.data(), out.data()));
    return detail::unflat(out.data(), source.points.size());
}

}  // namespace nrr
