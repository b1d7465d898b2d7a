// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle_math.hpp header). A plain
// single-threaded CPU restatement of the reference hot path
// (/root/reference/proj/include/nrr, "nrr", arXiv 2206.03410) written without
// Eigen. Every function cites the reference file:line it follows. It is the
// checker for the CUDA path, never the thing measured or shipped.
//
// Parity pin: the reference stores no golden vectors on disk and cannot be
// compiled here (Eigen, Catch2, CLI11 absent), so this restatement is pinned
// against the reference tests' known-answer tests and properties
// (tests/test_oracle_kats.py lists each with its reference file:line).
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <deque>
#include <limits>
#include <numeric>
#include <queue>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include "oracle_math.hpp"

namespace oracle {

// =================================================================== welsch.hpp
// welsch.hpp:11-13
inline double welsch(double x, double nu) { return 1.0 - std::exp(-(x * x) / (2.0 * nu * nu)); }
// welsch.hpp:16-18
inline double welsch_sq(double x2, double nu) { return 1.0 - std::exp(-x2 / (2.0 * nu * nu)); }
// welsch.hpp:22-25
inline double welsch_weight_sq(double y2, double nu) {
    const double two_nu2 = 2.0 * nu * nu;
    return std::exp(-y2 / two_nu2) / two_nu2;
}
// welsch.hpp:30-33
inline double welsch_surrogate(double x, double y, double nu) {
    const double psi_y = welsch(y, nu);
    return psi_y + (1.0 - psi_y) / (2.0 * nu * nu) * (x * x - y * y);
}

// ================================================================== surface.hpp
// surface.hpp:17-46
struct Surface {
    std::vector<Vec3> points;
    std::vector<std::array<int, 3>> faces;
    std::vector<std::pair<int, int>> edges;
    double avg_edge_length = 0.0;
    std::vector<std::vector<std::pair<int, double>>> adjacency;

    int point_count() const { return static_cast<int>(points.size()); }

    void finalize_edges() {
        const int n = point_count();
        adjacency.assign(n, {});
        double total = 0.0;
        for (const auto& [a, b] : edges) {
            if (a < 0 || b < 0 || a >= n || b >= n)
                throw NumericalError("surface edge index out of range");
            if (a == b) throw NumericalError("surface edge is a self-loop");
            const double len = (points[a] - points[b]).norm();
            adjacency[a].emplace_back(b, len);
            adjacency[b].emplace_back(a, len);
            total += len;
        }
        for (auto& nb : adjacency) std::sort(nb.begin(), nb.end());
        avg_edge_length = edges.empty() ? 0.0 : total / static_cast<double>(edges.size());
    }
};

// surface.hpp:49-65
inline std::vector<std::pair<int, int>> edges_from_faces(
    const std::vector<std::array<int, 3>>& faces, int point_count) {
    std::vector<std::pair<int, int>> edges;
    edges.reserve(faces.size() * 3);
    for (const auto& f : faces)
        for (int c = 0; c < 3; ++c) {
            const int a = f[c], b = f[(c + 1) % 3];
            if (a < 0 || b < 0 || a >= point_count || b >= point_count)
                throw NumericalError("face index out of range");
            if (a == b) throw NumericalError("degenerate face with repeated vertex");
            edges.emplace_back(std::min(a, b), std::max(a, b));
        }
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    return edges;
}

// surface.hpp:70-94 (exhaustive; ties toward the smaller index)
inline std::vector<std::pair<int, int>> knn_edges(const std::vector<Vec3>& points, int k) {
    const int n = static_cast<int>(points.size());
    if (k < 1) throw ConfigError("knn_edges: k must be >= 1");
    if (k >= n) throw ConfigError("knn_edges: k must be smaller than the point count");
    std::vector<std::pair<int, int>> edges;
    std::vector<std::pair<double, int>> dist;
    for (int i = 0; i < n; ++i) {
        dist.clear();
        for (int j = 0; j < n; ++j)
            if (j != i) dist.emplace_back((points[i] - points[j]).squaredNorm(), j);
        std::partial_sort(dist.begin(), dist.begin() + k, dist.end());
        for (int t = 0; t < k; ++t) {
            const int j = dist[t].second;
            edges.emplace_back(std::min(i, j), std::max(i, j));
        }
    }
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    return edges;
}

// surface.hpp:98-110
inline Surface make_surface(std::vector<Vec3> points, std::vector<std::array<int, 3>> faces = {},
                            int knn_k = 6) {
    Surface s;
    s.points = std::move(points);
    s.faces = std::move(faces);
    if (!s.faces.empty())
        s.edges = edges_from_faces(s.faces, s.point_count());
    else if (s.point_count() > 1)
        s.edges = knn_edges(s.points, std::min(knn_k, s.point_count() - 1));
    s.finalize_edges();
    return s;
}

// surface.hpp:113-149
struct Normalization {
    double scale = 1.0;
    Vec3 center;
    Vec3 apply(const Vec3& v) const { return (v - center) * scale; }
    Vec3 invert(const Vec3& v) const { return v / scale + center; }  // surface.hpp:118
};
inline Normalization normalize_pair(Surface& source, Surface& target) {
    if (source.points.empty() || target.points.empty())
        throw NumericalError("normalize_pair: empty surface");
    Vec3 lo = source.points[0], hi = source.points[0];
    for (const auto* pts : {&source.points, &target.points})
        for (const auto& p : *pts) {
            lo = cwiseMin(lo, p);
            hi = cwiseMax(hi, p);
        }
    const double diag = (hi - lo).norm();
    if (!(diag > 0.0)) throw NumericalError("normalize_pair: degenerate joint bounding box");
    Normalization nm;
    nm.scale = 1.0 / diag;
    nm.center = (lo + hi) * 0.5;
    for (auto& p : source.points) p = nm.apply(p);
    for (auto& p : target.points) p = nm.apply(p);
    source.finalize_edges();
    target.finalize_edges();
    return nm;
}

// ================================================================= geodesic.hpp
/// geodesic.hpp:22-84. Same BFS ball + restricted Dijkstra (ties pop by
/// vertex index); the O(n) per-call buffers are replaced by a reusable
/// scratch with touched-list reset, which does not change any result.
struct GeodesicScratch {
    std::vector<char> in_ball, done;
    std::vector<double> dist;
    void ensure(int n) {
        if (static_cast<int>(in_ball.size()) != n) {
            in_ball.assign(n, 0);
            done.assign(n, 0);
            dist.assign(n, std::numeric_limits<double>::infinity());
        }
    }
};

inline std::vector<std::pair<int, double>> limited_geodesic(const Surface& surface, int source_index,
                                                            double radius, GeodesicScratch& sc) {
    const int n = surface.point_count();
    if (source_index < 0 || source_index >= n)
        throw ConfigError("limited_geodesic: source index out of range");
    if (!(radius > 0.0)) throw ConfigError("limited_geodesic: radius must be positive");
    if (surface.adjacency.empty() && n > 0)
        throw NumericalError("limited_geodesic: surface adjacency not built");
    sc.ensure(n);
    const Vec3 src = surface.points[source_index];
    std::vector<int> ball;
    std::queue<int> frontier;
    sc.in_ball[source_index] = 1;
    ball.push_back(source_index);
    frontier.push(source_index);
    while (!frontier.empty()) {
        const int v = frontier.front();
        frontier.pop();
        for (const auto& [w, len] : surface.adjacency[v]) {
            (void)len;
            if (sc.in_ball[w]) continue;
            if ((surface.points[w] - src).norm() < radius) {
                sc.in_ball[w] = 1;
                ball.push_back(w);
                frontier.push(w);
            }
        }
    }
    using Entry = std::pair<double, int>;
    std::priority_queue<Entry, std::vector<Entry>, std::greater<Entry>> heap;
    sc.dist[source_index] = 0.0;
    heap.emplace(0.0, source_index);
    while (!heap.empty()) {
        const auto [d, v] = heap.top();
        heap.pop();
        if (sc.done[v] || d > sc.dist[v]) continue;
        sc.done[v] = 1;
        if (d >= radius) continue;
        for (const auto& [w, len] : surface.adjacency[v]) {
            if (!sc.in_ball[w] || sc.done[w]) continue;
            const double cand = d + len;
            if (cand < sc.dist[w]) {
                sc.dist[w] = cand;
                heap.emplace(cand, w);
            }
        }
    }
    std::vector<std::pair<int, double>> result;
    std::sort(ball.begin(), ball.end());
    for (int v : ball)
        if (sc.dist[v] < radius) result.emplace_back(v, sc.dist[v]);
    for (int v : ball) {
        sc.in_ball[v] = 0;
        sc.done[v] = 0;
        sc.dist[v] = std::numeric_limits<double>::infinity();
    }
    return result;
}

// ======================================================== deformation_graph.hpp
/// deformation_graph.hpp:17-38 — 4N x 3 column-major; rows 4j..4j+3 = [A_j^T; t_j^T].
struct NodeTransforms {
    int nodes = 0;
    std::vector<double> stacked;  // column-major (4N x 3): stacked[c*4N + row]

    static NodeTransforms identity(int n) {
        NodeTransforms x;
        x.nodes = n;
        x.stacked.assign(static_cast<size_t>(12) * n, 0.0);
        for (int j = 0; j < n; ++j)
            for (int c = 0; c < 3; ++c) x.at(4 * j + c, c) = 1.0;
        return x;
    }
    static NodeTransforms zeros(int n) {
        NodeTransforms x;
        x.nodes = n;
        x.stacked.assign(static_cast<size_t>(12) * n, 0.0);
        return x;
    }
    int node_count() const { return nodes; }
    double& at(int row, int c) { return stacked[static_cast<size_t>(c) * 4 * nodes + row]; }
    double at(int row, int c) const { return stacked[static_cast<size_t>(c) * 4 * nodes + row]; }
    Mat3 affine(int j) const {
        Mat3 a;
        for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r) a(c, r) = at(4 * j + r, c);
        return a;
    }
    Vec3 translation(int j) const { return {at(4 * j + 3, 0), at(4 * j + 3, 1), at(4 * j + 3, 2)}; }
    void set(int j, const Mat3& a, const Vec3& t) {
        for (int c = 0; c < 3; ++c) {
            for (int r = 0; r < 3; ++r) at(4 * j + r, c) = a(c, r);
            at(4 * j + 3, c) = t[c];
        }
    }
    bool all_finite() const {
        for (double v : stacked)
            if (!std::isfinite(v)) return false;
        return true;
    }
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
    int node_count() const { return static_cast<int>(node_positions.size()); }
    int directed_pair_count() const { return static_cast<int>(reg_pairs.size()); }
    int edge_count() const { return static_cast<int>(graph_edges.size()); }
};

/// deformation_graph.hpp:73-106
inline std::vector<int> pca_order(const std::vector<Vec3>& points) {
    const int n = static_cast<int>(points.size());
    if (n == 0) throw ConfigError("pca_order: empty point set");
    Vec3 mean;
    for (const auto& p : points) mean += p;
    mean = mean * (1.0 / static_cast<double>(n));
    double cov[9] = {0};
    for (const auto& p : points) {
        const Vec3 d = p - mean;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) cov[r * 3 + c] += d[r] * d[c];
    }
    double ev[3], vecs[9];
    sym_eigen(cov, 3, ev, vecs);
    Vec3 axis(vecs[0 * 3 + 2], vecs[1 * 3 + 2], vecs[2 * 3 + 2]);
    if (!axis.finite()) axis = Vec3(1, 0, 0);
    for (int c = 0; c < 3; ++c)
        if (axis[c] != 0.0) {
            if (axis[c] < 0.0) axis = axis * -1.0;
            break;
        }
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::vector<double> proj(n);
    for (int i = 0; i < n; ++i) proj[i] = points[i].dot(axis);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        if (proj[a] != proj[b]) return proj[a] < proj[b];
        return a < b;
    });
    return order;
}

/// deformation_graph.hpp:111-125
inline std::vector<double> influence_weights(const std::vector<double>& distances, double radius) {
    if (distances.empty()) throw ConfigError("influence_weights: empty influence set");
    std::vector<double> w(distances.size());
    double total = 0.0;
    for (size_t k = 0; k < distances.size(); ++k) {
        const double ratio = 1.0 - (distances[k] * distances[k]) / (radius * radius);
        if (!(ratio > 0.0)) throw NumericalError("influence_weights: distance not below radius");
        w[k] = ratio * ratio * ratio;
        total += w[k];
    }
    for (auto& v : w) v /= total;
    return w;
}

/// deformation_graph.hpp:130-148
inline void reg_weight_table(DeformationGraph& g) {
    g.reg_pairs.clear();
    g.reg_weights.clear();
    if (g.graph_edges.empty()) return;
    double inv_sum = 0.0;
    for (int i = 0; i < g.node_count(); ++i)
        for (int j : g.node_neighbors[i]) {
            const double len = (g.node_positions[i] - g.node_positions[j]).norm();
            if (!(len > 0.0)) throw NumericalError("reg_weight_table: coincident node positions");
            g.reg_pairs.emplace_back(i, j);
            g.reg_weights.push_back(1.0 / len);
            inv_sum += 1.0 / len;
        }
    const double scale = static_cast<double>(g.reg_pairs.size()) / inv_sum;
    for (auto& c : g.reg_weights) c *= scale;
}

/// deformation_graph.hpp:157-210
inline DeformationGraph build_graph(const Surface& source, double radius) {
    const int n = source.point_count();
    if (n == 0) throw ConfigError("build_graph: empty source surface");
    if (!(radius > 0.0)) throw ConfigError("build_graph: radius must be positive");
    DeformationGraph g;
    g.radius = radius;
    std::vector<std::vector<std::pair<int, double>>> raw(n);
    GeodesicScratch sc;
    for (int idx : pca_order(source.points)) {
        if (!g.node_indices.empty() && !raw[idx].empty()) continue;
        const int node_id = g.node_count();
        g.node_indices.push_back(idx);
        g.node_positions.push_back(source.points[idx]);
        for (const auto& [q, dist] : limited_geodesic(source, idx, radius, sc))
            raw[q].emplace_back(node_id, dist);
    }
    std::vector<std::pair<int, int>> edges;
    for (int i = 0; i < n; ++i) {
        const auto& list = raw[i];
        for (size_t a = 0; a < list.size(); ++a)
            for (size_t b = a + 1; b < list.size(); ++b)
                edges.emplace_back(list[a].first, list[b].first);
    }
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    g.graph_edges = std::move(edges);
    g.node_neighbors.assign(g.node_count(), {});
    for (const auto& [a, b] : g.graph_edges) {
        g.node_neighbors[a].push_back(b);
        g.node_neighbors[b].push_back(a);
    }
    for (auto& nb : g.node_neighbors) std::sort(nb.begin(), nb.end());
    g.influence.assign(n, {});
    std::vector<double> dists;
    for (int i = 0; i < n; ++i) {
        if (raw[i].empty()) throw NumericalError("build_graph: point left without influencing nodes");
        dists.clear();
        for (const auto& [node, d] : raw[i]) dists.push_back(d);
        const std::vector<double> w = influence_weights(dists, radius);
        g.influence[i].resize(raw[i].size());
        for (size_t k = 0; k < raw[i].size(); ++k)
            g.influence[i][k] = {raw[i][k].first, w[k], raw[i][k].second};
    }
    reg_weight_table(g);
    return g;
}

/// deformation_graph.hpp:214-222
inline Vec3 deformed_position(const Vec3& v, const std::vector<InfluenceEntry>& inf,
                              const DeformationGraph& g, const NodeTransforms& x) {
    Vec3 out;
    for (const auto& e : inf) {
        const Vec3& p = g.node_positions[e.node];
        out += e.weight * (x.affine(e.node) * (v - p) + p + x.translation(e.node));
    }
    return out;
}

/// deformation_graph.hpp:225-245
inline std::vector<Vec3> deform_points(const std::vector<Vec3>& source, const DeformationGraph& g,
                                       const NodeTransforms& x) {
    const int m = g.node_count();
    std::vector<Mat3> rot(m);
    std::vector<Vec3> shift(m);
    for (int j = 0; j < m; ++j) {
        rot[j] = x.affine(j);
        shift[j] = g.node_positions[j] + x.translation(j);
    }
    std::vector<Vec3> out(source.size());
    for (size_t i = 0; i < source.size(); ++i) {
        Vec3 acc;
        for (const auto& e : g.influence[i])
            acc += e.weight * (rot[e.node] * (source[i] - g.node_positions[e.node]) + shift[e.node]);
        out[i] = acc;
    }
    return out;
}

// ================================================================== kd_tree.hpp
/// kd_tree.hpp:17-107 — exact NN, median split, leaf size 8, ties -> smallest
/// index (:88), non-strict far-side prune (:99-100), distance = sqrt(best_d2) (:37).
class SpatialIndex {
public:
    struct Hit {
        int index = -1;
        double distance = 0.0;
    };
    explicit SpatialIndex(std::vector<Vec3> points) : points_(std::move(points)) {
        if (points_.empty()) throw NumericalError("SpatialIndex: cannot index an empty point set");
        order_.resize(points_.size());
        std::iota(order_.begin(), order_.end(), 0);
        nodes_.reserve(2 * points_.size() / kLeaf + 2);
        root_ = build(0, static_cast<int>(points_.size()));
    }
    Hit nearest(const Vec3& q) const {
        int bi = -1;
        double bd2 = std::numeric_limits<double>::infinity();
        search(root_, q, bi, bd2);
        return {bi, std::sqrt(bd2)};
    }
    const std::vector<Vec3>& points() const { return points_; }
    int size() const { return static_cast<int>(points_.size()); }

private:
    static constexpr int kLeaf = 8;
    struct Node {
        int axis = -1;
        double split = 0.0;
        int left = -1, right = -1, begin = 0, end = 0;
    };
    int build(int begin, int end) {
        Node node;
        if (end - begin <= kLeaf) {
            node.begin = begin;
            node.end = end;
            nodes_.push_back(node);
            return static_cast<int>(nodes_.size()) - 1;
        }
        Vec3 lo = points_[order_[begin]], hi = lo;
        for (int i = begin + 1; i < end; ++i) {
            lo = cwiseMin(lo, points_[order_[i]]);
            hi = cwiseMax(hi, points_[order_[i]]);
        }
        const Vec3 ext = hi - lo;
        int axis = 0;
        if (ext.y > ext[axis]) axis = 1;
        if (ext.z > ext[axis]) axis = 2;
        const int mid = begin + (end - begin) / 2;
        std::nth_element(order_.begin() + begin, order_.begin() + mid, order_.begin() + end,
                         [&](int a, int b) { return points_[a][axis] < points_[b][axis]; });
        node.axis = axis;
        node.split = points_[order_[mid]][axis];
        nodes_.push_back(node);
        const int self = static_cast<int>(nodes_.size()) - 1;
        const int l = build(begin, mid);
        const int r = build(mid, end);
        nodes_[self].left = l;
        nodes_[self].right = r;
        return self;
    }
    void search(int id, const Vec3& q, int& bi, double& bd2) const {
        const Node& node = nodes_[id];
        if (node.axis < 0) {
            for (int i = node.begin; i < node.end; ++i) {
                const int idx = order_[i];
                const double d2 = (points_[idx] - q).squaredNorm();
                if (d2 < bd2 || (d2 == bd2 && idx < bi)) {
                    bd2 = d2;
                    bi = idx;
                }
            }
            return;
        }
        const double diff = q[node.axis] - node.split;
        const int near = diff < 0.0 ? node.left : node.right;
        const int far = diff < 0.0 ? node.right : node.left;
        search(near, q, bi, bd2);
        if (diff * diff <= bd2) search(far, q, bi, bd2);
    }
    std::vector<Vec3> points_;
    std::vector<int> order_;
    std::vector<Node> nodes_;
    int root_ = -1;
};

// =================================================================== energy.hpp
struct Correspondences {  // energy.hpp:20-26
    std::vector<int> target_index;
    std::vector<Vec3> target_point;
    std::vector<double> squared_distance;
    int size() const { return static_cast<int>(target_index.size()); }
};

/// energy.hpp:28-42 (squared_distance = distance^2, distance = sqrt(d2))
inline Correspondences find_correspondences(const std::vector<Vec3>& deformed,
                                            const SpatialIndex& target) {
    Correspondences c;
    const int n = static_cast<int>(deformed.size());
    c.target_index.resize(n);
    c.target_point.resize(n);
    c.squared_distance.resize(n);
    for (int i = 0; i < n; ++i) {
        const auto hit = target.nearest(deformed[i]);
        c.target_index[i] = hit.index;
        c.target_point[i] = target.points()[hit.index];
        c.squared_distance[i] = hit.distance * hit.distance;
    }
    return c;
}

/// energy.hpp:47-56 (degenerate when sigma_min < 1e-12)
inline std::vector<Mat3> project_rotations(const NodeTransforms& x, int* degenerate = nullptr) {
    std::vector<Mat3> rot(x.node_count());
    for (int j = 0; j < x.node_count(); ++j) {
        double smin = 0.0;
        rot[j] = project_to_rotation(x.affine(j), &smin);
        if (degenerate && smin < 1e-12) ++*degenerate;
    }
    return rot;
}

struct EnergyParams {  // energy.hpp:58-63
    double alpha = 0.0, beta = 0.0, nu_a = 1.0, nu_r = 1.0;
};
struct EnergyBreakdown {  // energy.hpp:65-72
    double align = 0, reg = 0, rot = 0, total = 0;
    double alpha = 0, beta = 0, nu_a = 0, nu_r = 0;
};

/// energy.hpp:77-84
inline Vec3 reg_difference(const DeformationGraph& g, const NodeTransforms& x, int e) {
    const auto [i, j] = g.reg_pairs[e];
    const double c = g.reg_weights[e];
    const Vec3& pi = g.node_positions[i];
    const Vec3& pj = g.node_positions[j];
    return c * (x.affine(j) * (pi - pj) + pj + x.translation(j) - pi - x.translation(i));
}

inline double frob2_diff(const Mat3& a, const Mat3& b) {
    double s = 0;
    for (int k = 0; k < 9; ++k) s += (a.m[k] - b.m[k]) * (a.m[k] - b.m[k]);
    return s;
}

/// energy.hpp:92-116
inline EnergyBreakdown evaluate_energy(const std::vector<Vec3>& deformed, const NodeTransforms& x,
                                       const DeformationGraph& g, const Correspondences& corr,
                                       const std::vector<Mat3>& rotations, const EnergyParams& prm) {
    if (corr.size() != static_cast<int>(deformed.size()))
        throw NumericalError("evaluate_energy: correspondence count mismatch");
    if (static_cast<int>(rotations.size()) != g.node_count())
        throw NumericalError("evaluate_energy: rotation count mismatch");
    EnergyBreakdown e;
    for (size_t i = 0; i < deformed.size(); ++i)
        e.align += welsch_sq((deformed[i] - corr.target_point[i]).squaredNorm(), prm.nu_a);
    for (int k = 0; k < g.directed_pair_count(); ++k)
        e.reg += welsch_sq(reg_difference(g, x, k).squaredNorm(), prm.nu_r);
    for (int j = 0; j < g.node_count(); ++j) e.rot += frob2_diff(x.affine(j), rotations[j]);
    e.total = e.align + prm.alpha * e.reg + prm.beta * e.rot;
    e.alpha = prm.alpha;
    e.beta = prm.beta;
    e.nu_a = prm.nu_a;
    e.nu_r = prm.nu_r;
    return e;
}

struct Landmark {  // energy.hpp:125-128
    int source_index = -1;
    Vec3 target_position;
};

/// Block-sparse 4N x 4N matrix with the reference's fixed pattern: a 4x4
/// diagonal block per node plus both halves of every graph edge
/// (energy.hpp:264-279). Block row a holds the sorted column list
/// {a} U neighbors(a); values row-major per block.
struct BlockSparse {
    int nodes = 0;
    std::vector<int> row_ptr, col;  // block CSR
    std::vector<double> val;        // 16 per block, row-major 4x4
    int find(int a, int b) const {
        const auto lo = col.begin() + row_ptr[a], hi = col.begin() + row_ptr[a + 1];
        const auto it = std::lower_bound(lo, hi, b);
        if (it == hi || *it != b) return -1;
        return static_cast<int>(it - col.begin());
    }
    double& at(int row, int colm) {
        const int b = find(row / 4, colm / 4);
        if (b < 0) throw NumericalError("oracle: entry outside the fixed pattern");
        return val[static_cast<size_t>(b) * 16 + (row % 4) * 4 + (colm % 4)];
    }
    double get(int row, int colm) const {
        const int b = find(row / 4, colm / 4);
        return b < 0 ? 0.0 : val[static_cast<size_t>(b) * 16 + (row % 4) * 4 + (colm % 4)];
    }
    // y = K x for a 4N x 3 column-major block of right-hand sides
    std::vector<double> multiply(const std::vector<double>& x) const {
        const size_t dim = static_cast<size_t>(4) * nodes;
        std::vector<double> y(dim * 3, 0.0);
        for (int a = 0; a < nodes; ++a)
            for (int k = row_ptr[a]; k < row_ptr[a + 1]; ++k) {
                const int b = col[k];
                const double* v = &val[static_cast<size_t>(k) * 16];
                for (int c = 0; c < 3; ++c)
                    for (int r = 0; r < 4; ++r) {
                        double s = 0;
                        for (int q = 0; q < 4; ++q) s += v[r * 4 + q] * x[c * dim + 4 * b + q];
                        y[c * dim + 4 * a + r] += s;
                    }
            }
        return y;
    }
};

struct LinearSystem {  // energy.hpp:118-121
    BlockSparse K;
    std::vector<double> B;  // 4N x 3 column-major
};

/// Envelope (skyline) LDL^T over the scalar 4N system with a reverse
/// Cuthill-McKee node ordering. Stands in for Eigen::SimplicialLDLT
/// (energy.hpp:234-238, 394): the factorization fails exactly when a pivot
/// D_ii is exactly zero, as SimplicialLDLT's numeric factorization does.
/// Node ordering of the direct solve: 0 = reverse Cuthill-McKee (default),
/// 1 = natural order. The reference's Eigen SimplicialLDLT uses yet another
/// (AMD) order; the parity tests use the spread between two valid orders as
/// the reference's own rounding-level reproducibility.
inline int& ldlt_ordering() {
    static int mode = 0;
    return mode;
}

class EnvelopeLDLT {
public:
    void analyze(const BlockSparse& k) {
        n_nodes_ = k.nodes;
        const int N = k.nodes;
        if (ldlt_ordering() == 1) {
            perm_.resize(N);
            std::iota(perm_.begin(), perm_.end(), 0);
            finish_analysis(k);
            return;
        }
        // RCM over the node graph, component by component, min-degree start
        perm_.clear();
        std::vector<char> seen(N, 0);
        std::vector<int> deg(N);
        for (int a = 0; a < N; ++a) deg[a] = k.row_ptr[a + 1] - k.row_ptr[a];
        std::vector<int> by_deg(N);
        std::iota(by_deg.begin(), by_deg.end(), 0);
        std::stable_sort(by_deg.begin(), by_deg.end(), [&](int a, int b) { return deg[a] < deg[b]; });
        for (int start : by_deg) {
            if (seen[start]) continue;
            size_t head = perm_.size();
            perm_.push_back(start);
            seen[start] = 1;
            while (head < perm_.size()) {
                const int v = perm_[head++];
                std::vector<int> nb;
                for (int e = k.row_ptr[v]; e < k.row_ptr[v + 1]; ++e)
                    if (!seen[k.col[e]]) nb.push_back(k.col[e]);
                std::stable_sort(nb.begin(), nb.end(), [&](int a, int b) { return deg[a] < deg[b]; });
                for (int w : nb) {
                    seen[w] = 1;
                    perm_.push_back(w);
                }
            }
        }
        std::reverse(perm_.begin(), perm_.end());
        finish_analysis(k);
    }

    void finish_analysis(const BlockSparse& k) {
        const int N = k.nodes;
        inv_.assign(N, 0);
        for (int i = 0; i < N; ++i) inv_[perm_[i]] = i;
        // first column (in permuted scalar order) of each permuted scalar row
        const int n = 4 * N;
        first_.assign(n, 0);
        for (int pi = 0; pi < N; ++pi) {
            const int a = perm_[pi];
            int fmin = pi;
            for (int e = k.row_ptr[a]; e < k.row_ptr[a + 1]; ++e) fmin = std::min(fmin, inv_[k.col[e]]);
            for (int r = 0; r < 4; ++r) first_[4 * pi + r] = 4 * fmin;
        }
        offs_.assign(n + 1, 0);
        for (int i = 0; i < n; ++i) offs_[i + 1] = offs_[i] + (i - first_[i]);
        analyzed_ = true;
    }
    bool analyzed() const { return analyzed_; }

    /// Returns false if a pivot is exactly zero.
    bool factorize(const BlockSparse& k) {
        const int N = n_nodes_, n = 4 * N;
        L_.assign(offs_[n], 0.0);
        D_.assign(n, 0.0);
        std::vector<double> diag(n, 0.0);
        // scatter lower triangle (permuted) into the envelope
        for (int a = 0; a < N; ++a)
            for (int e = k.row_ptr[a]; e < k.row_ptr[a + 1]; ++e) {
                const int b = k.col[e];
                const double* v = &k.val[static_cast<size_t>(e) * 16];
                for (int r = 0; r < 4; ++r)
                    for (int c = 0; c < 4; ++c) {
                        const int i = 4 * inv_[a] + r, j = 4 * inv_[b] + c;
                        if (j < i) L_[offs_[i] + (j - first_[i])] = v[r * 4 + c];
                        else if (i == j) diag[i] = v[r * 4 + c];
                    }
            }
        for (int i = 0; i < n; ++i) {
            const int fi = first_[i];
            double* li = &L_[offs_[i]];  // li[j - fi], j in [fi, i)
            for (int j = fi; j < i; ++j) {
                const int fj = first_[j];
                const double* lj = &L_[offs_[j]];
                double s = li[j - fi];
                for (int q = std::max(fi, fj); q < j; ++q) s -= li[q - fi] * lj[q - fj];
                li[j - fi] = s;  // = L_ij * D_j
            }
            double d = diag[i];
            for (int j = fi; j < i; ++j) {
                const double t = li[j - fi];
                const double l = t / D_[j];
                li[j - fi] = l;
                d -= t * l;
            }
            if (d == 0.0 || !std::isfinite(d)) return false;
            D_[i] = d;
        }
        return true;
    }

    /// Solves for a 4N x 3 column-major right-hand side.
    std::vector<double> solve(const std::vector<double>& b) const {
        const int N = n_nodes_, n = 4 * N;
        std::vector<double> x(b.size());
        std::vector<double> y(n);
        for (int c = 0; c < 3; ++c) {
            for (int pi = 0; pi < N; ++pi)
                for (int r = 0; r < 4; ++r) y[4 * pi + r] = b[static_cast<size_t>(c) * n + 4 * perm_[pi] + r];
            for (int i = 0; i < n; ++i) {
                const double* li = &L_[offs_[i]];
                double s = y[i];
                for (int j = first_[i]; j < i; ++j) s -= li[j - first_[i]] * y[j];
                y[i] = s;
            }
            for (int i = 0; i < n; ++i) y[i] /= D_[i];
            for (int i = n - 1; i >= 0; --i) {
                const double* li = &L_[offs_[i]];
                const double yi = y[i];
                for (int j = first_[i]; j < i; ++j) y[j] -= li[j - first_[i]] * yi;
            }
            for (int pi = 0; pi < N; ++pi)
                for (int r = 0; r < 4; ++r) x[static_cast<size_t>(c) * n + 4 * perm_[pi] + r] = y[4 * pi + r];
        }
        return x;
    }

private:
    int n_nodes_ = 0;
    bool analyzed_ = false;
    std::vector<int> perm_, inv_, first_;
    std::vector<long long> offs_;
    std::vector<double> L_, D_;
};

inline double max_abs(const std::vector<double>& v) {
    double m = 0;
    for (double x : v) m = std::max(m, std::abs(x));
    return m;
}

/// energy.hpp:329-340
inline std::string describe_failure(const BlockSparse& k) {
    for (int j = 0; j < k.nodes; ++j) {
        double blk[16], ev[4], vecs[16];
        const int b = k.find(j, j);
        for (int i = 0; i < 16; ++i) blk[i] = k.val[static_cast<size_t>(b) * 16 + i];
        sym_eigen(blk, 4, ev, vecs);
        if (ev[0] <= 0.0) return "singular diagonal block at node " + std::to_string(j);
    }
    return "indefinite coupling between node blocks";
}

/// The residual check + single refinement of energy.hpp:245-252 / :399-406.
inline NodeTransforms solve_with_check(const LinearSystem& sys, EnvelopeLDLT& ldlt, bool describe) {
    if (!ldlt.analyzed()) ldlt.analyze(sys.K);
    if (!ldlt.factorize(sys.K))
        throw NumericalError(describe ? "linear system not positive definite (" +
                                            describe_failure(sys.K) + ")"
                                      : "linear system not positive definite");
    NodeTransforms x = NodeTransforms::zeros(sys.K.nodes);
    x.stacked = ldlt.solve(sys.B);
    const double tol = 1e-8 * (1.0 + max_abs(sys.B));
    std::vector<double> kx = sys.K.multiply(x.stacked);
    std::vector<double> res(sys.B.size());
    for (size_t i = 0; i < res.size(); ++i) res[i] = sys.B[i] - kx[i];
    if (max_abs(res) > tol) {
        const std::vector<double> dx = ldlt.solve(res);
        for (size_t i = 0; i < res.size(); ++i) x.stacked[i] += dx[i];
        kx = sys.K.multiply(x.stacked);
        for (size_t i = 0; i < res.size(); ++i) res[i] = sys.B[i] - kx[i];
        if (max_abs(res) > tol) throw NumericalError("linear solve residual above tolerance");
    }
    return x;
}

/// energy.hpp:137-359, program-free: the values of the reference's
/// contribution program (energy.hpp:290-327) recomputed directly in the same
/// order (points, then directed pairs, then landmarks, then beta), so each K
/// entry receives the same sequence of additions as the reference fill.
class SystemAssembler {
public:
    SystemAssembler(const std::vector<Vec3>& source, const DeformationGraph& g,
                    std::vector<Landmark> landmarks = {})
        : source_(&source), g_(&g), landmarks_(std::move(landmarks)) {
        const int n = static_cast<int>(source.size());
        const int N = g.node_count();
        for (const auto& lm : landmarks_)
            if (lm.source_index < 0 || lm.source_index >= n)
                throw ConfigError("landmark source index out of range");
        // energy.hpp:150-161
        point_f_.resize(n);
        anchor_.assign(n, Vec3());
        for (int i = 0; i < n; ++i) {
            const auto& inf = g.influence[i];
            point_f_[i].resize(inf.size());
            for (size_t a = 0; a < inf.size(); ++a) {
                const Vec3 d = source[i] - g.node_positions[inf[a].node];
                const double w = inf[a].weight;
                point_f_[i][a] = {w * d.x, w * d.y, w * d.z, w};
                anchor_[i] += w * g.node_positions[inf[a].node];
            }
        }
        // energy.hpp:164-173
        const int P = g.directed_pair_count();
        pair_g_.resize(P);
        pair_y_.resize(P);
        for (int e = 0; e < P; ++e) {
            const auto [i, j] = g.reg_pairs[e];
            const double c = g.reg_weights[e];
            const Vec3 d = g.node_positions[i] - g.node_positions[j];
            pair_g_[e] = {c * d.x, c * d.y, c * d.z, c};
            pair_y_[e] = c * d;
        }
        // pattern (energy.hpp:264-279)
        BlockSparse& K = sys_.K;
        K.nodes = N;
        std::vector<std::vector<int>> cols(N);
        for (int j = 0; j < N; ++j) cols[j].push_back(j);
        for (const auto& [a, b] : g.graph_edges) {
            cols[a].push_back(b);
            cols[b].push_back(a);
        }
        K.row_ptr.assign(N + 1, 0);
        for (int j = 0; j < N; ++j) {
            std::sort(cols[j].begin(), cols[j].end());
            cols[j].erase(std::unique(cols[j].begin(), cols[j].end()), cols[j].end());
            K.row_ptr[j + 1] = K.row_ptr[j] + static_cast<int>(cols[j].size());
        }
        K.col.reserve(K.row_ptr[N]);
        for (int j = 0; j < N; ++j) K.col.insert(K.col.end(), cols[j].begin(), cols[j].end());
        K.val.assign(static_cast<size_t>(K.row_ptr[N]) * 16, 0.0);
        sys_.B.assign(static_cast<size_t>(12) * N, 0.0);
        // resolve every block a point touches once (the reference's slot())
        point_blocks_.resize(n);
        for (int i = 0; i < n; ++i) {
            const auto& inf = g.influence[i];
            const size_t k = inf.size();
            point_blocks_[i].resize(k * k);
            for (size_t a = 0; a < k; ++a)
                for (size_t b = 0; b < k; ++b) {
                    const int blk = K.find(inf[a].node, inf[b].node);
                    if (blk < 0)
                        throw NumericalError("assemble: co-influencing node pair is not a graph edge");
                    point_blocks_[i][a * k + b] = blk;
                }
        }
        pair_blocks_.resize(P);
        for (int e = 0; e < P; ++e) {
            const auto [i, j] = g.reg_pairs[e];
            pair_blocks_[e] = {K.find(j, j), K.find(j, i), K.find(i, j), K.find(i, i)};
        }
    }

    /// energy.hpp:182-228
    void fill(const Correspondences& corr, const std::vector<Mat3>& rotations,
              const std::vector<double>& w_align, const std::vector<double>& w_reg, double beta,
              double landmark_weight = 0.0) {
        const int n = static_cast<int>(source_->size());
        const int N = g_->node_count();
        if (corr.size() != n) throw NumericalError("assemble: correspondence count mismatch");
        if (static_cast<int>(w_align.size()) != n)
            throw NumericalError("assemble: alignment weight count mismatch");
        if (static_cast<int>(w_reg.size()) != g_->directed_pair_count())
            throw NumericalError("assemble: regularization weight count mismatch");
        if (static_cast<int>(rotations.size()) != N)
            throw NumericalError("assemble: rotation count mismatch");
        double* val = sys_.K.val.data();
        std::fill(sys_.K.val.begin(), sys_.K.val.end(), 0.0);
        for (int i = 0; i < n; ++i) emit_point(i, w_align[i], val);
        for (int e = 0; e < g_->directed_pair_count(); ++e) {
            const auto& gg = pair_g_[e];
            const double c = g_->reg_weights[e];
            const auto& pb = pair_blocks_[e];
            const double w = w_reg[e];
            for (int r = 0; r < 4; ++r)
                for (int cc = 0; cc < 4; ++cc) val[pb[0] * 16 + r * 4 + cc] += w * (gg[r] * gg[cc]);
            for (int r = 0; r < 4; ++r) {
                val[pb[1] * 16 + r * 4 + 3] += w * (gg[r] * -c);
                val[pb[2] * 16 + 3 * 4 + r] += w * (-c * gg[r]);
            }
            val[pb[3] * 16 + 15] += w * (c * c);
        }
        if (landmark_weight != 0.0)
            for (const auto& lm : landmarks_) emit_point(lm.source_index, landmark_weight, val);
        for (int j = 0; j < N; ++j) {
            const int b = sys_.K.find(j, j);
            for (int r = 0; r < 3; ++r) val[b * 16 + r * 4 + r] += beta;
        }
        std::vector<double>& B = sys_.B;
        std::fill(B.begin(), B.end(), 0.0);
        const size_t dim = static_cast<size_t>(4) * N;
        for (int i = 0; i < n; ++i) {
            const Vec3 q = corr.target_point[i] - anchor_[i];
            const auto& inf = g_->influence[i];
            for (size_t a = 0; a < inf.size(); ++a)
                for (int r = 0; r < 4; ++r) {
                    const double wf = w_align[i] * point_f_[i][a][r];
                    for (int c = 0; c < 3; ++c) B[c * dim + 4 * inf[a].node + r] += wf * q[c];
                }
        }
        for (int e = 0; e < g_->directed_pair_count(); ++e) {
            const auto [i, j] = g_->reg_pairs[e];
            const double c = g_->reg_weights[e];
            for (int r = 0; r < 4; ++r) {
                const double wg = w_reg[e] * pair_g_[e][r];
                for (int cc = 0; cc < 3; ++cc) B[cc * dim + 4 * j + r] += wg * pair_y_[e][cc];
            }
            const double wc = w_reg[e] * -c;
            for (int cc = 0; cc < 3; ++cc) B[cc * dim + 4 * i + 3] += wc * pair_y_[e][cc];
        }
        for (int j = 0; j < N; ++j)
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) B[c * dim + 4 * j + r] += beta * rotations[j](c, r);
        if (landmark_weight != 0.0)
            for (const auto& lm : landmarks_) {
                const int i = lm.source_index;
                const Vec3 q = lm.target_position - anchor_[i];
                const auto& inf = g_->influence[i];
                for (size_t a = 0; a < inf.size(); ++a)
                    for (int r = 0; r < 4; ++r) {
                        const double wf = landmark_weight * point_f_[i][a][r];
                        for (int c = 0; c < 3; ++c) B[c * dim + 4 * inf[a].node + r] += wf * q[c];
                    }
            }
    }

    const LinearSystem& system() const { return sys_; }
    LinearSystem& system() { return sys_; }

    /// energy.hpp:233-254
    NodeTransforms solve() { return solve_with_check(sys_, ldlt_, true); }

    const std::vector<std::vector<std::array<double, 4>>>& point_f() const { return point_f_; }
    const std::vector<Vec3>& anchor() const { return anchor_; }

private:
    void emit_point(int i, double w, double* val) const {  // energy.hpp:313-327
        const auto& f = point_f_[i];
        const size_t k = f.size();
        for (size_t a = 0; a < k; ++a)
            for (size_t b = 0; b < k; ++b) {
                double* blk = val + static_cast<size_t>(point_blocks_[i][a * k + b]) * 16;
                for (int r = 0; r < 4; ++r)
                    for (int c = 0; c < 4; ++c) blk[r * 4 + c] += w * (f[a][r] * f[b][c]);
            }
    }

    const std::vector<Vec3>* source_;
    const DeformationGraph* g_;
    std::vector<Landmark> landmarks_;
    std::vector<std::vector<std::array<double, 4>>> point_f_;
    std::vector<Vec3> anchor_;
    std::vector<std::array<double, 4>> pair_g_;
    std::vector<Vec3> pair_y_;
    std::vector<std::vector<int>> point_blocks_;
    std::vector<std::array<int, 4>> pair_blocks_;
    LinearSystem sys_;
    EnvelopeLDLT ldlt_;
};

/// energy.hpp:363-368
inline std::vector<double> alignment_weights(const Correspondences& corr, double nu_a) {
    std::vector<double> w(corr.size());
    for (int i = 0; i < corr.size(); ++i) w[i] = welsch_weight_sq(corr.squared_distance[i], nu_a);
    return w;
}
/// energy.hpp:371-378
inline std::vector<double> regularization_weights(const DeformationGraph& g, const NodeTransforms& x,
                                                  double nu_r, double alpha) {
    std::vector<double> w(g.directed_pair_count());
    for (int e = 0; e < g.directed_pair_count(); ++e)
        w[e] = alpha * welsch_weight_sq(reg_difference(g, x, e).squaredNorm(), nu_r);
    return w;
}
/// energy.hpp:393-408
inline NodeTransforms solve_system(const LinearSystem& sys) {
    EnvelopeLDLT ldlt;
    return solve_with_check(sys, ldlt, false);
}

// ================================================================= anderson.hpp
struct AndersonEntry {  // anderson.hpp:12-15
    std::vector<double> g, f;
};

/// anderson.hpp:22-46
inline std::vector<double> anderson_combine(const std::deque<AndersonEntry>& h, int m,
                                            int* rank_out = nullptr) {
    if (h.empty()) throw NumericalError("anderson_combine: empty history");
    const int n = static_cast<int>(h.size());
    const int mk = std::min(n - 1, m);
    const std::vector<double>& g_last = h[n - 1].g;
    if (mk <= 0) return g_last;
    const size_t dim = g_last.size();
    std::vector<double> df(dim * mk), dg(dim * mk);
    for (int j = 1; j <= mk; ++j)
        for (size_t i = 0; i < dim; ++i) {
            df[(j - 1) * dim + i] = h[n - j].f[i] - h[n - j - 1].f[i];
            dg[(j - 1) * dim + i] = h[n - j].g[i] - h[n - j - 1].g[i];
        }
    std::vector<double> theta;
    ColPivQR qr(df, static_cast<int>(dim), mk);
    const int rk = qr.rank();
    if (rank_out) *rank_out = rk;
    if (rk == mk) {
        theta = qr.solve(h[n - 1].f);
    } else {
        std::vector<double> normal(mk * mk), rhs(mk);
        for (int a = 0; a < mk; ++a) {
            for (int b = 0; b < mk; ++b) {
                double s = 0;
                for (size_t i = 0; i < dim; ++i) s += df[a * dim + i] * df[b * dim + i];
                normal[a * mk + b] = s;
            }
            normal[a * mk + a] += 1e-10;
            double s = 0;
            for (size_t i = 0; i < dim; ++i) s += df[a * dim + i] * h[n - 1].f[i];
            rhs[a] = s;
        }
        theta = ldlt_solve(normal, mk, rhs);
    }
    std::vector<double> out(g_last);
    for (int j = 0; j < mk; ++j)
        for (size_t i = 0; i < dim; ++i) out[i] -= dg[j * dim + i] * theta[j];
    return out;
}

/// anderson.hpp:50-73
class AndersonWindow {
public:
    explicit AndersonWindow(int m) : m_(m) {
        if (m < 0) throw ConfigError("AndersonWindow: window must be >= 0");
    }
    void reset() { h_.clear(); }
    void push(std::vector<double> g, std::vector<double> f) {
        h_.push_back({std::move(g), std::move(f)});
        while (static_cast<int>(h_.size()) > m_ + 1) h_.pop_front();
    }
    bool extrapolating() const { return m_ > 0 && h_.size() > 1; }
    std::vector<double> combine() const { return anderson_combine(h_, m_); }
    int size() const { return static_cast<int>(h_.size()); }

private:
    int m_;
    std::deque<AndersonEntry> h_;
};

// =================================================================== solver.hpp
struct SolverConfig {  // solver.hpp:16-39
    double k_alpha = 100.0, k_beta = 1.0, eps = 1e-5;
    int i_max = 100, aa_window = 5;
    double nu_a_init = std::numeric_limits<double>::quiet_NaN();
    double nu_a_min = std::numeric_limits<double>::quiet_NaN();
    double nu_r_init = std::numeric_limits<double>::quiet_NaN();
    double nu_r_floor = 1e-8;
    std::vector<Landmark> landmarks;
    void validate() const {
        if (!(eps > 0.0)) throw ConfigError("eps must be positive");
        if (i_max < 1) throw ConfigError("i_max must be at least 1");
        if (aa_window < 0) throw ConfigError("aa_window must be >= 0");
        if (k_alpha < 0.0 || k_beta < 0.0) throw ConfigError("k_alpha and k_beta must be non-negative");
    }
};

struct SolverParams {  // solver.hpp:42-49
    double nu_a = 0, nu_r = 0, nu_a_min = 0, alpha = 0, beta = 0;
    bool alpha_forced_zero = false;
};
struct AnnealResult {
    double nu_a = 0, nu_r = 0;
    bool done = false;
};
// solver.hpp:60-64
inline AnnealResult anneal(double nu_a, double nu_r, double nu_a_min, double nu_r_floor = 1e-8) {
    if (nu_a == nu_a_min) return {nu_a, nu_r, true};
    return {std::max(nu_a / 2.0, nu_a_min), std::max(nu_r / 2.0, nu_r_floor), false};
}
// solver.hpp:68-80
inline void update_term_weights(SolverParams& p, int point_count, const DeformationGraph& g,
                                const SolverConfig& cfg) {
    if (g.edge_count() == 0) {
        p.alpha = 0.0;
        p.alpha_forced_zero = true;
    } else {
        p.alpha = cfg.k_alpha * (static_cast<double>(point_count) / g.edge_count()) *
                  (p.nu_r * p.nu_r) / (p.nu_a * p.nu_a);
    }
    p.beta = cfg.k_beta * (static_cast<double>(point_count) / g.node_count()) / (2.0 * p.nu_a * p.nu_a);
}
// solver.hpp:86-106
inline SolverParams init_parameters(const std::vector<Vec3>& source, double avg_edge_length,
                                    const SpatialIndex& target, const DeformationGraph& g,
                                    const SolverConfig& cfg) {
    std::vector<double> dist(source.size());
    for (size_t i = 0; i < source.size(); ++i) dist[i] = target.nearest(source[i]).distance;
    std::sort(dist.begin(), dist.end());
    const size_t n = dist.size();
    const double median = n % 2 == 1 ? dist[n / 2] : 0.5 * (dist[n / 2 - 1] + dist[n / 2]);
    const double l_bar = avg_edge_length;
    SolverParams p;
    p.nu_a_min = std::isnan(cfg.nu_a_min) ? l_bar / std::sqrt(3.0) : cfg.nu_a_min;
    p.nu_a = std::isnan(cfg.nu_a_init) ? std::max(median, p.nu_a_min) : cfg.nu_a_init;
    p.nu_r = std::isnan(cfg.nu_r_init) ? 3.0 * l_bar : cfg.nu_r_init;
    if (!(p.nu_a > 0.0) || !(p.nu_r > 0.0))
        throw NumericalError("init_parameters: Welsch parameters must be positive");
    update_term_weights(p, static_cast<int>(source.size()), g, cfg);
    return p;
}

struct IterationRecord {  // solver.hpp:108-116
    double e_total = 0, e_align = 0, e_reg = 0, e_rot = 0, e_landmark = 0;
    bool aa_accepted = false;
    double max_disp = 0;
};
struct StageRecord {  // solver.hpp:118-124
    double nu_a = 0, nu_r = 0, alpha = 0, beta = 0;
    int reverts = 0;
    bool converged = false;
    std::vector<IterationRecord> iterations;
};
struct RegistrationReport {  // solver.hpp:126-138
    std::vector<StageRecord> stages;
    int degenerate_rotations = 0;
    bool alpha_forced_zero = false;
    double solve_seconds = 0.0;
    int total_iterations() const {
        int n = 0;
        for (const auto& s : stages) n += static_cast<int>(s.iterations.size());
        return n;
    }
};
struct RegistrationResult {  // solver.hpp:140-144
    NodeTransforms transforms;
    std::vector<Vec3> deformed_points;
    RegistrationReport report;
};

// solver.hpp:146-154 — flatten is the column-major storage itself.
inline std::vector<double> flatten(const NodeTransforms& x) { return x.stacked; }
inline NodeTransforms unflatten(const std::vector<double>& v, int nodes) {
    NodeTransforms x;
    x.nodes = nodes;
    x.stacked = v;
    return x;
}

/// solver.hpp:159-169
inline NodeTransforms mm_step(const std::vector<Vec3>& source, const DeformationGraph& g,
                              const SpatialIndex& target, const NodeTransforms& x,
                              const SolverParams& prm) {
    const auto deformed = deform_points(source, g, x);
    const Correspondences corr = find_correspondences(deformed, target);
    const auto rotations = project_rotations(x);
    SystemAssembler as(source, g);
    as.fill(corr, rotations, alignment_weights(corr, prm.nu_a),
            regularization_weights(g, x, prm.nu_r, prm.alpha), prm.beta);
    return as.solve();
}

/// Optional per-pass observer (test instrumentation only): called on every
/// evaluated pass with the pass's correspondences and energy, before the
/// accept/revert decision.
struct PassObserver {
    virtual ~PassObserver() = default;
    virtual void on_pass(int stage, int pass, const Correspondences&, const EnergyBreakdown&,
                         bool reverted) = 0;
};

/// solver.hpp:180-304
inline RegistrationResult register_surfaces(const std::vector<Vec3>& source, double src_avg_edge,
                                            const std::vector<Vec3>& target,
                                            const DeformationGraph& g, const SolverConfig& cfg,
                                            PassObserver* obs = nullptr) {
    cfg.validate();
    if (source.empty() || target.empty()) throw NumericalError("register_surfaces: empty surface");
    const auto t0 = std::chrono::steady_clock::now();
    const SpatialIndex tindex(target);
    SolverParams prm = init_parameters(source, src_avg_edge, tindex, g, cfg);
    RegistrationResult res;
    RegistrationReport& rep = res.report;
    rep.alpha_forced_zero = prm.alpha_forced_zero;
    SystemAssembler as(source, g, cfg.landmarks);
    AndersonWindow window(cfg.aa_window);
    NodeTransforms x = NodeTransforms::identity(g.node_count());
    std::vector<Vec3> v_hat = deform_points(source, g, x);
    NodeTransforms x_mm = x;
    bool current_is_aa = false;
    auto landmark_energy = [&](const std::vector<Vec3>& pts) {
        double e = 0.0;
        for (const auto& lm : cfg.landmarks) e += (pts[lm.source_index] - lm.target_position).squaredNorm();
        return e;
    };
    for (int si = 0;; ++si) {
        StageRecord stage;
        stage.nu_a = prm.nu_a;
        stage.nu_r = prm.nu_r;
        stage.alpha = prm.alpha;
        stage.beta = prm.beta;
        const double lm_w = (si == 0 && !cfg.landmarks.empty()) ? 1.0 : 0.0;
        window.reset();
        double e_prev = std::numeric_limits<double>::infinity();
        int accepted = 0, passes = 0;
        while (true) {
            if (++passes > 2 * cfg.i_max + 4) throw NumericalError("solver stage failed to make progress");
            const Correspondences corr = find_correspondences(v_hat, tindex);
            const auto rotations = project_rotations(x, &rep.degenerate_rotations);
            const EnergyBreakdown e =
                evaluate_energy(v_hat, x, g, corr, rotations, {prm.alpha, prm.beta, prm.nu_a, prm.nu_r});
            const double e_lm = lm_w != 0.0 ? landmark_energy(v_hat) : 0.0;
            const double e_accept = e.total + lm_w * e_lm;
            if (!std::isfinite(e_accept)) throw NumericalError("solver aborted: energy is not finite");
            const bool revert = e_accept > e_prev && current_is_aa;
            if (obs) obs->on_pass(si, passes, corr, e, revert);
            if (revert) {
                x = x_mm;
                v_hat = deform_points(source, g, x);
                current_is_aa = false;
                ++stage.reverts;
                continue;
            }
            e_prev = e_accept;
            IterationRecord rec;
            rec.e_total = e.total;
            rec.e_align = e.align;
            rec.e_reg = e.reg;
            rec.e_rot = e.rot;
            rec.e_landmark = e_lm;
            rec.aa_accepted = current_is_aa;
            as.fill(corr, rotations, alignment_weights(corr, prm.nu_a),
                    regularization_weights(g, x, prm.nu_r, prm.alpha), prm.beta, lm_w);
            x_mm = as.solve();
            if (!x_mm.all_finite()) throw NumericalError("solver aborted: iterate is not finite");
            std::vector<double> gv = flatten(x_mm), fv(gv.size());
            for (size_t i = 0; i < gv.size(); ++i) fv[i] = gv[i] - x.stacked[i];
            window.push(gv, fv);
            current_is_aa = window.extrapolating();
            NodeTransforms x_next = unflatten(window.combine(), g.node_count());
            if (!x_next.all_finite()) throw NumericalError("solver aborted: iterate is not finite");
            std::vector<Vec3> v_next = deform_points(source, g, x_next);
            double max_disp = 0.0;
            for (size_t i = 0; i < v_next.size(); ++i) max_disp = std::max(max_disp, (v_next[i] - v_hat[i]).norm());
            rec.max_disp = max_disp;
            stage.iterations.push_back(rec);
            x = std::move(x_next);
            v_hat = std::move(v_next);
            ++accepted;
            if (max_disp < cfg.eps) {
                stage.converged = true;
                break;
            }
            if (accepted >= cfg.i_max) break;
        }
        rep.stages.push_back(std::move(stage));
        const AnnealResult nx = anneal(prm.nu_a, prm.nu_r, prm.nu_a_min, cfg.nu_r_floor);
        if (nx.done) break;
        prm.nu_a = nx.nu_a;
        prm.nu_r = nx.nu_r;
        update_term_weights(prm, static_cast<int>(source.size()), g, cfg);
    }
    rep.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    res.transforms = std::move(x);
    res.deformed_points = std::move(v_hat);
    return res;
}

// ============================================== reference test fixtures (helpers.hpp)
// These regenerate the reference tests' seeded fixtures with the same
// libstdc++ distributions (helpers.hpp:74-135).
struct Quat {
    double w, x, y, z;
    Quat(double a, double b, double c, double d) : w(a), x(b), y(c), z(d) {}
};
inline Mat3 quat_to_rot(double w, double x, double y, double z) {
    Mat3 r;
    r(0, 0) = 1 - 2 * (y * y + z * z);
    r(0, 1) = 2 * (x * y - w * z);
    r(0, 2) = 2 * (x * z + w * y);
    r(1, 0) = 2 * (x * y + w * z);
    r(1, 1) = 1 - 2 * (x * x + z * z);
    r(1, 2) = 2 * (y * z - w * x);
    r(2, 0) = 2 * (x * z - w * y);
    r(2, 1) = 2 * (y * z + w * x);
    r(2, 2) = 1 - 2 * (x * x + y * y);
    return r;
}
// helpers.hpp:74-79
inline Mat3 random_rotation(std::mt19937_64& rng) {
    std::normal_distribution<double> gauss(0.0, 1.0);
    // same argument-expression form as the fixture, so the compiler draws in
    // the same (unspecified) evaluation order as the reference build
    const Quat q(gauss(rng), gauss(rng), gauss(rng), gauss(rng));
    const double nrm = std::sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
    return quat_to_rot(q.w / nrm, q.x / nrm, q.y / nrm, q.z / nrm);
}
// helpers.hpp:81-86
inline std::vector<Vec3> random_points(std::mt19937_64& rng, int n, double extent = 1.0) {
    std::uniform_real_distribution<double> uni(-extent, extent);
    std::vector<Vec3> pts(n);
    for (auto& p : pts) p = Vec3(uni(rng), uni(rng), uni(rng));
    return pts;
}
// helpers.hpp:89-105
inline Surface make_strip(int nx, int ny, double len_x = 1.0, double len_y = 0.5) {
    std::vector<Vec3> pts;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) pts.emplace_back(len_x * i / (nx - 1), len_y * j / (ny - 1), 0.0);
    std::vector<std::array<int, 3>> faces;
    for (int j = 0; j + 1 < ny; ++j)
        for (int i = 0; i + 1 < nx; ++i) {
            const int a = j * nx + i, b = j * nx + i + 1, c = (j + 1) * nx + i, d = (j + 1) * nx + i + 1;
            faces.push_back({a, b, d});
            faces.push_back({a, d, c});
        }
    return make_surface(std::move(pts), std::move(faces));
}
struct WarpParams {  // helpers.hpp:107-112
    double amplitude = 0.05, frequency = 1.0, phase = 0.0, tilt = 0.0;
};
// helpers.hpp:114-122
inline WarpParams random_warp(std::mt19937_64& rng, double amplitude_scale = 1.0) {
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    WarpParams w;
    w.amplitude = amplitude_scale * (0.03 + 0.05 * uni(rng));
    w.frequency = 0.6 + 0.9 * uni(rng);
    w.phase = uni(rng);
    w.tilt = 0.3 * uni(rng);
    return w;
}
// helpers.hpp:124-128
inline Vec3 warp_point(const Vec3& p, const WarpParams& w) {
    const double z = w.amplitude * std::sin(2.0 * M_PI * (w.frequency * p.x + w.phase)) +
                     w.tilt * w.amplitude * std::sin(2.0 * M_PI * p.y);
    return {p.x, p.y, p.z + z};
}
// helpers.hpp:130-135
inline Surface warped_copy(const Surface& s, const WarpParams& w) {
    Surface out = s;
    for (auto& p : out.points) p = warp_point(p, w);
    out.finalize_edges();
    return out;
}

}  // namespace oracle
