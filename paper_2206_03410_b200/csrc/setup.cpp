// Setup side of the drop-in API (CPU, once per registration; outside the
// per-iteration hot path): surface connectivity,
// normalization, deformation-graph construction and the seeded synthetic
// configs that stand in for BASELINE.json's datasets.
//
// Semantics follow the reference exactly so graphs are identical to it:
//   edges_from_faces  surface.hpp:49-65      knn_edges   surface.hpp:70-94
//   finalize_edges    surface.hpp:29-45      normalize   surface.hpp:125-149
//   limited_geodesic  geodesic.hpp:22-84     pca_order   deformation_graph.hpp:73-106
//   influence weights :111-125               reg table   :130-148
//   build_graph       :157-210
// Differences are implementation only: a uniform-grid exact kNN instead of the
// O(n^2) scan, and touched-list scratch buffers instead of O(n) allocations
// per geodesic query.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <queue>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "errors.hpp"
#include "nrr_cuda.h"
#include "setup.hpp"
#include "nrr_synth.hpp"

namespace nrr_b200 {
namespace {

struct P3 {
    double x, y, z;
};
inline P3 sub(const P3& a, const P3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline double sqn(const P3& a) { return a.x * a.x + a.y * a.y + a.z * a.z; }
inline double nrm(const P3& a) { return std::sqrt(sqn(a)); }
inline P3 at3(const double* p, int i) { return {p[3 * i], p[3 * i + 1], p[3 * i + 2]}; }

// ------------------------------------------------------------------ surface
std::vector<std::pair<int, int>> faces_to_edges(const int32_t* faces, int nf, int n) {
    std::vector<std::pair<int, int>> e;
    e.reserve(static_cast<size_t>(nf) * 3);
    for (int f = 0; f < nf; ++f)
        for (int c = 0; c < 3; ++c) {
            const int a = faces[3 * f + c], b = faces[3 * f + (c + 1) % 3];
            if (a < 0 || b < 0 || a >= n || b >= n) throw NumericalError("face index out of range");
            if (a == b) throw NumericalError("degenerate face with repeated vertex");
            e.emplace_back(std::min(a, b), std::max(a, b));
        }
    std::sort(e.begin(), e.end());
    e.erase(std::unique(e.begin(), e.end()), e.end());
    return e;
}

// exact symmetric kNN on a uniform hash grid; neighbour order is the
// lexicographic (squared distance, index) order of the reference's sort
std::vector<std::pair<int, int>> grid_knn_edges(const double* pts, int n, int k) {
    if (k < 1) throw ConfigError("knn_edges: k must be >= 1");
    if (k >= n) throw ConfigError("knn_edges: k must be smaller than the point count");
    P3 lo = at3(pts, 0), hi = lo;
    for (int i = 1; i < n; ++i) {
        const P3 p = at3(pts, i);
        lo = {std::min(lo.x, p.x), std::min(lo.y, p.y), std::min(lo.z, p.z)};
        hi = {std::max(hi.x, p.x), std::max(hi.y, p.y), std::max(hi.z, p.z)};
    }
    const P3 ext = sub(hi, lo);
    const double vol = std::max(ext.x, 1e-12) * std::max(ext.y, 1e-12) * std::max(ext.z, 1e-12);
    double h = std::cbrt(vol * 2.0 / n);
    const double maxe = std::max(ext.x, std::max(ext.y, ext.z));
    h = std::max(h, maxe / 512.0);
    if (!(h > 0)) h = 1.0;
    const int gx = std::max(1, static_cast<int>(ext.x / h) + 1);
    const int gy = std::max(1, static_cast<int>(ext.y / h) + 1);
    const int gz = std::max(1, static_cast<int>(ext.z / h) + 1);
    auto cell_of = [&](const P3& p, int& cx, int& cy, int& cz) {
        cx = std::min(gx - 1, std::max(0, static_cast<int>((p.x - lo.x) / h)));
        cy = std::min(gy - 1, std::max(0, static_cast<int>((p.y - lo.y) / h)));
        cz = std::min(gz - 1, std::max(0, static_cast<int>((p.z - lo.z) / h)));
    };
    std::unordered_map<int64_t, std::vector<int>> cells;
    auto key = [&](int cx, int cy, int cz) {
        return (static_cast<int64_t>(cz) * gy + cy) * gx + cx;
    };
    for (int i = 0; i < n; ++i) {
        int cx, cy, cz;
        cell_of(at3(pts, i), cx, cy, cz);
        cells[key(cx, cy, cz)].push_back(i);
    }
    std::vector<std::pair<int, int>> edges;
    edges.reserve(static_cast<size_t>(n) * k);
    std::vector<std::pair<double, int>> best;
    for (int i = 0; i < n; ++i) {
        const P3 q = at3(pts, i);
        int cx, cy, cz;
        cell_of(q, cx, cy, cz);
        best.clear();
        const int maxs = std::max(gx, std::max(gy, gz));
        for (int s = 0; s <= maxs; ++s) {
            for (int dz = -s; dz <= s; ++dz)
                for (int dy = -s; dy <= s; ++dy)
                    for (int dx = -s; dx <= s; ++dx) {
                        if (std::max(std::abs(dx), std::max(std::abs(dy), std::abs(dz))) != s) continue;
                        const int x = cx + dx, y = cy + dy, z = cz + dz;
                        if (x < 0 || y < 0 || z < 0 || x >= gx || y >= gy || z >= gz) continue;
                        const auto it = cells.find(key(x, y, z));
                        if (it == cells.end()) continue;
                        for (int j : it->second) {
                            if (j == i) continue;
                            const P3 pj = at3(pts, j);
                            const P3 d = sub(q, pj);
                            best.emplace_back(sqn(d), j);
                        }
                    }
            if (static_cast<int>(best.size()) >= k) {
                std::nth_element(best.begin(), best.begin() + (k - 1), best.end());
                std::sort(best.begin(), best.begin() + k);
                best.resize(k);
                // every unvisited point lies outside the (2s+1)^3 cell box
                const double bx = std::min(q.x - (lo.x + (cx - s) * h), (lo.x + (cx + s + 1) * h) - q.x);
                const double by = std::min(q.y - (lo.y + (cy - s) * h), (lo.y + (cy + s + 1) * h) - q.y);
                const double bz = std::min(q.z - (lo.z + (cz - s) * h), (lo.z + (cz + s + 1) * h) - q.z);
                const double bound = std::min(bx, std::min(by, bz)) * (1.0 - 1e-12);
                if (best[k - 1].first < bound * bound) break;
            }
        }
        for (int t = 0; t < k; ++t) {
            const int j = best[t].second;
            edges.emplace_back(std::min(i, j), std::max(i, j));
        }
    }
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    return edges;
}

struct Adjacency {  // Surface::adjacency, sorted (neighbor, length) per vertex
    std::vector<int> off, nb;
    std::vector<double> len;
    double avg = 0.0;
};
Adjacency finalize(const double* pts, int n, const int32_t* edges, int ne) {
    Adjacency a;
    std::vector<std::vector<std::pair<int, double>>> tmp(n);
    double total = 0.0;
    for (int e = 0; e < ne; ++e) {
        const int u = edges[2 * e], v = edges[2 * e + 1];
        if (u < 0 || v < 0 || u >= n || v >= n) throw NumericalError("surface edge index out of range");
        if (u == v) throw NumericalError("surface edge is a self-loop");
        const double l = nrm(sub(at3(pts, u), at3(pts, v)));
        tmp[u].emplace_back(v, l);
        tmp[v].emplace_back(u, l);
        total += l;
    }
    a.off.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) {
        std::sort(tmp[i].begin(), tmp[i].end());
        a.off[i + 1] = a.off[i] + static_cast<int>(tmp[i].size());
    }
    a.nb.resize(a.off[n]);
    a.len.resize(a.off[n]);
    for (int i = 0; i < n; ++i)
        for (size_t t = 0; t < tmp[i].size(); ++t) {
            a.nb[a.off[i] + t] = tmp[i][t].first;
            a.len[a.off[i] + t] = tmp[i][t].second;
        }
    a.avg = ne == 0 ? 0.0 : total / static_cast<double>(ne);
    return a;
}

// ----------------------------------------------------------------- geodesic
class Geodesic {
public:
    Geodesic(const double* pts, int n, const Adjacency& adj)
        : pts_(pts), adj_(adj), in_ball_(n, 0), done_(n, 0), dist_(n, kInf) {}

    // vertices with edge-graph distance < radius, ascending vertex index
    void query(int src_idx, double radius, std::vector<std::pair<int, double>>& out) {
        out.clear();
        const P3 src = at3(pts_, src_idx);
        ball_.clear();
        in_ball_[src_idx] = 1;
        ball_.push_back(src_idx);
        size_t head = 0;
        while (head < ball_.size()) {  // BFS order == the reference's FIFO queue order
            const int v = ball_[head++];
            for (int t = adj_.off[v]; t < adj_.off[v + 1]; ++t) {
                const int w = adj_.nb[t];
                if (in_ball_[w]) continue;
                if (nrm(sub(at3(pts_, w), src)) < radius) {
                    in_ball_[w] = 1;
                    ball_.push_back(w);
                }
            }
        }
        using Entry = std::pair<double, int>;
        std::priority_queue<Entry, std::vector<Entry>, std::greater<Entry>> heap;
        dist_[src_idx] = 0.0;
        heap.emplace(0.0, src_idx);
        while (!heap.empty()) {
            const auto [d, v] = heap.top();
            heap.pop();
            if (done_[v] || d > dist_[v]) continue;
            done_[v] = 1;
            if (d >= radius) continue;
            for (int t = adj_.off[v]; t < adj_.off[v + 1]; ++t) {
                const int w = adj_.nb[t];
                if (!in_ball_[w] || done_[w]) continue;
                const double cand = d + adj_.len[t];
                if (cand < dist_[w]) {
                    dist_[w] = cand;
                    heap.emplace(cand, w);
                }
            }
        }
        std::sort(ball_.begin(), ball_.end());
        for (int v : ball_)
            if (dist_[v] < radius) out.emplace_back(v, dist_[v]);
        for (int v : ball_) {
            in_ball_[v] = 0;
            done_[v] = 0;
            dist_[v] = kInf;
        }
    }

private:
    static constexpr double kInf = std::numeric_limits<double>::infinity();
    const double* pts_;
    const Adjacency& adj_;
    std::vector<char> in_ball_, done_;
    std::vector<double> dist_;
    std::vector<int> ball_;
};

// ---------------------------------------------------------------- pca order
// 3x3 symmetric cyclic Jacobi (stands in for SelfAdjointEigenSolver); returns
// the eigenvector of the largest eigenvalue.
P3 dominant_axis(const double cov_in[9]) {
    double a[9], v[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    std::memcpy(a, cov_in, sizeof a);
    auto rot = [](double x, double y, double z, double& c, double& s) {
        const double deno = 2.0 * std::abs(y);
        if (deno < std::numeric_limits<double>::min()) {
            c = 1;
            s = 0;
            return;
        }
        const double tau = (x - z) / deno, w = std::sqrt(tau * tau + 1.0);
        const double t = tau > 0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
        const double n = 1.0 / std::sqrt(t * t + 1.0);
        s = -(t > 0 ? 1.0 : -1.0) * (y / std::abs(y)) * std::abs(t) * n;
        c = n;
    };
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0, diag = 0;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) (i == j ? diag : off) += a[i * 3 + j] * a[i * 3 + j];
        const double e2 = std::numeric_limits<double>::epsilon() * std::numeric_limits<double>::epsilon();
        if (off <= 1e-300 || off <= e2 * diag * 1e-4) break;
        for (int p = 0; p < 3; ++p)
            for (int q = p + 1; q < 3; ++q) {
                if (a[p * 3 + q] == 0.0) continue;
                double c, s;
                rot(a[p * 3 + p], a[p * 3 + q], a[q * 3 + q], c, s);
                // rows p,q by J^T = (c,-s): x' = c x - s y, y' = s x + c y
                for (int k = 0; k < 3; ++k) {
                    const double x = a[p * 3 + k], y = a[q * 3 + k];
                    a[p * 3 + k] = c * x - s * y;
                    a[q * 3 + k] = s * x + c * y;
                }
                // columns p,q of a and v by J (applied as J^T on the right)
                for (double* m : {a, v})
                    for (int k = 0; k < 3; ++k) {
                        const double x = m[k * 3 + p], y = m[k * 3 + q];
                        m[k * 3 + p] = c * x - s * y;
                        m[k * 3 + q] = s * x + c * y;
                    }
            }
    }
    int best = 0;
    for (int k = 1; k < 3; ++k)
        if (a[k * 3 + k] >= a[best * 3 + best]) best = k;
    // eigenvalues ascending with a stable order: the largest is the last of
    // the ascending sort, i.e. the last index among equal maxima
    int idx[3] = {0, 1, 2};
    std::sort(idx, idx + 3, [&](int x, int y) { return a[x * 3 + x] < a[y * 3 + y]; });
    best = idx[2];
    return {v[0 * 3 + best], v[1 * 3 + best], v[2 * 3 + best]};
}

}  // namespace

// pca_order's moments (deformation_graph.hpp:79-89): mean, then the
// covariance, both summed sequentially in point order
void pca_moments(const double* pts, int n, double cov[9]) {
    P3 mean{0, 0, 0};
    for (int i = 0; i < n; ++i) {
        mean.x += pts[3 * i];
        mean.y += pts[3 * i + 1];
        mean.z += pts[3 * i + 2];
    }
    const double inv = 1.0 / static_cast<double>(n);
    mean = {mean.x * inv, mean.y * inv, mean.z * inv};
    for (int k = 0; k < 9; ++k) cov[k] = 0.0;
    for (int i = 0; i < n; ++i) {
        const P3 d = sub(at3(pts, i), mean);
        const double dd[3] = {d.x, d.y, d.z};
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) cov[r * 3 + c] += dd[r] * dd[c];
    }
}

namespace {

std::vector<int> pca_order(const double* pts, int n) {
    if (n == 0) throw ConfigError("pca_order: empty point set");
    double cov[9];
    pca_moments(pts, n, cov);
    P3 axis = dominant_axis(cov);
    if (!std::isfinite(axis.x) || !std::isfinite(axis.y) || !std::isfinite(axis.z)) axis = {1, 0, 0};
    const double comp[3] = {axis.x, axis.y, axis.z};
    for (int c = 0; c < 3; ++c)
        if (comp[c] != 0.0) {
            if (comp[c] < 0.0) axis = {-axis.x, -axis.y, -axis.z};
            break;
        }
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::vector<double> proj(n);
    for (int i = 0; i < n; ++i) proj[i] = pts[3 * i] * axis.x + pts[3 * i + 1] * axis.y + pts[3 * i + 2] * axis.z;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        if (proj[a] != proj[b]) return proj[a] < proj[b];
        return a < b;
    });
    return order;
}

}  // namespace

// limited_geodesic (geodesic.hpp:22-84) over the adjacency of (pts, edges)
std::vector<std::pair<int, double>> limited_geodesic_impl(const double* pts, int n, const int32_t* edges, int ne,
                                                          int source, double radius) {
    if (source < 0 || source >= n) throw ConfigError("limited_geodesic: source index out of range");
    if (!(radius > 0.0)) throw ConfigError("limited_geodesic: radius must be positive");
    const Adjacency adj = finalize(pts, n, edges, ne);
    Geodesic geo(pts, n, adj);
    std::vector<std::pair<int, double>> out;
    geo.query(source, radius, out);
    return out;
}

// pca_order's axis (deformation_graph.hpp:86-95) from an accumulated
// covariance: the dominant eigenvector, (1,0,0) if not finite, sign fixed so
// the first nonzero component is positive (used by the device build)
void pca_axis(const double cov[9], double out[3]) {
    P3 axis = dominant_axis(cov);
    if (!std::isfinite(axis.x) || !std::isfinite(axis.y) || !std::isfinite(axis.z)) axis = {1, 0, 0};
    const double comp[3] = {axis.x, axis.y, axis.z};
    for (int c = 0; c < 3; ++c)
        if (comp[c] != 0.0) {
            if (comp[c] < 0.0) axis = {-axis.x, -axis.y, -axis.z};
            break;
        }
    out[0] = axis.x;
    out[1] = axis.y;
    out[2] = axis.z;
}

GraphData build_graph_impl(const double* pts, int n, const int32_t* sedges, int ne, double radius) {
    if (n == 0) throw ConfigError("build_graph: empty source surface");
    if (!(radius > 0.0)) throw ConfigError("build_graph: radius must be positive");
    const Adjacency adj = finalize(pts, n, sedges, ne);
    Geodesic geo(pts, n, adj);
    GraphData g;
    std::vector<std::vector<std::pair<int, double>>> raw(n);
    std::vector<std::pair<int, double>> ball;
    for (int idx : pca_order(pts, n)) {
        if (!g.node_indices.empty() && !raw[idx].empty()) continue;
        const int node_id = static_cast<int>(g.node_indices.size());
        g.node_indices.push_back(idx);
        for (int c = 0; c < 3; ++c) g.node_positions.push_back(pts[3 * idx + c]);
        geo.query(idx, radius, ball);
        for (const auto& [q, d] : ball) raw[q].emplace_back(node_id, d);
    }
    const int N = static_cast<int>(g.node_indices.size());
    for (int i = 0; i < n; ++i)
        for (size_t a = 0; a < raw[i].size(); ++a)
            for (size_t b = a + 1; b < raw[i].size(); ++b) g.edges.emplace_back(raw[i][a].first, raw[i][b].first);
    std::sort(g.edges.begin(), g.edges.end());
    g.edges.erase(std::unique(g.edges.begin(), g.edges.end()), g.edges.end());
    std::vector<std::vector<int>> nbrs(N);
    for (const auto& [a, b] : g.edges) {
        nbrs[a].push_back(b);
        nbrs[b].push_back(a);
    }
    for (auto& v : nbrs) std::sort(v.begin(), v.end());
    g.infl_off.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) {
        if (raw[i].empty()) throw NumericalError("build_graph: point left without influencing nodes");
        double total = 0.0;
        const size_t base = g.infl_w.size();
        for (const auto& [node, d] : raw[i]) {
            const double ratio = 1.0 - (d * d) / (radius * radius);
            if (!(ratio > 0.0)) throw NumericalError("influence_weights: distance not below radius");
            const double w = ratio * ratio * ratio;
            g.infl_node.push_back(node);
            g.infl_w.push_back(w);
            g.infl_d.push_back(d);
            total += w;
        }
        for (size_t t = base; t < g.infl_w.size(); ++t) g.infl_w[t] /= total;
        g.infl_off[i + 1] = static_cast<int>(g.infl_w.size());
    }
    if (!g.edges.empty()) {
        double inv_sum = 0.0;
        for (int i = 0; i < N; ++i)
            for (int j : nbrs[i]) {
                const P3 d = sub(at3(g.node_positions.data(), i), at3(g.node_positions.data(), j));
                const double len = nrm(d);
                if (!(len > 0.0)) throw NumericalError("reg_weight_table: coincident node positions");
                g.pairs.push_back(i);
                g.pairs.push_back(j);
                g.pair_w.push_back(1.0 / len);
                inv_sum += 1.0 / len;
            }
        const double scale = static_cast<double>(g.pair_w.size()) / inv_sum;
        for (auto& c : g.pair_w) c *= scale;
    }
    return g;
}

// ==================================================================== synth
void synth_config(int which, uint64_t seed, double scale, std::vector<double>& src, std::vector<int32_t>& faces,
                  std::vector<double>& tgt) {
    try {
        nrr_synth::synth_config(which, seed, scale, src, faces, tgt);
    } catch (const std::invalid_argument& e) {
        throw ConfigError(e.what());
    }
}

std::vector<std::pair<int, int>> edges_from_faces(const int32_t* faces, int nf, int n) {
    return faces_to_edges(faces, nf, n);
}
std::vector<std::pair<int, int>> knn_edges(const double* pts, int n, int k) { return grid_knn_edges(pts, n, k); }
double avg_edge_length(const double* pts, int n, const int32_t* edges, int ne) {
    return finalize(pts, n, edges, ne).avg;
}

}  // namespace nrr_b200
