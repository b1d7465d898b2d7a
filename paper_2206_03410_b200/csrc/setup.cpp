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

std::vector<int> pca_order(const double* pts, int n) {
    if (n == 0) throw ConfigError("pca_order: empty point set");
    P3 mean{0, 0, 0};
    for (int i = 0; i < n; ++i) {
        mean.x += pts[3 * i];
        mean.y += pts[3 * i + 1];
        mean.z += pts[3 * i + 2];
    }
    const double inv = 1.0 / static_cast<double>(n);
    mean = {mean.x * inv, mean.y * inv, mean.z * inv};
    double cov[9] = {0};
    for (int i = 0; i < n; ++i) {
        const P3 d = sub(at3(pts, i), mean);
        const double dd[3] = {d.x, d.y, d.z};
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) cov[r * 3 + c] += dd[r] * dd[c];
    }
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
namespace {
struct Rng {  // mt19937_64 with explicit, portable transforms
    uint64_t mt[312];
    int idx = 313;
    explicit Rng(uint64_t seed) {
        mt[0] = seed;
        for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
        idx = 312;
    }
    uint64_t next() {
        if (idx >= 312) {
            for (int i = 0; i < 312; ++i) {
                const uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
                uint64_t xa = x >> 1;
                if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
                mt[i] = mt[(i + 156) % 312] ^ xa;
            }
            idx = 0;
        }
        uint64_t y = mt[idx++];
        y ^= (y >> 29) & 0x5555555555555555ULL;
        y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
        y ^= (y << 37) & 0xFFF7EEE000000000ULL;
        y ^= y >> 43;
        return y;
    }
    double uni() { return static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0); }
    double uni(double a, double b) { return a + (b - a) * uni(); }
    double gauss() {  // Box-Muller
        double u1 = uni();
        while (u1 <= 0.0) u1 = uni();
        const double u2 = uni();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
    }
};

struct Cloud {
    std::vector<double> pts;  // k*3
    std::vector<int32_t> faces;
    void add(double x, double y, double z) {
        pts.push_back(x);
        pts.push_back(y);
        pts.push_back(z);
    }
    int count() const { return static_cast<int>(pts.size() / 3); }
};

void rotate_axis_angle(double* p, int n, const double ax[3], double ang, const double ctr[3]) {
    const double c = std::cos(ang), s = std::sin(ang), t = 1 - c;
    const double x = ax[0], y = ax[1], z = ax[2];
    const double R[9] = {t * x * x + c,     t * x * y - s * z, t * x * z + s * y,
                         t * x * y + s * z, t * y * y + c,     t * y * z - s * x,
                         t * x * z - s * y, t * y * z + s * x, t * z * z + c};
    for (int i = 0; i < n; ++i) {
        const double v[3] = {p[3 * i] - ctr[0], p[3 * i + 1] - ctr[1], p[3 * i + 2] - ctr[2]};
        for (int r = 0; r < 3; ++r) p[3 * i + r] = ctr[r] + R[r * 3] * v[0] + R[r * 3 + 1] * v[1] + R[r * 3 + 2] * v[2];
    }
}

void random_unit(Rng& rng, double out[3]) {
    double n2 = 0;
    do {
        for (int k = 0; k < 3; ++k) out[k] = rng.gauss();
        n2 = out[0] * out[0] + out[1] * out[1] + out[2] * out[2];
    } while (n2 < 1e-12);
    const double inv = 1.0 / std::sqrt(n2);
    for (int k = 0; k < 3; ++k) out[k] *= inv;
}

// area-uniform torus samples (R, r): rejection on the tube angle
void torus_samples(Rng& rng, int count, double R, double r, Cloud& out) {
    while (out.count() < count) {
        const double u = rng.uni(0, 2 * M_PI), v = rng.uni(0, 2 * M_PI);
        if (rng.uni() * (R + r) > R + r * std::cos(v)) continue;
        const double w = R + r * std::cos(v);
        out.add(w * std::cos(u), w * std::sin(u), r * std::sin(v));
    }
}

// Gaussian RBF displacement field: sum_k a_k exp(-|p-c_k|^2 / 2 sigma^2)
void rbf_warp(double* p, int n, const std::vector<double>& centers, const std::vector<double>& amps, double sigma) {
    const int K = static_cast<int>(centers.size() / 3);
    for (int i = 0; i < n; ++i) {
        double d[3] = {0, 0, 0};
        for (int k = 0; k < K; ++k) {
            const double dx = p[3 * i] - centers[3 * k], dy = p[3 * i + 1] - centers[3 * k + 1],
                         dz = p[3 * i + 2] - centers[3 * k + 2];
            const double g = std::exp(-(dx * dx + dy * dy + dz * dz) / (2 * sigma * sigma));
            for (int c = 0; c < 3; ++c) d[c] += amps[3 * k + c] * g;
        }
        for (int c = 0; c < 3; ++c) p[3 * i + c] += d[c];
    }
}

void add_uniform_outliers(Rng& rng, Cloud& c, int count, double enlarge) {
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int i = 0; i < c.count(); ++i)
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], c.pts[3 * i + k]);
            hi[k] = std::max(hi[k], c.pts[3 * i + k]);
        }
    for (int k = 0; k < 3; ++k) {
        const double mid = 0.5 * (lo[k] + hi[k]), half = 0.5 * (hi[k] - lo[k]) * enlarge;
        lo[k] = mid - half;
        hi[k] = mid + half;
    }
    for (int t = 0; t < count; ++t) c.add(rng.uni(lo[0], hi[0]), rng.uni(lo[1], hi[1]), rng.uni(lo[2], hi[2]));
}

// drop points on the far side of a random plane so that `frac` is removed
void halfspace_crop(Rng& rng, Cloud& c, double frac, bool planar_dir) {
    double dir[3];
    random_unit(rng, dir);
    if (planar_dir) {
        dir[2] = 0;
        const double l = std::hypot(dir[0], dir[1]);
        dir[0] /= l;
        dir[1] /= l;
    }
    const int n = c.count();
    std::vector<double> proj(n);
    for (int i = 0; i < n; ++i) proj[i] = c.pts[3 * i] * dir[0] + c.pts[3 * i + 1] * dir[1] + c.pts[3 * i + 2] * dir[2];
    std::vector<double> sorted(proj);
    const int cut = std::min(n - 1, static_cast<int>(frac * n));
    std::nth_element(sorted.begin(), sorted.begin() + cut, sorted.end());
    const double thr = sorted[cut];
    Cloud out;
    for (int i = 0; i < n; ++i)
        if (proj[i] >= thr) out.add(c.pts[3 * i], c.pts[3 * i + 1], c.pts[3 * i + 2]);
    c = std::move(out);
}

struct HeightField {
    double a[6], fx[6], fy[6], ph[6];
    int waves = 6;
    double z(double x, double y) const {
        double s = 0;
        for (int k = 0; k < waves; ++k) s += a[k] * std::sin(2 * M_PI * (fx[k] * x + fy[k] * y) + ph[k]);
        return s;
    }
};

HeightField random_height(Rng& rng) {
    HeightField h;
    for (int k = 0; k < 6; ++k) {
        h.a[k] = rng.uni(0.05, 0.2);
        const double f = rng.uni(1.0, 4.0), th = rng.uni(0, 2 * M_PI);
        h.fx[k] = f * std::cos(th);
        h.fy[k] = f * std::sin(th);
        h.ph[k] = rng.uni(0, 2 * M_PI);
    }
    return h;
}

// configs 2 and 4: height field grid source; warped, jittered, holed (or
// cropped) and outlier-polluted target
void height_pair(Rng& rng, int side, int holes, double hole_area, double crop_frac, double outlier_frac,
                 Cloud& src, Cloud& tgt) {
    const HeightField hf = random_height(rng);
    const double h = 2.0 / (side - 1);
    for (int j = 0; j < side; ++j)
        for (int i = 0; i < side; ++i) {
            const double x = -1.0 + i * h, y = -1.0 + j * h;
            src.add(x, y, hf.z(x, y));
        }
    for (int j = 0; j + 1 < side; ++j)
        for (int i = 0; i + 1 < side; ++i) {
            const int a = j * side + i, b = a + 1, c = a + side, d = c + 1;
            src.faces.insert(src.faces.end(), {a, b, d, a, d, c});
        }
    // 16-centre RBF warp of the analytic surface, sigma 0.25, |d| = 0.08
    std::vector<double> centers, amps;
    for (int k = 0; k < 16; ++k) {
        const double x = rng.uni(-1, 1), y = rng.uni(-1, 1);
        centers.insert(centers.end(), {x, y, hf.z(x, y)});
        double d[3];
        random_unit(rng, d);
        amps.insert(amps.end(), {0.08 * d[0], 0.08 * d[1], 0.08 * d[2]});
    }
    // elliptical holes totalling hole_area of the [-1,1]^2 domain
    std::vector<std::array<double, 5>> ell;  // cx, cy, a, b, angle
    for (int k = 0; k < holes; ++k) {
        const double area = hole_area * 4.0 / holes, aspect = rng.uni(1.0, 2.0);
        const double b = std::sqrt(area / (M_PI * aspect)), a = aspect * b;
        ell.push_back({rng.uni(-0.7, 0.7), rng.uni(-0.7, 0.7), a, b, rng.uni(0, M_PI)});
    }
    for (int j = 0; j < side; ++j)
        for (int i = 0; i < side; ++i) {
            const double x = -1.0 + (i + rng.uni(-0.5, 0.5)) * h, y = -1.0 + (j + rng.uni(-0.5, 0.5)) * h;
            bool in_hole = false;
            for (const auto& e : ell) {
                const double dx = x - e[0], dy = y - e[1], c = std::cos(e[4]), s = std::sin(e[4]);
                const double u = (c * dx + s * dy) / e[2], v = (-s * dx + c * dy) / e[3];
                if (u * u + v * v < 1.0) in_hole = true;
            }
            if (!in_hole) tgt.add(x, y, hf.z(x, y));
        }
    rbf_warp(tgt.pts.data(), tgt.count(), centers, amps, 0.25);
    if (crop_frac > 0) halfspace_crop(rng, tgt, crop_frac, true);
    add_uniform_outliers(rng, tgt, static_cast<int>(outlier_frac * src.count()), 1.0);
}

// configs 0 and 3: torus pair (R=1, r=0.35) with an 8-centre RBF warp, a
// rotation of at most 15 degrees and N(0, 0.002^2) noise
void torus_pair(Rng& rng, int count, Cloud& src, Cloud& tgt) {
    torus_samples(rng, count, 1.0, 0.35, src);
    torus_samples(rng, count, 1.0, 0.35, tgt);
    Cloud ctr;
    torus_samples(rng, 8, 1.0, 0.35, ctr);
    std::vector<double> amps(24);
    for (auto& a : amps) a = 0.1 * rng.gauss();
    rbf_warp(tgt.pts.data(), tgt.count(), ctr.pts, amps, 0.3);
    double ax[3];
    random_unit(rng, ax);
    const double ang = rng.uni(0, 15.0 * M_PI / 180.0), zero[3] = {0, 0, 0};
    rotate_axis_angle(tgt.pts.data(), tgt.count(), ax, ang, zero);
    for (auto& v : tgt.pts) v += 0.002 * rng.gauss();
}

// config 1: chain of 5 capsules (radius 0.15, segment 0.6) along x; target
// bent at each joint by U(-40, 40) degrees, 30% half-space crop, 5% outliers
void capsule_pair(Rng& rng, int count, Cloud& src, Cloud& tgt) {
    const int segs = 5;
    const double rad = 0.15, len = 0.6;
    auto sample_chain = [&](Cloud& c, std::vector<int>& seg_of) {
        const double cyl = 2 * M_PI * rad * len, cap = 4 * M_PI * rad * rad;
        while (c.count() < count) {
            const int s = std::min(segs - 1, static_cast<int>(rng.uni() * segs));
            const double x0 = s * len;
            if (rng.uni() * (cyl + cap) < cyl) {
                const double t = rng.uni(0, len), th = rng.uni(0, 2 * M_PI);
                c.add(x0 + t, rad * std::cos(th), rad * std::sin(th));
            } else {
                double d[3];
                random_unit(rng, d);
                const double xe = d[0] < 0 ? x0 : x0 + len;
                c.add(xe + rad * d[0], rad * d[1], rad * d[2]);
            }
            seg_of.push_back(s);
        }
    };
    std::vector<int> ss, ts;
    sample_chain(src, ss);
    sample_chain(tgt, ts);
    // forward kinematics from the tail: joint k (at x = k*len on the straight
    // chain) rotates every segment >= k; applying k = segs-1 .. 1 keeps each
    // joint centre at its original position when it is used
    double angles[segs], axes[segs][3];
    for (int k = 1; k < segs; ++k) {
        angles[k] = rng.uni(-40.0, 40.0) * M_PI / 180.0;
        axes[k][0] = 0;
        axes[k][1] = rng.gauss();
        axes[k][2] = rng.gauss();
        const double l = std::hypot(axes[k][1], axes[k][2]);
        axes[k][1] /= l;
        axes[k][2] /= l;
    }
    for (int k = segs - 1; k >= 1; --k) {
        std::vector<int> ids;
        for (int i = 0; i < tgt.count(); ++i)
            if (ts[i] >= k) ids.push_back(i);
        std::vector<double> moved(ids.size() * 3);
        for (size_t t = 0; t < ids.size(); ++t)
            for (int c = 0; c < 3; ++c) moved[3 * t + c] = tgt.pts[3 * ids[t] + c];
        const double jc[3] = {k * len, 0, 0};
        rotate_axis_angle(moved.data(), static_cast<int>(ids.size()), axes[k], angles[k], jc);
        for (size_t t = 0; t < ids.size(); ++t)
            for (int c = 0; c < 3; ++c) tgt.pts[3 * ids[t] + c] = moved[3 * t + c];
    }
    halfspace_crop(rng, tgt, 0.30, false);
    // replace 5% of the remaining points by uniform outliers in 1.2x the bbox
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int i = 0; i < tgt.count(); ++i)
        for (int c = 0; c < 3; ++c) {
            lo[c] = std::min(lo[c], tgt.pts[3 * i + c]);
            hi[c] = std::max(hi[c], tgt.pts[3 * i + c]);
        }
    for (int c = 0; c < 3; ++c) {
        const double mid = 0.5 * (lo[c] + hi[c]), half = 0.6 * (hi[c] - lo[c]);
        lo[c] = mid - half;
        hi[c] = mid + half;
    }
    const int cnt = tgt.count(), n_out = static_cast<int>(0.05 * cnt);
    std::vector<int> perm(cnt);
    std::iota(perm.begin(), perm.end(), 0);
    for (int t = 0; t < n_out; ++t) {
        const int j = t + static_cast<int>(rng.uni() * (cnt - t)) % (cnt - t);
        std::swap(perm[t], perm[j]);
        const int i = perm[t];
        for (int c = 0; c < 3; ++c) tgt.pts[3 * i + c] = rng.uni(lo[c], hi[c]);
    }
}
}  // namespace

void synth_config(int which, uint64_t seed, double scale, std::vector<double>& src, std::vector<int32_t>& faces,
                  std::vector<double>& tgt) {
    if (!(scale > 0.0 && scale <= 1.0)) throw ConfigError("synth: scale must be in (0, 1]");
    Rng rng(seed);
    Cloud s, t;
    switch (which) {
        case 0:
            torus_pair(rng, std::max(64, static_cast<int>(5000 * scale)), s, t);
            break;
        case 1:
            capsule_pair(rng, std::max(64, static_cast<int>(50000 * scale)), s, t);
            break;
        case 2:
            height_pair(rng, std::max(8, static_cast<int>(std::lround(316 * std::sqrt(scale)))), 3, 0.10, 0.0, 0.10, s,
                        t);
            break;
        case 3:
            torus_pair(rng, std::max(64, static_cast<int>(20000 * scale)), s, t);
            break;
        case 4:
            height_pair(rng, std::max(8, static_cast<int>(std::lround(1000 * std::sqrt(scale)))), 0, 0.0, 0.20, 0.08,
                        s, t);
            break;
        default:
            throw ConfigError("synth: config must be 0..4");
    }
    src = std::move(s.pts);
    faces = std::move(s.faces);
    tgt = std::move(t.pts);
}

std::vector<std::pair<int, int>> edges_from_faces(const int32_t* faces, int nf, int n) {
    return faces_to_edges(faces, nf, n);
}
std::vector<std::pair<int, int>> knn_edges(const double* pts, int n, int k) { return grid_knn_edges(pts, n, k); }
double avg_edge_length(const double* pts, int n, const int32_t* edges, int ne) {
    return finalize(pts, n, edges, ne).avg;
}

}  // namespace nrr_b200
