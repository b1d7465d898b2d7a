// Surface sample sets (reference surface.hpp:17-149). Connectivity and
// normalisation run on the host through the C ABI setup entry points.
#pragma once

#include <array>
#include <utility>
#include <vector>

#include "nrr/common.hpp"

namespace nrr {

struct Surface {
    std::vector<Vec3> points;
    std::vector<std::array<int, 3>> faces;
    std::vector<std::pair<int, int>> edges;
    double avg_edge_length = 0.0;
    /// per vertex: (neighbour, edge length), sorted (surface.hpp:24)
    std::vector<std::vector<std::pair<int, double>>> adjacency;

    int point_count() const { return static_cast<int>(points.size()); }

    /// surface.hpp:29-45: mean edge length (C ABI, which also range-checks the
    /// edges) and the sorted adjacency lists
    void finalize_edges() {
        const auto f = detail::flat(points);
        std::vector<int32_t> e(2 * edges.size());
        for (size_t i = 0; i < edges.size(); ++i) {
            e[2 * i] = edges[i].first;
            e[2 * i + 1] = edges[i].second;
        }
        detail::check(nrr_avg_edge_length(f.data(), point_count(), e.data(), static_cast<int32_t>(edges.size()),
                                          &avg_edge_length));
        adjacency.assign(points.size(), {});
        for (const auto& [a, b] : edges) {
            const double len = (points[a] - points[b]).norm();
            adjacency[a].emplace_back(b, len);
            adjacency[b].emplace_back(a, len);
        }
        for (auto& nb : adjacency) std::sort(nb.begin(), nb.end());
    }
};

inline std::vector<std::pair<int, int>> edges_from_faces(const std::vector<std::array<int, 3>>& faces,
                                                         int point_count) {  // surface.hpp:49-65
    std::vector<int32_t> f(3 * faces.size()), out(6 * faces.size() + 2);
    for (size_t i = 0; i < faces.size(); ++i)
        for (int k = 0; k < 3; ++k) f[3 * i + k] = faces[i][k];
    int32_t cnt = 0;
    detail::check(nrr_edges_from_faces(f.data(), static_cast<int32_t>(faces.size()), point_count, out.data(),
                                       static_cast<int32_t>(out.size() / 2), &cnt));
    std::vector<std::pair<int, int>> e(cnt);
    for (int i = 0; i < cnt; ++i) e[i] = {out[2 * i], out[2 * i + 1]};
    return e;
}

/// surface.hpp:70-94 (device build when a B200 is visible, k <= 32)
inline std::vector<std::pair<int, int>> knn_edges(const std::vector<Vec3>& points, int k) {
    const auto f = detail::flat(points);
    std::vector<int32_t> out(2 * points.size() * std::max(k, 1) + 2);
    int32_t cnt = 0;
    if (detail::setup_on_device() && k >= 1 && k <= 32)
        detail::check(nrr_knn_edges_gpu(0, f.data(), static_cast<int32_t>(points.size()), k, out.data(),
                                        static_cast<int32_t>(out.size() / 2), &cnt));
    else
        detail::check(nrr_knn_edges(f.data(), static_cast<int32_t>(points.size()), k, out.data(),
                                    static_cast<int32_t>(out.size() / 2), &cnt));
    std::vector<std::pair<int, int>> e(cnt);
    for (int i = 0; i < cnt; ++i) e[i] = {out[2 * i], out[2 * i + 1]};
    return e;
}

inline Surface make_surface(std::vector<Vec3> points, std::vector<std::array<int, 3>> faces = {},
                            int knn_k = 6) {  // surface.hpp:98-110
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

struct Normalization {  // surface.hpp:113-119
    double scale = 1.0;
    Vec3 center = Vec3::Zero();
    Vec3 apply(const Vec3& v) const { return (v - center) * scale; }
    Vec3 invert(const Vec3& v) const { return v / scale + center; }
};

inline Normalization normalize_pair(Surface& source, Surface& target) {  // surface.hpp:125-149
    auto s = detail::flat(source.points), t = detail::flat(target.points);
    double out4[4];
    detail::check(nrr_normalize_pair(s.data(), source.point_count(), t.data(), target.point_count(), out4));
    source.points = detail::unflat(s.data(), source.points.size());
    target.points = detail::unflat(t.data(), target.points.size());
    source.finalize_edges();
    target.finalize_edges();
    Normalization n;
    n.scale = out4[0];
    n.center = Vec3(out4[1], out4[2], out4[3]);
    return n;
}

}  // namespace nrr
