// Edge-graph geodesic ball (reference geodesic.hpp:22-84): every vertex whose
// shortest path along the surface edges from `source_index` is < radius, as
// (vertex, distance) sorted by vertex, the source at 0. Host code through the
// C ABI (the device graph build computes the same balls in setup_graph.cu).
#pragma once

#include <utility>
#include <vector>

#include "nrr/common.hpp"
#include "nrr/surface.hpp"

namespace nrr {

inline std::vector<std::pair<int, double>> limited_geodesic(const Surface& surface, int source_index, double radius) {
    const auto pts = detail::flat(surface.points);
    std::vector<int32_t> e(2 * surface.edges.size());
    for (size_t i = 0; i < surface.edges.size(); ++i) {
        e[2 * i] = surface.edges[i].first;
        e[2 * i + 1] = surface.edges[i].second;
    }
    const int32_t ne = static_cast<int32_t>(surface.edges.size());
    int32_t cnt = 0;
    detail::check(nrr_limited_geodesic(pts.data(), surface.point_count(), e.data(), ne, source_index, radius, nullptr,
                                       nullptr, 0, &cnt));
    std::vector<int32_t> idx(cnt);
    std::vector<double> dist(cnt);
    detail::check(nrr_limited_geodesic(pts.data(), surface.point_count(), e.data(), ne, source_index, radius,
                                       idx.data(), dist.data(), cnt, &cnt));
    std::vector<std::pair<int, double>> out(cnt);
    for (int t = 0; t < cnt; ++t) out[t] = {idx[t], dist[t]};
    return out;
}

}  // namespace nrr
