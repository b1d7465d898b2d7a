// Exact nearest-neighbour index (reference kd_tree.hpp:17-119) backed by the
// device BVH (csrc/nn.cu): same results as an exhaustive FP64 scan, ties to the
// smallest index.
#pragma once

#include <memory>
#include <utility>
#include <vector>

#include "nrr/common.hpp"

namespace nrr {

class SpatialIndex {
public:
    struct Hit {
        int index = -1;
        double distance = 0.0;
    };
    explicit SpatialIndex(std::vector<Vec3> points) : points_(std::move(points)), ctx_(std::make_shared<detail::Context>(0)) {
        if (points_.empty()) throw NumericalError("SpatialIndex: cannot index an empty point set");
        const auto f = detail::flat(points_);
        detail::check(nrr_ctx_set_target(ctx_->get(), f.data(), static_cast<int32_t>(points_.size())));
    }
    Hit nearest(const Vec3& q) const {
        const auto hits = nearest_batch({q});
        return hits[0];
    }
    /// batched queries: one kernel launch for all of them
    std::vector<Hit> nearest_batch(const std::vector<Vec3>& queries) const {
        const auto f = detail::flat(queries);
        std::vector<int32_t> idx(queries.size());
        std::vector<double> dist(queries.size());
        if (!queries.empty())
            detail::check(nrr_nearest(ctx_->get(), f.data(), static_cast<int32_t>(queries.size()), idx.data(), dist.data()));
        std::vector<Hit> out(queries.size());
        for (size_t i = 0; i < queries.size(); ++i) out[i] = {idx[i], dist[i]};
        return out;
    }
    const std::vector<Vec3>& points() const { return points_; }
    int size() const { return static_cast<int>(points_.size()); }

private:
    std::vector<Vec3> points_;
    std::shared_ptr<detail::Context> ctx_;
};

inline SpatialIndex build_spatial_index(std::vector<Vec3> points) { return SpatialIndex(std::move(points)); }

inline std::pair<int, double> closest_point(const SpatialIndex& index, const Vec3& q) {
    const auto hit = index.nearest(q);
    return {hit.index, hit.distance};
}

}  // namespace nrr
