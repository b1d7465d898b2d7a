// Correspondences, rotation projections, energy and the linear system
// (reference energy.hpp:19-410) on the device.
#pragma once

#include <algorithm>
#include <memory>
#include <vector>

#include "nrr/common.hpp"
#include "nrr/deformation_graph.hpp"
#include "nrr/kd_tree.hpp"
#include "nrr/rotation.hpp"
#include "nrr/welsch.hpp"

namespace nrr {

struct Correspondences {  // energy.hpp:20-26
    std::vector<int> target_index;
    std::vector<Vec3> target_point;
    std::vector<double> squared_distance;
    int size() const { return static_cast<int>(target_index.size()); }
};

/// energy.hpp:28-42: one batched device query (squared_distance = distance^2)
inline Correspondences find_correspondences(const std::vector<Vec3>& deformed, const SpatialIndex& target) {
    const auto hits = target.nearest_batch(deformed);
    Correspondences c;
    c.target_index.resize(hits.size());
    c.target_point.resize(hits.size());
    c.squared_distance.resize(hits.size());
    for (size_t i = 0; i < hits.size(); ++i) {
        c.target_index[i] = hits[i].index;
        c.target_point[i] = target.points()[hits[i].index];
        c.squared_distance[i] = hits[i].distance * hits[i].distance;
    }
    return c;
}

/// energy.hpp:47-56: all node projections in one launch
inline std::vector<Mat3> project_rotations(const NodeTransforms& x, int* degenerate_count = nullptr) {
    const int N = x.node_count();
    std::vector<double> R(9 * static_cast<size_t>(N));
    int32_t deg = 0;
    if (!x.all_finite()) throw NumericalError("project_to_rotation: non-finite input matrix");
    detail::check(nrr_project_rotations(detail::default_context(), x.stacked.data(), N, R.data(), &deg));
    std::vector<Mat3> out(N);
    for (int j = 0; j < N; ++j)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) out[j](r, c) = R[9 * j + r * 3 + c];
    if (degenerate_count) *degenerate_count += deg;
    return out;
}

struct EnergyParams {  // energy.hpp:58-63
    double alpha = 0.0, beta = 0.0, nu_a = 1.0, nu_r = 1.0;
};
struct EnergyBreakdown {  // energy.hpp:65-72
    double align = 0.0, reg = 0.0, rot = 0.0, total = 0.0;
    double alpha = 0.0, beta = 0.0, nu_a = 0.0, nu_r = 0.0;
};

/// energy.hpp:74-86
inline Vec3 reg_difference(const DeformationGraph& graph, const NodeTransforms& x, int pair_index) {
    const auto [i, j] = graph.reg_pairs[pair_index];
    const double c = graph.reg_weights[pair_index];
    const Vec3& pi = graph.node_positions[i];
    const Vec3& pj = graph.node_positions[j];
    return c * (x.affine(j) * (pi - pj) + pj + x.translation(j) - pi - x.translation(i));
}

namespace detail {
inline nrr_energy_terms_in terms_in(const DeformationGraph& graph, const NodeTransforms& x,
                                    std::vector<double>& pos, std::vector<int32_t>& pairs) {
    nrr_energy_terms_in in{};
    pos = flat(graph.node_positions);
    pairs.clear();
    for (const auto& [i, j] : graph.reg_pairs) {
        pairs.push_back(i);
        pairs.push_back(j);
    }
    in.node_count = graph.node_count();
    in.X = x.stacked.data();
    in.node_positions = pos.data();
    in.pair_count = graph.directed_pair_count();
    in.reg_pairs = pairs.data();
    in.reg_weights = graph.reg_weights.data();
    return in;
}
}  // namespace detail

/// energy.hpp:92-116 against caller-held correspondences and rotations, on
/// the device (api_terms.cu: per point / pair / node terms, fixed-order sums;
/// inside register_surfaces the same sums come from terms_kernel)
inline EnergyBreakdown evaluate_energy(const std::vector<Vec3>& deformed, const NodeTransforms& x,
                                       const DeformationGraph& graph, const Correspondences& corr,
                                       const std::vector<Mat3>& rotations, const EnergyParams& prm) {
    if (corr.size() != static_cast<int>(deformed.size()))
        throw NumericalError("evaluate_energy: correspondence count mismatch");
    if (static_cast<int>(rotations.size()) != graph.node_count())
        throw NumericalError("evaluate_energy: rotation count mismatch");
    std::vector<double> pos, R(9 * rotations.size());
    std::vector<int32_t> pairs;
    nrr_energy_terms_in in = detail::terms_in(graph, x, pos, pairs);
    const auto d = detail::flat(deformed), u = detail::flat(corr.target_point);
    for (size_t j = 0; j < rotations.size(); ++j)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) R[9 * j + 3 * r + c] = rotations[j](r, c);
    in.n = static_cast<int32_t>(deformed.size());
    in.deformed = d.data();
    in.corr_points = u.data();
    in.nu_a = prm.nu_a;
    in.nu_r = prm.nu_r;
    in.rotations = R.data();
    double sums[3];
    detail::check(nrr_energy_terms(detail::default_context(), &in, nullptr, nullptr, sums));
    EnergyBreakdown e;
    e.align = sums[0];
    e.reg = sums[1];
    e.rot = sums[2];
    e.total = e.align + prm.alpha * e.reg + prm.beta * e.rot;
    e.alpha = prm.alpha;
    e.beta = prm.beta;
    e.nu_a = prm.nu_a;
    e.nu_r = prm.nu_r;
    return e;
}

/// energy.hpp:118-121: K (4N x 4N, the fixed pattern: diagonal + both halves
/// of every graph edge) and B (4N x 3). The device assembles K as 4x4 blocks
/// in pattern order (block_row_ptr / block_cols / values, 16 per block
/// row-major); K is their scalar CSC image, refreshed by every fill (the
/// reference's Eigen::SparseMatrix member, read by callers and tests).
struct LinearSystem {
    SparseMatrix K;
    MatrixX B;  // 4N x 3
    std::vector<int> block_row_ptr;
    std::vector<int> block_cols;
    std::vector<double> values;
    std::vector<int> csc_from_block;       // K.val[q] = values[csc_from_block[q]]
    std::shared_ptr<detail::Context> ctx;  // device copy of the system

    int rows() const { return B.rows(); }
    double coeff(int r, int c) const { return K.coeff(r, c); }

    // scalar CSC pattern of the block pattern (K is symmetric: column c of
    // block column b lists rows 4a + i for the blocks a of node b, ascending)
    void build_pattern() {
        const int N = static_cast<int>(block_row_ptr.size()) - 1;
        K = SparseMatrix(4 * N, 4 * N);
        csc_from_block.clear();
        for (int b = 0; b < N; ++b)
            for (int j = 0; j < 4; ++j) {
                for (int k = block_row_ptr[b]; k < block_row_ptr[b + 1]; ++k)
                    for (int i = 0; i < 4; ++i) {
                        K.inner.push_back(4 * block_cols[k] + i);
                        // K(4a+i, 4b+j) = block (b, a) entry (j, i) by symmetry
                        csc_from_block.push_back(16 * k + 4 * j + i);
                    }
                K.outer[4 * b + j + 1] = static_cast<int>(K.inner.size());
            }
        K.val.assign(K.inner.size(), 0.0);
    }
    void refresh_K() {
        for (size_t q = 0; q < csc_from_block.size(); ++q) K.val[q] = values[csc_from_block[q]];
    }
};

struct Landmark {  // energy.hpp:125-128
    int source_index = -1;
    Vec3 target_position = Vec3::Zero();
};

namespace detail {
struct LandmarkArrays {
    std::vector<int32_t> idx;
    std::vector<double> pos;
    nrr_solver_config cfg{};
    explicit LandmarkArrays(const std::vector<Landmark>& lms) {
        for (const auto& lm : lms) {
            idx.push_back(lm.source_index);
            for (int k = 0; k < 3; ++k) pos.push_back(lm.target_position[k]);
        }
        cfg.landmark_count = static_cast<int32_t>(idx.size());
        cfg.landmark_index = idx.empty() ? nullptr : idx.data();
        cfg.landmark_pos = pos.empty() ? nullptr : pos.data();
    }
};
}  // namespace detail

/// energy.hpp:137-360: the pattern and the assembly plan are built once on
/// the device (nrr_ctx_set_problem); fill() runs the assembly kernel
/// (mirrored writes, fixed order, bitwise symmetric K); solve() runs the FP64
/// block-Jacobi + aggregation PCG instead of the sparse LDLT, with the same
/// residual bar and failure messages.
class SystemAssembler {
public:
    SystemAssembler(const Surface& source, const DeformationGraph& graph, std::vector<Landmark> landmarks = {})
        : source_(&source), graph_(&graph), landmarks_(std::move(landmarks)),
          ctx_(std::make_shared<detail::Context>(0)) {
        for (const auto& lm : landmarks_)
            if (lm.source_index < 0 || lm.source_index >= source.point_count())
                throw ConfigError("landmark source index out of range");
        detail::ProblemArrays pa(source, nullptr, graph);
        detail::check(nrr_ctx_set_problem(ctx_->get(), &pa.view));
        const int N = graph.node_count();
        std::vector<std::vector<int>> cols(N);
        for (int j = 0; j < N; ++j) cols[j].push_back(j);
        for (const auto& [a, b] : graph.graph_edges) {
            cols[a].push_back(b);
            cols[b].push_back(a);
        }
        system_.block_row_ptr.push_back(0);
        for (auto& c : cols) {
            std::sort(c.begin(), c.end());
            system_.block_cols.insert(system_.block_cols.end(), c.begin(), c.end());
            system_.block_row_ptr.push_back(static_cast<int>(system_.block_cols.size()));
        }
        system_.values.assign(16 * system_.block_cols.size(), 0.0);
        system_.B.setZero(4 * N, 3);
        system_.build_pattern();
        system_.ctx = ctx_;
    }

    /// energy.hpp:182-228
    void fill(const Correspondences& corr, const std::vector<Mat3>& rotations, const std::vector<double>& w_align,
              const std::vector<double>& w_reg, double beta, double landmark_weight = 0.0) {
        const int n = source_->point_count();
        if (corr.size() != n) throw NumericalError("assemble: correspondence count mismatch");
        if (static_cast<int>(w_align.size()) != n || static_cast<int>(w_reg.size()) != graph_->directed_pair_count())
            throw NumericalError("assemble: weight count mismatch");
        if (static_cast<int>(rotations.size()) != graph_->node_count())
            throw NumericalError("assemble: rotation count mismatch");
        const auto q = detail::flat(corr.target_point);
        std::vector<double> R(9 * rotations.size());
        for (size_t j = 0; j < rotations.size(); ++j)
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) R[9 * j + 3 * r + c] = rotations[j](r, c);
        detail::LandmarkArrays la(landmarks_);
        detail::check(nrr_assemble(ctx_->get(), q.data(), w_align.data(), w_reg.data(), R.data(), beta,
                                   landmark_weight, landmarks_.empty() ? nullptr : &la.cfg, system_.values.data(),
                                   system_.B.data()));
        system_.refresh_K();
    }

    const LinearSystem& system() const { return system_; }

    /// energy.hpp:233-254: solve the resident system on the device
    NodeTransforms solve() {
        NodeTransforms x;
        x.stacked.setZero(system_.B.rows(), 3);
        detail::check(nrr_solve(ctx_->get(), nullptr, nullptr, nullptr, x.stacked.data()));
        return x;
    }

private:
    const Surface* source_;
    const DeformationGraph* graph_;
    std::vector<Landmark> landmarks_;
    std::shared_ptr<detail::Context> ctx_;
    LinearSystem system_;
};

/// energy.hpp:363-369 on the device (api_terms.cu)
inline std::vector<double> alignment_weights(const Correspondences& corr, double nu_a) {
    std::vector<double> w(corr.size());
    if (w.empty()) return w;
    nrr_energy_terms_in in{};
    in.n = corr.size();
    in.corr_sqdist = corr.squared_distance.data();
    in.nu_a = nu_a;
    detail::check(nrr_energy_terms(detail::default_context(), &in, w.data(), nullptr, nullptr));
    return w;
}

/// energy.hpp:371-379 on the device (api_terms.cu)
inline std::vector<double> regularization_weights(const DeformationGraph& graph, const NodeTransforms& x, double nu_r,
                                                  double alpha) {
    std::vector<double> w(graph.directed_pair_count());
    if (w.empty()) return w;
    std::vector<double> pos;
    std::vector<int32_t> pairs;
    nrr_energy_terms_in in = detail::terms_in(graph, x, pos, pairs);
    in.nu_r = nu_r;
    in.alpha = alpha;
    detail::check(nrr_energy_terms(detail::default_context(), &in, nullptr, w.data(), nullptr));
    return w;
}

/// energy.hpp:381-391
inline LinearSystem assemble_system(const NodeTransforms& x, const Surface& source, const DeformationGraph& graph,
                                    const Correspondences& corr, const std::vector<Mat3>& rotations,
                                    const EnergyParams& prm) {
    SystemAssembler assembler(source, graph);
    assembler.fill(corr, rotations, alignment_weights(corr, prm.nu_a),
                   regularization_weights(graph, x, prm.nu_r, prm.alpha), prm.beta);
    return assembler.system();
}

/// energy.hpp:393-409: K X = B on the device PCG (K must be positive definite)
inline NodeTransforms solve_system(const LinearSystem& system) {
    if (!system.ctx) throw ConfigError("solve_system: system was not assembled by this library");
    // the block values from K (a caller may have edited K, as the reference's
    // tests do with B): every block entry is one CSC entry of K
    std::vector<double> values(system.values.size());
    for (size_t q = 0; q < system.csc_from_block.size(); ++q) values[system.csc_from_block[q]] = system.K.val[q];
    NodeTransforms x;
    x.stacked.setZero(system.B.rows(), 3);
    detail::check(nrr_solve(system.ctx->get(), values.data(), system.B.data(), nullptr, x.stacked.data()));
    return x;
}

}  // namespace nrr
