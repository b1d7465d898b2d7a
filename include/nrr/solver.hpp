// Registration driver (reference solver.hpp:16-304): register_surfaces runs
// the whole MM loop on the device (nrr_register) -- NN, Welsch weights,
// assembly, PCG, rotation projection, Anderson with the energy safeguard,
// annealing -- with host copies only at entry and exit. The parameter helpers
// are the reference's formulas on the host.
#pragma once

#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "nrr/anderson.hpp"
#include "nrr/deformation_graph.hpp"
#include "nrr/energy.hpp"
#include "nrr/kd_tree.hpp"
#include "nrr/surface.hpp"

namespace nrr {

struct SolverConfig {  // solver.hpp:16-39
    double k_alpha = 100.0;
    double k_beta = 1.0;
    double eps = 1e-5;
    int i_max = 100;
    int aa_window = 5;
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
    double nu_a = 0.0, nu_r = 0.0, nu_a_min = 0.0, alpha = 0.0, beta = 0.0;
    bool alpha_forced_zero = false;
};

struct AnnealResult {  // solver.hpp:54-58
    double nu_a = 0.0, nu_r = 0.0;
    bool done = false;
};

/// solver.hpp:60-64
inline AnnealResult anneal(double nu_a, double nu_r, double nu_a_min, double nu_r_floor = 1e-8) {
    if (nu_a == nu_a_min) return {nu_a, nu_r, true};
    return {std::max(nu_a / 2.0, nu_a_min), std::max(nu_r / 2.0, nu_r_floor), false};
}

/// solver.hpp:68-81
inline void update_term_weights(SolverParams& p, int point_count, const DeformationGraph& graph,
                                const SolverConfig& cfg) {
    if (graph.edge_count() == 0) {
        p.alpha = 0.0;
        p.alpha_forced_zero = true;
    } else {
        p.alpha = cfg.k_alpha * (static_cast<double>(point_count) / graph.edge_count()) * (p.nu_r * p.nu_r) /
                  (p.nu_a * p.nu_a);
    }
    p.beta = cfg.k_beta * (static_cast<double>(point_count) / graph.node_count()) / (2.0 * p.nu_a * p.nu_a);
}

/// solver.hpp:87-106: the median source->target distance from one batched
/// device query
inline SolverParams init_parameters(const Surface& source, const SpatialIndex& target, const DeformationGraph& graph,
                                    const SolverConfig& cfg) {
    const auto hits = target.nearest_batch(source.points);
    std::vector<double> dist(hits.size());
    for (size_t i = 0; i < hits.size(); ++i) dist[i] = hits[i].distance;
    std::sort(dist.begin(), dist.end());
    const size_t n = dist.size();
    const double median = n % 2 == 1 ? dist[n / 2] : 0.5 * (dist[n / 2 - 1] + dist[n / 2]);
    const double l_bar = source.avg_edge_length;
    SolverParams p;
    p.nu_a_min = std::isnan(cfg.nu_a_min) ? l_bar / std::sqrt(3.0) : cfg.nu_a_min;
    p.nu_a = std::isnan(cfg.nu_a_init) ? std::max(median, p.nu_a_min) : cfg.nu_a_init;
    p.nu_r = std::isnan(cfg.nu_r_init) ? 3.0 * l_bar : cfg.nu_r_init;
    if (!(p.nu_a > 0.0) || !(p.nu_r > 0.0)) throw NumericalError("init_parameters: Welsch parameters must be positive");
    update_term_weights(p, source.point_count(), graph, cfg);
    return p;
}

struct IterationRecord {  // solver.hpp:108-116
    double e_total = 0.0, e_align = 0.0, e_reg = 0.0, e_rot = 0.0, e_landmark = 0.0;
    bool aa_accepted = false;
    double max_disp = 0.0;
};

struct StageRecord {  // solver.hpp:118-124
    double nu_a = 0.0, nu_r = 0.0;
    double alpha = 0.0, beta = 0.0;
    int reverts = 0;
    bool converged = false;
    std::vector<IterationRecord> iterations;
};

struct RegistrationReport {  // solver.hpp:126-138
    std::vector<StageRecord> stages;
    int degenerate_rotations = 0;
    bool alpha_forced_zero = false;
    double solve_seconds = 0.0;
    double graph_seconds = 0.0;
    int linear_iterations = 0;  // device path: PCG iterations over the run

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

/// solver.hpp:146-154: the 4N x 3 column-major block as the AA state vector
inline VectorX flatten(const NodeTransforms& x) { return x.stacked.d; }
inline NodeTransforms unflatten(const VectorX& v, int node_count) {
    if (v.size() != static_cast<size_t>(12) * node_count) throw NumericalError("unflatten: size mismatch");
    NodeTransforms x;
    x.stacked.setZero(4 * node_count, 3);
    x.stacked.d = v;
    return x;
}

/// solver.hpp:159-170: one evaluation of the fixed-point map, teacher-forced
/// at x (nrr_step: deform, NN, projections, weights, assembly, PCG on the
/// device)
inline NodeTransforms mm_step(const Surface& source, const DeformationGraph& graph, const SpatialIndex& target,
                              const NodeTransforms& x, const SolverParams& prm) {
    detail::ProblemArrays pa(source, &target.points(), graph);
    nrr_ctx* c = detail::default_context();
    detail::use_problem(c, pa);
    const double p4[4] = {prm.alpha, prm.beta, prm.nu_a, prm.nu_r};
    NodeTransforms out;
    out.stacked.setZero(4 * graph.node_count(), 3);
    detail::check(nrr_step(c, x.stacked.data(), p4, 0.0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                           out.stacked.data()));
    return out;
}

/// register_surfaces (solver.hpp:180-292) on the device
inline RegistrationResult register_surfaces(const Surface& source, const Surface& target,
                                            const DeformationGraph& graph, const SolverConfig& cfg) {
    cfg.validate();
    if (source.point_count() == 0 || target.point_count() == 0)
        throw NumericalError("register_surfaces: empty surface");
    detail::ProblemArrays pa(source, &target.points, graph);
    detail::LandmarkArrays la(cfg.landmarks);
    nrr_solver_config c = la.cfg;
    c.k_alpha = cfg.k_alpha;
    c.k_beta = cfg.k_beta;
    c.eps = cfg.eps;
    c.i_max = cfg.i_max;
    c.aa_window = cfg.aa_window;
    c.nu_a_init = cfg.nu_a_init;
    c.nu_a_min = cfg.nu_a_min;
    c.nu_r_init = cfg.nu_r_init;
    c.nu_r_floor = cfg.nu_r_floor;

    detail::Context ctx(0);
    RegistrationResult res;
    res.transforms.stacked.setZero(4 * graph.node_count(), 3);
    std::vector<double> deformed(3 * static_cast<size_t>(source.point_count()));
    detail::check(nrr_register(ctx.get(), &pa.view, &c, res.transforms.stacked.data(), deformed.data()));
    res.deformed_points = detail::unflat(deformed.data(), source.points.size());

    nrr_report_summary s{};
    detail::check(nrr_ctx_report(ctx.get(), &s, nullptr, 0, nullptr, 0, nullptr, 0, nullptr));
    std::vector<nrr_stage_record> st(s.stage_count);
    std::vector<nrr_iteration_record> it(s.total_iterations);
    detail::check(nrr_ctx_report(ctx.get(), &s, st.data(), s.stage_count, it.data(), s.total_iterations, nullptr, 0,
                                 nullptr));
    RegistrationReport& rep = res.report;
    rep.degenerate_rotations = s.degenerate_rotations;
    rep.alpha_forced_zero = s.alpha_forced_zero != 0;
    rep.solve_seconds = s.solve_seconds;
    rep.linear_iterations = s.linear_iterations;
    for (const auto& sr : st) {
        StageRecord r;
        r.nu_a = sr.nu_a;
        r.nu_r = sr.nu_r;
        r.alpha = sr.alpha;
        r.beta = sr.beta;
        r.reverts = sr.reverts;
        r.converged = sr.converged != 0;
        for (int k = sr.first_iteration; k < sr.first_iteration + sr.iteration_count; ++k) {
            const auto& ir = it[k];
            IterationRecord rec;
            rec.e_total = ir.e_total;
            rec.e_align = ir.e_align;
            rec.e_reg = ir.e_reg;
            rec.e_rot = ir.e_rot;
            rec.e_landmark = ir.e_landmark;
            rec.aa_accepted = ir.aa_accepted != 0;
            rec.max_disp = ir.max_disp;
            r.iterations.push_back(rec);
        }
        rep.stages.push_back(std::move(r));
    }
    return res;
}

/// solver.hpp:296-302
inline RegistrationResult register_surfaces(const Surface& source, const Surface& target, double radius,
                                            const SolverConfig& cfg) {
    const DeformationGraph graph = build_graph(source, radius);
    return register_surfaces(source, target, graph, cfg);
}

}  // namespace nrr
