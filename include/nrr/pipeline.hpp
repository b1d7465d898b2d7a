// The `register` pipeline (reference pipeline.hpp:19-262): load the pair,
// normalise it to a unit joint bounding-box diagonal, build the deformation
// graph, register on the device (register_surfaces: the whole MM loop runs in
// libnrr_b200.so), map the result back to the original units, attach metrics
// when ground truth is given, write the deformed mesh and the JSON report.
// Same RunConfig fields and defaults, same validation and error classes, same
// report document (json_export.hpp) as the reference; runs with identical
// inputs produce byte-identical outputs apart from `timings` (the device path
// is deterministic: fixed-order reductions, no atomics in the sums).
#pragma once

#include <chrono>
#include <cstdint>
#include <fstream>
#include <limits>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "nrr/common.hpp"
#include "nrr/json.hpp"
#include "nrr/json_export.hpp"
#include "nrr/mesh_io.hpp"
#include "nrr/metrics.hpp"
#include "nrr/solver.hpp"

namespace nrr {

enum class GroundTruthMode { None, IndexIdentity, Flow };

/// pipeline.hpp:22-66
struct RunConfig {
    std::string source_path, target_path, output_path, report_path;
    double k_alpha = 100.0;
    double k_beta = 1.0;
    double radius_multiplier = 5.0;  // R = multiplier * mean source edge length
    double eps = 1e-5;
    int i_max = 100;
    int aa_window = 5;
    int knn = 6;
    uint64_t seed = 0;
    bool binary_ply = false;
    bool error_channel = false;
    double nu_a_init = std::numeric_limits<double>::quiet_NaN();
    double nu_a_min = std::numeric_limits<double>::quiet_NaN();
    double nu_r_init = std::numeric_limits<double>::quiet_NaN();
    GroundTruthMode gt_mode = GroundTruthMode::None;
    std::string flow_path, complete_target_path, mask_path, landmarks_path;

    SolverConfig solver_config() const {
        SolverConfig sc;
        sc.k_alpha = k_alpha;
        sc.k_beta = k_beta;
        sc.eps = eps;
        sc.i_max = i_max;
        sc.aa_window = aa_window;
        sc.nu_a_init = nu_a_init;
        sc.nu_a_min = nu_a_min;
        sc.nu_r_init = nu_r_init;
        return sc;
    }
    void validate() const {
        if (source_path.empty() || target_path.empty()) throw ConfigError("source and target paths are required");
        if (output_path.empty()) throw ConfigError("output path is required");
        if (!(radius_multiplier > 0.0)) throw ConfigError("radius multiplier must be positive");
        if (knn < 1) throw ConfigError("knn must be at least 1");
        if (gt_mode == GroundTruthMode::Flow && flow_path.empty())
            throw ConfigError("flow ground truth requires a flow file");
        solver_config().validate();
    }
};

namespace io_detail {
// line-oriented record files: blank lines and '#' comments are skipped; a
// record whose fields do not parse is "path:line: malformed <what> record"
template <typename Fn>
inline void for_each_record(const std::string& path, const char* kind, Fn&& fn) {
    std::ifstream in(path);
    if (!in) throw IoError(std::string("cannot open ") + kind + " file '" + path + "'");
    std::string line;
    for (size_t lineno = 1; std::getline(in, line); ++lineno) {
        if (blank_or_comment(line)) continue;
        std::istringstream ls(line);
        if (!fn(ls)) fail(path, lineno, std::string("malformed ") + kind + " record");
    }
}
}  // namespace io_detail

/// pipeline.hpp:69-90: `index tx ty tz` per line
inline std::vector<SceneFlow> read_flow_file(const std::string& path) {
    std::vector<SceneFlow> flows;
    std::ifstream probe(path);
    if (!probe) throw IoError("cannot open flow file '" + path + "'");
    std::string line;
    for (size_t lineno = 1; std::getline(probe, line); ++lineno) {
        if (io_detail::blank_or_comment(line)) continue;
        std::istringstream ls(line);
        SceneFlow f;
        double x, y, z;
        if (!(ls >> f.index >> x >> y >> z)) io_detail::fail(path, lineno, "malformed flow record");
        if (f.index < 0) io_detail::fail(path, lineno, "negative flow index");
        f.flow = Vec3(x, y, z);
        flows.push_back(f);
    }
    return flows;
}

/// pipeline.hpp:93-113: `source_index target_index` per line
inline std::vector<std::pair<int, int>> read_landmark_file(const std::string& path) {
    std::vector<std::pair<int, int>> pairs;
    io_detail::for_each_record(path, "landmark", [&](std::istringstream& ls) {
        int s, t;
        if (!(ls >> s >> t)) return false;
        pairs.emplace_back(s, t);
        return true;
    });
    return pairs;
}

/// pipeline.hpp:116-123: one 0/1 per target vertex
inline std::vector<char> read_mask_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open mask file '" + path + "'");
    std::vector<char> mask;
    for (int v; in >> v;) mask.push_back(v != 0 ? 1 : 0);
    return mask;
}

inline void write_mask_file(const std::string& path, const std::vector<char>& mask) {
    std::ofstream out(path);
    if (!out) throw IoError("cannot open '" + path + "' for writing");
    for (char m : mask) out << (m ? '1' : '0') << '\n';
    if (!out) throw IoError("write to '" + path + "' failed");
}

/// pipeline.hpp:133-137
struct PipelineResult {
    RegistrationResult registration;
    nlohmann::json document;
    std::vector<Vec3> deformed_original_units;
};

namespace pipeline_detail {
using clock = std::chrono::steady_clock;
inline double since(clock::time_point t) { return std::chrono::duration<double>(clock::now() - t).count(); }

// metrics in original units (pipeline.hpp:206-230); fills the per-vertex
// errors when the index-identity ground truth is used
inline nlohmann::json metrics(const RunConfig& cfg, const Surface& source_original, const Surface& target_original,
                              const std::vector<Vec3>& deformed, std::vector<double>& errors) {
    nlohmann::json m;
    if (cfg.gt_mode == GroundTruthMode::IndexIdentity) {
        Surface complete;
        const Surface* ref = &target_original;
        if (!cfg.complete_target_path.empty()) {
            complete = load_surface(cfg.complete_target_path, cfg.knn);
            ref = &complete;
        }
        if (ref->point_count() < source_original.point_count())
            throw ConfigError("ground-truth target has fewer vertices than the source");
        const std::vector<Vec3> gt(ref->points.begin(), ref->points.begin() + static_cast<long>(deformed.size()));
        errors = pointwise_error(deformed, gt);
        m["rmse"] = rmse(errors);
    } else if (cfg.gt_mode == GroundTruthMode::Flow) {
        m["rs"] = scene_flow_rmse(deformed, source_original.points, read_flow_file(cfg.flow_path));
    }
    if (!cfg.mask_path.empty()) m["overlap"] = overlap_ratio(read_mask_file(cfg.mask_path), source_original.point_count());
    return m;
}
}  // namespace pipeline_detail

/// pipeline.hpp:141-262
inline PipelineResult run_pipeline(const RunConfig& cfg) {
    using namespace pipeline_detail;
    cfg.validate();
    const auto t0 = clock::now();
    const Surface source_original = load_surface(cfg.source_path, cfg.knn);
    const Surface target_original = load_surface(cfg.target_path, cfg.knn);
    const double load_s = since(t0);

    Surface source = source_original, target = target_original;
    const Normalization norm = normalize_pair(source, target);
    if (!(source.avg_edge_length > 0.0)) throw NumericalError("source surface has no usable edges");

    const auto t_graph = clock::now();
    const DeformationGraph graph = build_graph(source, cfg.radius_multiplier * source.avg_edge_length);
    const double graph_s = since(t_graph);

    SolverConfig sc = cfg.solver_config();
    if (!cfg.landmarks_path.empty()) {
        for (const auto& [s, t] : read_landmark_file(cfg.landmarks_path)) {
            if (s < 0 || s >= source.point_count() || t < 0 || t >= target.point_count())
                throw ConfigError("landmark index out of range");
            Landmark lm;
            lm.source_index = s;
            lm.target_position = target.points[t];
            sc.landmarks.push_back(lm);
        }
    }

    const auto t_reg = clock::now();
    PipelineResult out;
    out.registration = register_surfaces(source, target, graph, sc);
    out.registration.report.graph_seconds = graph_s;
    const double register_s = since(t_reg);

    const auto& dn = out.registration.deformed_points;
    out.deformed_original_units.reserve(dn.size());
    for (const Vec3& p : dn) out.deformed_original_units.push_back(norm.invert(p));

    std::vector<double> errors;
    const nlohmann::json met = metrics(cfg, source_original, target_original, out.deformed_original_units, errors);

    Surface deformed_mesh = source_original;
    deformed_mesh.points = out.deformed_original_units;
    deformed_mesh.finalize_edges();
    SaveOptions so;
    so.binary_ply = cfg.binary_ply;
    save_surface(deformed_mesh, cfg.output_path, cfg.error_channel ? errors : std::vector<double>{}, so);

    nlohmann::json doc = nlohmann::json::object();
    nlohmann::json c = nlohmann::json::object();
    c["source"] = cfg.source_path;
    c["target"] = cfg.target_path;
    c["output"] = cfg.output_path;
    c["k_alpha"] = cfg.k_alpha;
    c["k_beta"] = cfg.k_beta;
    c["radius_multiplier"] = cfg.radius_multiplier;
    c["eps"] = cfg.eps;
    c["i_max"] = cfg.i_max;
    c["aa_window"] = cfg.aa_window;
    c["knn"] = cfg.knn;
    c["seed"] = cfg.seed;
    doc["config"] = std::move(c);
    nlohmann::json g = nlohmann::json::object();
    g["node_count"] = graph.node_count();
    g["edge_count"] = graph.edge_count();
    g["radius"] = graph.radius;
    doc["graph"] = std::move(g);
    nlohmann::json nz = nlohmann::json::object();
    nz["scale"] = norm.scale;
    nz["center"] = {norm.center.x(), norm.center.y(), norm.center.z()};
    doc["normalization"] = std::move(nz);
    const nlohmann::json rep = report_to_json(out.registration.report, !sc.landmarks.empty());
    doc["stages"] = rep.at("stages");
    nlohmann::json so_json = nlohmann::json::object();
    so_json["degenerate_rotations"] = rep.at("degenerate_rotations");
    so_json["alpha_forced_zero"] = rep.at("alpha_forced_zero");
    so_json["total_iterations"] = rep.at("total_iterations");
    doc["solver"] = std::move(so_json);
    if (!met.is_null()) doc["metrics"] = met;
    nlohmann::json tm = nlohmann::json::object();
    tm["load_s"] = load_s;
    tm["graph_s"] = graph_s;
    tm["register_s"] = register_s;
    tm["total_s"] = since(t0);
    doc["timings"] = std::move(tm);

    if (!cfg.report_path.empty()) {
        std::ofstream rf(cfg.report_path);
        if (!rf) throw IoError("cannot open '" + cfg.report_path + "' for writing");
        rf << doc.dump(2) << '\n';
        if (!rf) throw IoError("write to '" + cfg.report_path + "' failed");
    }
    out.document = std::move(doc);
    return out;
}

}  // namespace nrr
