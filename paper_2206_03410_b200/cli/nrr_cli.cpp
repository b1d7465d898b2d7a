// `nrr` command-line front end over the drop-in API (reference
// proj/tools/nrr_cli.cpp:149-280): `register` (run_pipeline, the MM loop on
// the B200), `metrics` and `graph-dump`. Same option names, defaults, error
// document on stderr ({"error": {"kind", "message", "code"}}) and exit codes
// (2 io, 3 numerical/internal, 4 config) as the reference. CLI11 is not in
// this image, so options are parsed here: `--name value`, `--name=value`, the
// short aliases -s/-t/-o, flags, and `--config file` with `name = value`
// lines (CLI11's config-file form; '#' / ';' comments, [section] headers
// ignored). The reference's `synth-noise` / `synth-crop` generate test
// inputs (synthesis.hpp) and are outside this build's scope.
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "nrr/nrr.hpp"

namespace {

struct ParseError : std::runtime_error {
    explicit ParseError(const std::string& m) : std::runtime_error(m) {}
};

void emit_error(const std::string& kind, const std::string& message, int code) {
    nlohmann::json inner = nlohmann::json::object();
    inner["kind"] = kind;
    inner["message"] = message;
    inner["code"] = code;
    nlohmann::json err = nlohmann::json::object();
    err["error"] = inner;
    std::cerr << err.dump() << std::endl;
}

// one subcommand's options: name -> setter; flags take no value
class Options {
public:
    explicit Options(std::string sub) : sub_(std::move(sub)) {}
    template <typename T>
    void value(const std::string& names, T& target, const std::string& help, bool required = false) {
        add(names, help, required, false, [&target, names](const std::string& v) { assign(target, v, names); });
    }
    void flag(const std::string& names, bool& target, const std::string& help) {
        add(names, help, false, true, [&target](const std::string& v) { target = v.empty() || v == "true" || v == "1"; });
    }
    void choice(const std::string& names, std::string& target, std::set<std::string> allowed, const std::string& help) {
        add(names, help, false, false, [&target, allowed, names](const std::string& v) {
            if (!allowed.count(v)) throw ParseError(names + ": " + v + " not in {" + join(allowed) + "}");
            target = v;
        });
    }

    void parse(const std::vector<std::string>& args) {
        for (size_t i = 0; i < args.size(); ++i) {
            std::string a = args[i], v;
            bool has_value = false;
            const size_t eq = a.find('=');
            if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
                v = a.substr(eq + 1);
                a = a.substr(0, eq);
                has_value = true;
            }
            if (a == "--config") {
                if (!has_value) {
                    if (i + 1 >= args.size()) throw ParseError("--config: 1 required argument missing");
                    v = args[++i];
                }
                read_config(v);
                continue;
            }
            auto it = by_name_.find(a);
            if (it == by_name_.end()) throw ParseError("The following argument was not expected: " + args[i]);
            Opt& o = opts_[it->second];
            if (o.is_flag) {
                o.set(has_value ? v : "");
            } else {
                if (!has_value) {
                    if (i + 1 >= args.size()) throw ParseError(o.names + ": 1 required argument missing");
                    v = args[++i];
                }
                o.set(v);
            }
            o.seen = true;
        }
        for (const Opt& o : opts_)
            if (o.required && !o.seen) throw ParseError(o.names + " is required");
    }

    std::string usage() const {
        std::ostringstream os;
        os << "Usage: nrr " << sub_ << " [OPTIONS]\n\nOptions:\n  --config TEXT  Read options from a key=value config file\n";
        for (const Opt& o : opts_)
            os << "  " << o.names << (o.is_flag ? "" : " VALUE") << (o.required ? " REQUIRED" : "") << "  " << o.help
               << "\n";
        return os.str();
    }

private:
    struct Opt {
        std::string names, help;
        bool required = false, is_flag = false, seen = false;
        std::function<void(const std::string&)> set;
    };

    static std::string join(const std::set<std::string>& s) {
        std::string out;
        for (const auto& x : s) out += (out.empty() ? "" : ",") + x;
        return out;
    }
    template <typename T>
    static void assign(T& target, const std::string& v, const std::string& names) {
        std::istringstream is(v);
        T x{};
        if constexpr (std::is_same_v<T, std::string>) {
            target = v;
            return;
        } else {
            if (!(is >> x) || !(is >> std::ws).eof())
                throw ParseError(names + ": Value " + v + " could not be converted");
            target = x;
        }
    }
    void add(const std::string& names, const std::string& help, bool required, bool is_flag,
             std::function<void(const std::string&)> set) {
        Opt o;
        o.names = names;
        o.help = help;
        o.required = required;
        o.is_flag = is_flag;
        o.set = std::move(set);
        std::istringstream ns(names);
        for (std::string n; std::getline(ns, n, ',');) {
            by_name_[n] = opts_.size();
            if (n.rfind("--", 0) == 0) config_key_[n.substr(2)] = opts_.size();
        }
        opts_.push_back(std::move(o));
    }
    void read_config(const std::string& path) {
        std::ifstream in(path);
        if (!in) throw ParseError("File does not exist: " + path);
        std::string line;
        while (std::getline(in, line)) {
            const size_t b = line.find_first_not_of(" \t\r");
            if (b == std::string::npos || line[b] == '#' || line[b] == ';' || line[b] == '[') continue;
            const size_t eq = line.find('=');
            if (eq == std::string::npos) throw ParseError("config line without '=': " + line);
            auto trim = [](std::string s) {
                const size_t x = s.find_first_not_of(" \t\r\""), y = s.find_last_not_of(" \t\r\"");
                return x == std::string::npos ? std::string() : s.substr(x, y - x + 1);
            };
            std::string key = trim(line.substr(0, eq)), val = trim(line.substr(eq + 1));
            for (char& ch : key)
                if (ch == '_') ch = '-';
            auto it = config_key_.find(key);
            if (it == config_key_.end()) throw ParseError("The following argument was not expected: " + key);
            opts_[it->second].set(val);
            opts_[it->second].seen = true;
        }
    }

    std::string sub_;
    std::vector<Opt> opts_;
    std::map<std::string, size_t> by_name_, config_key_;
};

// reference nrr_cli.cpp:80-124
struct MetricsArgs {
    std::string deformed, gt_target, source, flow_file, mask_file, report, per_vertex_out;
    int knn = 6;
};

void write_doc(const nlohmann::json& doc, const std::string& path) {
    if (path.empty()) {
        std::cout << doc.dump(2) << std::endl;
        return;
    }
    std::ofstream out(path);
    if (!out) throw nrr::IoError("cannot open '" + path + "' for writing");
    out << doc.dump(2) << '\n';
}

void run_metrics(const MetricsArgs& a) {
    const nrr::Surface deformed = nrr::load_surface(a.deformed, a.knn);
    nlohmann::json metrics;
    std::vector<double> errors;
    if (!a.gt_target.empty()) {
        const nrr::Surface gt = nrr::load_surface(a.gt_target, a.knn);
        if (gt.point_count() < deformed.point_count())
            throw nrr::ConfigError("ground-truth target has fewer vertices than the result");
        const std::vector<nrr::Vec3> ref(gt.points.begin(), gt.points.begin() + deformed.point_count());
        errors = nrr::pointwise_error(deformed.points, ref);
        metrics["rmse"] = nrr::rmse(errors);
        if (!a.mask_file.empty()) {
            const std::vector<char> mask = nrr::read_mask_file(a.mask_file);
            metrics["overlap"] = nrr::overlap_ratio(mask, deformed.point_count());
            std::vector<double> inside;
            for (size_t i = 0; i < errors.size() && i < mask.size(); ++i)
                if (mask[i]) inside.push_back(errors[i]);
            if (!inside.empty()) metrics["rmse_overlap"] = nrr::rmse(inside);
        }
    }
    if (!a.flow_file.empty()) {
        if (a.source.empty()) throw nrr::ConfigError("flow metrics need --source for the undeformed points");
        const nrr::Surface source = nrr::load_surface(a.source, a.knn);
        metrics["rs"] = nrr::scene_flow_rmse(deformed.points, source.points, nrr::read_flow_file(a.flow_file));
    }
    if (metrics.is_null()) throw nrr::ConfigError("no ground truth given to metrics");
    if (!a.per_vertex_out.empty() && !errors.empty()) nrr::save_surface(deformed, a.per_vertex_out, errors);
    nlohmann::json doc = nlohmann::json::object();
    doc["metrics"] = metrics;
    write_doc(doc, a.report);
}

// reference nrr_cli.cpp:126-146
struct GraphDumpArgs {
    std::string in, out;
    double radius_mult = 5.0;
    int knn = 6;
};

void run_graph_dump(const GraphDumpArgs& a) {
    const nrr::Surface surface = nrr::load_surface(a.in, a.knn);
    if (!(surface.avg_edge_length > 0.0)) throw nrr::NumericalError("surface has no usable edges");
    write_doc(nrr::graph_to_json(nrr::build_graph(surface, a.radius_mult * surface.avg_edge_length)), a.out);
}

const char* kTop =
    "Robust non-rigid registration of a source surface to a target point set\n"
    "Usage: nrr SUBCOMMAND [OPTIONS]\n\nSubcommands:\n"
    "  register    Register a source surface to a target\n"
    "  metrics     Evaluate a registration result\n"
    "  graph-dump  Export the deformation graph as JSON\n";

}  // namespace

int main(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    if (args.empty()) {
        std::cerr << kTop;
        emit_error("config", "A subcommand is required", 4);
        return 4;
    }
    if (args[0] == "--help" || args[0] == "-h") {
        std::cout << kTop;
        return 0;
    }
    const std::string sub = args[0];
    args.erase(args.begin());
    const bool help = [&] {
        for (const auto& a : args)
            if (a == "--help" || a == "-h") return true;
        return false;
    }();

    nrr::RunConfig reg;
    std::string gt_mode = "none";
    MetricsArgs met;
    GraphDumpArgs gd;
    Options opt(sub);
    if (sub == "register") {  // nrr_cli.cpp:154-192
        opt.value("--source,-s", reg.source_path, "Source mesh or point cloud", true);
        opt.value("--target,-t", reg.target_path, "Target mesh or point cloud", true);
        opt.value("--out,-o", reg.output_path, "Deformed source output path", true);
        opt.value("--report", reg.report_path, "JSON report output path");
        opt.value("--k-alpha", reg.k_alpha, "Regularization weight multiplier");
        opt.value("--k-beta", reg.k_beta, "Rotation term weight multiplier");
        opt.value("--radius-mult", reg.radius_multiplier, "Graph sampling radius as a multiple of the mean edge length");
        opt.value("--eps", reg.eps, "Convergence threshold on max point displacement");
        opt.value("--i-max", reg.i_max, "Max iterations per annealing stage");
        opt.value("--aa-window", reg.aa_window, "Anderson window size (0 disables)");
        opt.value("--knn", reg.knn, "Neighbors for point-cloud connectivity");
        opt.value("--seed", reg.seed, "Random seed (echoed into the report)");
        opt.flag("--binary-ply", reg.binary_ply, "Write binary PLY output");
        opt.flag("--error-channel", reg.error_channel, "Store per-vertex error in the output mesh (needs ground truth)");
        opt.value("--nu-a-init", reg.nu_a_init, "Override the initial alignment nu");
        opt.value("--nu-a-min", reg.nu_a_min, "Override the final alignment nu");
        opt.value("--nu-r-init", reg.nu_r_init, "Override the initial smoothness nu");
        opt.choice("--gt", gt_mode, {"none", "index", "flow"}, "Ground-truth mode: none, index, flow");
        opt.value("--flow-file", reg.flow_path, "Scene-flow ground-truth file");
        opt.value("--complete-target", reg.complete_target_path, "Uncropped target used as the index-identity reference");
        opt.value("--mask-file", reg.mask_path, "Target vertex membership mask for the overlap ratio");
        opt.value("--landmarks", reg.landmarks_path, "Fixed corresponding pairs, applied in the first stage");
    } else if (sub == "metrics") {  // nrr_cli.cpp:223-236
        opt.value("--deformed", met.deformed, "Deformed source mesh", true);
        opt.value("--gt-target", met.gt_target, "Index-identity ground-truth target mesh");
        opt.value("--source", met.source, "Undeformed source (for flow metrics)");
        opt.value("--flow-file", met.flow_file, "Scene-flow ground-truth file");
        opt.value("--mask", met.mask_file, "Target vertex membership mask");
        opt.value("--report", met.report, "JSON output path (stdout if omitted)");
        opt.value("--per-vertex-out", met.per_vertex_out, "Mesh output carrying the per-vertex error channel");
        opt.value("--knn", met.knn, "Neighbors for point-cloud connectivity");
    } else if (sub == "graph-dump") {  // nrr_cli.cpp:238-244
        opt.value("--in", gd.in, "Input mesh", true);
        opt.value("--out", gd.out, "JSON output path (stdout if omitted)");
        opt.value("--radius-mult", gd.radius_mult, "Sampling radius as a multiple of the mean edge length");
        opt.value("--knn", gd.knn, "Neighbors for point-cloud connectivity");
    } else if (sub == "synth-noise" || sub == "synth-crop") {
        emit_error("config", sub + " (synthetic test-case generation) is not part of this build", 4);
        return 4;
    } else {
        std::cerr << kTop;
        emit_error("config", "The following argument was not expected: " + sub, 4);
        return 4;
    }
    if (help) {
        std::cout << opt.usage();
        return 0;
    }
    try {
        opt.parse(args);
    } catch (const ParseError& e) {
        emit_error("config", e.what(), 4);
        return 4;
    }

    try {  // nrr_cli.cpp:254-278
        if (sub == "register") {
            if (gt_mode == "index") reg.gt_mode = nrr::GroundTruthMode::IndexIdentity;
            else if (gt_mode == "flow") reg.gt_mode = nrr::GroundTruthMode::Flow;
            nrr::run_pipeline(reg);
        } else if (sub == "metrics") {
            run_metrics(met);
        } else {
            run_graph_dump(gd);
        }
    } catch (const nrr::IoError& e) {
        emit_error("io", e.what(), 2);
        return 2;
    } catch (const nrr::ConfigError& e) {
        emit_error("config", e.what(), 4);
        return 4;
    } catch (const nrr::NumericalError& e) {
        emit_error("numerical", e.what(), 3);
        return 3;
    } catch (const std::exception& e) {
        emit_error("internal", e.what(), 3);
        return 3;
    }
    return 0;
}
