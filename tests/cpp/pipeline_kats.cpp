// Report / pipeline / mesh-file / metrics layer of the drop-in API (§8 f3, f4):
// re-derived from the reference's own tests (proj/tests/pipeline_tests.cpp,
// mesh_io_tests.cpp, metrics_tests.cpp; each TEST names what it restates).
// Cases named "cpu: ..." need no GPU (host I/O, JSON, metrics, validation);
// "gpu: ..." run the whole pipeline, i.e. the MM loop on the B200.
#include <array>
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <random>
#include <sstream>

#include "check.hpp"
#include "nrr/nrr.hpp"

using namespace nrr;

namespace {

std::filesystem::path tmp_dir() {
    const auto d = std::filesystem::temp_directory_path() / "nrr_b200_pipeline_kats";
    std::filesystem::create_directories(d);
    return d;
}
std::string tmp(const std::string& name) { return (tmp_dir() / name).string(); }
std::string write_text(const std::string& name, const std::string& body) {
    std::ofstream(tmp(name)) << body;
    return tmp(name);
}
std::string file_bytes(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    return {std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
}

// flat grid strip of nx x ny vertices over [0,len_x] x [0,len_y], two
// triangles per cell (the reference tests' helpers.hpp make_strip layout)
Surface strip(int nx, int ny, double len_x = 1.0, double len_y = 0.5) {
    std::vector<Vec3> p;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) p.emplace_back(len_x * i / (nx - 1), len_y * j / (ny - 1), 0.0);
    std::vector<std::array<int, 3>> f;
    for (int j = 0; j + 1 < ny; ++j)
        for (int i = 0; i + 1 < nx; ++i) {
            const int a = j * nx + i, b = a + 1, c = a + nx, d = c + 1;
            f.push_back({a, b, d});
            f.push_back({a, d, c});
        }
    return make_surface(std::move(p), std::move(f));
}

// smooth out-of-plane bend z = A sin(2 pi (f x + phase)) + tilt A sin(2 pi y)
Surface bent(const Surface& s, double amp, double freq, double phase, double tilt) {
    Surface o = s;
    for (auto& q : o.points)
        q = Vec3(q.x(), q.y(),
                 q.z() + amp * std::sin(2.0 * M_PI * (freq * q.x() + phase)) + tilt * amp * std::sin(2.0 * M_PI * q.y()));
    o.finalize_edges();
    return o;
}

Surface jittered(uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-0.2, 0.2);
    Surface s = strip(7, 4);
    for (auto& q : s.points) q += Vec3(u(rng), u(rng), u(rng));
    s.finalize_edges();
    return s;
}

}  // namespace

// ------------------------------------------------------------------ JSON format
TEST("cpu: json dump follows nlohmann's layout, key order and number format") {
    nlohmann::json j = nlohmann::json::object();
    j["b"] = 1.0;
    j["a"] = {1, 2.5, "x"};
    j["c"] = nlohmann::json::object();
    j["d"] = true;
    j["e"] = nlohmann::json::array();
    CHECK(j.dump() == "{\"a\":[1,2.5,\"x\"],\"b\":1.0,\"c\":{},\"d\":true,\"e\":[]}");
    CHECK(j.dump(2) == "{\n  \"a\": [\n    1,\n    2.5,\n    \"x\"\n  ],\n  \"b\": 1.0,\n  \"c\": {},\n  \"d\": true,\n"
                       "  \"e\": []\n}");
    CHECK(nlohmann::json(1e-5).dump() == "1e-05");
    CHECK(nlohmann::json(0.0001).dump() == "0.0001");
    CHECK(nlohmann::json(1e14).dump() == "100000000000000.0");
    CHECK(nlohmann::json(1e15).dump() == "1e+15");
    CHECK(nlohmann::json(1e16).dump() == "1e+16");
    CHECK(nlohmann::json(123456.789).dump() == "123456.789");
    CHECK(nlohmann::json(-0.1).dump() == "-0.1");
    CHECK(nlohmann::json(0.1 + 0.2).dump() == "0.30000000000000004");
    CHECK(nlohmann::json(2.5e-300).dump() == "2.5e-300");
    CHECK(nlohmann::json(std::nan("")).dump() == "null");
    CHECK(nlohmann::json(uint64_t(18446744073709551615ull)).dump() == "18446744073709551615");
    CHECK(nlohmann::json("q\"\\\n\t\x01").dump() == "\"q\\\"\\\\\\n\\t\\u0001\"");
    nlohmann::json o = {{"k", 1}, {"center", {0.5, 1.5, 2.5}}};
    CHECK(o.is_object() && o.at("center").is_array() && o.at("center").size() == 3);
    CHECK(o.contains("k") && !o.contains("z"));
    o.erase("k");
    CHECK(o.dump() == "{\"center\":[0.5,1.5,2.5]}");
    CHECK(o.at("center").at(1).get<double>() == 1.5);
    CHECK_THROWS_AS(o.at("missing"), std::exception);
}

TEST("cpu: report_to_json carries the reference schema (json_export.hpp:12-37)") {
    RegistrationReport r;
    StageRecord s;
    s.nu_a = 0.1;
    s.nu_r = 0.2;
    s.alpha = 3.0;
    s.beta = 4.0;
    s.reverts = 2;
    s.converged = true;
    IterationRecord it;
    it.e_total = 1.5;
    it.e_align = 1.0;
    it.e_reg = 0.25;
    it.e_rot = 0.25;
    it.e_landmark = 0.125;
    it.aa_accepted = true;
    it.max_disp = 1e-6;
    s.iterations = {it, it};
    r.stages = {s};
    r.degenerate_rotations = 1;
    const auto j = report_to_json(r);
    CHECK(j.at("total_iterations").get<int>() == 2);
    CHECK(j.at("degenerate_rotations").get<int>() == 1);
    CHECK(j.at("alpha_forced_zero").get<bool>() == false);
    const auto& i0 = j.at("stages").at(0).at("iterations").at(0);
    for (const char* k : {"E", "E_align", "E_reg", "E_rot", "aa_accepted", "max_disp"}) CHECK(i0.contains(k));
    CHECK(!i0.contains("E_landmark"));
    CHECK(report_to_json(r, true).at("stages").at(0).at("iterations").at(1).at("E_landmark").get<double>() == 0.125);
    CHECK(j.at("stages").at(0).dump() ==
          "{\"alpha\":3.0,\"beta\":4.0,\"converged\":true,\"iterations\":[{\"E\":1.5,\"E_align\":1.0,\"E_reg\":0.25,"
          "\"E_rot\":0.25,\"aa_accepted\":true,\"max_disp\":1e-06},{\"E\":1.5,\"E_align\":1.0,\"E_reg\":0.25,\"E_rot\":"
          "0.25,\"aa_accepted\":true,\"max_disp\":1e-06}],\"nu_a\":0.1,\"nu_r\":0.2,\"reverts\":2}");
}

TEST("cpu: graph_to_json dumps nodes, edges, influence and weights (json_export.hpp:41-69)") {
    const Surface s = strip(8, 5);
    const DeformationGraph g = build_graph(s, 3.0 * s.avg_edge_length);
    const auto j = graph_to_json(g);
    CHECK(j.at("node_indices").size() == static_cast<size_t>(g.node_count()));
    CHECK(j.at("node_positions").size() == static_cast<size_t>(g.node_count()));
    CHECK(j.at("edges").size() == static_cast<size_t>(g.edge_count()));
    CHECK(j.at("influence").size() == static_cast<size_t>(s.point_count()));
    CHECK(j.at("reg_weights").size() == static_cast<size_t>(g.directed_pair_count()));
    double csum = 0.0;
    for (size_t k = 0; k < j.at("reg_weights").size(); ++k) csum += j.at("reg_weights").at(k).at("c").get<double>();
    CHECK_APPROX(csum / g.directed_pair_count(), 1.0, 1e-12, 0.0);  // mean c is 1 (deformation_graph.hpp:146-147)
    for (size_t v = 0; v < j.at("influence").size(); ++v) {
        double w = 0.0;
        for (size_t k = 0; k < j.at("influence").at(v).size(); ++k)
            w += j.at("influence").at(v).at(k).at("weight").get<double>();
        CHECK_APPROX(w, 1.0, 1e-12, 0.0);
    }
    CHECK(j.at("radius").get<double>() == g.radius);
}

// ------------------------------------------------------------------ mesh files (mesh_io_tests.cpp)
TEST("cpu: obj minimal triangle, texture/normal indices and fan triangulation") {
    const Surface s = load_surface(write_text("tri.obj", "# comment\nv 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n"));
    CHECK(s.point_count() == 3 && s.faces.size() == 1 && s.edges.size() == 3);
    const Surface q = load_surface(write_text("quad.obj", "v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nf 1/1 2/2/2 3//3 4\n"));
    CHECK(q.point_count() == 4);
    CHECK(q.faces.size() == 2);
    CHECK((q.faces[0] == std::array<int, 3>{0, 1, 2}));
    CHECK((q.faces[1] == std::array<int, 3>{0, 2, 3}));
    CHECK(q.adjacency.size() == 4 && q.adjacency[0].size() == 3);
}

TEST("cpu: obj malformed records report the line") {
    CHECK_THROWS_WITH(load_surface(write_text("bad_v.obj", "v 0 0 0\nv 1 2\n")), IoError, ":2:");
    CHECK_THROWS_WITH(load_surface(write_text("bad_f.obj", "v 0 0 0\nv 1 0 0\nf 1 2 5\n")), IoError, "out of range");
    CHECK_THROWS_WITH(load_surface(write_text("bad_t.obj", "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 x 3\n")), IoError, ":4:");
}

TEST("cpu: ply ascii point cloud falls back to kNN connectivity; unknown properties skipped") {
    std::string body = "ply\nformat ascii 1.0\nelement vertex 10\nproperty float x\nproperty float y\nproperty float z\n"
                       "end_header\n";
    std::mt19937_64 rng(5);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    for (int i = 0; i < 10; ++i) body += std::to_string(u(rng)) + " " + std::to_string(u(rng)) + " " + std::to_string(u(rng)) + "\n";
    const Surface s = load_surface(write_text("cloud.ply", body));
    CHECK(s.point_count() == 10 && s.faces.empty() && !s.edges.empty());
    std::vector<int> deg(10, 0);
    for (const auto& [a, b] : s.edges) ++deg[a], ++deg[b];
    for (int d : deg) CHECK(d >= 6);
    const Surface e = load_surface(write_text("extra.ply", "ply\nformat ascii 1.0\nelement vertex 2\nproperty float x\n"
                                                          "property float y\nproperty float z\nproperty float confidence\n"
                                                          "end_header\n1 2 3 0.5\n4 5 6 0.25\n"),
                                   1);
    CHECK(e.point_count() == 2 && e.points[0] == Vec3(1, 2, 3) && e.points[1] == Vec3(4, 5, 6));
}

TEST("cpu: obj and ply (ascii, binary) round trips are bitwise") {
    const Surface m = jittered(11);
    for (const char* name : {"rt.obj", "rt_a.ply", "rt_b.ply"}) {
        SaveOptions o;
        o.binary_ply = std::string(name) == "rt_b.ply";
        save_surface(m, tmp(name), {}, o);
        const Surface b = load_surface(tmp(name));
        CHECK(b.point_count() == m.point_count());
        CHECK(b.faces == m.faces);
        for (int i = 0; i < m.point_count(); ++i) CHECK(b.points[i] == m.points[i]);
    }
}

TEST("cpu: scalar channels (ply quality, obj colours) and write errors") {
    const Surface m = jittered(13);
    std::vector<double> q(m.point_count());
    for (int i = 0; i < m.point_count(); ++i) q[i] = 0.01 * i;
    save_surface(m, tmp("quality.ply"), q);
    CHECK(file_bytes(tmp("quality.ply")).find("property double quality") != std::string::npos);
    CHECK(load_surface(tmp("quality.ply")).point_count() == m.point_count());
    std::vector<double> err(m.point_count(), 0.0);
    err.back() = 1.0;
    save_surface(m, tmp("colored.obj"), err);
    std::ifstream in(tmp("colored.obj"));
    std::string line, tag;
    std::getline(in, line);
    std::istringstream ls(line);
    ls >> tag;
    int fields = 0;
    for (double v; ls >> v;) ++fields;
    CHECK(fields == 6);
    CHECK_THROWS_AS(save_surface(m, tmp("bad.ply"), {1.0, 2.0}), ConfigError);
    CHECK_THROWS_AS(load_surface(tmp("mesh.stl")), IoError);
    CHECK_THROWS_AS(load_surface(tmp("does_not_exist.obj")), IoError);
    CHECK_THROWS_AS(save_surface(m, tmp("mesh.stl")), IoError);
}

TEST("cpu: ply binary mixed types, big-endian rejected, CR headers, truncation offset") {
    {
        std::ofstream out(tmp("mixed.ply"), std::ios::binary);
        out << "ply\nformat binary_little_endian 1.0\nelement vertex 3\nproperty float x\nproperty float y\n"
               "property float z\nelement face 1\nproperty list uchar int vertex_indices\nend_header\n";
        const float c[9] = {0, 0, 0, 1, 0, 0, 0, 1, 0};
        out.write(reinterpret_cast<const char*>(c), sizeof c);
        const uint8_t cnt = 3;
        const int32_t idx[3] = {0, 1, 2};
        out.write(reinterpret_cast<const char*>(&cnt), 1);
        out.write(reinterpret_cast<const char*>(idx), sizeof idx);
    }
    const Surface s = load_surface(tmp("mixed.ply"));
    CHECK(s.point_count() == 3 && s.faces.size() == 1);
    CHECK_THROWS_WITH(load_surface(write_text("be.ply", "ply\nformat binary_big_endian 1.0\nelement vertex 0\nend_header\n")),
                      IoError, "unsupported PLY format");
    const Surface cr = load_surface(write_text("crlf.ply", "ply\r\nformat ascii 1.0\r\nelement vertex 1\r\nproperty float x\r\n"
                                                           "property float y\r\nproperty float z\r\nend_header\r\n1 2 3\r\n"),
                                    1);
    CHECK(cr.point_count() == 1 && cr.points[0] == Vec3(1, 2, 3));
    {
        std::ofstream out(tmp("trunc.ply"), std::ios::binary);
        out << "ply\nformat binary_little_endian 1.0\nelement vertex 2\nproperty double x\nproperty double y\n"
               "property double z\nend_header\n";
        const double one = 1.0;
        out.write(reinterpret_cast<const char*>(&one), 8);
    }
    CHECK_THROWS_WITH(load_surface(tmp("trunc.ply")), IoError, "offset");
}

// ------------------------------------------------------------------ metrics (metrics_tests.cpp)
TEST("cpu: pointwise error, rmse, scene-flow rmse, overlap ratio") {
    const std::vector<Vec3> a{Vec3(1, 2, 3), Vec3(4, 5, 6)};
    CHECK(pointwise_error(a, a) == (std::vector<double>{0.0, 0.0}));
    const std::vector<Vec3> mv{Vec3(1, 2.75, 4), Vec3(4, 5, 6)};
    CHECK_APPROX(pointwise_error(mv, a)[0], 1.25, 1e-15, 0.0);
    CHECK_THROWS_AS(pointwise_error({Vec3(0, 0, 0)}, a), NumericalError);
    CHECK(rmse({0.0, 0.0, 0.0}) == 0.0);
    CHECK_APPROX(rmse({3.0, 4.0}), 3.5355339059327378, 1e-15, 0.0);
    CHECK_APPROX(rmse({0.7, 0.7, 0.7, 0.7}), 0.7, 1e-15, 0.0);
    CHECK_THROWS_AS(rmse({}), NumericalError);
    const std::vector<Vec3> src{Vec3(0, 0, 0), Vec3(1, 0, 0)};
    CHECK(scene_flow_rmse(src, src, {{0, Vec3(0, 0, 0)}, {1, Vec3(0, 0, 0)}}) == 0.0);
    CHECK_APPROX(scene_flow_rmse(src, src, {{0, Vec3(1, 0, 0)}}), 1.0, 1e-15, 0.0);
    CHECK_THROWS_AS(scene_flow_rmse(src, src, {}), NumericalError);
    CHECK_THROWS_AS(scene_flow_rmse(src, src, {{5, Vec3(0, 0, 0)}}), NumericalError);
    CHECK(overlap_ratio(std::vector<char>{1, 1, 1, 1}, 4) == 1.0);
    CHECK(overlap_ratio(std::vector<char>{1, 1, 0, 0}, 4) == 0.5);
    CHECK_APPROX(overlap_ratio(std::vector<char>{0, 1, 1, 1}, std::vector<int>{3, 3, 0}), 2.0 / 3.0, 1e-15, 0.0);
    CHECK_THROWS_AS(overlap_ratio(std::vector<char>{1}, std::vector<int>{2}), NumericalError);
}

// ------------------------------------------------------------------ record files / config (pipeline_tests.cpp)
TEST("cpu: flow / landmark / mask files and RunConfig validation") {
    CHECK_THROWS_WITH(read_flow_file(write_text("bad.flow", "0 0 0 0\n1 nope 0 0\n")), IoError, ":2:");
    const auto fl = read_flow_file(write_text("ok.flow", "# c\n\n3 0.5 0 -1\n"));
    CHECK(fl.size() == 1 && fl[0].index == 3 && fl[0].flow == Vec3(0.5, 0, -1));
    CHECK_THROWS_WITH(read_flow_file(write_text("neg.flow", "-1 0 0 0\n")), IoError, "negative flow index");
    const auto lm = read_landmark_file(write_text("ok.landmarks", "0 1\n# x\n5 7\n"));
    CHECK(lm.size() == 2 && lm[1] == std::make_pair(5, 7));
    CHECK_THROWS_WITH(read_landmark_file(write_text("bad.landmarks", "0\n")), IoError, ":1:");
    std::vector<char> mask{1, 0, 1, 1};
    write_mask_file(tmp("m.mask"), mask);
    CHECK(read_mask_file(tmp("m.mask")) == mask);
    CHECK_THROWS_AS(read_mask_file(tmp("none.mask")), IoError);
    RunConfig cfg;
    CHECK_THROWS_AS(cfg.validate(), ConfigError);
    cfg.source_path = "a.obj";
    cfg.target_path = "b.obj";
    cfg.output_path = "c.obj";
    cfg.radius_multiplier = 0.0;
    CHECK_THROWS_AS(cfg.validate(), ConfigError);
    cfg.radius_multiplier = 5.0;
    cfg.gt_mode = GroundTruthMode::Flow;
    CHECK_THROWS_AS(cfg.validate(), ConfigError);
    cfg.gt_mode = GroundTruthMode::None;
    cfg.i_max = 0;
    CHECK_THROWS_AS(cfg.validate(), ConfigError);
    cfg.i_max = 10;
    cfg.validate();
    CHECK_THROWS_AS(run_pipeline(cfg), IoError);  // a.obj does not exist
}

// ------------------------------------------------------------------ the pipeline on the GPU (pipeline_tests.cpp)
TEST("gpu: identity pair registers with near-zero error; error channel; report schema") {
    const Surface s = strip(12, 6);
    save_surface(s, tmp("ident_src.obj"));
    save_surface(s, tmp("ident_tgt.obj"));
    RunConfig cfg;
    cfg.source_path = tmp("ident_src.obj");
    cfg.target_path = tmp("ident_tgt.obj");
    cfg.output_path = tmp("ident_out.obj");
    cfg.report_path = tmp("ident_report.json");
    cfg.gt_mode = GroundTruthMode::IndexIdentity;
    cfg.error_channel = true;
    const PipelineResult r = run_pipeline(cfg);
    CHECK(r.document.at("metrics").at("rmse").get<double>() < 1e-6);
    CHECK(std::filesystem::exists(cfg.output_path) && std::filesystem::exists(cfg.report_path));
    std::ifstream mesh(cfg.output_path);
    std::string first, tag;
    std::getline(mesh, first);
    std::istringstream ls(first);
    ls >> tag;
    int fields = 0;
    for (double v; ls >> v;) ++fields;
    CHECK(fields == 6);
    const auto& st = r.document.at("stages");
    CHECK(st.is_array() && !st.empty());
    const auto& it0 = st.at(0).at("iterations").at(0);
    for (const char* k : {"E", "E_align", "E_reg", "E_rot", "aa_accepted", "max_disp"}) CHECK(it0.contains(k));
    // the report file is the document, dumped with indent 2
    CHECK(file_bytes(cfg.report_path) == r.document.dump(2) + "\n");
    for (const char* k : {"config", "graph", "normalization", "solver", "timings"}) CHECK(r.document.contains(k));
    CHECK(r.document.at("solver").at("total_iterations").get<int>() == r.registration.report.total_iterations());
}

TEST("gpu: runs are byte-identical apart from timings") {
    const Surface src = strip(14, 7);
    const Surface tgt = bent(src, 0.06, 0.9, 0.3, 0.2);
    save_surface(src, tmp("det_src.obj"));
    save_surface(tgt, tmp("det_tgt.obj"));
    auto once = [&](const std::string& tag) {
        RunConfig cfg;
        cfg.source_path = tmp("det_src.obj");
        cfg.target_path = tmp("det_tgt.obj");
        cfg.output_path = tmp("det_out_" + tag + ".obj");
        cfg.report_path = tmp("det_rep_" + tag + ".json");
        cfg.gt_mode = GroundTruthMode::IndexIdentity;
        cfg.seed = 7;
        return run_pipeline(cfg);
    };
    const PipelineResult a = once("a"), b = once("b");
    CHECK(file_bytes(tmp("det_out_a.obj")) == file_bytes(tmp("det_out_b.obj")));
    nlohmann::json da = a.document, db = b.document;
    for (auto* d : {&da, &db}) {
        d->erase("timings");
        d->erase("config");
    }
    CHECK(da.dump() == db.dump());
    CHECK(a.document.at("config").at("seed").get<uint64_t>() == 7);
}

TEST("gpu: normalization round trip matches the saved result") {
    const Surface src = strip(10, 5);
    save_surface(src, tmp("norm_src.obj"));
    save_surface(bent(src, 0.05, 1.1, 0.1, 0.1), tmp("norm_tgt.obj"));
    RunConfig cfg;
    cfg.source_path = tmp("norm_src.obj");
    cfg.target_path = tmp("norm_tgt.obj");
    cfg.output_path = tmp("norm_out.obj");
    const PipelineResult r = run_pipeline(cfg);
    Normalization nz;
    nz.scale = r.document.at("normalization").at("scale").get<double>();
    const auto& c = r.document.at("normalization").at("center");
    nz.center = Vec3(c.at(0).get<double>(), c.at(1).get<double>(), c.at(2).get<double>());
    double worst = 0.0;
    for (size_t i = 0; i < r.deformed_original_units.size(); ++i)
        worst = std::max(worst, (nz.apply(r.deformed_original_units[i]) - r.registration.deformed_points[i]).norm());
    CHECK(worst < 1e-12);
    CHECK(!r.document.contains("metrics"));
}

TEST("gpu: point clouds register through kNN connectivity") {
    const Surface s = strip(30, 15);
    const Surface w = bent(s, 0.05, 0.7, 0.3, 0.2);
    save_surface(make_surface(s.points, {}, 6), tmp("cloud_src.ply"));
    save_surface(make_surface(w.points, {}, 6), tmp("cloud_tgt.ply"));
    RunConfig cfg;
    cfg.source_path = tmp("cloud_src.ply");
    cfg.target_path = tmp("cloud_tgt.ply");
    cfg.output_path = tmp("cloud_out.ply");
    cfg.gt_mode = GroundTruthMode::IndexIdentity;
    cfg.k_alpha = 1.0;
    cfg.k_beta = 0.1;
    const PipelineResult r = run_pipeline(cfg);
    CHECK(r.document.at("metrics").at("rmse").get<double>() < 0.02);
    CHECK(r.document.at("graph").at("node_count").get<int>() > 1);
}

TEST("gpu: flow ground truth, mask overlap, landmarks (E_landmark) and a bad landmark index") {
    const Surface s = strip(8, 4);
    save_surface(s, tmp("flow_src.obj"));
    RunConfig cfg;
    cfg.source_path = tmp("flow_src.obj");
    cfg.target_path = tmp("flow_src.obj");
    cfg.output_path = tmp("flow_out.obj");
    cfg.gt_mode = GroundTruthMode::Flow;
    cfg.flow_path = write_text("zero.flow", "# zero flows on three points\n0 0 0 0\n5 0 0 0\n7 0 0 0\n");
    CHECK(run_pipeline(cfg).document.at("metrics").at("rs").get<double>() < 1e-6);

    std::vector<char> mask(s.point_count(), 0);
    for (int i = 0; i < s.point_count() / 2; ++i) mask[i] = 1;
    write_mask_file(tmp("half.mask"), mask);
    RunConfig mc;
    mc.source_path = mc.target_path = tmp("flow_src.obj");
    mc.output_path = tmp("mask_out.obj");
    mc.mask_path = tmp("half.mask");
    CHECK_APPROX(run_pipeline(mc).document.at("metrics").at("overlap").get<double>(), 0.5, 1e-15, 0.0);

    RunConfig lc = mc;
    lc.mask_path.clear();
    lc.output_path = tmp("lm_out.obj");
    lc.landmarks_path = write_text("ok.lm", "0 0\n3 3\n");
    const PipelineResult lr = run_pipeline(lc);
    CHECK(lr.document.at("stages").at(0).at("iterations").at(0).contains("E_landmark"));
    lc.landmarks_path = write_text("bad.lm", "0 0\n999 0\n");
    CHECK_THROWS_AS(run_pipeline(lc), ConfigError);
}

KAT_MAIN
