// Pins the CPU oracle (oracle/nrr_oracle.hpp) against the known-answer tests
// and properties of the reference test suite (/root/reference/proj/tests).
// Every TEST names the reference test it re-derives (file:line). The fixtures
// are regenerated with the same seeds and libstdc++ distributions.
#include <random>
#include <set>

#include "../../oracle/nrr_oracle.hpp"
#include "check.hpp"

using namespace oracle;

namespace {

// ------------------------------------------------------------ independent oracles
// helpers.hpp:25-37 brute-force NN (first index wins ties)
std::pair<int, double> brute_force_nearest(const std::vector<Vec3>& pts, const Vec3& q) {
    int best = -1;
    double bd2 = std::numeric_limits<double>::infinity();
    for (size_t i = 0; i < pts.size(); ++i) {
        const double d2 = (pts[i] - q).squaredNorm();
        if (d2 < bd2) {
            bd2 = d2;
            best = static_cast<int>(i);
        }
    }
    return {best, std::sqrt(bd2)};
}

Surface surface_from_edges(std::vector<Vec3> pts, std::vector<std::pair<int, int>> edges) {
    Surface s;
    s.points = std::move(pts);
    s.edges = std::move(edges);
    s.finalize_edges();
    return s;
}

Vec3 deform_one(const std::vector<Vec3>& src, const DeformationGraph& g, const NodeTransforms& x, int i) {
    Vec3 v;
    for (const auto& e : g.influence[i]) {
        const Vec3& p = g.node_positions[e.node];
        v += e.weight * (x.affine(e.node) * (src[i] - p) + p + x.translation(e.node));
    }
    return v;
}
Vec3 reg_diff(const DeformationGraph& g, const NodeTransforms& t, size_t k) {
    const auto [i, j] = g.reg_pairs[k];
    return g.reg_weights[k] * (t.affine(j) * (g.node_positions[i] - g.node_positions[j]) +
                               g.node_positions[j] + t.translation(j) - g.node_positions[i] - t.translation(i));
}

// helpers.hpp:211-240
double scalar_energy(const std::vector<Vec3>& src, const DeformationGraph& g, const NodeTransforms& x,
                     const std::vector<Vec3>& cp, const std::vector<Mat3>& rot, double alpha, double beta,
                     double nu_a, double nu_r) {
    auto psi = [](double v, double nu) { return 1.0 - std::exp(-v * v / (2.0 * nu * nu)); };
    double ea = 0, er = 0, et = 0;
    for (size_t i = 0; i < src.size(); ++i) ea += psi((deform_one(src, g, x, i) - cp[i]).norm(), nu_a);
    for (size_t k = 0; k < g.reg_pairs.size(); ++k) er += psi(reg_diff(g, x, k).norm(), nu_r);
    for (int j = 0; j < g.node_count(); ++j) et += frob2_diff(x.affine(j), rot[j]);
    return ea + alpha * er + beta * et;
}

// helpers.hpp:244-283 (constants dropped)
double surrogate_dropped(const std::vector<Vec3>& src, const DeformationGraph& g, const NodeTransforms& x,
                         const NodeTransforms& anchor, const std::vector<Vec3>& cp,
                         const std::vector<Mat3>& arot, double alpha, double beta, double nu_a,
                         double nu_r) {
    double total = 0;
    for (size_t i = 0; i < src.size(); ++i) {
        const double r2 = (deform_one(src, g, anchor, i) - cp[i]).squaredNorm();
        const double w = std::exp(-r2 / (2 * nu_a * nu_a)) / (2 * nu_a * nu_a);
        total += w * (deform_one(src, g, x, i) - cp[i]).squaredNorm();
    }
    for (size_t k = 0; k < g.reg_pairs.size(); ++k) {
        const double d2 = reg_diff(g, anchor, k).squaredNorm();
        const double w = std::exp(-d2 / (2 * nu_r * nu_r)) / (2 * nu_r * nu_r);
        total += alpha * w * reg_diff(g, x, k).squaredNorm();
    }
    for (int j = 0; j < g.node_count(); ++j) total += beta * frob2_diff(x.affine(j), arot[j]);
    return total;
}
// helpers.hpp:288-321
double surrogate_constant(const std::vector<Vec3>& src, const DeformationGraph& g, const NodeTransforms& anchor,
                          const std::vector<Vec3>& cp, double alpha, double nu_a, double nu_r) {
    auto psi = [](double v2, double nu) { return 1.0 - std::exp(-v2 / (2.0 * nu * nu)); };
    double c = 0;
    for (size_t i = 0; i < src.size(); ++i) {
        const double r2 = (deform_one(src, g, anchor, i) - cp[i]).squaredNorm();
        const double w = std::exp(-r2 / (2 * nu_a * nu_a)) / (2 * nu_a * nu_a);
        c += psi(r2, nu_a) - w * r2;
    }
    for (size_t k = 0; k < g.reg_pairs.size(); ++k) {
        const double d2 = reg_diff(g, anchor, k).squaredNorm();
        const double w = std::exp(-d2 / (2 * nu_r * nu_r)) / (2 * nu_r * nu_r);
        c += alpha * (psi(d2, nu_r) - w * d2);
    }
    return c;
}

// robust_energy_tests.cpp:12-45
struct Instance {
    Surface source, target;
    DeformationGraph graph;
    NodeTransforms anchor;
    Correspondences corr;
    std::vector<Mat3> rotations;
    EnergyParams prm;
};
Instance make_instance(uint64_t seed, double perturb = 0.15) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    Instance in;
    in.source = make_strip(10, 5);
    in.target = warped_copy(in.source, random_warp(rng));
    in.graph = build_graph(in.source, 4.0 * in.source.avg_edge_length);
    in.anchor = NodeTransforms::identity(in.graph.node_count());
    for (int j = 0; j < in.graph.node_count(); ++j) {
        Mat3 a = Mat3::identity();
        for (int k = 0; k < 9; ++k) a(k / 3, k % 3) += perturb * uni(rng);
        const Vec3 t = 0.1 * Vec3(uni(rng), uni(rng), uni(rng));
        in.anchor.set(j, a, t);
    }
    const SpatialIndex idx(in.target.points);
    in.corr = find_correspondences(deform_points(in.source.points, in.graph, in.anchor), idx);
    in.rotations = project_rotations(in.anchor);
    in.prm = {0.8, 1.7, 0.09, 0.12};
    return in;
}
// robust_energy_tests.cpp:47-57
NodeTransforms random_transforms(int nodes, uint64_t seed, double scale = 0.3) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    NodeTransforms x = NodeTransforms::identity(nodes);
    for (int j = 0; j < nodes; ++j) {
        Mat3 a = Mat3::identity();
        for (int k = 0; k < 9; ++k) a(k / 3, k % 3) += scale * uni(rng);
        x.set(j, a, scale * Vec3(uni(rng), uni(rng), uni(rng)));
    }
    return x;
}
// robust_energy_tests.cpp:59-63: tr(X^T K X) - 2 tr(B^T X)
double quadratic_form(const LinearSystem& s, const NodeTransforms& x) {
    const auto kx = s.K.multiply(x.stacked);
    double a = 0, b = 0;
    for (size_t i = 0; i < kx.size(); ++i) {
        a += x.stacked[i] * kx[i];
        b += s.B[i] * x.stacked[i];
    }
    return a - 2.0 * b;
}
LinearSystem assemble_system(const NodeTransforms& x, const Surface& src, const DeformationGraph& g,
                             const Correspondences& corr, const std::vector<Mat3>& rot, const EnergyParams& p) {
    SystemAssembler as(src.points, g);
    as.fill(corr, rot, alignment_weights(corr, p.nu_a), regularization_weights(g, x, p.nu_r, p.alpha), p.beta);
    return as.system();
}
double max_abs_diff(const Mat3& a, const Mat3& b) {
    double m = 0;
    for (int k = 0; k < 9; ++k) m = std::max(m, std::abs(a.m[k] - b.m[k]));
    return m;
}
double ortho_err(const Mat3& r) {
    const Mat3 p = r * r.transpose();
    return max_abs_diff(p, Mat3::identity());
}
double frob(const Mat3& a, const Mat3& b) { return std::sqrt(frob2_diff(a, b)); }
double rmse_pts(const std::vector<Vec3>& a, const std::vector<Vec3>& b) {
    double s = 0;
    for (size_t i = 0; i < a.size(); ++i) s += (a[i] - b[i]).squaredNorm();
    return std::sqrt(s / static_cast<double>(a.size()));
}

// linear contraction with spectral radius `radius` (solver_tests.cpp:11-18
// scales by the largest eigenvalue modulus). Without Eigen's eigensolver the
// spectral radius is taken as lim ||A^(2^p)||^(1/2^p) by repeated squaring.
double spectral_radius(const std::vector<double>& a, int dim) {
    std::vector<double> b(a), t(dim * dim);
    double logscale = 0.0;
    for (int p = 0; p < 40; ++p) {
        for (int i = 0; i < dim; ++i)
            for (int j = 0; j < dim; ++j) {
                double s = 0;
                for (int k = 0; k < dim; ++k) s += b[i * dim + k] * b[k * dim + j];
                t[i * dim + j] = s;
            }
        double nrm = 0;
        for (double x : t) nrm += x * x;
        nrm = std::sqrt(nrm);
        for (int i = 0; i < dim * dim; ++i) b[i] = t[i] / nrm;
        logscale = 2.0 * logscale + std::log(nrm);
    }
    return std::exp(logscale / std::ldexp(1.0, 40));
}
std::vector<double> random_contraction(std::mt19937_64& rng, int dim, double radius) {
    std::normal_distribution<double> gauss(0.0, 1.0);
    std::vector<double> a(dim * dim);
    for (int i = 0; i < dim; ++i)
        for (int j = 0; j < dim; ++j) a[i * dim + j] = gauss(rng);
    const double rho = spectral_radius(a, dim);
    for (auto& x : a) x *= radius / rho;
    return a;
}
std::vector<double> solve_dense(std::vector<double> a, int n, std::vector<double> b) {
    for (int k = 0; k < n; ++k) {
        int p = k;
        for (int i = k + 1; i < n; ++i)
            if (std::abs(a[i * n + k]) > std::abs(a[p * n + k])) p = i;
        for (int j = 0; j < n; ++j) std::swap(a[k * n + j], a[p * n + j]);
        std::swap(b[k], b[p]);
        for (int i = k + 1; i < n; ++i) {
            const double l = a[i * n + k] / a[k * n + k];
            for (int j = k; j < n; ++j) a[i * n + j] -= l * a[k * n + j];
            b[i] -= l * b[k];
        }
    }
    std::vector<double> x(n);
    for (int i = n - 1; i >= 0; --i) {
        double s = b[i];
        for (int j = i + 1; j < n; ++j) s -= a[i * n + j] * x[j];
        x[i] = s / a[i * n + i];
    }
    return x;
}
double inf_norm_diff(const std::vector<double>& a, const std::vector<double>& b) {
    double m = 0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}

}  // namespace

// =========================================================================== welsch
TEST("welsch: declared values and bound (robust_energy_tests.cpp:67-78)") {
    CHECK(welsch(0.0, 0.5) == 0.0);
    CHECK_APPROX(welsch(1.0, 1.0), 0.393469, 0, 1e-6);
    CHECK_APPROX(welsch(10.0, 1.0), 1.0, 0, 1e-9);
    double prev = -1.0;
    for (int k = 0; k <= 50; ++k) {
        const double v = welsch(0.1 * k, 0.7);
        CHECK(v > prev);
        CHECK(v < 1.0);
        prev = v;
    }
}
TEST("welsch surrogate: touch point and value 0.090204 (robust_energy_tests.cpp:80-83)") {
    for (double y : {0.0, 0.3, 1.7}) CHECK(welsch_surrogate(y, y, 0.8) == welsch(y, 0.8));
    CHECK_APPROX(welsch_surrogate(0.0, 1.0, 1.0), 0.090204, 0, 1e-6);
}
TEST("welsch surrogate dominates, 1000 samples seed 42 (robust_energy_tests.cpp:85-94)") {
    std::mt19937_64 rng(42);
    std::uniform_real_distribution<double> uni(0.0, 3.0), nud(0.05, 2.0);
    for (int k = 0; k < 1000; ++k) {
        const double x = uni(rng), y = uni(rng), nu = nud(rng);
        CHECK(welsch_surrogate(x, y, nu) >= welsch(x, nu) - 1e-15);
        CHECK(std::abs(welsch_surrogate(y, y, nu) - welsch(y, nu)) < 1e-12);
    }
}
TEST("acceptance 1: majorization on 1e4 triples (acceptance_main.cpp:77-95)") {
    std::mt19937_64 rng(11);
    std::uniform_real_distribution<double> arg(0.0, 4.0), nud(0.02, 2.5);
    int bad = 0;
    double gap = 0;
    for (int k = 0; k < 10000; ++k) {
        const double x = arg(rng), y = arg(rng), nu = nud(rng);
        if (welsch_surrogate(x, y, nu) < welsch(x, nu)) ++bad;
        gap = std::max(gap, std::abs(welsch_surrogate(y, y, nu) - welsch(y, nu)));
    }
    CHECK(bad == 0);
    CHECK(gap < 1e-12);
}

// ============================================================== spatial index / NN
TEST("NN: single point, distance sqrt(75) (geometry_core_tests.cpp:11-16)") {
    SpatialIndex idx({Vec3(0, 0, 0)});
    const auto h = idx.nearest(Vec3(5, 5, 5));
    CHECK(h.index == 0);
    CHECK_APPROX(h.distance, std::sqrt(75.0), 1e-12, 0);
}
TEST("NN: nearer of two (geometry_core_tests.cpp:18-21)") {
    SpatialIndex idx({Vec3(0, 0, 0), Vec3(1, 0, 0)});
    CHECK(idx.nearest(Vec3(0.4, 0, 0)).index == 0);
}
TEST("NN: query on an indexed point, idx 17 dist 0 (geometry_core_tests.cpp:23-30)") {
    std::mt19937_64 rng(11);
    const auto pts = random_points(rng, 64);
    SpatialIndex idx(pts);
    const auto h = idx.nearest(pts[17]);
    CHECK(h.index == 17);
    CHECK(h.distance == 0.0);
}
TEST("NN: equidistant -> smallest index, both tree sides (geometry_core_tests.cpp:32-44)") {
    std::vector<Vec3> pts(10, Vec3(5, 5, 5));
    pts[3] = Vec3(1, 2, 0);
    pts[7] = Vec3(-1, -2, 0);
    CHECK(SpatialIndex(pts).nearest(Vec3(0, 0, 0)).index == 3);
    std::swap(pts[3], pts[7]);
    CHECK(SpatialIndex(pts).nearest(Vec3(0, 0, 0)).index == 3);
}
TEST("NN: matches exhaustive scan n in {10,200,2000,10000} seed 2024 (geometry_core_tests.cpp:46-60)") {
    std::mt19937_64 rng(2024);
    for (int n : {10, 200, 2000, 10000}) {
        const auto pts = random_points(rng, n);
        SpatialIndex idx(pts);
        const int queries = n == 10000 ? 200 : 50;
        for (int q = 0; q < queries; ++q) {
            const Vec3 qq = random_points(rng, 1, 1.2)[0];
            const auto [bi, bd] = brute_force_nearest(pts, qq);
            const auto h = idx.nearest(qq);
            CHECK(h.index == bi);
            CHECK(h.distance == bd);
        }
    }
}
TEST("NN: empty input throws (geometry_core_tests.cpp:62-64)") {
    CHECK_THROWS_AS(SpatialIndex(std::vector<Vec3>{}), NumericalError);
}
TEST("correspondences: exact vs brute force, seed 3 (robust_energy_tests.cpp:96-108)") {
    std::mt19937_64 rng(3);
    const auto targets = random_points(rng, 120);
    const auto queries = random_points(rng, 60);
    const SpatialIndex idx(targets);
    const Correspondences c = find_correspondences(queries, idx);
    for (size_t i = 0; i < queries.size(); ++i) {
        const auto [bi, bd] = brute_force_nearest(targets, queries[i]);
        CHECK(c.target_index[i] == bi);
        CHECK_APPROX(c.squared_distance[i], bd * bd, 0, 1e-15);
        CHECK((c.target_point[i] - targets[bi]).squaredNorm() == 0.0);
    }
}

// ========================================================================= rotation
TEST("rotation projection: I, diag(2,1,.5), 3*R90 (geometry_core_tests.cpp:172-181)") {
    CHECK(max_abs_diff(project_to_rotation(Mat3::identity()), Mat3::identity()) < 1e-12);
    Mat3 d;
    d(0, 0) = 2.0;
    d(1, 1) = 1.0;
    d(2, 2) = 0.5;
    CHECK(max_abs_diff(project_to_rotation(d), Mat3::identity()) < 1e-12);
    Mat3 r90;
    r90(0, 1) = -1;
    r90(1, 0) = 1;
    r90(2, 2) = 1;
    Mat3 s3 = r90;
    for (double& v : s3.m) v *= 3.0;
    CHECK(max_abs_diff(project_to_rotation(s3), r90) < 1e-12);
}
TEST("rotation projection: fixed point and minimality, seed 31 (geometry_core_tests.cpp:183-200)") {
    std::mt19937_64 rng(31);
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (int t = 0; t < 100; ++t) {
        const Mat3 r = random_rotation(rng);
        CHECK(max_abs_diff(project_to_rotation(r), r) < 1e-9);
    }
    for (int t = 0; t < 30; ++t) {
        Mat3 a;
        for (int i = 0; i < 9; ++i) a(i / 3, i % 3) = gauss(rng);
        const Mat3 p = project_to_rotation(a);
        CHECK(ortho_err(p) < 1e-9);
        CHECK(p.determinant() > 0.0);
        const double best = frob(a, p);
        for (int q = 0; q < 100; ++q) CHECK(best <= frob(a, random_rotation(rng)) + 1e-12);
    }
}
TEST("rotation projection: NaN throws (geometry_core_tests.cpp:202-206)") {
    Mat3 bad = Mat3::identity();
    bad(1, 1) = std::numeric_limits<double>::quiet_NaN();
    CHECK_THROWS_AS(project_to_rotation(bad), NumericalError);
}
TEST("acceptance 7: 1e4 random matrices, seed 707 (acceptance_main.cpp:301-331)") {
    std::mt19937_64 rng(707);
    std::normal_distribution<double> gauss(0.0, 1.0);
    double worst = 0;
    bool det_ok = true, min_ok = true;
    for (int k = 0; k < 10000; ++k) {
        Mat3 a;
        for (int i = 0; i < 9; ++i) a(i / 3, i % 3) = gauss(rng);
        const Mat3 r = project_to_rotation(a);
        worst = std::max(worst, ortho_err(r));
        if (r.determinant() <= 0) det_ok = false;
        const double best = frob(a, r);
        for (int q = 0; q < 20; ++q)
            if (best > frob(a, random_rotation(rng)) + 1e-12) min_ok = false;
    }
    CHECK(det_ok);
    CHECK(min_ok);
    CHECK(worst <= 1e-9);
}
TEST("rotation projections: degenerate count = 1 (robust_energy_tests.cpp:170-183)") {
    NodeTransforms x = NodeTransforms::identity(3);
    Mat3 rank1;
    rank1(0, 0) = 2.0;
    x.set(1, rank1, Vec3());
    int deg = 0;
    const auto rot = project_rotations(x, &deg);
    CHECK(deg == 1);
    CHECK(rot.size() == 3);
    for (const auto& r : rot) {
        CHECK(ortho_err(r) < 1e-9);
        CHECK(r.determinant() > 0.0);
    }
}

// ====================================================================== deformation
TEST("deform: identity reproduces points (deformation_graph_tests.cpp:227-234)") {
    Surface strip = make_strip(12, 6);
    const DeformationGraph g = build_graph(strip, 5.0 * strip.avg_edge_length);
    const auto d = deform_points(strip.points, g, NodeTransforms::identity(g.node_count()));
    for (int i = 0; i < strip.point_count(); ++i) CHECK((d[i] - strip.points[i]).norm() < 1e-14);
}
TEST("deform: single node translation (deformation_graph_tests.cpp:236-245)") {
    Surface s;
    s.points = {Vec3(1, 2, 3)};
    s.finalize_edges();
    const DeformationGraph g = build_graph(s, 1.0);
    NodeTransforms x = NodeTransforms::identity(1);
    x.set(0, Mat3::identity(), Vec3(1, 0, 0));
    CHECK((deformed_position(s.points[0], g.influence[0], g, x) - Vec3(2, 2, 3)).norm() < 1e-15);
}
TEST("deform: two-node blend = (2.5,2,2) (deformation_graph_tests.cpp:247-260)") {
    DeformationGraph g;
    g.radius = 10.0;
    g.node_indices = {0, 1};
    g.node_positions = {Vec3(1, 2, 2), Vec3(2, 1, 2)};
    g.influence.resize(1);
    g.influence[0] = {{0, 0.5, 0.0}, {1, 0.5, 0.0}};
    NodeTransforms x = NodeTransforms::identity(2);
    Mat3 two = Mat3::identity();
    for (double& v : two.m) v *= 2.0;
    x.set(0, two, Vec3());
    CHECK((deformed_position(Vec3(2, 2, 2), g.influence[0], g, x) - Vec3(2.5, 2, 2)).norm() < 1e-15);
}

// ======================================================================= graph setup
TEST("influence weights: 1, 1/2, 64/91 27/91, 1/3 (deformation_graph_tests.cpp:71-88)") {
    CHECK(influence_weights({0.4}, 1.0) == std::vector<double>{1.0});
    const auto eq = influence_weights({0.3, 0.3}, 1.0);
    CHECK_APPROX(eq[0], 0.5, 1e-12, 0);
    const auto pr = influence_weights({0.0, 0.5}, 1.0);
    CHECK_APPROX(pr[0], 64.0 / 91.0, 1e-9, 0);
    CHECK_APPROX(pr[1], 27.0 / 91.0, 1e-9, 0);
    for (double w : influence_weights({0.0, 0.0, 0.0}, 1.0)) CHECK_APPROX(w, 1.0 / 3.0, 1e-12, 0);
    CHECK_THROWS_AS(influence_weights({}, 1.0), ConfigError);
}
TEST("reg weight table: lengths 1 and 2 -> 4/3, 2/3 (deformation_graph_tests.cpp:104-118)") {
    DeformationGraph g;
    g.node_indices = {0, 1, 2};
    g.node_positions = {Vec3(0, 0, 0), Vec3(1, 0, 0), Vec3(3, 0, 0)};
    g.graph_edges = {{0, 1}, {1, 2}};
    g.node_neighbors = {{1}, {0, 2}, {1}};
    reg_weight_table(g);
    CHECK(g.reg_pairs.size() == 4);
    CHECK_APPROX(g.reg_weights[0], 4.0 / 3.0, 1e-12, 0);
    CHECK_APPROX(g.reg_weights[3], 2.0 / 3.0, 1e-12, 0);
}
TEST("pca order: x-axis points sort by coordinate (deformation_graph_tests.cpp:25-28)") {
    CHECK((pca_order({Vec3(3, 0, 0), Vec3(1, 0, 0), Vec3(2, 0, 0)}) == std::vector<int>{1, 2, 0}));
    CHECK((pca_order(std::vector<Vec3>(5, Vec3(0.3, -0.7, 2.0))) == std::vector<int>{0, 1, 2, 3, 4}));
}
TEST("acceptance 6: collinear sweeps R=2.5/3.5 (acceptance_main.cpp:247-297)") {
    std::vector<Vec3> line;
    for (int i = 0; i < 6; ++i) line.emplace_back(i, 0.0, 0.0);
    const Surface col = surface_from_edges(line, {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {4, 5}});
    const DeformationGraph t = build_graph(col, 2.5), w = build_graph(col, 3.5);
    CHECK((t.node_indices == std::vector<int>{0, 3}));
    CHECK((t.graph_edges == std::vector<std::pair<int, int>>{{0, 1}}));
    CHECK((w.node_indices == std::vector<int>{0, 4}));
    CHECK((w.graph_edges == std::vector<std::pair<int, int>>{{0, 1}}));
}

// ============================================================================ energy
TEST("energy: exact alignment at identity is zero (robust_energy_tests.cpp:110-124)") {
    Surface strip = make_strip(8, 4);
    const DeformationGraph g = build_graph(strip, 4.0 * strip.avg_edge_length);
    const NodeTransforms x = NodeTransforms::identity(g.node_count());
    const auto d = deform_points(strip.points, g, x);
    const SpatialIndex idx(strip.points);
    const auto c = find_correspondences(d, idx);
    const auto e = evaluate_energy(d, x, g, c, project_rotations(x), {1.0, 1.0, 0.1, 0.1});
    CHECK(std::abs(e.align) <= 1e-18);
    CHECK(std::abs(e.reg) <= 1e-18);
    CHECK(std::abs(e.rot) <= 1e-22);
    CHECK(std::abs(e.total) <= 1e-17);
}
TEST("energy: pure rotation has no rigidity cost (robust_energy_tests.cpp:126-141)") {
    Surface s;
    s.points = {Vec3(0, 0, 0)};
    s.finalize_edges();
    const DeformationGraph g = build_graph(s, 1.0);
    Mat3 r90;
    r90(0, 1) = -1;
    r90(1, 0) = 1;
    r90(2, 2) = 1;
    NodeTransforms x = NodeTransforms::identity(1);
    x.set(0, r90, Vec3());
    const auto d = deform_points(s.points, g, x);
    const auto c = find_correspondences(d, SpatialIndex(s.points));
    const auto e = evaluate_energy(d, x, g, c, project_rotations(x), {1, 1, 0.5, 0.5});
    CHECK(std::abs(e.rot) <= 1e-18);
}
TEST("energy: matches the scalar-loop oracle at 1e-12 (robust_energy_tests.cpp:143-159)") {
    const Instance in = make_instance(8);
    const NodeTransforms x = random_transforms(in.graph.node_count(), 77);
    const auto d = deform_points(in.source.points, in.graph, x);
    const auto rot = project_rotations(x);
    const auto e = evaluate_energy(d, x, in.graph, in.corr, rot, in.prm);
    const double o = scalar_energy(in.source.points, in.graph, x, in.corr.target_point, rot, in.prm.alpha,
                                   in.prm.beta, in.prm.nu_a, in.prm.nu_r);
    CHECK_APPROX(e.total, o, 1e-12, 0);
    CHECK_APPROX(e.total, e.align + in.prm.alpha * e.reg + in.prm.beta * e.rot, 1e-14, 0);
    CHECK(e.align <= in.source.point_count());
    CHECK(e.reg <= 2.0 * in.graph.edge_count());
    CHECK(e.rot >= 0.0);
}
TEST("energy: dimension mismatch throws (robust_energy_tests.cpp:161-168)") {
    const Instance in = make_instance(9);
    const auto d = deform_points(in.source.points, in.graph, in.anchor);
    const std::vector<Mat3> too_few(1, Mat3::identity());
    CHECK_THROWS_AS(evaluate_energy(d, in.anchor, in.graph, in.corr, too_few, in.prm), NumericalError);
}

// ==================================================================== assembly/solve
TEST("assemble: K bitwise symmetric (robust_energy_tests.cpp:185-196)") {
    const Instance in = make_instance(21);
    const LinearSystem s = assemble_system(in.anchor, in.source, in.graph, in.corr, in.rotations, in.prm);
    double mx = 0;
    const int n4 = 4 * in.graph.node_count();
    for (int r = 0; r < n4; ++r)
        for (int c = 0; c < n4; ++c) mx = std::max(mx, std::abs(s.K.get(r, c) - s.K.get(c, r)));
    CHECK(mx == 0.0);
}
TEST("assemble: one node one point vs dense, solve 1e-10 (robust_energy_tests.cpp:223-258)") {
    std::vector<Vec3> pts = {Vec3(0.2, 0.3, 0.4)};
    DeformationGraph g;
    g.radius = 2.0;
    g.node_indices = {0};
    g.node_positions = {Vec3(0, 0, 0)};
    g.influence = {{{0, 1.0, 0.7}}};
    Correspondences corr;
    corr.target_index = {0};
    corr.target_point = {Vec3(1, 2, 3)};
    corr.squared_distance = {(Vec3(0.2, 0.3, 0.4) - Vec3(1, 2, 3)).squaredNorm()};
    const EnergyParams prm{0.0, 0.5, 0.7, 1.0};
    SystemAssembler as(pts, g);
    as.fill(corr, {Mat3::identity()}, alignment_weights(corr, prm.nu_a),
            regularization_weights(g, NodeTransforms::identity(1), prm.nu_r, prm.alpha), prm.beta);
    const LinearSystem& s = as.system();
    const double f[4] = {0.2, 0.3, 0.4, 1.0};
    const double w = welsch_weight_sq(corr.squared_distance[0], prm.nu_a);
    const double q[3] = {1, 2, 3};
    double mk = 0, mb = 0;
    std::vector<double> kd(16), bd(12);
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            kd[r * 4 + c] = w * f[r] * f[c] + (r == c && r < 3 ? prm.beta : 0.0);
            mk = std::max(mk, std::abs(s.K.get(r, c) - kd[r * 4 + c]));
        }
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 3; ++c) {
            bd[c * 4 + r] = w * f[r] * q[c] + (r == c ? prm.beta : 0.0);
            mb = std::max(mb, std::abs(s.B[c * 4 + r] - bd[c * 4 + r]));
        }
    CHECK(mk < 1e-15);
    CHECK(mb < 1e-15);
    const NodeTransforms x = solve_system(s);
    double mx = 0;
    for (int c = 0; c < 3; ++c) {
        std::vector<double> rhs(4);
        for (int r = 0; r < 4; ++r) rhs[r] = bd[c * 4 + r];
        const auto xd = solve_dense(kd, 4, rhs);
        for (int r = 0; r < 4; ++r) mx = std::max(mx, std::abs(x.at(r, c) - xd[r]));
    }
    CHECK(mx < 1e-10);
}
TEST("assemble: quadratic form = scalar surrogate at 1e-9 (robust_energy_tests.cpp:260-277)") {
    const Instance in = make_instance(33);
    const LinearSystem s = assemble_system(in.anchor, in.source, in.graph, in.corr, in.rotations, in.prm);
    const NodeTransforms zero = NodeTransforms::zeros(in.graph.node_count());
    auto sur = [&](const NodeTransforms& x) {
        return surrogate_dropped(in.source.points, in.graph, x, in.anchor, in.corr.target_point, in.rotations,
                                 in.prm.alpha, in.prm.beta, in.prm.nu_a, in.prm.nu_r);
    };
    const double constant = sur(zero);
    for (uint64_t seed : {1, 2, 3, 4, 5}) {
        const NodeTransforms x = random_transforms(in.graph.node_count(), seed);
        CHECK_APPROX(quadratic_form(s, x) + constant, sur(x), 1e-9, 0);
    }
}
TEST("solve: recovers a constructed solution at 1e-8 (robust_energy_tests.cpp:279-287)") {
    const Instance in = make_instance(44);
    LinearSystem s = assemble_system(in.anchor, in.source, in.graph, in.corr, in.rotations, in.prm);
    const NodeTransforms ex = random_transforms(in.graph.node_count(), 123);
    s.B = s.K.multiply(ex.stacked);
    CHECK(inf_norm_diff(solve_system(s).stacked, ex.stacked) < 1e-8);
}
TEST("solve: one step never increases bound or energy (robust_energy_tests.cpp:289-315)") {
    for (uint64_t seed : {6, 7, 8}) {
        const Instance in = make_instance(seed);
        const LinearSystem s = assemble_system(in.anchor, in.source, in.graph, in.corr, in.rotations, in.prm);
        const NodeTransforms nx = solve_system(s);
        auto sur = [&](const NodeTransforms& x) {
            return surrogate_dropped(in.source.points, in.graph, x, in.anchor, in.corr.target_point,
                                     in.rotations, in.prm.alpha, in.prm.beta, in.prm.nu_a, in.prm.nu_r);
        };
        CHECK(sur(nx) <= sur(in.anchor) + 1e-12);
        const SpatialIndex idx(in.target.points);
        const auto dn = deform_points(in.source.points, in.graph, nx);
        const auto cn = find_correspondences(dn, idx);
        const auto en = evaluate_energy(dn, nx, in.graph, cn, project_rotations(nx), in.prm);
        const auto da = deform_points(in.source.points, in.graph, in.anchor);
        const auto ea = evaluate_energy(da, in.anchor, in.graph, in.corr, in.rotations, in.prm);
        CHECK(en.total <= ea.total + 1e-12);
    }
}
TEST("majorization: restored-constant bound dominates (robust_energy_tests.cpp:317-341)") {
    const Instance in = make_instance(55);
    const double c = surrogate_constant(in.source.points, in.graph, in.anchor, in.corr.target_point,
                                        in.prm.alpha, in.prm.nu_a, in.prm.nu_r);
    auto full = [&](const NodeTransforms& x) {
        return c + surrogate_dropped(in.source.points, in.graph, x, in.anchor, in.corr.target_point,
                                     in.rotations, in.prm.alpha, in.prm.beta, in.prm.nu_a, in.prm.nu_r);
    };
    auto fixed = [&](const NodeTransforms& x) {
        return scalar_energy(in.source.points, in.graph, x, in.corr.target_point, in.rotations, in.prm.alpha,
                             in.prm.beta, in.prm.nu_a, in.prm.nu_r);
    };
    CHECK_APPROX(full(in.anchor), fixed(in.anchor), 1e-10, 0);
    for (uint64_t seed = 200; seed < 240; ++seed) {
        const NodeTransforms x = random_transforms(in.graph.node_count(), seed, 0.5);
        CHECK(full(x) >= fixed(x) - 1e-10);
    }
}
TEST("solve: unconstrained block names node 0 (robust_energy_tests.cpp:343-361)") {
    Surface s;
    s.points = {Vec3(0, 0, 0)};
    s.finalize_edges();
    const DeformationGraph g = build_graph(s, 1.0);
    Correspondences corr;
    corr.target_index = {0};
    corr.target_point = {Vec3(0.1, 0, 0)};
    corr.squared_distance = {0.01};
    LinearSystem sys;
    {
        SystemAssembler as(s.points, g);
        as.fill(corr, {Mat3::identity()}, alignment_weights(corr, 0.5), std::vector<double>{}, 0.0);
        sys = as.system();
    }
    CHECK_THROWS_WITH(solve_system(sys), NumericalError, "positive definite");
    SystemAssembler as(s.points, g);
    as.fill(corr, {Mat3::identity()}, alignment_weights(corr, 0.5), std::vector<double>{}, 0.0);
    CHECK_THROWS_WITH(as.solve(), NumericalError, "node 0");
}

// ========================================================================= anderson
TEST("anderson: empty history throws (solver_tests.cpp:22-24)") {
    CHECK_THROWS_AS(anderson_combine({}, 5), NumericalError);
}
TEST("anderson: single entry / window 0 = plain update (solver_tests.cpp:26-38)") {
    std::deque<AndersonEntry> h{{{1.0, 2.0}, {-0.5, 0.25}}};
    CHECK((anderson_combine(h, 5) == std::vector<double>{1.0, 2.0}));
    h.push_back({{0.5, 1.0}, {-0.25, 0.125}});
    CHECK((anderson_combine(h, 0) == std::vector<double>{0.5, 1.0}));
}
TEST("anderson: halving map exact after two evaluations (solver_tests.cpp:40-55)") {
    AndersonWindow w(1);
    std::vector<double> x{1.0};
    std::vector<double> g{0.5 * x[0]};
    w.push(g, {g[0] - x[0]});
    x = w.combine();
    CHECK_APPROX(x[0], 0.5, 1e-12, 0);
    g = {0.5 * x[0]};
    w.push(g, {g[0] - x[0]});
    x = w.combine();
    CHECK(std::abs(x[0]) <= 1e-15);
}
TEST("anderson: linear contractions within dim+1, seed 17 (solver_tests.cpp:57-80)") {
    std::mt19937_64 rng(17);
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (int dim : {2, 5, 11}) {
        const auto a = random_contraction(rng, dim, 0.85);
        std::vector<double> b(dim);
        for (auto& v : b) v = gauss(rng);
        std::vector<double> ima(dim * dim);
        for (int i = 0; i < dim; ++i)
            for (int j = 0; j < dim; ++j) ima[i * dim + j] = (i == j ? 1.0 : 0.0) - a[i * dim + j];
        const auto fixed = solve_dense(ima, dim, b);
        AndersonWindow w(dim);
        std::vector<double> x(dim, 0.0);
        int used = 0;
        for (int it = 1; it <= dim + 4; ++it) {
            std::vector<double> g(dim), f(dim);
            for (int i = 0; i < dim; ++i) {
                g[i] = b[i];
                for (int j = 0; j < dim; ++j) g[i] += a[i * dim + j] * x[j];
                f[i] = g[i] - x[i];
            }
            w.push(g, f);
            x = w.combine();
            used = it;
            if (inf_norm_diff(x, fixed) < 1e-9) break;
        }
        CHECK(used <= dim + 1);
        CHECK(inf_norm_diff(x, fixed) < 1e-9);
    }
}
TEST("anderson: degenerate differences stay finite (solver_tests.cpp:82-92)") {
    AndersonWindow w(3);
    for (int k = 0; k < 3; ++k) w.push({1.0, -1.0}, {0.5, 0.5});
    const auto x = w.combine();
    CHECK(std::isfinite(x[0]) && std::isfinite(x[1]));
}
TEST("acceptance 4: AA on 10 contractions, seed 404 (acceptance_main.cpp:148-197)") {
    std::mt19937_64 rng(404);
    std::normal_distribution<double> gauss(0.0, 1.0);
    std::uniform_int_distribution<int> dimd(2, 20);
    std::uniform_real_distribution<double> radd(0.8, 0.9);
    for (int trial = 0; trial < 10; ++trial) {
        const int dim = dimd(rng);
        const auto a = random_contraction(rng, dim, radd(rng));
        std::vector<double> b(dim);
        for (auto& v : b) v = gauss(rng);
        std::vector<double> ima(dim * dim);
        for (int i = 0; i < dim; ++i)
            for (int j = 0; j < dim; ++j) ima[i * dim + j] = (i == j ? 1.0 : 0.0) - a[i * dim + j];
        const auto fixed = solve_dense(ima, dim, b);
        AndersonWindow w(dim);
        std::vector<double> x(dim, 0.0);
        auto apply = [&](const std::vector<double>& v) {
            std::vector<double> g(b);
            for (int i = 0; i < dim; ++i)
                for (int j = 0; j < dim; ++j) g[i] += a[i * dim + j] * v[j];
            return g;
        };
        int aa = 0;
        for (int it = 1; it <= dim + 2; ++it) {
            const auto g = apply(x);
            std::vector<double> f(dim);
            for (int i = 0; i < dim; ++i) f[i] = g[i] - x[i];
            w.push(g, f);
            x = w.combine();
            aa = it;
            if (inf_norm_diff(x, fixed) <= 1e-8) break;
        }
        CHECK(inf_norm_diff(x, fixed) <= 1e-8);
        std::vector<double> plain(dim, 0.0);
        int pi = 0;
        while (inf_norm_diff(plain, fixed) > 1e-8 && pi < 100000) {
            plain = apply(plain);
            ++pi;
        }
        CHECK(pi >= 3 * aa);
    }
}

// ========================================================================== solver
TEST("anneal: bound terminates; halving clamps; nu_r floor (solver_tests.cpp:94-121)") {
    CHECK(anneal(0.01, 0.5, 0.01).done);
    double a = 0.08, r = 0.24;
    std::vector<double> seq{a};
    while (true) {
        const auto n = anneal(a, r, 0.01);
        if (n.done) break;
        a = n.nu_a;
        r = n.nu_r;
        seq.push_back(a);
    }
    CHECK((seq == std::vector<double>{0.08, 0.04, 0.02, 0.01}));
    const auto first = anneal(0.03, 0.09, 0.02);
    CHECK(!first.done);
    CHECK(first.nu_a == 0.02);
    CHECK(anneal(first.nu_a, first.nu_r, 0.02).done);
    CHECK(anneal(1.0, 1.5e-8, 1e-12, 1e-8).nu_r == 1e-8);
}
TEST("init parameters: identical pair clamps; median 0.03; formulas (solver_tests.cpp:123-179)") {
    {
        Surface strip = make_strip(8, 4);
        const DeformationGraph g = build_graph(strip, 4.0 * strip.avg_edge_length);
        const SolverParams p = init_parameters(strip.points, strip.avg_edge_length, SpatialIndex(strip.points), g, {});
        CHECK(p.nu_a == p.nu_a_min);
        CHECK_APPROX(p.nu_a_min, strip.avg_edge_length / std::sqrt(3.0), 1e-12, 0);
    }
    {
        std::vector<Vec3> src, tgt;
        const double d[5] = {0.01, 0.02, 0.03, 0.04, 0.05};
        for (int i = 0; i < 5; ++i) {
            src.emplace_back(i, 0.0, 0.0);
            tgt.emplace_back(i, d[i], 0.0);
        }
        Surface s = surface_from_edges(src, {{0, 1}, {1, 2}, {2, 3}, {3, 4}});
        const DeformationGraph g = build_graph(s, 2.5);
        SolverConfig cfg;
        cfg.nu_a_min = 1e-4;
        CHECK_APPROX(init_parameters(s.points, s.avg_edge_length, SpatialIndex(tgt), g, cfg).nu_a, 0.03, 1e-12, 0);
    }
    {
        Surface pr = surface_from_edges({Vec3(0, 0, 0), Vec3(0.01, 0, 0)}, {{0, 1}});
        CHECK_APPROX(pr.avg_edge_length, 0.01, 1e-12, 0);
        const DeformationGraph g = build_graph(pr, 0.05);
        const SpatialIndex idx(std::vector<Vec3>{Vec3(0.5, 0, 0), Vec3(0.6, 0, 0)});
        const SolverParams p = init_parameters(pr.points, pr.avg_edge_length, idx, g, {});
        CHECK_APPROX(p.nu_a_min, 0.0057735, 0, 1e-7);
        CHECK_APPROX(p.nu_r, 0.03, 1e-12, 0);
        SolverConfig cfg;
        cfg.k_alpha = 2.0;
        cfg.k_beta = 3.0;
        const SolverParams q = init_parameters(pr.points, pr.avg_edge_length, idx, g, cfg);
        const double v = 2.0, e = g.edge_count(), m = g.node_count();
        if (e > 0) CHECK_APPROX(q.alpha, 2.0 * (v / e) * q.nu_r * q.nu_r / (q.nu_a * q.nu_a), 1e-12, 0);
        CHECK_APPROX(q.beta, 3.0 * (v / m) / (2.0 * q.nu_a * q.nu_a), 1e-12, 0);
    }
    {
        Surface s;
        s.points = {Vec3(0, 0, 0)};
        s.finalize_edges();
        const DeformationGraph g = build_graph(s, 1.0);
        const SolverParams p = init_parameters(s.points, 0.01, SpatialIndex(std::vector<Vec3>{Vec3(1, 0, 0)}), g, {});
        CHECK(p.alpha == 0.0);
        CHECK(p.alpha_forced_zero);
    }
}
TEST("register: identity pair, one stage, RMSE<1e-6 (solver_tests.cpp:181-193)") {
    Surface src = make_strip(12, 6), tgt = src;
    normalize_pair(src, tgt);
    const DeformationGraph g = build_graph(src, 5.0 * src.avg_edge_length);
    const auto r = register_surfaces(src.points, src.avg_edge_length, tgt.points, g, {});
    CHECK(r.report.stages.size() == 1);
    CHECK(r.report.stages[0].converged);
    CHECK(rmse_pts(r.deformed_points, tgt.points) < 1e-6);
}
TEST("register: monotone energy per stage, halving (solver_tests.cpp:195-218)") {
    std::mt19937_64 rng(4242);
    Surface src = make_strip(24, 10);
    Surface tgt = warped_copy(src, random_warp(rng, 2.5));
    normalize_pair(src, tgt);
    const DeformationGraph g = build_graph(src, 5.0 * src.avg_edge_length);
    const auto r = register_surfaces(src.points, src.avg_edge_length, tgt.points, g, {});
    CHECK(r.report.stages.size() >= 2);
    for (const auto& st : r.report.stages)
        for (size_t k = 1; k < st.iterations.size(); ++k)
            CHECK(st.iterations[k].e_total + st.iterations[k].e_landmark <=
                  st.iterations[k - 1].e_total + st.iterations[k - 1].e_landmark + 1e-12);
    for (size_t s = 1; s < r.report.stages.size(); ++s) {
        const auto &p = r.report.stages[s - 1], &c = r.report.stages[s];
        CHECK_APPROX(c.nu_a, std::max(p.nu_a / 2.0, r.report.stages.back().nu_a), 1e-12, 0);
        CHECK_APPROX(c.nu_r, p.nu_r / 2.0, 1e-12, 0);
    }
}
TEST("register: converged iterate is a fixed point <= 10 eps (solver_tests.cpp:220-239)") {
    std::mt19937_64 rng(515);
    Surface src = make_strip(16, 7);
    Surface tgt = warped_copy(src, random_warp(rng));
    normalize_pair(src, tgt);
    const DeformationGraph g = build_graph(src, 5.0 * src.avg_edge_length);
    SolverConfig cfg;
    const auto r = register_surfaces(src.points, src.avg_edge_length, tgt.points, g, cfg);
    CHECK(r.report.stages.back().converged);
    const auto& last = r.report.stages.back();
    SolverParams prm;
    prm.nu_a = last.nu_a;
    prm.nu_r = last.nu_r;
    prm.alpha = last.alpha;
    prm.beta = last.beta;
    const NodeTransforms gx = mm_step(src.points, g, SpatialIndex(tgt.points), r.transforms, prm);
    CHECK(inf_norm_diff(gx.stacked, r.transforms.stacked) <= 10.0 * cfg.eps);
}
TEST("register: aa_window=0 -> no reverts, no AA flags (solver_tests.cpp:241-254)") {
    std::mt19937_64 rng(808);
    Surface src = make_strip(14, 6);
    Surface tgt = warped_copy(src, random_warp(rng));
    normalize_pair(src, tgt);
    const DeformationGraph g = build_graph(src, 5.0 * src.avg_edge_length);
    SolverConfig cfg;
    cfg.aa_window = 0;
    const auto r = register_surfaces(src.points, src.avg_edge_length, tgt.points, g, cfg);
    for (const auto& st : r.report.stages) {
        CHECK(st.reverts == 0);
        for (const auto& it : st.iterations) CHECK(!it.aa_accepted);
    }
}
TEST("register: landmarks act in the first stage only (solver_tests.cpp:256-275)") {
    Surface src = make_strip(10, 5), tgt = src;
    for (auto& p : tgt.points) p += Vec3(0.04, 0.0, 0.0);
    tgt.finalize_edges();
    normalize_pair(src, tgt);
    const DeformationGraph g = build_graph(src, 5.0 * src.avg_edge_length);
    SolverConfig cfg;
    cfg.nu_a_min = 1e-3;
    cfg.landmarks.push_back({0, tgt.points[0]});
    cfg.landmarks.push_back({9, tgt.points[9]});
    const auto r = register_surfaces(src.points, src.avg_edge_length, tgt.points, g, cfg);
    CHECK(r.report.stages.size() >= 2);
    for (size_t s = 1; s < r.report.stages.size(); ++s)
        for (const auto& it : r.report.stages[s].iterations) CHECK(it.e_landmark == 0.0);
    CHECK((r.deformed_points[0] - tgt.points[0]).norm() < 0.01);
}
TEST("solver config validation (solver_tests.cpp:277-290)") {
    SolverConfig c;
    c.eps = 0.0;
    CHECK_THROWS_AS(c.validate(), ConfigError);
    c = {};
    c.i_max = 0;
    CHECK_THROWS_AS(c.validate(), ConfigError);
    c = {};
    c.aa_window = -1;
    CHECK_THROWS_AS(c.validate(), ConfigError);
    c = {};
    c.k_alpha = -0.5;
    CHECK_THROWS_AS(c.validate(), ConfigError);
}

// ===================================================== acceptance 2/3/5 (strip pool)
namespace {
struct Warp {
    Surface src, tgt;
    DeformationGraph g;
    RegistrationResult annealed;
};
std::vector<Warp>& pool() {  // acceptance_main.cpp:41-60
    static std::vector<Warp> p;
    if (!p.empty()) return p;
    std::mt19937_64 rng(90210);
    std::uniform_int_distribution<int> verts(200, 2000);
    for (int k = 0; k < 20; ++k) {
        const int total = verts(rng);
        const int nx = std::max(8, static_cast<int>(std::sqrt(2.0 * total)));
        const int ny = std::max(5, total / nx);
        Warp w;
        w.src = make_strip(nx, ny);
        w.tgt = warped_copy(w.src, random_warp(rng, 1.5));
        normalize_pair(w.src, w.tgt);
        w.g = build_graph(w.src, 5.0 * w.src.avg_edge_length);
        w.annealed = register_surfaces(w.src.points, w.src.avg_edge_length, w.tgt.points, w.g, {});
        p.push_back(std::move(w));
    }
    return p;
}
}  // namespace
TEST("acceptance 2+3: MM monotone, fixed point on 20 strips (acceptance_main.cpp:99-144)") {
    double worst = 0;
    for (auto& w : pool()) {
        for (const auto& st : w.annealed.report.stages)
            for (size_t k = 1; k < st.iterations.size(); ++k)
                CHECK(st.iterations[k].e_total <= st.iterations[k - 1].e_total + 1e-12);
        const auto& last = w.annealed.report.stages.back();
        SolverParams prm;
        prm.nu_a = last.nu_a;
        prm.nu_r = last.nu_r;
        prm.alpha = last.alpha;
        prm.beta = last.beta;
        const NodeTransforms gx = mm_step(w.src.points, w.g, SpatialIndex(w.tgt.points), w.annealed.transforms, prm);
        worst = std::max(worst, inf_norm_diff(gx.stacked, w.annealed.transforms.stacked));
    }
    CHECK(worst <= 10.0 * 1e-5);
}
TEST("acceptance 5: AA benefit >= 80%, ratio <= 1.2 (acceptance_main.cpp:201-243)") {
    int not_worse = 0;
    double worst_ratio = 0;
    const int cap = 500;
    auto first_reach = [](const std::vector<double>& t, double thr) {
        for (size_t i = 0; i < t.size(); ++i)
            if (t[i] <= thr) return static_cast<int>(i);
        return static_cast<int>(t.size());
    };
    auto trace = [](const RegistrationReport& r) {
        std::vector<double> t;
        for (const auto& s : r.stages)
            for (const auto& it : s.iterations) t.push_back(it.e_total);
        return t;
    };
    for (auto& w : pool()) {
        const SolverParams init = init_parameters(w.src.points, w.src.avg_edge_length, SpatialIndex(w.tgt.points), w.g, {});
        SolverConfig fc;
        fc.nu_a_init = init.nu_a;
        fc.nu_a_min = init.nu_a;
        fc.nu_r_init = init.nu_r;
        fc.eps = 1e-12;
        fc.i_max = cap;
        SolverConfig ac = fc;
        ac.aa_window = 5;
        const auto at = trace(register_surfaces(w.src.points, w.src.avg_edge_length, w.tgt.points, w.g, ac).report);
        SolverConfig mc = fc;
        mc.aa_window = 0;
        const auto mt = trace(register_surfaces(w.src.points, w.src.avg_edge_length, w.tgt.points, w.g, mc).report);
        const double es = at.back();
        const int a = first_reach(at, es + 1e-6);
        const int m = std::min(cap, first_reach(mt, es + 1e-6));
        if (a <= m) ++not_worse;
        worst_ratio = std::max(worst_ratio, static_cast<double>(a) / std::max(1, m));
    }
    const int n = static_cast<int>(pool().size());
    CHECK(not_worse >= (8 * n + 9) / 10);
    CHECK(worst_ratio <= 1.2);
}

KAT_MAIN
