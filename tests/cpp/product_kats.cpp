// GPU known-answer checks of the drop-in C++ API (include/nrr/*.hpp over
// libnrr_b200.so) against the CPU oracle (oracle/nrr_oracle.hpp, test
// infrastructure only). Mirrors the reference's per-module tests
// (tests/test_kd_tree.cpp, test_deformation_graph.cpp, test_energy.cpp,
// test_anderson.cpp, test_solver.cpp): same cases, the product on one side,
// the oracle on the other.
#include <random>

#include "../../oracle/nrr_oracle.hpp"
#include "check.hpp"
#include "nrr/nrr.hpp"

namespace {

nrr::Vec3 P(const oracle::Vec3& v) { return {v.x, v.y, v.z}; }
std::vector<nrr::Vec3> P(const std::vector<oracle::Vec3>& v) {
    std::vector<nrr::Vec3> o;
    for (const auto& p : v) o.push_back(P(p));
    return o;
}

nrr::Surface P(const oracle::Surface& s) {
    return nrr::make_surface(P(s.points), s.faces);
}

oracle::NodeTransforms random_transforms(std::mt19937_64& rng, int N, double amp) {
    std::normal_distribution<double> g(0.0, 1.0);
    oracle::NodeTransforms x = oracle::NodeTransforms::identity(N);
    for (double& v : x.stacked) v += amp * g(rng);
    return x;
}
nrr::NodeTransforms P(const oracle::NodeTransforms& x) {
    nrr::NodeTransforms o;
    o.stacked.setZero(4 * x.node_count(), 3);
    o.stacked.d = x.stacked;
    return o;
}

struct Case {
    oracle::Surface src, tgt;
    oracle::DeformationGraph og;
    nrr::Surface psrc, ptgt;
    nrr::DeformationGraph pg;
};

Case strip_case(uint64_t seed, int nx = 24, int ny = 12) {
    std::mt19937_64 rng(seed);
    Case c;
    c.src = oracle::make_strip(nx, ny);
    c.tgt = oracle::warped_copy(c.src, oracle::random_warp(rng));
    const double radius = 4.0 * c.src.avg_edge_length;
    c.og = oracle::build_graph(c.src, radius);
    c.psrc = P(c.src);
    c.ptgt = P(c.tgt);
    c.pg = nrr::build_graph(c.psrc, radius);
    return c;
}

double max_abs_diff(const std::vector<double>& a, const std::vector<double>& b) {
    double m = 0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}

}  // namespace

TEST("graph: build_graph matches the oracle bitwise") {
    const Case c = strip_case(1);
    CHECK(c.pg.node_indices == c.og.node_indices);
    CHECK(c.pg.graph_edges == c.og.graph_edges);
    CHECK(c.pg.reg_weights == c.og.reg_weights);
    bool infl = c.pg.influence.size() == c.og.influence.size();
    for (size_t i = 0; infl && i < c.og.influence.size(); ++i) {
        infl = c.pg.influence[i].size() == c.og.influence[i].size();
        for (size_t k = 0; infl && k < c.og.influence[i].size(); ++k)
            infl = c.pg.influence[i][k].node == c.og.influence[i][k].node &&
                   c.pg.influence[i][k].weight == c.og.influence[i][k].weight;
    }
    CHECK(infl);
}

TEST("kd_tree: nearest_batch equals exhaustive search, ties to the smallest index") {
    std::mt19937_64 rng(7);
    const auto pts = oracle::random_points(rng, 5000);
    const auto qs = oracle::random_points(rng, 3000, 1.2);
    nrr::SpatialIndex index(P(pts));
    const auto hits = index.nearest_batch(P(qs));
    int bad = 0;
    for (size_t i = 0; i < qs.size(); ++i) {
        int bi = -1;
        double bd = 1e300;
        for (size_t k = 0; k < pts.size(); ++k) {
            const double d = (qs[i] - pts[k]).squaredNorm();
            if (d < bd) bd = d, bi = static_cast<int>(k);
        }
        if (hits[i].index != bi || hits[i].distance != std::sqrt(bd)) ++bad;
    }
    CHECK(bad == 0);
    // duplicated points: the smallest index wins
    std::vector<nrr::Vec3> dup = {{0, 0, 0}, {1, 0, 0}, {1, 0, 0}, {0.5, 0, 0}};
    nrr::SpatialIndex di(dup);
    CHECK(di.nearest({2, 0, 0}).index == 1);
    CHECK(di.nearest({0.75, 0, 0}).index == 1);  // equidistant to 1 and 3
    CHECK(nrr::closest_point(di, {0.2, 0, 0}).first == 0);
}

TEST("deformation: deform_points matches the oracle") {
    const Case c = strip_case(2);
    std::mt19937_64 rng(3);
    const auto x = random_transforms(rng, c.og.node_count(), 0.05);
    const auto ref = oracle::deform_points(c.src.points, c.og, x);
    const auto got = nrr::deform_points(c.psrc, c.pg, P(x));
    double m = 0;
    for (size_t i = 0; i < ref.size(); ++i) m = std::max(m, (P(ref[i]) - got[i]).norm());
    CHECK(m <= 1e-13);
}

TEST("energy: project_rotations matches the oracle and counts degenerate blocks") {
    std::mt19937_64 rng(4);
    auto x = random_transforms(rng, 200, 0.3);
    x.set(5, oracle::Mat3(), {0, 0, 0});  // rank 0: degenerate
    int deg_o = 0, deg_p = 0;
    const auto ro = oracle::project_rotations(x, &deg_o);
    const auto rp = nrr::project_rotations(P(x), &deg_p);
    double m = 0;
    for (int j = 0; j < 200; ++j)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) m = std::max(m, std::abs(ro[j](r, c) - rp[j](r, c)));
    CHECK(m <= 1e-12);
    CHECK(deg_o == deg_p);
    CHECK(deg_p >= 1);
}

TEST("energy: SystemAssembler fill/solve match the oracle's K, B and solution") {
    const Case c = strip_case(5);
    std::mt19937_64 rng(6);
    const auto x = random_transforms(rng, c.og.node_count(), 0.02);
    const auto deformed = oracle::deform_points(c.src.points, c.og, x);
    const oracle::SpatialIndex ti(c.tgt.points);
    const auto corr = oracle::find_correspondences(deformed, ti);
    const auto rot = oracle::project_rotations(x);
    const double nu_a = 0.05, nu_r = 0.1, alpha = 3.0, beta = 0.7;
    const auto wa = oracle::alignment_weights(corr, nu_a);
    const auto wr = oracle::regularization_weights(c.og, x, nu_r, alpha);
    oracle::SystemAssembler oa(c.src.points, c.og);
    oa.fill(corr, rot, wa, wr, beta);
    const auto xo = oa.solve();

    nrr::Correspondences pc;
    pc.target_index = corr.target_index;
    pc.target_point = P(corr.target_point);
    pc.squared_distance = corr.squared_distance;
    std::vector<nrr::Mat3> prot(rot.size());
    for (size_t j = 0; j < rot.size(); ++j)
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k) prot[j](r, k) = rot[j](r, k);
    nrr::SystemAssembler pa(c.psrc, c.pg);
    pa.fill(pc, prot, wa, wr, beta);
    const auto& sys = pa.system();
    CHECK(sys.block_row_ptr == oa.system().K.row_ptr);
    CHECK(sys.block_cols == oa.system().K.col);
    const double kmax = std::max(1.0, max_abs_diff(oa.system().K.val, std::vector<double>(oa.system().K.val.size())));
    CHECK(max_abs_diff(sys.values, oa.system().K.val) <= 1e-13 * kmax);
    CHECK(max_abs_diff(sys.B.d, oa.system().B) <= 1e-13 * (1.0 + max_abs_diff(oa.system().B, std::vector<double>(oa.system().B.size()))));
    // K bitwise symmetric (energy.hpp:131-136)
    bool sym = true;
    for (int r = 0; r < sys.rows() && sym; ++r)
        for (int k = sys.block_row_ptr[r / 4]; k < sys.block_row_ptr[r / 4 + 1]; ++k)
            for (int q = 0; q < 4; ++q) {
                const int col = 4 * sys.block_cols[k] + q;
                if (sys.coeff(r, col) != sys.coeff(col, r)) sym = false;
            }
    CHECK(sym);
    // the reference's LinearSystem::K view (robust_energy_tests.cpp:60,185-214,252)
    CHECK(sys.K.rows() == sys.rows() && sys.K.cols() == sys.rows());
    CHECK(sys.K.nonZeros() == 16 * static_cast<int>(sys.block_cols.size()));
    CHECK((sys.K - sys.K.transpose()).norm() == 0.0);
    {
        double worst = 0.0;
        for (int a = 0; a + 1 < static_cast<int>(sys.block_row_ptr.size()); ++a)
            for (int k = sys.block_row_ptr[a]; k < sys.block_row_ptr[a + 1]; ++k)
                for (int i = 0; i < 4; ++i)
                    for (int j = 0; j < 4; ++j)
                        worst = std::max(worst, std::abs(sys.K.coeff(4 * a + i, 4 * sys.block_cols[k] + j) -
                                                         sys.values[16 * static_cast<size_t>(k) + 4 * i + j]));
        CHECK(worst == 0.0);
        const nrr::MatrixX Kx = sys.K * sys.B;  // sparse x dense
        const nrr::MatrixX Kd = sys.K.toDense();
        double dd = 0.0;
        for (int r = 0; r < sys.rows(); ++r)
            for (int q = 0; q < 3; ++q) {
                double v = 0.0;
                for (int cc = 0; cc < sys.rows(); ++cc) v += Kd(r, cc) * sys.B(cc, q);
                dd = std::max(dd, std::abs(v - Kx(r, q)));
            }
        CHECK(dd <= 1e-9 * (1.0 + kmax));
    }
    const auto xp = pa.solve();
    CHECK(max_abs_diff(xp.stacked.d, xo.stacked) <= 1e-9);
    // solve_system on the returned LinearSystem
    const auto xs = nrr::solve_system(sys);
    CHECK(max_abs_diff(xs.stacked.d, xo.stacked) <= 1e-9);
    // evaluate_energy (host utility) agrees with the oracle
    const auto eo = oracle::evaluate_energy(deformed, x, c.og, corr, rot, {alpha, beta, nu_a, nu_r});
    const auto ep = nrr::evaluate_energy(P(deformed), P(x), c.pg, pc, prot, {alpha, beta, nu_a, nu_r});
    CHECK_APPROX(ep.total, eo.total, 1e-13, 0.0);
}

TEST("energy: a singular system fails with the reference's message") {
    const Case c = strip_case(8, 10, 6);
    nrr::SystemAssembler pa(c.psrc, c.pg);
    nrr::Correspondences pc;
    pc.target_index.assign(c.psrc.point_count(), 0);
    pc.target_point.assign(c.psrc.point_count(), nrr::Vec3());
    pc.squared_distance.assign(c.psrc.point_count(), 0.0);
    std::vector<nrr::Mat3> rot(c.pg.node_count(), nrr::Mat3::Identity());
    pa.fill(pc, rot, std::vector<double>(c.psrc.point_count(), 0.0),
            std::vector<double>(c.pg.directed_pair_count(), 0.0), 0.0);
    bool threw = false;
    try {
        pa.solve();
    } catch (const nrr::NumericalError& e) {
        threw = std::string(e.what()).find("linear system not positive definite") != std::string::npos;
    }
    CHECK(threw);
}

TEST("energy: the failing block named is the first non-PD one, at a node j != 0") {
    // beta > 0 makes every A-part PD; a node's translation pivot is exactly 0
    // when all points it influences have zero alignment weight and the reg
    // weights are zero: describe_failure (energy.hpp:329-340) names the first
    // such node
    const Case c = strip_case(8, 10, 6);
    const int N = c.pg.node_count(), n = c.psrc.point_count();
    const int j = N - 1;
    std::vector<double> w(n, 1.0);
    for (int i = 0; i < n; ++i)
        for (const auto& e : c.pg.influence[i])
            if (e.node == j) w[i] = 0.0;
    int expect = -1;
    for (int k = 0; k < N && expect < 0; ++k) {
        bool any = false;
        for (int i = 0; i < n; ++i)
            for (const auto& e : c.pg.influence[i])
                if (e.node == k && w[i] != 0.0) any = true;
        if (!any) expect = k;
    }
    CHECK(expect > 0);
    nrr::SystemAssembler pa(c.psrc, c.pg);
    nrr::Correspondences pc;
    pc.target_index.assign(n, 0);
    pc.target_point.assign(n, nrr::Vec3());
    pc.squared_distance.assign(n, 0.0);
    std::vector<nrr::Mat3> rot(N, nrr::Mat3::Identity());
    pa.fill(pc, rot, w, std::vector<double>(c.pg.directed_pair_count(), 0.0), 1.0);
    std::string msg;
    try {
        pa.solve();
    } catch (const nrr::NumericalError& e) {
        msg = e.what();
    }
    CHECK(msg.find("linear system not positive definite") != std::string::npos);
    CHECK(msg.find("node " + std::to_string(expect) + ")") != std::string::npos);
}

TEST("anderson: anderson_combine and AndersonWindow match the oracle") {
    std::mt19937_64 rng(9);
    std::normal_distribution<double> g(0.0, 1.0);
    const int dim = 600;
    oracle::AndersonWindow ow(5);
    nrr::AndersonWindow pw(5);
    std::vector<double> x(dim, 0.0);
    for (int it = 0; it < 9; ++it) {
        std::vector<double> gv(dim);
        for (int i = 0; i < dim; ++i) gv[i] = 0.7 * x[i] + 0.1 * g(rng) + 1.0;
        std::vector<double> f(dim);
        for (int i = 0; i < dim; ++i) f[i] = gv[i] - x[i];
        ow.push(gv, f);
        pw.push(gv, f);
        const auto co = ow.combine();
        const auto cp = pw.combine();
        double scale = 1.0;
        for (double v : co) scale = std::max(scale, std::abs(v));
        CHECK(max_abs_diff(co, cp) <= 1e-10 * scale);
        CHECK(ow.extrapolating() == pw.extrapolating());
        x = co;
    }
}

TEST("solver: mm_step matches the oracle's fixed-point map") {
    const Case c = strip_case(10);
    nrr::SpatialIndex pti(c.ptgt.points);
    oracle::SpatialIndex oti(c.tgt.points);
    oracle::SolverConfig oc;
    nrr::SolverConfig pc;
    const auto op = oracle::init_parameters(c.src.points, c.src.avg_edge_length, oti, c.og, oc);
    const auto pp = nrr::init_parameters(c.psrc, pti, c.pg, pc);
    CHECK_APPROX(pp.nu_a, op.nu_a, 1e-15, 0.0);
    CHECK_APPROX(pp.alpha, op.alpha, 1e-15, 0.0);
    CHECK_APPROX(pp.beta, op.beta, 1e-15, 0.0);
    const auto x = oracle::NodeTransforms::identity(c.og.node_count());
    const auto xo = oracle::mm_step(c.src.points, c.og, oti, x, op);
    const auto xp = nrr::mm_step(c.psrc, c.pg, pti, P(x), pp);
    CHECK(max_abs_diff(xp.stacked.d, xo.stacked) <= 1e-9);
}

TEST("solver: register_surfaces (plain MM) follows the oracle's trajectory") {
    const Case c = strip_case(11);
    oracle::SolverConfig oc;
    oc.aa_window = 0;
    oc.i_max = 30;
    nrr::SolverConfig pc;
    pc.aa_window = 0;
    pc.i_max = 30;
    const auto ro = oracle::register_surfaces(c.src.points, c.src.avg_edge_length, c.tgt.points, c.og, oc);
    const auto rp = nrr::register_surfaces(c.psrc, c.ptgt, c.pg, pc);
    CHECK(rp.report.stages.size() == ro.report.stages.size());
    CHECK(rp.report.total_iterations() == ro.report.total_iterations());
    double worst = 0;
    for (size_t s = 0; s < std::min(rp.report.stages.size(), ro.report.stages.size()); ++s) {
        const auto& a = rp.report.stages[s].iterations;
        const auto& b = ro.report.stages[s].iterations;
        for (size_t k = 0; k < std::min(a.size(), b.size()); ++k)
            worst = std::max(worst, std::abs(a[k].e_total - b[k].e_total) / std::max(1e-300, std::abs(b[k].e_total)));
    }
    CHECK(worst <= 1e-6);
    double diag = 0;
    {
        nrr::Vec3 lo = rp.deformed_points[0], hi = lo;
        for (const auto& p : c.psrc.points) lo = lo.cwiseMin(p), hi = hi.cwiseMax(p);
        diag = (hi - lo).norm();
    }
    double m = 0;
    for (size_t i = 0; i < rp.deformed_points.size(); ++i)
        m = std::max(m, (rp.deformed_points[i] - P(ro.deformed_points[i])).norm());
    CHECK(m <= 1e-5 * diag);
}

TEST("solver: register_surfaces with Anderson acceleration, teacher-forced at every pass") {
    // AA trajectories are chaotic in floating point, so the
    // device run is checked pass by pass at its OWN iterates (the pass trace,
    // nrr_ctx_trace): at every evaluated X the oracle's correspondences must
    // be the device's (ties excepted), its energies within the north_star's
    // 1e-6, and every accept/revert decision the reference's rule
    // (solver.hpp:239) on the oracle energies, outside the tolerance band
    const Case c = strip_case(12);
    const oracle::SolverConfig oc;
    const auto ro = oracle::register_surfaces(c.src.points, c.src.avg_edge_length, c.tgt.points, c.og, oc);
    nrr::detail::ProblemArrays pa(c.psrc, &c.ptgt.points, c.pg);
    nrr::detail::LandmarkArrays la({});
    nrr_solver_config cfg = la.cfg;
    const nrr::SolverConfig pc;
    cfg.k_alpha = pc.k_alpha;
    cfg.k_beta = pc.k_beta;
    cfg.eps = pc.eps;
    cfg.i_max = pc.i_max;
    cfg.aa_window = pc.aa_window;
    cfg.nu_a_init = pc.nu_a_init;
    cfg.nu_a_min = pc.nu_a_min;
    cfg.nu_r_init = pc.nu_r_init;
    cfg.nu_r_floor = pc.nu_r_floor;
    nrr_ctx* ctx = nullptr;
    CHECK(nrr_ctx_create(0, &ctx) == 0);
    nrr_solve_options so{1e-13, 20000, 3, 0};
    CHECK(nrr_ctx_set_options(ctx, &so) == 0);
    const int N = c.pg.node_count(), n = c.psrc.point_count();
    std::vector<double> X(12 * static_cast<size_t>(N)), V(3 * static_cast<size_t>(n));
    CHECK(nrr_register(ctx, &pa.view, &cfg, X.data(), V.data()) == 0);
    nrr_report_summary sum{};
    CHECK(nrr_ctx_report(ctx, &sum, nullptr, 0, nullptr, 0, nullptr, 0, nullptr) == 0);
    std::vector<nrr_stage_record> st(sum.stage_count);
    CHECK(nrr_ctx_report(ctx, &sum, st.data(), sum.stage_count, nullptr, 0, nullptr, 0, nullptr) == 0);
    CHECK(static_cast<int>(st.size()) == static_cast<int>(ro.report.stages.size()));
    int passes = 0;
    CHECK(nrr_ctx_trace_count(ctx, &passes) == 0);
    CHECK(passes >= sum.total_iterations);
    const oracle::SpatialIndex ti(c.tgt.points);
    double worst_e = 0.0;
    int nn_diff = 0, flips = 0, checked = 0;
    double e_prev = INFINITY;
    int prev_stage = -1, accepted_in_stage = 0;
    bool after_revert = false;
    std::vector<double> xe(12 * static_cast<size_t>(N)), xm(12 * static_cast<size_t>(N));
    std::vector<int32_t> nn(n);
    for (int k = 0; k < passes; ++k) {
        nrr_pass_trace tr{};
        CHECK(nrr_ctx_trace(ctx, k, &tr, xe.data(), xm.data(), nn.data()) == 0);
        const auto& sr = st[tr.stage];
        oracle::NodeTransforms x = oracle::NodeTransforms::zeros(N);
        x.stacked = xe;
        const auto deformed = oracle::deform_points(c.src.points, c.og, x);
        const auto corr = oracle::find_correspondences(deformed, ti);
        for (int i = 0; i < n; ++i)
            if (corr.target_index[i] != nn[i]) {
                const auto d = c.tgt.points[nn[i]] - deformed[i];
                const double dg = d.squaredNorm(), dor = corr.squared_distance[i];
                if (std::abs(dg - dor) > 1e-6 * dor) ++nn_diff;  // only distance ties may differ
            }
        const auto rot = oracle::project_rotations(x);
        const auto e = oracle::evaluate_energy(deformed, x, c.og, corr, rot, {sr.alpha, sr.beta, sr.nu_a, sr.nu_r});
        worst_e = std::max(worst_e, std::abs(tr.e_total - e.total) / std::abs(e.total));
        // the safeguard: an AA iterate is rejected iff E > E_prev (solver.hpp:239)
        if (tr.stage != prev_stage) {  // window and E_prev reset per stage (solver.hpp:219-220)
            e_prev = INFINITY;
            accepted_in_stage = 0;
            after_revert = false;
            prev_stage = tr.stage;
        }
        // the iterate is an AA extrapolation once the window holds two
        // entries (anderson.hpp:64), and never right after a revert (x_mm)
        const bool is_aa = !after_revert && accepted_in_stage >= 2 && cfg.aa_window > 0;
        if (is_aa) {
            const bool rule = e.total > e_prev;
            if (rule != (tr.reverted != 0) && std::abs(e.total - e_prev) > 1e-6 * std::abs(e_prev)) ++flips;
        } else if (tr.reverted) {
            ++flips;  // plain iterates are always accepted (solver.hpp:240-243)
        }
        if (!tr.reverted) {
            e_prev = e.total;
            ++accepted_in_stage;
        }
        after_revert = tr.reverted != 0;
        ++checked;
    }
    nrr_ctx_destroy(ctx);
    CHECK(checked == passes);
    CHECK(nn_diff == 0);
    CHECK(worst_e <= 1e-6);
    CHECK(flips == 0);
    CHECK(sum.total_iterations > 0);
    std::printf("    AA teacher-forced: %d passes, worst energy rel %.2e, NN diffs %d, decision flips %d\n", passes,
                worst_e, nn_diff, flips);
}

TEST("errors: configuration and input errors use the reference's classes") {
    const Case c = strip_case(13, 8, 5);
    nrr::SolverConfig bad;
    bad.eps = 0.0;
    bool cfg = false;
    try {
        nrr::register_surfaces(c.psrc, c.ptgt, c.pg, bad);
    } catch (const nrr::ConfigError&) {
        cfg = true;
    }
    CHECK(cfg);
    bool empty = false;
    try {
        nrr::register_surfaces(c.psrc, nrr::Surface{}, c.pg, nrr::SolverConfig{});
    } catch (const nrr::NumericalError&) {
        empty = true;
    }
    CHECK(empty);
    nrr::SolverConfig lm;
    lm.landmarks.push_back({c.psrc.point_count() + 5, nrr::Vec3()});
    bool range = false;
    try {
        nrr::register_surfaces(c.psrc, c.ptgt, c.pg, lm);
    } catch (const nrr::ConfigError&) {
        range = true;
    }
    CHECK(range);
}

int main(int argc, char** argv) { return kat::run_all(argc, argv); }
