// dropin_test — the C++ drop-in path end to end: the UNMODIFIED reference
// (built against oracle/shim) sets up a problem and evaluates its own rhs();
// the same objects go through include/swedg_b200.hpp (C ABI -> CUDA) and the
// results are compared in-process.  TEST INFRASTRUCTURE (built into
// oracle/_ref/, linked against paper_2005_02516_b200/libswedg_b200.so, run by
// tests/test_dropin.py on the GPU).
//
// Exit code = number of failed checks; one line per check on stdout.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>

#include "swedg/run.hpp"
#include "swedg/solver.hpp"
#include "swedg_b200.hpp"
#include "swedg_b200_run.hpp"

using namespace swedg;

static int failures = 0;
static void check(bool ok, const std::string& what, double v = 0.0) {
    std::printf("%s %s %.3e\n", ok ? "PASS" : "FAIL", what.c_str(), v);
    if (!ok) ++failures;
}

static double max_rel(const std::vector<Mat>& a, const std::vector<Mat>& b) {
    double d = 0.0, s = 0.0;
    for (size_t k = 0; k < a.size(); ++k) {
        d = std::max(d, (a[k] - b[k]).cwiseAbs().maxCoeff());
        s = std::max(s, b[k].cwiseAbs().maxCoeff());
    }
    return d / (1.0 + s);
}

// tests/test_solver.cpp:14-25
static State smooth_state(const Mesh& mesh, int N, unsigned seed) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> amp(-0.1, 0.1);
    double a1 = amp(rng), a2 = amp(rng), a3 = amp(rng);
    ExactFn fn = [=](double x, double y, double) -> ConsState {
        double h = 1.5 + a1 * std::sin(M_PI * x) * std::cos(M_PI * y);
        double u = a2 * std::cos(M_PI * x);
        double v = a3 * std::sin(M_PI * y);
        return {h, h * u, h * v};
    };
    return make_state(mesh, N, fn, lake_bathymetry);
}

int main() {
    // ---- hybridized N = 4, curved periodic mesh (test_solver.cpp Fixture)
    for (int N : {3, 4}) {
        RefOperators ref = build_ref_operators(N);
        Mesh mesh = uniform_tri_mesh(6, 6, {0, 0, 2, 2});
        set_mapping_degree(mesh, N);
        warp_mesh(mesh, 0.1);
        Connectivity conn = connect(mesh, true, true);
        Geometry geo = build_geometry(mesh, ref);
        FaceMatch fm = match_faces(mesh, conn, geo, ref);
        SolverOps ops = precompute_element_ops(ref, mesh, geo, conn, fm, 9.81);
        State st = smooth_state(mesh, N, 23);
        set_bathymetry(ops, st.b);
        auto du_ref = rhs(ops, st);

        std::string tag = "N=" + std::to_string(N);
        auto par = swedg_b200::precompute_element_ops(ref, mesh, geo, conn, fm, 9.81, SWEDG_PENALTY_LF,
                                                      swedg_b200::Mode::Parity, 0, &ops);
        swedg_b200::set_bathymetry(par, st.b);
        auto du_par = swedg_b200::rhs(par, st);
        check(max_rel(du_par, du_ref) == 0.0, tag + " parity rhs bitwise == reference rhs", max_rel(du_par, du_ref));
        auto proj_ref = entropy_projection(ops, st);
        auto proj_par = swedg_b200::entropy_projection(par, st);
        check(max_rel(proj_par, proj_ref) == 0.0, tag + " parity entropy_projection bitwise", max_rel(proj_par, proj_ref));

        auto fast = swedg_b200::precompute_element_ops(ref, mesh, geo, conn, fm, 9.81);  // Mh_inv formed in the adapter
        swedg_b200::set_bathymetry(fast, st.b);
        auto du_fast = swedg_b200::rhs(fast, st);
        check(max_rel(du_fast, du_ref) <= 1e-12, tag + " fast rhs within 1e-12", max_rel(du_fast, du_ref));

        // five LSRK45 steps: reference loop vs device-resident steps
        double dt = compute_dt(mesh, N, 0.125);
        State s_ref = st, s_gpu = st, s_par = st;
        std::vector<Mat> res;
        for (int i = 0; i < 5; ++i) step_lsrk45(s_ref, [&](const State& s) { return rhs(ops, s); }, dt, res);
        swedg_b200::step_lsrk45(s_par, par, dt, 5);
        swedg_b200::step_lsrk45(s_gpu, fast, dt, 5);
        check(max_rel(s_par.u, s_ref.u) == 0.0, tag + " parity 5 LSRK45 steps bitwise", max_rel(s_par.u, s_ref.u));
        check(max_rel(s_gpu.u, s_ref.u) <= 1e-12, tag + " fast 5 LSRK45 steps within 1e-12", max_rel(s_gpu.u, s_ref.u));
        check(std::abs(s_gpu.t - s_ref.t) == 0.0, tag + " time bookkeeping", s_gpu.t - s_ref.t);
    }

    // ---- error convention: negative height in element 1 (test_solver.cpp:355-371)
    {
        int N = 2;
        RefOperators ref = build_ref_operators(N);
        Mesh mesh = uniform_tri_mesh(2, 2, {0, 0, 2, 2});
        set_mapping_degree(mesh, N);
        Connectivity conn = connect(mesh, true, true);
        Geometry geo = build_geometry(mesh, ref);
        FaceMatch fm = match_faces(mesh, conn, geo, ref);
        int K = mesh.num_elements();
        std::vector<Vec> b(K, Vec::Zero(ref.Np));
        State st;
        st.N = N;
        for (int k = 0; k < K; ++k) {
            Mat u = Mat::Zero(ref.Np, 3);
            u(0, 0) = std::sqrt(2.0);
            st.u.push_back(u);
            st.b.push_back(b[k]);
        }
        st.u[1](0, 0) = -std::sqrt(2.0);
        auto dops = swedg_b200::precompute_element_ops(ref, mesh, geo, conn, fm, 9.81);
        swedg_b200::set_bathymetry(dops, b);
        bool threw = false;
        try {
            swedg_b200::rhs(dops, st);
        } catch (const std::runtime_error& e) {
            threw = std::string(e.what()).find("element 1") != std::string::npos;
            std::printf("     message: %s\n", e.what());
        }
        check(threw, "positivity failure reports element 1");
        bool inv = false;
        try {
            swedg_b200::step_lsrk45(st, dops, -1.0);
        } catch (const std::invalid_argument&) {
            inv = true;
        }
        check(inv, "dt <= 0 throws invalid_argument");
    }

    // ---- SBP dam break N = 4 (walls, curved dam)
    {
        RunConfig cfg;
        cfg.problem = ProblemId::DamBreak;
        cfg.degree = 4;
        cfg.nx = cfg.ny = 12;
        cfg.scheme = Scheme::SbpLegendre;
        cfg.cfl = 0.0625;
        Case c = build_case(cfg);
        auto du_ref = rhs_sbp(c.sops, c.nstate);
        auto par = swedg_b200::precompute_sbp_ops(c.ref, *c.tsbp, c.mesh, c.geo, c.conn, c.fm, c.cfg.g,
                                                  SWEDG_PENALTY_LF, swedg_b200::Mode::Parity);
        swedg_b200::set_bathymetry(par, c.nstate.b);
        auto du_par = swedg_b200::rhs(par, c.nstate);
        check(max_rel(du_par, du_ref) == 0.0, "SBP N=4 dam parity rhs bitwise", max_rel(du_par, du_ref));
    }
    // ---- run() time loop + diagnostics (run.hpp:226-284) through swedg_b200_run.hpp
    struct RunCase {
        ProblemId p;
        Scheme s;
        int N, n;
        double warp, tfinal;
        const char* tag;
    };
    for (const RunCase& rc : {RunCase{ProblemId::Vortex, Scheme::Hybridized, 3, 8, 0.0, 0.2, "vortex N=3"},
                              RunCase{ProblemId::Lake, Scheme::Hybridized, 3, 6, 0.1, 0.05, "lake N=3 curved"},
                              RunCase{ProblemId::Lake, Scheme::SbpLegendre, 3, 4, 0.1, 0.02, "SBP lake N=3"},
                              RunCase{ProblemId::DamBreak, Scheme::SbpLegendre, 4, 10, 0.0, 0.02, "SBP dam N=4"}}) {
        RunConfig cfg;
        cfg.problem = rc.p;
        cfg.scheme = rc.s;
        cfg.degree = rc.N;
        cfg.nx = cfg.ny = rc.n;
        cfg.warp = rc.warp;
        cfg.tfinal = rc.tfinal;
        if (rc.p == ProblemId::DamBreak) cfg.cfl = 0.0625;
        Case cr = build_case(cfg), cd = build_case(cfg);
        FineQuad fq(cfg.degree);
        Invariants i_ref = compute_invariants(fq, cr.geo, cr.modal_solution(), cr.modal_bathymetry(), cr.cfg.g, cr.time());
        RunResult r_ref = run(cr);
        auto ops = swedg_b200::make_device_ops(cd, swedg_b200::Mode::Parity);
        Invariants i_dev = swedg_b200::compute_invariants(ops, cd);
        const std::string tag = rc.tag;
        auto rel = [](double a, double b) { return std::abs(a - b) / (1.0 + std::abs(b)); };
        double d0 = std::max({rel(i_dev.mass, i_ref.mass), rel(i_dev.momentum_x, i_ref.momentum_x),
                              rel(i_dev.momentum_y, i_ref.momentum_y), rel(i_dev.entropy, i_ref.entropy)});
        check(d0 <= 1e-13 && i_dev.min_h == i_ref.min_h, tag + " compute_invariants (exact sums vs serial)", d0);
        RunResult r_dev = swedg_b200::run(cd, ops);
        check(r_dev.steps == r_ref.steps && r_dev.series.size() == r_ref.series.size() && r_dev.dt == r_ref.dt,
              tag + " run(): steps and samples", (double)r_dev.steps);
        double ds = 0.0;
        bool times = true;
        for (size_t i = 0; i < std::min(r_dev.series.size(), r_ref.series.size()); ++i) {
            const Invariants &a = r_dev.series[i], &b = r_ref.series[i];
            times = times && a.t == b.t && a.min_h == b.min_h;
            ds = std::max({ds, rel(a.mass, b.mass), rel(a.momentum_x, b.momentum_x), rel(a.momentum_y, b.momentum_y),
                           rel(a.entropy, b.entropy)});
        }
        check(times && ds <= 1e-13, tag + " run(): invariant series", ds);
        const auto& ud = cd.sbp ? cd.nstate.u : cd.hstate.u;
        const auto& ur = cr.sbp ? cr.nstate.u : cr.hstate.u;
        check(max_rel(ud, ur) == 0.0 && cd.time() == cr.time(), tag + " run(): final state bitwise (parity)",
              max_rel(ud, ur));
        if (r_ref.has_error)
            check(r_dev.has_error && rel(r_dev.error.combined, r_ref.error.combined) <= 1e-11 &&
                      r_dev.error.h_mesh == r_ref.error.h_mesh,
                  tag + " run(): L2 error", rel(r_dev.error.combined, r_ref.error.combined));
    }
    std::printf("%s\n", failures ? "FAILURES" : "all drop-in checks passed");
    return failures;
}
