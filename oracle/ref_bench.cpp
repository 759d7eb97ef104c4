// swedg_refbench — times the UNMODIFIED reference CPU hot path (built against
// oracle/shim into oracle/_ref/) on the bench workload — TEST / BASELINE
// INFRASTRUCTURE ONLY (bench.py --impl reference and bench.py's cpu_baseline).
//
// Workload = bench.py's: modal ESDG (hybridized) degree N, smooth_state field
// (tests/test_solver.cpp:14-25 generator, seed 23) with lake bathymetry on the
// warped periodic [-1,1]^2 mesh, LSRK45 steps of the reference's own
// step_lsrk45 (solver.hpp:466-484) over rhs (solver.hpp:295) with
// ops.threads = T (parallel_for, parallel.hpp:14).  A bench "step" is one
// LSRK45 step (5 RHS stages).  Prints one JSON line.
//
//   swedg_refbench N K1D warmup steps threads [warp]
//   swedg_refbench ratio K threads     (bench.hpp ratio_sweep: the R_CPU study, CSV)
//   swedg_refbench run PROBLEM N SCHEME K1D warp cfl tfinal threads
//       the reference's build_case + run() (run.hpp:214-284) on lake|vortex|dambreak,
//       SCHEME hybridized|sbp (Gauss-Legendre edges): time to solution, one JSON line
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <thread>

#include "swedg/bench.hpp"
#include "swedg/run.hpp"
#include "swedg/solver.hpp"

using namespace swedg;

int main(int argc, char** argv) {
    if (argc >= 2 && std::string(argv[1]) == "ratio") {
        int K = argc > 2 ? std::atoi(argv[2]) : 64, threads = argc > 3 ? std::atoi(argv[3]) : 1;
        std::fputs(ratios_csv(ratio_sweep(default_bench_sizes(), K, threads, 0)).c_str(), stdout);
        return 0;
    }
    if (argc >= 2 && std::string(argv[1]) == "run") {
        if (argc < 10) {
            std::fprintf(stderr, "usage: swedg_refbench run PROBLEM N SCHEME K1D warp cfl tfinal threads\n");
            return 2;
        }
        RunConfig cfg;
        const std::string prob = argv[2], scheme = argv[4];
        cfg.problem = prob == "lake" ? ProblemId::Lake : prob == "vortex" ? ProblemId::Vortex : ProblemId::DamBreak;
        cfg.degree = std::atoi(argv[3]);
        cfg.scheme = scheme == "sbp" ? Scheme::SbpLegendre : Scheme::Hybridized;
        cfg.nx = cfg.ny = std::atoi(argv[5]);
        cfg.warp = std::atof(argv[6]);
        cfg.cfl = std::atof(argv[7]);
        cfg.tfinal = std::atof(argv[8]);
        cfg.threads = std::atoi(argv[9]);
        if (cfg.threads <= 0) cfg.threads = (int)std::thread::hardware_concurrency();
        cfg.validate();
        auto t0 = std::chrono::steady_clock::now();
        Case c = build_case(cfg);
        auto t1 = std::chrono::steady_clock::now();
        RunResult r = run(c);
        auto t2 = std::chrono::steady_clock::now();
        std::printf("{\"problem\": \"%s\", \"K\": %d, \"steps\": %d, \"dt\": %.17g, \"t\": %.17g, "
                    "\"run_s\": %.6g, \"setup_s\": %.6g, \"threads\": %d, \"samples\": %zu, "
                    "\"l2_h\": %.17g}\n",
                    prob.c_str(), c.num_elements(), r.steps, r.dt, c.time(),
                    std::chrono::duration<double>(t2 - t1).count(), std::chrono::duration<double>(t1 - t0).count(),
                    cfg.threads, r.series.size(), r.has_error ? r.error.err_h : -1.0);
        return 0;
    }
    if (argc < 6) {
        std::fprintf(stderr, "usage: swedg_refbench N K1D warmup steps threads [warp]\n");
        return 2;
    }
    int N = std::atoi(argv[1]), n = std::atoi(argv[2]), warm = std::atoi(argv[3]),
        steps = std::atoi(argv[4]), threads = std::atoi(argv[5]);
    double warp = argc > 6 ? std::atof(argv[6]) : 0.1;
    if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
    auto t0 = std::chrono::steady_clock::now();
    RefOperators ref = build_ref_operators(N);
    Mesh mesh = uniform_tri_mesh(n, n, {0, 0, 2, 2});
    set_mapping_degree(mesh, N);
    if (warp != 0.0) warp_mesh(mesh, warp);
    Connectivity conn = connect(mesh, true, true);
    Geometry geo = build_geometry(mesh, ref);
    FaceMatch fm = match_faces(mesh, conn, geo, ref);
    SolverOps ops = precompute_element_ops(ref, mesh, geo, conn, fm, 9.81, Penalty::LaxFriedrichs, threads);
    std::mt19937 rng(23);
    std::uniform_real_distribution<double> amp(-0.1, 0.1);
    double a1 = amp(rng), a2 = amp(rng), a3 = amp(rng);
    ExactFn fn = [=](double x, double y, double) -> ConsState {
        double h = 1.5 + a1 * std::sin(M_PI * x) * std::cos(M_PI * y);
        double u = a2 * std::cos(M_PI * x);
        double v = a3 * std::sin(M_PI * y);
        return {h, h * u, h * v};
    };
    State st = make_state(mesh, N, fn, lake_bathymetry);
    set_bathymetry(ops, st.b);
    double setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    double dt = compute_dt(mesh, N, 0.125);
    std::vector<Mat> res;
    auto rhs_fn = [&](const State& s) { return rhs(ops, s); };
    for (int i = 0; i < warm; ++i) step_lsrk45(st, rhs_fn, dt, res);
    auto t1 = std::chrono::steady_clock::now();
    for (int i = 0; i < steps; ++i) step_lsrk45(st, rhs_fn, dt, res);
    double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
    long K = mesh.num_elements();
    double dof = (double)K * ref.Np * 3;
    double gdofs = steps > 0 ? dof * 5.0 * steps / sec / 1e9 : 0.0;
    std::printf("{\"value\": %.6g, \"unit\": \"GDOF*stages/s\", \"ms_per_step\": %.6g, \"K\": %ld, \"N\": %d, "
                "\"K1D\": %d, \"threads\": %d, \"steps\": %d, \"warmup\": %d, \"setup_s\": %.3f, \"dt\": %.17g}\n",
                gdofs, steps > 0 ? sec * 1e3 / steps : 0.0, K, N, n, threads, steps, warm, setup_s, dt);
    return 0;
}
