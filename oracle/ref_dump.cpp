// swedg_dump — golden-vector generator built from the UNMODIFIED reference
// headers (/root/reference/proj/include) against oracle/shim — TEST
// INFRASTRUCTURE ONLY (built into oracle/_ref/ by oracle/Makefile.ref).
//
// Each sub-command builds one case exactly the way the reference's own tests
// and case builders do (tests/test_solver.cpp:27-45 Fixture, run.hpp:116-209
// build_*_case), evaluates the reference hot path (solver.hpp entropy_projection,
// rhs, rhs_sbp, step_lsrk45) and writes every input and output array to a
// simple binary container that tests/golden/make_golden.py converts to .npz.
//
// Container: repeated records
//   u32 name_len, name bytes, u8 dtype (0 = f64, 1 = i32), u32 ndim,
//   u64 dims[ndim], raw little-endian data (C order).
// Per-element Eigen matrices (column-major r x c) are stacked as [K][c][r].
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <iterator>
#include <string>
#include <vector>

#include "swedg/bench.hpp"
#include "swedg/run.hpp"
#include "swedg/solver.hpp"

using namespace swedg;

namespace {

struct Writer {
    std::ofstream out;
    explicit Writer(const std::string& path) : out(path, std::ios::binary) {
        if (!out) throw std::runtime_error("cannot open " + path);
    }
    void header(const std::string& name, uint8_t dtype, const std::vector<uint64_t>& dims) {
        uint32_t n = static_cast<uint32_t>(name.size());
        out.write(reinterpret_cast<const char*>(&n), 4);
        out.write(name.data(), n);
        out.write(reinterpret_cast<const char*>(&dtype), 1);
        uint32_t nd = static_cast<uint32_t>(dims.size());
        out.write(reinterpret_cast<const char*>(&nd), 4);
        for (uint64_t d : dims) out.write(reinterpret_cast<const char*>(&d), 8);
    }
    void f64(const std::string& name, const std::vector<uint64_t>& dims, const double* p) {
        header(name, 0, dims);
        uint64_t n = 1;
        for (auto d : dims) n *= d;
        out.write(reinterpret_cast<const char*>(p), static_cast<std::streamsize>(n * 8));
    }
    void i32(const std::string& name, const std::vector<uint64_t>& dims, const int* p) {
        header(name, 1, dims);
        uint64_t n = 1;
        for (auto d : dims) n *= d;
        out.write(reinterpret_cast<const char*>(p), static_cast<std::streamsize>(n * 4));
    }
    void scalar(const std::string& name, double v) { f64(name, {1}, &v); }
    void iscalar(const std::string& name, int v) { i32(name, {1}, &v); }
    void mat(const std::string& name, const Mat& m) {
        f64(name, {static_cast<uint64_t>(m.cols()), static_cast<uint64_t>(m.rows())}, m.data());
    }
    void vec(const std::string& name, const Vec& v) {
        f64(name, {static_cast<uint64_t>(v.size())}, v.data());
    }
    // stack per-element matrices as [K][c][r]
    void mats(const std::string& name, const std::vector<Mat>& ms) {
        uint64_t K = ms.size(), r = ms[0].rows(), c = ms[0].cols();
        std::vector<double> buf;
        buf.reserve(K * r * c);
        for (const auto& m : ms) buf.insert(buf.end(), m.data(), m.data() + r * c);
        f64(name, {K, c, r}, buf.data());
    }
    void vecs(const std::string& name, const std::vector<Vec>& vs) {
        uint64_t K = vs.size(), n = vs[0].size();
        std::vector<double> buf;
        buf.reserve(K * n);
        for (const auto& v : vs) buf.insert(buf.end(), v.data(), v.data() + n);
        f64(name, {K, n}, buf.data());
    }
};

// tests/test_solver.cpp:14-25 (identical generator, same seeds)
State smooth_state(const Mesh& mesh, int N, unsigned seed) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> amp(-0.1, 0.1);
    double a1 = amp(rng), a2 = amp(rng), a3 = amp(rng);
    ExactFn fn = [=](double x, double y, double) -> ConsState {
        double h = 1.5 + a1 * std::sin(M_PI * x) * std::cos(M_PI * y);
        double u = a2 * std::cos(M_PI * x);
        double v = a3 * std::sin(M_PI * y);
        return {h, h * u, h * v};
    };
    return make_state(mesh, N, fn, [](double, double) { return 0.0; });
}

// tests/test_solver.cpp:176-189 bathymetry in P^N
std::vector<Vec> entropy_test_bathymetry(const Mesh& mesh, int N, int Np) {
    LatticeInterp li(N);
    std::vector<Vec> b(mesh.num_elements());
    for (int k = 0; k < mesh.num_elements(); ++k) {
        Vec bv(Np);
        for (int i = 0; i < bv.size(); ++i) {
            double x = mesh.map_nodes[k](i, 0), y = mesh.map_nodes[k](i, 1);
            bv[i] = 0.05 * std::sin(M_PI * x) * std::sin(M_PI * y) + 0.1 * std::cos(M_PI * x);
        }
        b[k] = li.coeffs(bv);
    }
    return b;
}

void write_ref_ops(Writer& w, const RefOperators& ref) {
    w.iscalar("N", ref.N);
    w.iscalar("Np", ref.Np);
    w.iscalar("nq", ref.volq.size());
    w.iscalar("nf", ref.surfq.size());
    w.iscalar("npf", ref.surfq.nodes_per_face);
    w.mat("ref_Vq", ref.Vq);
    w.mat("ref_Vf", ref.Vf);
    w.mat("ref_Pq", ref.Pq);
    w.mat("ref_Qh_x", ref.Qh_x);
    w.mat("ref_Qh_y", ref.Qh_y);
    w.mat("ref_Qh_skew_x", ref.Qh_skew_x);
    w.mat("ref_Qh_skew_y", ref.Qh_skew_y);
    w.mat("ref_M", ref.M);
    w.mat("ref_Dx", ref.Dx);
    w.mat("ref_Dy", ref.Dy);
    w.vec("volq_x", ref.volq.x);
    w.vec("volq_y", ref.volq.y);
    w.vec("volq_w", ref.volq.w);
    w.vec("surfq_x", ref.surfq.x);
    w.vec("surfq_y", ref.surfq.y);
    w.vec("surfq_w", ref.surfq.w);
}

void write_mesh_geo(Writer& w, const Mesh& mesh, const Connectivity& conn, const Geometry& geo,
                    const FaceMatch& fm, int npf) {
    int K = mesh.num_elements();
    w.iscalar("K", K);
    std::vector<double> verts;
    for (auto& v : mesh.verts) verts.insert(verts.end(), {v[0], v[1]});
    w.f64("mesh_verts", {mesh.verts.size(), 2}, verts.data());
    std::vector<int> tris;
    for (auto& t : mesh.tris) tris.insert(tris.end(), {t[0], t[1], t[2]});
    w.i32("mesh_tris", {static_cast<uint64_t>(K), 3}, tris.data());
    w.mats("map_nodes", mesh.map_nodes);
    std::vector<Mat> gf, xys;
    std::vector<Vec> J, sJ, nx, ny;
    for (auto& e : geo.elems) {
        gf.push_back(e.gf);
        xys.push_back(e.xy_surf);
        J.push_back(e.J_vol);
        sJ.push_back(e.sJ);
        nx.push_back(e.nx);
        ny.push_back(e.ny);
    }
    w.mats("gf", gf);
    w.mats("xy_surf", xys);
    w.vecs("J_vol", J);
    w.vecs("sJ", sJ);
    w.vecs("nx", nx);
    w.vecs("ny", ny);
    std::vector<int> nbr, nbr_face, ftype, perm;
    std::vector<double> shift;
    for (int k = 0; k < K; ++k)
        for (int f = 0; f < 3; ++f) {
            const FaceInfo& fi = conn.faces[k][f];
            nbr.push_back(fi.type == FaceType::Wall ? -1 : fi.nbr_elem);
            nbr_face.push_back(fi.nbr_face);
            ftype.push_back(static_cast<int>(fi.type));
            shift.insert(shift.end(), {fi.shift[0], fi.shift[1]});
            for (int s = 0; s < npf; ++s)
                perm.push_back(fi.type == FaceType::Wall ? -1 : fm.perm[k][f][s]);
        }
    w.i32("nbr", {static_cast<uint64_t>(K), 3}, nbr.data());
    w.i32("nbr_face", {static_cast<uint64_t>(K), 3}, nbr_face.data());
    w.i32("face_type", {static_cast<uint64_t>(K), 3}, ftype.data());
    w.f64("face_shift", {static_cast<uint64_t>(K), 3, 2}, shift.data());
    w.i32("perm", {static_cast<uint64_t>(K), static_cast<uint64_t>(3 * npf)}, perm.data());
}

void write_elem_ops(Writer& w, const SolverOps& ops, int n_full_skew) {
    std::vector<Mat> Minv, Mh;
    std::vector<Vec> Bx, By, wsj, bs, sx, sy;
    for (auto& eo : ops.elem) {
        Minv.push_back(eo.Mh_inv);
        Mh.push_back(eo.Mh);
        Bx.push_back(eo.Bx);
        By.push_back(eo.By);
        wsj.push_back(eo.wf_sJ);
        bs.push_back(eo.b_stacked);
        sx.push_back(eo.src_x);
        sy.push_back(eo.src_y);
    }
    w.mats("Mh_inv", Minv);
    w.mats("Mh", Mh);
    w.vecs("Bx", Bx);
    w.vecs("By", By);
    w.vecs("wf_sJ", wsj);
    w.vecs("b_stacked", bs);
    w.vecs("src_x", sx);
    w.vecs("src_y", sy);
    std::vector<Mat> qx, qy;
    for (int k = 0; k < n_full_skew && k < static_cast<int>(ops.elem.size()); ++k) {
        qx.push_back(ops.elem[k].Qh_skew_x);
        qy.push_back(ops.elem[k].Qh_skew_y);
    }
    if (!qx.empty()) {
        w.mats("Qh_skew_x_elem", qx);
        w.mats("Qh_skew_y_elem", qy);
    }
}

// Modal (hybridized) fixture on the lake domain [-1,1]^2 (test_solver.cpp:27-45).
// bathy: 0 = zero, 1 = entropy-test bathymetry.  Evaluates proj, du(LF), du(EC),
// the entropy/conservation hooks and `nsteps` LSRK45 steps of size dt (LF).
int cmd_modal(const std::string& path, int N, int n, double warp, bool periodic, unsigned seed,
              int bathy, int nsteps, double dt) {
    Writer w(path);
    RefOperators ref = build_ref_operators(N);
    Mesh mesh = uniform_tri_mesh(n, n, {0, 0, 2, 2});
    set_mapping_degree(mesh, N);
    if (warp != 0.0) warp_mesh(mesh, warp);
    Connectivity conn = connect(mesh, periodic, periodic);
    Geometry geo = build_geometry(mesh, ref);
    FaceMatch fm = match_faces(mesh, conn, geo, ref);
    double g = 9.81;
    SolverOps ops = precompute_element_ops(ref, mesh, geo, conn, fm, g);
    int K = mesh.num_elements();
    std::vector<Vec> b = bathy == 1 ? entropy_test_bathymetry(mesh, N, ref.Np)
                                    : std::vector<Vec>(K, Vec::Zero(ref.Np));
    set_bathymetry(ops, b);
    State st = smooth_state(mesh, N, seed);
    st.b = b;

    write_ref_ops(w, ref);
    w.scalar("g", g);
    w.iscalar("scheme", 0);
    write_mesh_geo(w, mesh, conn, geo, fm, ref.surfq.nodes_per_face);
    write_elem_ops(w, ops, 4);
    w.mats("u", st.u);
    w.vecs("b", st.b);

    auto proj = entropy_projection(ops, st);
    w.mats("proj", proj);
    ops.penalty = Penalty::LaxFriedrichs;
    auto du_lf = rhs(ops, st, proj);
    w.mats("du_lf", du_lf);
    w.scalar("entropy_rate_lf", entropy_rate(ops, st, du_lf));
    auto cr = conservation_rate(ops, du_lf);
    w.f64("conservation_rate_lf", {3}, cr.data());
    ops.penalty = Penalty::EntropyConservative;
    auto du_ec = rhs(ops, st, proj);
    w.mats("du_ec", du_ec);
    w.scalar("entropy_rate_ec", entropy_rate(ops, st, du_ec));

    // volume-only accumulator of element 0..3 (skew kernel alone) for kernel parity
    {
        std::vector<Mat> accs;
        for (int k = 0; k < std::min(K, 4); ++k) {
            Mat acc = Mat::Zero(ref.n_stack(), 3);
            detail::skew_volume_kernel(ops.elem[k].Qh_skew_x, ops.elem[k].Qh_skew_y, proj[k],
                                       ref.volq.size(), g, acc);
            accs.push_back(acc);
        }
        w.mats("vol_acc_first4", accs);
    }

    if (nsteps > 0) {
        ops.penalty = Penalty::LaxFriedrichs;
        w.scalar("dt", dt);
        w.iscalar("nsteps", nsteps);
        std::vector<Mat> res;
        State s2 = st;
        for (int i = 0; i < nsteps; ++i)
            step_lsrk45(s2, [&](const State& s) { return rhs(ops, s); }, dt, res);
        w.mats("u_steps", s2.u);
        w.mats("res_steps", res);
        w.scalar("t_steps", s2.t);
    }
    return 0;
}

// compute_invariants and both l2_error forms of the case's current state, the
// way run() calls them (run.hpp:236-238, 264-270).
void dump_diagnostics(Writer& w, const Case& c, const FineQuad& fq, const std::string& p) {
    Invariants inv = compute_invariants(fq, c.geo, c.modal_solution(), c.modal_bathymetry(), c.cfg.g, c.time());
    double iv[6] = {inv.t, inv.mass, inv.momentum_x, inv.momentum_y, inv.entropy, inv.min_h};
    w.f64(p + "invariants", {6}, iv);
    if (!c.ref_state.empty()) {
        ErrorReport e = l2_error(fq, c.geo, c.modal_solution(), c.ref_state);
        double ev[4] = {e.err_h, e.err_hu, e.err_hv, e.combined};
        w.f64(p + "l2_ref", {4}, ev);
        w.mats(p + "ref_state", c.ref_state);
    }
    if (c.exact) {
        ErrorReport e = l2_error(fq, c.geo, c.modal_solution(), c.exact, c.time());
        double ev[4] = {e.err_h, e.err_hu, e.err_hv, e.combined};
        w.f64(p + "l2_exact", {4}, ev);
    }
}

// Named reference problems through run.hpp's builders and run() loop.
int cmd_problem(const std::string& path, const std::string& problem, int N,
                const std::string& scheme, int n, double warp, double cfl, double tfinal,
                int store_inputs) {
    Writer w(path);
    RunConfig cfg;
    cfg.problem = problem == "lake" ? ProblemId::Lake
                  : problem == "vortex" ? ProblemId::Vortex
                                        : ProblemId::DamBreak;
    cfg.degree = N;
    cfg.scheme = scheme == "sbp" ? Scheme::SbpLegendre : Scheme::Hybridized;
    cfg.nx = cfg.ny = n;
    cfg.warp = warp;
    cfg.cfl = cfl;
    cfg.tfinal = tfinal;
    Case c = build_case(cfg);
    int K = c.num_elements();
    int npf = c.ref.surfq.nodes_per_face;
    write_ref_ops(w, c.ref);
    w.scalar("g", c.cfg.g);
    w.iscalar("scheme", c.sbp ? 1 : 0);
    w.scalar("cfl", cfl);
    w.scalar("tfinal", tfinal);
    w.scalar("dt", compute_dt(c.mesh, N, cfl));
    w.scalar("min_edge", min_edge_length(c.mesh));
    if (store_inputs) {
        write_mesh_geo(w, c.mesh, c.conn, c.geo, c.fm, npf);
    } else {
        w.iscalar("K", K);
    }
    if (!c.sbp) {
        if (store_inputs) write_elem_ops(w, c.hops, 0);
        w.mats("u", c.hstate.u);
        w.vecs("b", c.hstate.b);
        auto du = rhs(c.hops, c.hstate);
        w.mats("du_lf", du);
    } else {
        const TraditionalSBP& t = *c.tsbp;
        w.mat("sbp_Qx", t.Q_SBP_x);
        w.mat("sbp_Qy", t.Q_SBP_y);
        w.vec("sbp_M_diag", t.M_diag);
        w.i32("sbp_face_index", {t.face_index.size()}, t.face_index.data());
        if (store_inputs) {
            std::vector<Vec> minv, sx, sy, bx, by, wsj;
            for (auto& eo : c.sops.elem) {
                minv.push_back(eo.Minv_diag);
                sx.push_back(eo.src_x);
                sy.push_back(eo.src_y);
                bx.push_back(eo.Bx);
                by.push_back(eo.By);
                wsj.push_back(eo.wf_sJ);
            }
            w.vecs("Minv_diag", minv);
            w.vecs("src_x", sx);
            w.vecs("src_y", sy);
            w.vecs("Bx", bx);
            w.vecs("By", by);
            w.vecs("wf_sJ", wsj);
        }
        w.mats("u", c.nstate.u);
        w.vecs("b", c.nstate.b);
        auto du = rhs_sbp(c.sops, c.nstate);
        w.mats("du_lf", du);
        c.sops.penalty = Penalty::EntropyConservative;
        auto du_ec = rhs_sbp(c.sops, c.nstate);
        w.mats("du_ec", du_ec);
        c.sops.penalty = Penalty::LaxFriedrichs;
    }
    // diagnostics inputs and outputs (diagnostics.hpp:142-267) on the initial state
    FineQuad fq(N);
    w.vec("fine_w", fq.rule.w);
    w.mat("fine_V", fq.V);
    w.mat("fine_Vr", fq.Vx);
    w.mat("fine_Vs", fq.Vy);
    {
        std::vector<Mat> mc;
        for (auto& e : c.geo.elems) mc.push_back(e.map_coeffs);
        w.mats("map_coeffs", mc);
    }
    dump_diagnostics(w, c, fq, "diag0_");
    if (tfinal > 0) {
        RunResult r = run(c);
        w.iscalar("run_steps", r.steps);
        w.scalar("run_dt", r.dt);
        w.scalar("run_t", c.time());
        w.scalar("run_err_combined", r.has_error ? r.error.combined : -1.0);
        std::vector<double> inv;
        for (auto& s : r.series)
            inv.insert(inv.end(), {s.t, s.mass, s.momentum_x, s.momentum_y, s.entropy, s.min_h});
        w.f64("run_invariants", {r.series.size(), 6}, inv.data());
        if (!c.sbp)
            w.mats("u_final", c.hstate.u);
        else
            w.mats("u_final", c.nstate.u);
        w.scalar("run_err_h", r.has_error ? r.error.err_h : -1.0);
        w.scalar("run_err_hu", r.has_error ? r.error.err_hu : -1.0);
        w.scalar("run_err_hv", r.has_error ? r.error.err_hv : -1.0);
        dump_diagnostics(w, c, fq, "diag1_");
    }
    return 0;
}

// Reference operator tables for N = 1..4 (modal rule and SBP-Legendre rule).
int cmd_ops(const std::string& path) {
    Writer w(path);
    for (int N = 1; N <= 4; ++N) {
        RefOperators ref = build_ref_operators(N);
        std::string p = "N" + std::to_string(N) + "_";
        w.mat(p + "Vq", ref.Vq);
        w.mat(p + "Vf", ref.Vf);
        w.mat(p + "Pq", ref.Pq);
        w.mat(p + "M", ref.M);
        w.mat(p + "Dx", ref.Dx);
        w.mat(p + "Dy", ref.Dy);
        w.mat(p + "Qh_x", ref.Qh_x);
        w.mat(p + "Qh_y", ref.Qh_y);
        w.vec(p + "volq_x", ref.volq.x);
        w.vec(p + "volq_y", ref.volq.y);
        w.vec(p + "volq_w", ref.volq.w);
        w.vec(p + "surfq_x", ref.surfq.x);
        w.vec(p + "surfq_y", ref.surfq.y);
        w.vec(p + "surfq_w", ref.surfq.w);
        auto sq = sbp_rule(N, EdgeFamily::GaussLegendre);
        RefOperators sref = build_ref_operators(N, sq.vol, sq.surf);
        TraditionalSBP t = build_traditional_sbp(sref, sq);
        w.vec(p + "sbp_x", sq.vol.x);
        w.vec(p + "sbp_y", sq.vol.y);
        w.vec(p + "sbp_w", sq.vol.w);
        w.mat(p + "sbp_Vq", sref.Vq);
        w.mat(p + "sbp_Pq", sref.Pq);
        w.mat(p + "sbp_Qx", t.Q_SBP_x);
        w.mat(p + "sbp_Qy", t.Q_SBP_y);
        w.i32(p + "sbp_face_index", {t.face_index.size()}, t.face_index.data());
    }
    // every tabulated volume rule used for N <= 7 and the fine rules (degree <= 16)
    for (int d = 1; d <= 16; ++d) {
        Quadrature2D q = volume_rule_by_degree(d);
        std::string p = "volrule_deg" + std::to_string(d) + "_";
        w.vec(p + "x", q.x);
        w.vec(p + "y", q.y);
        w.vec(p + "w", q.w);
        w.iscalar(p + "degree", q.degree);
    }
    return 0;
}

// The positivity-failure case of test_solver.cpp:355-371.
int cmd_positivity(const std::string& path) {
    Writer w(path);
    int N = 2;
    RefOperators ref = build_ref_operators(N);
    Mesh mesh = uniform_tri_mesh(2, 2, {0, 0, 2, 2});
    set_mapping_degree(mesh, N);
    Connectivity conn = connect(mesh, true, true);
    Geometry geo = build_geometry(mesh, ref);
    FaceMatch fm = match_faces(mesh, conn, geo, ref);
    SolverOps ops = precompute_element_ops(ref, mesh, geo, conn, fm, 9.81);
    int K = mesh.num_elements();
    std::vector<Vec> b(K, Vec::Zero(ref.Np));
    set_bathymetry(ops, b);
    State st;
    st.N = N;
    for (int k = 0; k < K; ++k) {
        Mat u = Mat::Zero(ref.Np, 3);
        u(0, 0) = std::sqrt(2.0) * 1.0;
        st.u.push_back(u);
        st.b.push_back(b[k]);
    }
    st.u[1](0, 0) = -std::sqrt(2.0);
    std::string msg;
    try {
        rhs(ops, st);
    } catch (const std::runtime_error& e) {
        msg = e.what();
    }
    write_ref_ops(w, ref);
    w.scalar("g", 9.81);
    w.iscalar("scheme", 0);
    write_mesh_geo(w, mesh, conn, geo, fm, ref.surfq.nodes_per_face);
    write_elem_ops(w, ops, 0);
    w.mats("u", st.u);
    w.vecs("b", st.b);
    std::vector<int> m(msg.begin(), msg.end());
    w.i32("error_message", {m.size()}, m.data());
    return 0;
}

// bench.hpp's volume-kernel cost study (kernel_matvec / kernel_fluxdiff /
// kernel_fluxdiff_skew, bench.hpp:55-128) on the ratio_sweep operators and
// states (random_operator / random_states, seeded as ratio_sweep does).
int cmd_ratio(const std::string& path) {
    Writer w(path);
    const double g = 9.81;
    const int K = 4;
    std::vector<int> sizes = {6, 10, 15, 21, 28, 36, 50};
    w.i32("sizes", {sizes.size()}, sizes.data());
    for (int n : sizes) {
        std::mt19937 rng(0u + static_cast<unsigned>(n));
        Mat Q = random_operator(n, rng);
        BenchStates s = random_states(n, K, rng);
        std::string p = "n" + std::to_string(n) + "_";
        w.mat(p + "Q", Q);
        w.mats(p + "u", s.u);
        w.mats(p + "y_dg", kernel_matvec(Q, s, g));
        w.mats(p + "y_esdg", kernel_fluxdiff(Q, s, g));
        // block-zero operator for the skew variant (nq = 2n/3)
        int nq = (2 * n) / 3;
        Mat Qz = Q;
        Qz.bottomRightCorner(n - nq, n - nq).setZero();
        w.iscalar(p + "nq", nq);
        w.mats(p + "y_skew", kernel_fluxdiff_skew(Qz, nq, s, g));
    }
    return 0;
}

// Output formats (diagnostics.hpp:272-375, mesh.hpp:462-493): the reference's own
// writers' bytes for small cases, with the inputs they were written from.
std::vector<int> file_bytes(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    std::string s((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    return std::vector<int>(s.begin(), s.end());
}

int cmd_io(const std::string& path, const std::string& tmpdir) {
    Writer w(path);
    auto text = [&](const std::string& name, const std::string& s) {
        std::vector<int> v(s.begin(), s.end());
        w.i32(name, {v.size()}, v.data());
    };
    {  // mesh text: the unwarped 8 x 8 lake mesh and a 6 x 6 dam-break mesh (wall faces)
        Mesh lake = uniform_tri_mesh(8, 8, {0.0, 0.0, 2.0, 2.0});
        std::ostringstream a;
        write_mesh_text(lake, a);
        text("mesh_lake_text", a.str());
        RunConfig cfg;
        cfg.problem = ProblemId::DamBreak;
        cfg.degree = 2;
        cfg.nx = cfg.ny = 6;
        Case c = build_case(cfg);
        std::ostringstream b;
        write_mesh_text(c.mesh, b);
        text("mesh_dam_text", b.str());
    }
    {  // run() output files of a small vortex case
        RunConfig cfg;
        cfg.problem = ProblemId::Vortex;
        cfg.degree = 2;
        cfg.nx = cfg.ny = 4;
        cfg.tfinal = 0.05;
        cfg.out_dir = tmpdir;
        Case c = build_case(cfg);
        w.mats("vtk_map_nodes", c.mesh.map_nodes);
        w.mats("u0", c.hstate.u);
        w.vecs("b", c.hstate.b);
        RunResult r = run(c);
        w.mats("u_final", c.hstate.u);
        w.scalar("t_final", c.time());
        std::vector<double> inv;
        for (auto& s : r.series) inv.insert(inv.end(), {s.t, s.mass, s.momentum_x, s.momentum_y, s.entropy, s.min_h});
        w.f64("series", {r.series.size(), 6}, inv.data());
        double er[6] = {(double)r.error.N, r.error.h_mesh, r.error.err_h, r.error.err_hu, r.error.err_hv,
                        r.error.combined};
        w.f64("error", {6}, er);
        std::ostringstream tag;
        tag << c.time();
        text("final_name", "solution_" + tag.str() + ".vtk");
        auto put = [&](const std::string& name, const std::string& file) {
            std::vector<int> v = file_bytes(tmpdir + "/" + file);
            w.i32(name, {v.size()}, v.data());
        };
        put("vtk0_text", "solution_0.vtk");
        put("vtk1_text", "solution_" + tag.str() + ".vtk");
        put("invariants_csv", "invariants.csv");
        put("errors_csv", "errors.csv");
    }
    return 0;
}

// Acceptance criterion 5 (acceptance.cpp:188-223): the reference's vortex
// convergence studies (run.hpp:287-332) — affine and curved hybridized N = 2, 3 and
// SBP-Legendre N = 2, nx x ny = 8 x 4 doubled twice, T = 0.5.
int cmd_convergence(const std::string& path) {
    Writer w(path);
    RunConfig base;
    base.problem = ProblemId::Vortex;
    base.nx = 8;
    base.ny = 4;
    base.tfinal = 0.5;
    std::vector<double> rows;  // variant, N, nx, ny, err_h, err_hu, err_hv, combined, order, h_mesh
    auto add = [&](int variant, const std::vector<ConvergenceRow>& rs) {
        for (const auto& r : rs)
            rows.insert(rows.end(), {(double)variant, (double)r.N, (double)r.nx, (double)r.ny, r.error.err_h,
                                     r.error.err_hu, r.error.err_hv, r.error.combined, r.order, r.error.h_mesh});
    };
    add(0, convergence_study(base, {2, 3}, 3));
    RunConfig curved = base;
    curved.warp = 0.1;
    add(1, convergence_study(curved, {2, 3}, 3));
    RunConfig sbp = base;
    sbp.scheme = Scheme::SbpLegendre;
    add(2, convergence_study(sbp, {2}, 3));
    w.f64("rows", {rows.size() / 10, 10}, rows.data());
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr,
                     "usage: swedg_dump ops OUT | modal OUT N n warp periodic seed bathy nsteps dt |"
                     " problem OUT name N scheme n warp cfl tfinal store_inputs | positivity OUT\n");
        return 2;
    }
    std::string cmd = argv[1], out = argv[2];
    try {
        if (cmd == "ops") return cmd_ops(out);
        if (cmd == "positivity") return cmd_positivity(out);
        if (cmd == "ratio") return cmd_ratio(out);
        if (cmd == "convergence") return cmd_convergence(out);
        if (cmd == "io" && argc == 4) return cmd_io(out, argv[3]);
        if (cmd == "modal" && argc == 11)
            return cmd_modal(out, std::atoi(argv[3]), std::atoi(argv[4]), std::atof(argv[5]),
                             std::atoi(argv[6]) != 0, static_cast<unsigned>(std::atoi(argv[7])),
                             std::atoi(argv[8]), std::atoi(argv[9]), std::atof(argv[10]));
        if (cmd == "problem" && argc == 11)
            return cmd_problem(out, argv[3], std::atoi(argv[4]), argv[5], std::atoi(argv[6]),
                               std::atof(argv[7]), std::atof(argv[8]), std::atof(argv[9]),
                               std::atoi(argv[10]));
    } catch (const std::exception& e) {
        std::fprintf(stderr, "swedg_dump: %s\n", e.what());
        return 1;
    }
    std::fprintf(stderr, "swedg_dump: bad arguments\n");
    return 2;
}
