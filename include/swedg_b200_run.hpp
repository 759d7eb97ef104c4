// swedg_b200_run.hpp — drop-in for the callers around the hot path: the
// reference's run() time loop and its diagnostics (run.hpp:226-284,
// diagnostics.hpp:142-267), on the device-resident solver of swedg_b200.hpp.
//
// Include it where the reference's headers are on the include path (it uses
// swedg::Case, FineQuad, Invariants, ErrorReport and RunResult directly):
//
//     swedg::Case c = swedg::build_case(cfg);
//     auto ops = swedg_b200::make_device_ops(c);        // operators, bathymetry, FineQuad
//     swedg::RunResult r = swedg_b200::run(c, ops);     // == swedg::run(c)
//
// run() keeps the state on the device for the whole integration: full-dt steps
// between samples replay a captured step graph, invariants are sampled by a
// device kernel into a device buffer, and the only host syncs are the final
// error check and the read-back (reference: a host round trip per step and
// per sample).  Invariant sums are exact (correctly rounded) where the
// reference sums serially; the difference is the reference's own summation
// rounding.  Output files (cfg.out_dir) are written by the reference's own
// writers from the host copies.
#pragma once

#include <algorithm>
#include <cmath>
#include <sstream>
#include <string>
#include <vector>

#include "swedg/run.hpp"
#include "swedg_b200.hpp"

namespace swedg_b200 {

// FineQuad operators and per-element mapping coefficients -> the device
// (FineQuad::element_geometry inputs, diagnostics.hpp:142-165).
inline void set_diagnostics(DeviceSolverOps& ops, const swedg::Case& c, const swedg::FineQuad& fq) {
    std::vector<double> w = detail::flat(fq.rule.w), V = detail::flat(fq.V), Vr = detail::flat(fq.Vx),
                        Vs = detail::flat(fq.Vy), map, Pq;
    const int Np = c.ref.Np;
    map.reserve((size_t)c.num_elements() * 2 * Np);
    for (const auto& e : c.geo.elems) map.insert(map.end(), e.map_coeffs.data(), e.map_coeffs.data() + 2 * Np);
    if (c.sbp) Pq = detail::flat(c.ref.Pq);
    swedg_diag_desc d{};
    d.nfine = static_cast<int>(fq.rule.w.size());
    d.w = w.data();
    d.V = V.data();
    d.Vr = Vr.data();
    d.Vs = Vs.data();
    d.map_coeffs = map.data();
    d.Pq = c.sbp ? Pq.data() : nullptr;
    throw_status(ops.handle(), swedg_set_diagnostics(ops.handle(), &d));
}

// Device ops for a built case: precompute_*_ops + set_bathymetry + FineQuad.
inline DeviceSolverOps make_device_ops(const swedg::Case& c, Mode mode = Mode::Fast, int device = 0) {
    const int pen = c.cfg.penalty == swedg::Penalty::LaxFriedrichs ? SWEDG_PENALTY_LF : SWEDG_PENALTY_EC;
    DeviceSolverOps ops = c.sbp ? precompute_sbp_ops(c.ref, *c.tsbp, c.mesh, c.geo, c.conn, c.fm, c.cfg.g, pen,
                                                     mode, device)
                                : precompute_element_ops(c.ref, c.mesh, c.geo, c.conn, c.fm, c.cfg.g, pen, mode,
                                                         device, &c.hops);
    if (c.sbp)
        set_bathymetry(ops, c.nstate.b);
    else
        set_bathymetry(ops, c.hstate.b);
    set_diagnostics(ops, c, swedg::FineQuad(c.cfg.degree));
    return ops;
}

namespace detail {
inline swedg::Invariants to_invariants(const double* v) {
    swedg::Invariants inv;
    inv.t = v[0];
    inv.mass = v[1];
    inv.momentum_x = v[2];
    inv.momentum_y = v[3];
    inv.entropy = v[4];
    inv.min_h = v[5];
    return inv;
}
inline std::vector<double> case_state(const swedg::Case& c) {
    return c.sbp ? pack_state(c.nstate, c.nstate.u.empty() ? 0 : (int)c.nstate.u[0].rows())
                 : pack_state(c.hstate, c.hstate.u.empty() ? 0 : (int)c.hstate.u[0].rows());
}
}  // namespace detail

// compute_invariants(fq, geo, c.modal_solution(), c.modal_bathymetry(), g, t) of the case's host state
inline swedg::Invariants compute_invariants(const DeviceSolverOps& ops, const swedg::Case& c) {
    std::vector<double> u = detail::case_state(c), out(6);
    throw_status(ops.handle(), swedg_compute_invariants(ops.handle(), u.data(), c.time(), out.data()));
    return detail::to_invariants(out.data());
}

// The L2 error run() reports (run.hpp:264-271): vs ref_state when present, else vs
// the exact solution (vortex: VortexParams with the case's g; lake: its initial state).
inline bool case_error(const DeviceSolverOps& ops, const swedg::Case& c, swedg::ErrorReport& rep) {
    std::vector<double> u = detail::case_state(c), out(4);
    int rc;
    if (!c.ref_state.empty()) {
        std::vector<double> ref;
        for (const auto& m : c.ref_state) ref.insert(ref.end(), m.data(), m.data() + m.size());
        rc = swedg_l2_error(ops.handle(), SWEDG_DIAG_L2_REF, u.data(), ref.data(), c.time(), out.data());
    } else if (c.exact && c.cfg.problem == swedg::ProblemId::Vortex) {
        swedg::VortexParams vp;
        vp.g = c.cfg.g;
        const double p[7] = {vp.h_inf, vp.u_inf, vp.v_inf, vp.beta, vp.g, vp.xc, vp.yc};
        rc = swedg_l2_error(ops.handle(), SWEDG_DIAG_L2_VORTEX, u.data(), p, c.time(), out.data());
    } else if (c.exact && c.cfg.problem == swedg::ProblemId::Lake) {
        rc = swedg_l2_error(ops.handle(), SWEDG_DIAG_L2_LAKE, u.data(), nullptr, c.time(), out.data());
    } else {
        return false;
    }
    throw_status(ops.handle(), rc);
    rep.N = c.cfg.degree;
    rep.err_h = out[0];
    rep.err_hu = out[1];
    rep.err_hv = out[2];
    rep.combined = out[3];
    rep.h_mesh = swedg::min_edge_length(c.mesh);
    return true;
}

// run(Case&) (run.hpp:226-284) on the device.  The case's host state is uploaded,
// integrated to cfg.tfinal and written back (with its time).
inline swedg::RunResult run(swedg::Case& c, DeviceSolverOps& ops) {
    const swedg::RunConfig& cfg = c.cfg;
    const double dt = swedg::compute_dt(c.mesh, cfg.degree, cfg.cfl);
    const int nsteps = cfg.tfinal > 0.0 ? static_cast<int>(std::ceil(cfg.tfinal / dt - 1e-12)) : 0;
    const int cadence = cfg.sample_every > 0 ? cfg.sample_every : std::max(1, nsteps / 100);
    swedg::RunResult res;
    res.dt = dt;
    if (!cfg.out_dir.empty())
        swedg::write_solution_vtk(cfg.out_dir + "/solution_0.vtk", c.mesh, cfg.degree, c.modal_solution(),
                                  c.modal_bathymetry());
    std::vector<double> u = detail::case_state(c);
    throw_status(ops.handle(), swedg_set_state(ops.handle(), u.data(), nullptr, c.time()));
    const int max_samples = nsteps / cadence + 2;
    std::vector<double> series((size_t)max_samples * 6);
    int ns = 0, done = 0;
    throw_status(ops.handle(), swedg_run(ops.handle(), dt, cfg.tfinal, cadence, max_samples, series.data(), &ns,
                                         &done));
    for (int i = 0; i < ns; ++i) res.series.push_back(detail::to_invariants(series.data() + 6 * i));
    res.steps = done;
    double t = 0.0;
    throw_status(ops.handle(), swedg_get_state(ops.handle(), u.data(), nullptr, &t));
    auto put = [&](auto& st) {
        const size_t n = (size_t)st.u[0].rows() * 3;
        for (size_t k = 0; k < st.u.size(); ++k) std::memcpy(st.u[k].data(), u.data() + k * n, sizeof(double) * n);
        st.t = t;
    };
    if (c.sbp)
        put(c.nstate);
    else
        put(c.hstate);
    res.has_error = case_error(ops, c, res.error);
    if (!cfg.out_dir.empty()) {
        swedg::write_invariants_csv(cfg.out_dir + "/invariants.csv", res.series);
        if (res.has_error) swedg::write_errors_csv(cfg.out_dir + "/errors.csv", {res.error}, {});
        std::ostringstream tag;
        tag << c.time();
        swedg::write_solution_vtk(cfg.out_dir + "/solution_" + tag.str() + ".vtk", c.mesh, cfg.degree,
                                  c.modal_solution(), c.modal_bathymetry());
    }
    return res;
}

}  // namespace swedg_b200
