// swedg_b200.hpp — C++ drop-in adapter: the reference's solver API
// (/root/reference/proj/include/swedg/solver.hpp) on top of the C ABI in
// swedg_b200.h.  Header-only and templated on the reference's own types, so a
// reference user includes it next to swedg/solver.hpp and swaps
//
//     swedg::SolverOps ops = swedg::precompute_element_ops(ref, mesh, geo, conn, fm, g);
//     swedg::set_bathymetry(ops, b);
//     auto du = swedg::rhs(ops, state);
//     swedg::step_lsrk45(state, [&](const State& s) { return swedg::rhs(ops, s); }, dt, res);
// for
//     auto dops = swedg_b200::precompute_element_ops(ref, mesh, geo, conn, fm, g);
//     swedg_b200::set_bathymetry(dops, b);
//     auto du = swedg_b200::rhs(dops, state);            // host-in / host-out, same layout
//     swedg_b200::step_lsrk45(state, dops, dt, nsteps);   // device-resident steps
//
// Errors surface as the reference's exception types and messages:
// std::runtime_error("entropy projection failed in element k at t = ..."),
// std::runtime_error("non-finite RHS in element k at t = ..."),
// std::invalid_argument("dt must be positive")  (solver.hpp:176-180, 288-290, 468).
#pragma once

#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "swedg_b200.h"

namespace swedg_b200 {

enum class Mode { Fast = SWEDG_MODE_FAST, Parity = SWEDG_MODE_PARITY };

inline void throw_status(swedg_handle h, int rc) {
    if (rc == SWEDG_OK) return;
    char msg[512] = {0};
    int code = rc;
    long elem = -1;
    double t = 0.0;
    swedg_last_error(h, &code, &elem, &t, msg, sizeof msg);
    std::string m = h ? std::string(msg) : std::string(swedg_create_error());
    if (rc == SWEDG_ERR_INVALID) throw std::invalid_argument(m);
    throw std::runtime_error(m);
}

// Device-resident replacement of swedg::SolverOps / swedg::SbpSolverOps.
class DeviceSolverOps {
public:
    DeviceSolverOps() = default;
    explicit DeviceSolverOps(const swedg_desc& d) : K_(d.K), nstate_(d.scheme == SWEDG_SCHEME_SBP ? d.nq : d.Np),
                                                     nh_(d.nq + d.nf), scheme_(d.scheme) {
        throw_status(nullptr, swedg_create(&d, &h_));
    }
    DeviceSolverOps(const DeviceSolverOps&) = delete;
    DeviceSolverOps& operator=(const DeviceSolverOps&) = delete;
    DeviceSolverOps(DeviceSolverOps&& o) noexcept { *this = std::move(o); }
    DeviceSolverOps& operator=(DeviceSolverOps&& o) noexcept {
        std::swap(h_, o.h_);
        K_ = o.K_;
        nstate_ = o.nstate_;
        nh_ = o.nh_;
        scheme_ = o.scheme_;
        return *this;
    }
    ~DeviceSolverOps() {
        if (h_) swedg_destroy(h_);
    }
    swedg_handle handle() const { return h_; }
    int K() const { return K_; }
    int nstate() const { return nstate_; }
    int nh() const { return nh_; }
    int scheme() const { return scheme_; }
    void set_penalty(int p) { throw_status(h_, swedg_set_penalty(h_, p)); }
    void set_mode(Mode m) { throw_status(h_, swedg_set_mode(h_, static_cast<int>(m))); }

private:
    swedg_handle h_ = nullptr;
    int K_ = 0, nstate_ = 0, nh_ = 0, scheme_ = 0;
};

namespace detail {

template <class Vec>
std::vector<double> flat(const Vec& v) {
    return std::vector<double>(v.data(), v.data() + v.size());
}

// per-element geometry + connectivity of the reference objects into ABI arrays
struct Packed {
    std::vector<double> Vq, Vf, Pq, Qr, Qs, wf, M_diag, gf, sJ, nx, ny, J_vol, Mh_inv;
    std::vector<int> face_index, nbr, perm;
};

template <class Geo, class Conn, class FM>
void pack_mesh(Packed& p, const Geo& geo, const Conn& conn, const FM& fm, int K, int nf, int npf, int nrow,
               int nq) {
    p.gf.reserve((size_t)K * 4 * nrow);
    for (int k = 0; k < K; ++k) {
        const auto& e = geo.elems[k];
        p.gf.insert(p.gf.end(), e.gf.data(), e.gf.data() + 4 * nrow);       // Eigen column-major nrow x 4
        p.sJ.insert(p.sJ.end(), e.sJ.data(), e.sJ.data() + nf);
        p.nx.insert(p.nx.end(), e.nx.data(), e.nx.data() + nf);
        p.ny.insert(p.ny.end(), e.ny.data(), e.ny.data() + nf);
        p.J_vol.insert(p.J_vol.end(), e.J_vol.data(), e.J_vol.data() + nq);
        for (int f = 0; f < 3; ++f) {
            const auto& fi = conn.faces[k][f];
            const bool wall = static_cast<int>(fi.type) == 2;  // FaceType::Wall (mesh.hpp:143)
            p.nbr.push_back(wall ? -1 : fi.nbr_elem);
            for (int s = 0; s < npf; ++s) p.perm.push_back(wall ? 0 : fm.perm[k][f][s]);
        }
    }
}

}  // namespace detail

// precompute_element_ops (solver.hpp:84-123) — reads the reference's setup
// objects; M_h^{-1} is taken from an existing swedg::SolverOps when given
// (bitwise the reference's), otherwise formed here with the reference's formula.
template <class Ref, class Mesh, class Geo, class Conn, class FM, class HostOps = std::nullptr_t>
DeviceSolverOps precompute_element_ops(const Ref& ref, const Mesh& mesh, const Geo& geo, const Conn& conn,
                                       const FM& fm, double g, int penalty = SWEDG_PENALTY_LF,
                                       Mode mode = Mode::Fast, int device = 0, const HostOps* host_ops = nullptr) {
    const int K = mesh.num_elements(), nq = ref.volq.size(), nf = ref.surfq.size(), Np = ref.Np;
    const int npf = ref.surfq.nodes_per_face;
    detail::Packed p;
    p.Vq = detail::flat(ref.Vq);
    p.Vf = detail::flat(ref.Vf);
    p.Pq = detail::flat(ref.Pq);
    p.Qr = detail::flat(ref.Qh_x);
    p.Qs = detail::flat(ref.Qh_y);
    p.wf = detail::flat(ref.surfq.w);
    detail::pack_mesh(p, geo, conn, fm, K, nf, npf, nq + nf, nq);
    p.Mh_inv.reserve((size_t)K * Np * Np);
    for (int k = 0; k < K; ++k) {
        if constexpr (!std::is_same_v<HostOps, std::nullptr_t>) {
            if (host_ops) {
                const auto& m = host_ops->elem[k].Mh_inv;
                p.Mh_inv.insert(p.Mh_inv.end(), m.data(), m.data() + Np * Np);
                continue;
            }
        }
        // solver.hpp:118-120
        const auto& eg = geo.elems[k];
        auto Mh = (ref.Vq.transpose() * (ref.volq.w.cwiseProduct(eg.J_vol)).asDiagonal() * ref.Vq).eval();
        auto Minv = Mh.llt().solve(decltype(Mh)::Identity(Np, Np)).eval();
        p.Mh_inv.insert(p.Mh_inv.end(), Minv.data(), Minv.data() + Np * Np);
    }
    swedg_desc d{};
    d.abi_version = SWEDG_ABI_VERSION;
    d.scheme = SWEDG_SCHEME_HYBRIDIZED;
    d.penalty = penalty;
    d.mode = static_cast<int>(mode);
    d.N = ref.N;
    d.Np = Np;
    d.nq = nq;
    d.nf = nf;
    d.npf = npf;
    d.K = K;
    d.g = g;
    d.device = device;
    d.Vq = p.Vq.data();
    d.Vf = p.Vf.data();
    d.Pq = p.Pq.data();
    d.Qr = p.Qr.data();
    d.Qs = p.Qs.data();
    d.wf = p.wf.data();
    d.gf = p.gf.data();
    d.sJ = p.sJ.data();
    d.nx = p.nx.data();
    d.ny = p.ny.data();
    d.J_vol = p.J_vol.data();
    d.Mh_inv = p.Mh_inv.data();
    d.nbr = p.nbr.data();
    d.perm = p.perm.data();
    return DeviceSolverOps(d);
}

// precompute_sbp_ops (solver.hpp:322-360)
template <class Ref, class Sbp, class Mesh, class Geo, class Conn, class FM>
DeviceSolverOps precompute_sbp_ops(const Ref& ref, const Sbp& sbp, const Mesh& mesh, const Geo& geo,
                                   const Conn& conn, const FM& fm, double g, int penalty = SWEDG_PENALTY_LF,
                                   Mode mode = Mode::Fast, int device = 0) {
    const int K = mesh.num_elements(), nq = ref.volq.size(), nf = ref.surfq.size();
    const int npf = ref.surfq.nodes_per_face;
    detail::Packed p;
    p.Qr = detail::flat(sbp.Q_SBP_x);
    p.Qs = detail::flat(sbp.Q_SBP_y);
    p.wf = detail::flat(ref.surfq.w);
    p.M_diag = detail::flat(sbp.M_diag);
    p.face_index.assign(sbp.face_index.begin(), sbp.face_index.end());
    detail::pack_mesh(p, geo, conn, fm, K, nf, npf, nq + nf, nq);
    swedg_desc d{};
    d.abi_version = SWEDG_ABI_VERSION;
    d.scheme = SWEDG_SCHEME_SBP;
    d.penalty = penalty;
    d.mode = static_cast<int>(mode);
    d.N = ref.N;
    d.Np = ref.Np;
    d.nq = nq;
    d.nf = nf;
    d.npf = npf;
    d.K = K;
    d.g = g;
    d.device = device;
    d.Qr = p.Qr.data();
    d.Qs = p.Qs.data();
    d.wf = p.wf.data();
    d.M_diag = p.M_diag.data();
    d.face_index = p.face_index.data();
    d.gf = p.gf.data();
    d.sJ = p.sJ.data();
    d.nx = p.nx.data();
    d.ny = p.ny.data();
    d.J_vol = p.J_vol.data();
    d.nbr = p.nbr.data();
    d.perm = p.perm.data();
    return DeviceSolverOps(d);
}

// set_bathymetry (solver.hpp:127-141 / 362-367): per-element modal (or nodal) b
template <class VecList>
void set_bathymetry(DeviceSolverOps& ops, const VecList& b) {
    std::vector<double> flat;
    flat.reserve((size_t)ops.K() * ops.nstate());
    for (const auto& v : b) flat.insert(flat.end(), v.data(), v.data() + v.size());
    throw_status(ops.handle(), swedg_set_bathymetry(ops.handle(), flat.data()));
}

namespace detail {
template <class StateT>
std::vector<double> pack_state(const StateT& st, int n) {
    std::vector<double> u;
    u.reserve(st.u.size() * 3 * (size_t)n);
    for (const auto& m : st.u) u.insert(u.end(), m.data(), m.data() + 3 * n);  // Eigen n x 3 column-major
    return u;
}
template <class MatT>
std::vector<MatT> unpack(const std::vector<double>& flat, int K, int rows) {
    std::vector<MatT> out(K);
    for (int k = 0; k < K; ++k) {
        out[k].resize(rows, 3);
        std::memcpy(out[k].data(), flat.data() + (size_t)k * 3 * rows, sizeof(double) * 3 * rows);
    }
    return out;
}
}  // namespace detail

// rhs(ops, state) (solver.hpp:295-297) and rhs_sbp(ops, state) (:369-434)
template <class StateT>
auto rhs(const DeviceSolverOps& ops, const StateT& state) {
    using MatT = std::decay_t<decltype(state.u[0])>;
    std::vector<double> u = detail::pack_state(state, ops.nstate());
    std::vector<double> du(u.size());
    throw_status(ops.handle(), swedg_rhs(ops.handle(), u.data(), state.t, du.data()));
    return detail::unpack<MatT>(du, ops.K(), ops.nstate());
}

// entropy_projection(ops, state) (solver.hpp:170-183): stacked (nq+nf) x 3 per element
template <class StateT>
auto entropy_projection(const DeviceSolverOps& ops, const StateT& state) {
    using MatT = std::decay_t<decltype(state.u[0])>;
    std::vector<double> u = detail::pack_state(state, ops.nstate());
    std::vector<double> proj((size_t)ops.K() * 3 * ops.nh());
    throw_status(ops.handle(), swedg_entropy_projection(ops.handle(), u.data(), state.t, proj.data()));
    return detail::unpack<MatT>(proj, ops.K(), ops.nh());
}

// step_lsrk45(state, rhs, dt, res) (solver.hpp:466-484), nsteps device-resident steps.
// Signature differs from the reference's step_lsrk45(state, rhs_fn, dt, res): the RHS
// functor is the device ops and the LSRK register lives on the device.  It is reset
// to zero on every call (swedg_set_state with res = NULL), which matches the
// reference's result because Lsrk45::a[0] == 0 (solver.hpp:442): stage 0 sets
// res = dt * du whatever res held.
template <class StateT>
void step_lsrk45(StateT& state, DeviceSolverOps& ops, double dt, int nsteps = 1) {
    if (!(dt > 0.0)) throw std::invalid_argument("dt must be positive");
    std::vector<double> u = detail::pack_state(state, ops.nstate());
    throw_status(ops.handle(), swedg_set_state(ops.handle(), u.data(), nullptr, state.t));
    throw_status(ops.handle(), swedg_step_lsrk45(ops.handle(), dt, nsteps, 1));
    double t = state.t;
    throw_status(ops.handle(), swedg_get_state(ops.handle(), u.data(), nullptr, &t));
    const int n = ops.nstate();
    for (size_t k = 0; k < state.u.size(); ++k)
        std::memcpy(state.u[k].data(), u.data() + k * 3 * (size_t)n, sizeof(double) * 3 * n);
    state.t = t;
}

// ---- multi-rank ---------------------------------------------
// A rank's DeviceSolverOps is built over its element partition (owned elements;
// neighbour ids K.. address the halo slots, desc.n_halo).  Give it the exchange map
// and a transport; step_lsrk45 then runs every stage with the cut-face exchange
// overlapped with the interior volume kernel (swedg_b200.h, multi-rank stepping).
inline void set_halo(DeviceSolverOps& ops, const swedg_halo_desc& d) {
    throw_status(ops.handle(), swedg_set_halo(ops.handle(), &d));
}
// nccl_comm: an ncclComm_t over the ranks named in the halo map (or swedg_nccl_comm_init)
inline void set_nccl_comm(DeviceSolverOps& ops, void* nccl_comm) {
    throw_status(ops.handle(), swedg_set_nccl_comm(ops.handle(), nccl_comm));
}
// any other transport (MPI, a test's device copies): called once per stage at enqueue time
inline void set_exchange(DeviceSolverOps& ops, swedg_exchange_fn fn, void* user) {
    throw_status(ops.handle(), swedg_set_exchange(ops.handle(), fn, user));
}

}  // namespace swedg_b200
