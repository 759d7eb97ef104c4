// multirank_test — the multi-rank path through the C ABI from C++ (TEST
// INFRASTRUCTURE; built by __graft_entry__.build() into tests/cpp/, run on the GPU
// by tests/test_multirank_cpp.py).
//
//  1. P = 1, 2, 3 logical partitions of one mesh on one GPU (strong y-strips from the
//     native setup; modal and SBP schemes, N = 3, 4), one host thread per rank, each stepping its DeviceSolverOps with
//     swedg_step_lsrk45.  The transport is a swedg_exchange_fn that pushes the
//     rank's packed cut-face messages into its peers' halo slots with device copies,
//     ordered by CUDA events (a copy into a peer starts once the peer reached the
//     stage's exchange; a rank's interface kernel waits for every copy into it).
//     The gathered state must equal the unpartitioned run bit for bit.
//  2. One rank whose halo is its own periodic cut, with a one-rank NCCL communicator
//     (ncclSend/ncclRecv to itself inside the captured step graph): bitwise equal to
//     the unpartitioned run.
//  3. The same rank with the peer-memory transport against itself (swedg_p2p_export +
//     swedg_set_p2p: pack-and-store into its halo slots, stream-ordered flags, graph
//     replay): bitwise equal to the unpartitioned run.
// Exit code = number of failed checks; one PASS/FAIL line per check.
#include <cuda_runtime.h>

#include <algorithm>
#include <barrier>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "swedg_b200.hpp"
#include "swedg_setup.h"

static int failures = 0;
static void check(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
    std::fflush(stdout);
    if (!ok) ++failures;
}

struct Case {
    swedg_case c = nullptr;
    explicit Case(const swedg_case_config& cfg) {
        if (swedg_case_build(&cfg, &c) != SWEDG_OK) throw std::runtime_error(swedg_case_error());
    }
    ~Case() { swedg_case_destroy(c); }
    int K() const { return swedg_case_K(c); }
    const double* u0() const { return swedg_case_array(c, "u0", nullptr); }
};

static swedg_case_config config(int N, int nx, int ny, int P, int strip, int scheme = SWEDG_SCHEME_HYBRIDIZED) {
    swedg_case_config cfg{};
    cfg.problem = SWEDG_PROBLEM_SMOOTH;
    cfg.scheme = scheme;
    cfg.N = N;
    cfg.nx = nx;
    cfg.ny = ny;
    cfg.warp = 0.1;
    cfg.cfl = 0.125;
    cfg.seed = 23;
    cfg.threads = 2;
    cfg.strips = P;
    cfg.strip = strip;
    cfg.partition = strip >= 0 ? SWEDG_PARTITION_STRONG : SWEDG_PARTITION_NONE;
    return cfg;
}

static swedg_b200::DeviceSolverOps make_ops(const Case& c) {
    swedg_desc d{};
    swedg_case_fill_desc(c.c, &d);
    d.penalty = SWEDG_PENALTY_LF;
    d.mode = SWEDG_MODE_FAST;
    d.device = 0;
    swedg_b200::DeviceSolverOps ops(d);
    const double* b = swedg_case_array(c.c, "b", nullptr);
    swedg_b200::throw_status(ops.handle(), swedg_set_bathymetry(ops.handle(), b));
    return ops;
}

static std::vector<double> run_steps(swedg_handle h, const double* u0, size_t n, double dt, int nsteps) {
    std::vector<double> u(u0, u0 + n);
    swedg_b200::throw_status(h, swedg_set_state(h, u.data(), nullptr, 0.0));
    swedg_b200::throw_status(h, swedg_step_lsrk45(h, dt, nsteps, 1));
    swedg_b200::throw_status(h, swedg_get_state(h, u.data(), nullptr, nullptr));
    return u;
}

// ---- exchange by device copies between logical partitions -------------------
struct Route {
    size_t send_off, dst_off, len;  // doubles
    int dst;
};
struct Group;
struct Rank {
    Group* g;
    int r;
    double *send = nullptr, *recv = nullptr;
    std::vector<Route> routes;
    cudaEvent_t ready = nullptr, copied = nullptr;
    std::vector<int> pushes_into_me;  // ranks that copy into this rank's halo slots
};
struct Group {
    std::vector<Rank> ranks;
    std::unique_ptr<std::barrier<>> bar;
};

static int push_exchange(void* user, int, const double*, double* recv, void* stream) {
    Rank& me = *static_cast<Rank*>(user);
    Group& g = *me.g;
    auto st = static_cast<cudaStream_t>(stream);
    me.recv = recv;  // this stage's halo slots (SBP: in the stage's input state buffer)
    if (cudaEventRecord(me.ready, st) != cudaSuccess) return 1;
    g.bar->arrive_and_wait();  // every rank's "ready" of this stage is recorded
    for (const Route& rt : me.routes) {
        if (cudaStreamWaitEvent(st, g.ranks[rt.dst].ready, 0) != cudaSuccess) return 1;
        if (cudaMemcpyAsync(g.ranks[rt.dst].recv + rt.dst_off, me.send + rt.send_off, rt.len * 8,
                            cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return 1;
    }
    if (cudaEventRecord(me.copied, st) != cudaSuccess) return 1;
    g.bar->arrive_and_wait();  // every copy of this stage is enqueued
    for (int q : me.pushes_into_me)
        if (cudaStreamWaitEvent(st, g.ranks[q].copied, 0) != cudaSuccess) return 1;
    return 0;
}

static std::vector<std::pair<size_t, size_t>> msg_offsets(const int* counts, int n, int nf) {
    std::vector<std::pair<size_t, size_t>> o;
    size_t off = 0;
    for (int m = 0; m < n; ++m) {
        const size_t len = (size_t)((counts[m] + 2) / 3) * 3 * nf;
        o.push_back({off, len});
        off += len;
    }
    return o;
}

// per element: state doubles per field (Np modal, nq SBP) and pseudo-element field stride
static void sizes(const Case& c, int* nstate, int* stride) {
    swedg_desc d{};
    swedg_case_fill_desc(c.c, &d);
    *nstate = d.scheme == SWEDG_SCHEME_SBP ? d.nq : d.Np;
    *stride = d.scheme == SWEDG_SCHEME_SBP ? d.nq : d.nf;
}

static std::string tag(int scheme, int N, int P) {
    return std::string(scheme == SWEDG_SCHEME_SBP ? "SBP" : "modal") + " N=" + std::to_string(N) + " P=" +
           std::to_string(P);
}

static void logical_partitions(int scheme, int N, int P) {
    const int nx = 8, ny = 9, nsteps = 3;
    Case global(config(N, nx, ny, 1, -1, scheme));
    auto gops = make_ops(global);
    std::vector<std::unique_ptr<Case>> cases;
    std::vector<swedg_b200::DeviceSolverOps> ops;
    double dt = 1e300;
    for (int r = 0; r < P; ++r) {
        cases.emplace_back(new Case(config(N, nx, ny, P, r, scheme)));
        ops.push_back(make_ops(*cases.back()));
        dt = std::min(dt, swedg_case_dt(cases.back()->c));
    }
    int Np, nf;  // state doubles per field, pseudo-element field stride
    sizes(global, &Np, &nf);
    check(dt == swedg_case_dt(global.c), tag(scheme, N, P) + " min over ranks of the owned dt == global dt");
    auto ug = run_steps(gops.handle(), global.u0(), (size_t)global.K() * 3 * Np, dt, nsteps);

    Group g;
    g.ranks.resize(P);
    g.bar = std::make_unique<std::barrier<>>(P);
    std::vector<swedg_halo_desc> halos(P);
    for (int r = 0; r < P; ++r) {
        swedg_case_fill_halo(cases[r]->c, &halos[r]);
        swedg_b200::set_halo(ops[r], halos[r]);
        Rank& rk = g.ranks[r];
        rk.g = &g;
        rk.r = r;
        swedg_halo_buffers(ops[r].handle(), &rk.send, nullptr, &rk.recv, nullptr);
        cudaEventCreateWithFlags(&rk.ready, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&rk.copied, cudaEventDisableTiming);
    }
    // the k-th message r -> q fills q's k-th receive message from r
    for (int r = 0; r < P; ++r) {
        const auto so = msg_offsets(halos[r].send_count, halos[r].n_send_msgs, nf);
        std::vector<int> used(P, 0);
        for (int m = 0; m < halos[r].n_send_msgs; ++m) {
            const int q = halos[r].send_peer[m];
            const auto ro = msg_offsets(halos[q].recv_count, halos[q].n_recv_msgs, nf);
            int k = used[q]++;
            for (int mm = 0; mm < halos[q].n_recv_msgs; ++mm)
                if (halos[q].recv_peer[mm] == r && k-- == 0) {
                    g.ranks[r].routes.push_back({so[m].first, ro[mm].first, so[m].second, q});
                    break;
                }
            auto& in = g.ranks[q].pushes_into_me;
            if (std::find(in.begin(), in.end(), r) == in.end()) in.push_back(r);
        }
        swedg_b200::set_exchange(ops[r], push_exchange, &g.ranks[r]);
    }
    std::vector<std::vector<double>> out(P);
    std::vector<std::string> err(P);
    std::vector<std::thread> th;
    for (int r = 0; r < P; ++r)
        th.emplace_back([&, r] {
            try {
                out[r] = run_steps(ops[r].handle(), cases[r]->u0(), (size_t)cases[r]->K() * 3 * Np, dt, nsteps);
            } catch (const std::exception& e) {
                err[r] = e.what();
            }
        });
    for (auto& t : th) t.join();
    size_t off = 0;
    bool same = true;
    for (int r = 0; r < P; ++r) {
        if (!err[r].empty()) {
            std::printf("rank %d: %s\n", r, err[r].c_str());
            same = false;
            continue;
        }
        same = same && std::memcmp(out[r].data(), ug.data() + off, out[r].size() * 8) == 0;
        off += out[r].size();
    }
    check(same && off == ug.size(),
          tag(scheme, N, P) + " logical partitions (exchange callback, device copies) == global, bitwise");
    for (auto& rk : g.ranks) {
        cudaEventDestroy(rk.ready);
        cudaEventDestroy(rk.copied);
    }
}

static void nccl_self(int scheme, int N) {
    Case global(config(N, 8, 9, 1, -1, scheme));
    Case strip(config(N, 8, 9, 1, 0, scheme));
    auto gops = make_ops(global);
    auto sops = make_ops(strip);
    int Np, stride;
    sizes(global, &Np, &stride);
    const double dt = swedg_case_dt(global.c);
    auto ug = run_steps(gops.handle(), global.u0(), (size_t)global.K() * 3 * Np, dt, 4);
    char id[128];
    void* comm = nullptr;
    if (swedg_nccl_unique_id(id) != SWEDG_OK || swedg_nccl_comm_init(1, id, 0, 0, &comm) != SWEDG_OK) {
        check(false, std::string("NCCL communicator: ") + swedg_create_error());
        return;
    }
    swedg_halo_desc hd;
    swedg_case_fill_halo(strip.c, &hd);
    swedg_b200::set_halo(sops, hd);
    swedg_b200::set_nccl_comm(sops, comm);
    std::vector<double> u;
    try {
        u = run_steps(sops.handle(), strip.u0(), (size_t)strip.K() * 3 * Np, dt, 4);  // graph replay
    } catch (const std::exception& e) {
        std::printf("%s\n", e.what());
    }
    check(u.size() == ug.size() && std::memcmp(u.data(), ug.data(), u.size() * 8) == 0,
          tag(scheme, N, 1) + " one-rank NCCL self exchange across the periodic cut == global, bitwise");
    swedg_b200::set_nccl_comm(sops, nullptr);  // drops the captured graph (NCCL work) before the comm goes
    swedg_nccl_comm_destroy(comm);
}

static void p2p_self(int scheme, int N) {
    Case global(config(N, 8, 9, 1, -1, scheme));
    Case strip(config(N, 8, 9, 1, 0, scheme));
    auto gops = make_ops(global);
    auto sops = make_ops(strip);
    int Np, stride;
    sizes(global, &Np, &stride);
    const double dt = swedg_case_dt(global.c);
    auto ug = run_steps(gops.handle(), global.u0(), (size_t)global.K() * 3 * Np, dt, 4);
    swedg_halo_desc hd;
    swedg_case_fill_halo(strip.c, &hd);
    swedg_b200::set_halo(sops, hd);
    std::vector<char> blob(SWEDG_P2P_BLOB_BYTES);
    if (swedg_p2p_export(sops.handle(), 0, blob.data()) != SWEDG_OK ||
        swedg_set_p2p(sops.handle(), 0, 1, blob.data()) != SWEDG_OK) {
        char msg[256] = {0};
        int code = 0;
        swedg_last_error(sops.handle(), &code, nullptr, nullptr, msg, sizeof(msg));
        check(false, tag(scheme, N, 1) + " peer-memory attach: " + msg);
        return;
    }
    std::vector<double> u;
    try {
        u = run_steps(sops.handle(), strip.u0(), (size_t)strip.K() * 3 * Np, dt, 4);  // graph replay
    } catch (const std::exception& e) {
        std::printf("%s\n", e.what());
    }
    check(u.size() == ug.size() && std::memcmp(u.data(), ug.data(), u.size() * 8) == 0,
          tag(scheme, N, 1) + " peer-memory self exchange across the periodic cut == global, bitwise");
}

int main(int argc, char** argv) {
    std::setvbuf(stdout, nullptr, _IOLBF, 0);
    // multirank_test [--no-nccl | --nccl-only N...]
    const std::string mode = argc > 1 ? argv[1] : "";
    try {
        const int schemes[2] = {SWEDG_SCHEME_HYBRIDIZED, SWEDG_SCHEME_SBP};
        if (mode == "--nccl-only") {
            for (int a = 2; a < argc; ++a) nccl_self(SWEDG_SCHEME_HYBRIDIZED, std::atoi(argv[a]));
        } else {
            for (int sc : schemes)
                for (int N : {3, 4})
                    for (int P : {1, 2, 3}) logical_partitions(sc, N, P);
            for (int sc : schemes)
                for (int N : {3, 4}) p2p_self(sc, N);
            if (mode != "--no-nccl")
                for (int sc : schemes)
                    for (int N : {3, 4}) nccl_self(sc, N);
        }
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        ++failures;
    }
    if (failures == 0) std::printf("all multi-rank checks passed\n");
    return failures;
}
