/*
 * swedg_b200.h — C ABI of the B200-native ESDG shallow-water RHS.
 *
 * Drop-in boundary for the reference's operator API (header-only C++,
 * /root/reference/proj/include/swedg/solver.hpp).  The reference has no FFI;
 * each entry point below replaces one reference function for a caller that
 * owns the reference's setup objects (RefOperators, Mesh, Geometry,
 * Connectivity, FaceMatch).  include/swedg_b200.hpp is the C++ adapter that
 * re-exposes the reference's signatures and exceptions over this ABI, and
 * INTEGRATION.md shows the binding.
 *
 *   reference (solver.hpp)                          replaced by
 *   precompute_element_ops(ref,mesh,geo,conn,fm,g)  swedg_create (scheme HYBRIDIZED)      :84-123
 *   precompute_sbp_ops(ref,sbp,mesh,geo,conn,fm,g)  swedg_create (scheme SBP)             :322-360
 *   set_bathymetry(SolverOps&, b)                   swedg_set_bathymetry                  :127-141
 *   set_bathymetry(SbpSolverOps&, b)                swedg_set_bathymetry                  :362-367
 *   entropy_projection(ops, state)                  swedg_entropy_projection              :170-183
 *   rhs(ops, state[, proj])                         swedg_rhs                             :237-297
 *   rhs_sbp(ops, state)                             swedg_rhs                             :369-434
 *   step_lsrk45(state, rhs_fn, dt, res)             swedg_step_lsrk45 (device-resident)  :466-484
 *   compute_invariants(fq, geo, u, b, g, t)         swedg_compute_invariants   diagnostics.hpp:237-267
 *   l2_error(fq, geo, u, exact | ref_state, t)      swedg_l2_error             diagnostics.hpp:176-226
 *   run(Case&) time loop + invariant sampling       swedg_run                  run.hpp:226-262
 *   exceptions (solver.hpp:176-180,288-290,468)     status codes + swedg_last_error
 *
 * Conventions
 *   - Plain pointers and sizes; no torch or CUDA types in signatures
 *     (streams are passed as void*).
 *   - All arrays are IEEE float64 / int32, C order, with per-element Eigen
 *     column-major blocks stacked: a per-element r x c Eigen matrix occupies
 *     [K][c][r].  So the modal state is u[K][3][Np] (Np x 3 column-major per
 *     element: (h, hu, hv) columns, solver.hpp:27-32), nodal SBP state
 *     u[K][3][nq], gf[K][4][nq+nf] (mesh.hpp:258-262), Mh_inv[K][Np][Np].
 *     Reference-element operators are column-major, exactly Eigen's .data().
 *   - Host-pointer entry points copy in/out and synchronise; the *_device
 *     entry points take device pointers and are stream-ordered.
 *   - Every call returns SWEDG_OK (0) or a negative status; the message,
 *     element id and stage time of the failure are returned by
 *     swedg_last_error.  A handle is not thread-safe; calls are
 *     stream-ordered on the handle's stream.
 */
#ifndef SWEDG_B200_H
#define SWEDG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWEDG_ABI_VERSION 5

/* status codes */
#define SWEDG_OK 0
#define SWEDG_ERR_INVALID (-1)     /* bad descriptor / argument (std::invalid_argument) */
#define SWEDG_ERR_POSITIVITY (-2)  /* nonpositive water height (PositivityError, solver.hpp:176) */
#define SWEDG_ERR_NONFINITE (-3)   /* non-finite RHS (solver.hpp:288, :429) */
#define SWEDG_ERR_CUDA (-4)        /* CUDA runtime failure / no device / extension missing */
#define SWEDG_ERR_UNSUPPORTED (-5) /* degree or size not compiled in */

/* scheme (solver.hpp:22) */
#define SWEDG_SCHEME_HYBRIDIZED 0
#define SWEDG_SCHEME_SBP 1
/* penalty (solver.hpp:23) */
#define SWEDG_PENALTY_EC 0
#define SWEDG_PENALTY_LF 1
/* arithmetic mode */
#define SWEDG_MODE_FAST 0   /* FMA-contracted, reassociated flux differencing (<= 1e-12 rel.) */
#define SWEDG_MODE_PARITY 1 /* reference evaluation order, no contraction (bitwise w/ oracle) */

typedef struct swedg_handle_s* swedg_handle;

/* Everything precompute_element_ops / precompute_sbp_ops read from the
 * reference's setup objects.  Sizes: nh = nq + nf, nrow = nq + nf. */
typedef struct {
    int abi_version;  /* = SWEDG_ABI_VERSION */
    int scheme;       /* SWEDG_SCHEME_* */
    int penalty;      /* SWEDG_PENALTY_* */
    int mode;         /* SWEDG_MODE_* */
    int N;            /* polynomial degree (RefOperators::N) */
    int Np;           /* basis_dim(N) = (N+1)(N+2)/2 */
    int nq;           /* volume nodes (volq.size(); SBP: M_diag.size()) */
    int nf;           /* surface nodes, 3*npf (surfq.size()) */
    int npf;          /* nodes per face (surfq.nodes_per_face) */
    int K;            /* elements on this rank (mesh.num_elements()) */
    double g;         /* gravity (SolverOps::g) */
    int device;       /* CUDA device ordinal */

    /* reference-element operators, column-major (refelem.hpp:123-139) */
    const double* Vq; /* nq x Np  (hybridized) */
    const double* Vf; /* nf x Np  (hybridized) */
    const double* Pq; /* Np x nq  (hybridized) */
    const double* Qr; /* hybridized: RefOperators::Qh_x (nh x nh); SBP: Q_SBP_x (nq x nq) */
    const double* Qs; /* hybridized: RefOperators::Qh_y;            SBP: Q_SBP_y          */
    const double* wf; /* nf: surfq.w (face Jacobian included, quadrature.hpp:202) */
    const int* face_index; /* SBP: nf surface slot -> volume node (TraditionalSBP::face_index) */
    const double* M_diag;  /* SBP: nq rule weights (TraditionalSBP::M_diag) */

    /* per-element geometry (mesh.hpp:251-329) */
    const double* gf;     /* [K][4][nq+nf]  ElemGeom::gf */
    const double* sJ;     /* [K][nf]        ElemGeom::sJ */
    const double* nx;     /* [K][nf]        ElemGeom::nx */
    const double* ny;     /* [K][nf]        ElemGeom::ny */
    const double* J_vol;  /* SBP: [K][nq]   ElemGeom::J_vol (Minv = 1/(M_diag*J)) */
    const double* Mh_inv; /* hybridized: [K][Np][Np] ElementOps::Mh_inv (solver.hpp:118-120) */

    /* connectivity (mesh.hpp:143-154, 333-373) */
    const int* nbr;  /* [K][3]  neighbour element of face f, -1 = wall (FaceType::Wall) */
    const int* perm; /* [K][nf] FaceMatch::perm[k][f][s]: neighbour surface slot (ignored on walls) */

    /* multi-rank (element partition): neighbour ids K..K+n_halo-1 address halo
     * slots of the face-trace buffer ([3][nf] pseudo-elements, each holding up to
     * three received cut faces in its face positions; perm selects the position and
     * node), filled by the per-stage exchange (swedg_set_halo).  0 for one rank. */
    int n_halo;
} swedg_desc;

/* Per-stage halo exchange of an element-partitioned mesh.  The only
 * cross-element read of the RHS is the exterior trace (solver.hpp:263-264), so a
 * rank sends the traces of its cut faces (3 fields x npf nodes per face) once per
 * RK stage.  Wire format of a message of n faces: ceil(n/3) pseudo-elements of
 * [3][nf] doubles, face i in pseudo-element i/3 at face position i%3 (so a
 * received message lands directly in the halo slots).  Receive message m fills
 * halo slots [sum_{q<m} ceil(recv_count[q]/3), ...).  Messages between the same
 * two ranks pair up in issue order (the k-th send from a to b matches b's k-th
 * receive from a). */
typedef struct {
    int n_send_msgs;
    const int* send_peer;   /* [n_send_msgs] destination rank */
    const int* send_count;  /* [n_send_msgs] faces per message */
    const int* send_elem;   /* [sum send_count] owned element of each sent face, message-major */
    const int* send_face;   /* [sum send_count] its local face 0..2 */
    int n_recv_msgs;
    const int* recv_peer;   /* [n_recv_msgs] source rank */
    const int* recv_count;  /* [n_recv_msgs] faces per message */
} swedg_halo_desc;

/* Custom transport: called once per RK stage on the host while the stage is
 * enqueued, after the cut faces were packed into `send` (device, the send messages
 * back to back in wire format; modal: projected traces, [3][nf] pseudo-elements;
 * SBP: the stage input's face-node states, [3][nq] pseudo-elements).  It must enqueue on `stream`
 * (cudaStream_t) whatever fills `recv` (device, the halo slots = receive messages
 * back to back) and return 0; the interface kernel waits on `stream`. */
typedef int (*swedg_exchange_fn)(void* user, int stage, const double* send, double* recv, void* stream);

/* ---- lifecycle ------------------------------------------------------------ */
int swedg_create(const swedg_desc* desc, swedg_handle* out);
int swedg_destroy(swedg_handle h);
/* Use an external CUDA stream (cudaStream_t passed as void*); NULL = handle's own. */
int swedg_set_stream(swedg_handle h, void* stream);
void* swedg_get_stream(swedg_handle h);
int swedg_set_penalty(swedg_handle h, int penalty);
int swedg_set_mode(swedg_handle h, int mode);

/* ---- bathymetry (solver.hpp:127-141 / :362-367) -------------------------- */
/* hybridized: b[K][Np] modal coefficients; SBP: b[K][nq] nodal values. */
int swedg_set_bathymetry(swedg_handle h, const double* b);

/* ---- host-in / host-out evaluation (parity and tests) -------------------- */
/* proj[K][3][nq+nf]: entropy-projected (h,hu,hv) at stacked points. */
int swedg_entropy_projection(swedg_handle h, const double* u, double t, double* proj);
/* du[K][3][Np] (SBP: [K][3][nq]) = rhs(ops, state) at time t (t only labels errors). */
int swedg_rhs(swedg_handle h, const double* u, double t, double* du);

/* ---- device-resident time stepping (the throughput path) ----------------- */
/* state u (and LSRK register res, zeroed when res == NULL) copied from host */
int swedg_set_state(swedg_handle h, const double* u, const double* res, double t);
int swedg_get_state(swedg_handle h, double* u, double* res, double* t);
/* nsteps LSRK45 steps of size dt on the device-resident state (solver.hpp:466-484).
 * Stream-ordered; errors are checked (one device sync) when sync != 0. */
int swedg_step_lsrk45(swedg_handle h, double dt, int nsteps, int sync);
/* The same steps on a HOST-resident state u_host [K][3][Np] (the reference's
 * calling pattern: state.u lives on the host between steps).  Each step reads
 * its input from u_host and writes its result back; the transfers are
 * pipelined with the compute in `nchunks` element chunks (0 = the default: 24 for the N = 4
 * FAST path, whose wavefront merges each tick's launches, 16 otherwise).  When every
 * element's neighbours lie in its own or an adjacent chunk (row-ordered meshes),
 * the chunks run through the stages and steps as a wavefront, so a chunk's
 * D2H, its H2D for the next step and other chunks' kernels all overlap;
 * otherwise only the first stage's volume kernel and the last stage's interface
 * kernel overlap the copies.  u_host should be pinned.  Syncs and checks errors
 * at the end; results are bit-for-bit those of swedg_step_lsrk45. */
int swedg_step_lsrk45_host(swedg_handle h, double* u_host, double dt, int nsteps, int nchunks);
/* Replay nsteps >= 2 as a captured one-step CUDA graph (default on; off while
 * per-kernel timers are enabled). */
int swedg_set_graphs(swedg_handle h, int on);
/* Raw device pointers of the resident state (for zero-copy interop). */
int swedg_state_device_ptr(swedg_handle h, double** u, double** res);
/* du = rhs(u) with device pointers, stream-ordered, no host sync. */
int swedg_rhs_device(swedg_handle h, const double* u_dev, double* du_dev, double t);
/* Stage-level stepping for multi-rank runs: one LSRK45 stage (0..4) split at the
 * halo exchange.  swedg_stage_volume runs the projection+volume kernel and
 * writes the owned elements' face traces; the caller then fills the halo trace
 * slots (device pointer below, layout [K + n_halo][3][nf]); swedg_stage_surface
 * runs the fused surface + lift + M^-1 + register update.  Stream-ordered. */
int swedg_stage_volume(swedg_handle h, int stage, double dt);
int swedg_stage_surface(swedg_handle h, int stage, double dt);
/* swedg_stage_volume on the element range [k0, k1) only, so boundary elements can
 * be computed first and their traces exchanged while the interior runs (the
 * projection + volume kernel is element-local).  The range starting at k0 == 0
 * opens the stage; the ranges of one stage must cover [0, K) before
 * swedg_stage_surface. */
int swedg_stage_volume_range(swedg_handle h, int stage, double dt, int k0, int k1);
/* swedg_stage_surface on [k0, k1) (e.g. to copy finished chunks out while the rest
 * runs); the range ending at k1 == K closes the step (advances t) for stage 4. */
int swedg_stage_surface_range(swedg_handle h, int stage, double dt, int k0, int k1);
int swedg_trace_device_ptr(swedg_handle h, double** trace, long long* n_owned, long long* n_halo);

/* ---- multi-rank stepping ------------------------------------------------------
 * With a halo map and a transport (NCCL communicator, peer memory or exchange callback),
 * swedg_step_lsrk45 runs every stage as: projection+volume kernel on the elements
 * owning sent faces -> pack -> exchange on a second stream, overlapped with the
 * interior volume kernel -> interface/update kernel after the exchange.  With NCCL or
 * peer memory the step is captured once into a CUDA graph and replayed.  Results are bitwise
 * independent of the partition (per-element arithmetic is unchanged). */
int swedg_set_halo(swedg_handle h, const swedg_halo_desc* d);
/* NCCL transport: comm is an ncclComm_t whose ranks are the peers of the halo map
 * (libnccl.so.2 is resolved at run time: the one already loaded, e.g. by torch, or
 * $SWEDG_NCCL_LIB).  NULL detaches (and drops the captured step graph, which holds
 * NCCL work): detach or destroy every handle using a communicator before the
 * communicator is destroyed. */
int swedg_set_nccl_comm(swedg_handle h, void* comm);
int swedg_set_exchange(swedg_handle h, swedg_exchange_fn fn, void* user);
/* Device pointers and sizes (doubles) of the packed send messages and the halo slots
 * (modal: in the face-trace buffer; SBP: in the state buffer — the SBP FAST path rotates
 * the stage input over three buffers, so its callbacks receive each stage's `recv`). */
int swedg_halo_buffers(swedg_handle h, double** send, size_t* n_send, double** recv, size_t* n_recv);
/* Pack the cut-face traces of the current stage into the send buffer (stage-level
 * API: after the volume ranges that own sent faces, before the exchange). */
int swedg_halo_pack(swedg_handle h);
/* The volume-kernel schedule of a multi-rank stage: ranges[2i], ranges[2i+1] = [k0, k1);
 * the first n_boundary ranges hold every element owning a sent face, the next
 * n_interior the rest (ranges NULL: counts only). */
int swedg_halo_ranges(swedg_handle h, int* ranges, int max_ranges, int* n_boundary, int* n_interior);
/* NCCL communicator helpers (so a caller without its own NCCL setup can build one):
 * id is 128 bytes (ncclUniqueId), created on one rank and shared with the others. */
int swedg_nccl_unique_id(void* id);
int swedg_nccl_comm_init(int nranks, const void* id, int rank, int device, void** comm);
int swedg_nccl_comm_destroy(void* comm);
/* Peer-memory transport (the ranks of one node, NVLink / NVSwitch): instead of a send
 * buffer and NCCL, the pack kernel stores each cut-face trace straight into the
 * destination rank's halo slot over peer memory, and 32-bit flags in the ranks' memory,
 * written and waited on by the streams themselves (cuStreamWriteValue32 /
 * cuStreamWaitValue32), order every stage's exchange: the sender waits until the
 * receiver consumed the previous stage's halo, stores, then raises the receiver's
 * "ready" flag; the receiver's interface (SBP: boundary RHS) kernel waits for it, then
 * raises the sender's "free" flag.  No host synchronisation; captured into the step graph.
 * swedg_p2p_export writes this rank's descriptor (SWEDG_P2P_BLOB_BYTES bytes: IPC
 * handles and addresses of its halo slots and flags, its receive table) and initialises
 * its flags; every rank gathers all descriptors (e.g. torch.distributed all_gather) and
 * passes them, concatenated in rank order, to swedg_set_p2p (after swedg_set_halo).
 * Peers in the same process are addressed directly, others through
 * cudaIpcOpenMemHandle.  Every rank must run the same stages; after an error, export
 * and attach again.  blobs NULL detaches. */
#define SWEDG_P2P_BLOB_BYTES 4096
int swedg_p2p_export(swedg_handle h, int rank, void* blob);
int swedg_set_p2p(swedg_handle h, int rank, int nranks, const void* blobs);
/* Check the device error record (syncs the stream). */
int swedg_check(swedg_handle h);

/* Bathymetry products of swedg_set_bathymetry, copied to host (testing):
 * b_stacked[K][nq+nf] (hybridized only, may be NULL), src[K][2][nq+nf] (SBP: [K][2][nq]). */
int swedg_debug_bathymetry(swedg_handle h, double* b_stacked, double* src);

/* ---- diagnostics on the device (diagnostics.hpp:142-267) ------------------
 * FineQuad evaluations of the resident (or a host) state.  Every per-point term
 * is computed in the reference's operation order (bit-for-bit the reference's
 * terms, except the exact-solution values of SWEDG_DIAG_L2_VORTEX/LAKE, which
 * use CUDA's exp/sincos); the sums are EXACT: fixed-point integer accumulators,
 * rounded once to nearest — independent of launch shape and of the number of
 * ranks, and within the reference's own serial-summation rounding of its result. */
#define SWEDG_DIAG_INVARIANTS 0 /* compute_invariants (diagnostics.hpp:237-267) */
#define SWEDG_DIAG_L2_REF 1     /* l2_error vs a discrete modal state (diagnostics.hpp:205-226) */
#define SWEDG_DIAG_L2_VORTEX 2  /* l2_error vs vortex_exact (diagnostics.hpp:41-53, 176-202) */
#define SWEDG_DIAG_L2_LAKE 3    /* l2_error vs the lake-at-rest state (run.hpp:125-127) */

typedef struct {
    int nfine;                /* FineQuad(N).rule.size(): volume_rule_by_degree(2N+2) */
    const double* w;          /* [nfine] rule weights */
    const double* V;          /* nfine x Np column-major: FineQuad::V */
    const double* Vr;         /* nfine x Np: FineQuad::Vx (d/dr) */
    const double* Vs;         /* nfine x Np: FineQuad::Vy (d/ds) */
    const double* map_coeffs; /* [K][2][Np]: ElemGeom::map_coeffs (Np x 2 column-major per element) */
    const double* Pq;         /* SBP: RefOperators::Pq (Np x nq) for project_nodal; hybridized: NULL */
} swedg_diag_desc;

int swedg_set_diagnostics(swedg_handle h, const swedg_diag_desc* d);
/* compute_invariants of u (host state in the scheme's layout; NULL = resident
 * state at the handle's t) with the bathymetry of swedg_set_bathymetry (SBP:
 * projected, Case::modal_bathymetry).  out[6] = {t, mass, momentum_x,
 * momentum_y, entropy, min_h} (Invariants).  h <= 0 at a fine point fails with
 * SWEDG_ERR_POSITIVITY (entropy() -> check_positive).  Syncs. */
int swedg_compute_invariants(swedg_handle h, const double* u, double t, double* out);
/* l2_error of u (NULL = resident) for what = SWEDG_DIAG_L2_*: aux = u_ref
 * [K][3][Np] (L2_REF), VortexParams {h_inf,u_inf,v_inf,beta,g,xc,yc} (L2_VORTEX),
 * NULL (L2_LAKE).  out[4] = {err_h, err_hu, err_hv, combined} (ErrorReport).  Syncs. */
int swedg_l2_error(swedg_handle h, int what, const double* u, const double* aux, double t, double* out);
/* Raw exact accumulators (multi-rank): one record of swedg_diag_raw_bytes()
 * bytes; swedg_diag_from_raw merges raw[nranks][n] records exactly (rank-count
 * independent, bitwise) and finishes them to out[n][6] (l2: first 4 used). */
size_t swedg_diag_raw_bytes(void);
int swedg_diag_raw(swedg_handle h, int what, const double* u, const double* aux, double t, void* raw);
int swedg_diag_from_raw(const void* raw, int nranks, int n, double* out);
/* Run-loop sampling without host syncs: invariants of the resident state at
 * the handle's t into device slot `slot`; read back n slots as out[n][6]. */
int swedg_sample_invariants(swedg_handle h, int slot);
int swedg_read_invariants(swedg_handle h, int n, double* out);
int swedg_read_invariants_raw(swedg_handle h, int n, void* raw);
/* run() (run.hpp:226-262) on the resident state: nsteps = ceil(tfinal/dt - 1e-12),
 * step_dt = min(dt, tfinal - t), invariants sampled at the start, every
 * sample_every steps (0 = max(1, nsteps/100)) and at the last step, into
 * series[max_samples][6].  One host sync at the end. */
int swedg_run(swedg_handle h, double dt, double tfinal, int sample_every, int max_samples, double* series,
              int* nsamples, int* nsteps_done);
/* Host reference of the exact accumulator: *out = correctly rounded sum of x[0..n). */
int swedg_exact_sum(const double* x, size_t n, double* out);

/* ---- volume-kernel cost study (bench.hpp:55-201) ---------
 * R_GPU = t_ESDG / t_DG of the reference's two study kernels on the device:
 * kernel_matvec (y = Q f(u), nodal x-flux) and kernel_fluxdiff
 * (y_i = sum_j 2 Q_ij f_S(u_i, u_j); nq < n: kernel_fluxdiff_skew, the block
 * j, i >= nq skipped).  Q n x n column-major (2 <= n <= 256), u/y [K][3][n].
 * Both kernels run 2 untimed + reps timed launches (CUDA events);
 * t_ms[2] = median {t_DG, t_ESDG}; y_dg / y_esdg (may be NULL) receive the
 * outputs.  mode PARITY = the reference's arithmetic bit for bit; FAST = FMA
 * and the reassociated EC flux.  No handle; stand-alone device buffers. */
int swedg_ratio_kernels(int device, int n, int nq, int K, const double* Q, const double* u, double g, int mode,
                        int reps, double* y_dg, double* y_esdg, double* t_ms);

/* ---- errors ----------------------------------------------------------------- */
/* Last failure: status code, element id (or -1), stage time, message. */
int swedg_last_error(swedg_handle h, int* code, long* elem, double* t, char* msg, size_t len);
/* Message of the last failure of swedg_create (no handle yet). */
const char* swedg_create_error(void);

/* ---- introspection ---------------------------------------------------------- */
/* Per-kernel CUDA-event timers on the handle's stream (off by default).  Kernel
 * classes: 0 = volume kernel (modal projection+volume / SBP rhs), 1 = surface +
 * update kernel (modal) / RK update (SBP).  swedg_read_timers syncs, returns the
 * summed milliseconds and launch counts since the last read, and resets them. */
int swedg_enable_timers(swedg_handle h, int on);
int swedg_read_timers(swedg_handle h, double* ms, long long* launches, int nclass);
/* Measured FP64 (DFMA) throughput of the device in TFLOP/s (FMA = 2 flops):
 * a register-resident DFMA chain kernel, best of `reps` timed launches. */
int swedg_probe_fp64_peak(int device, int reps, double* tflops);

/* Number of kernels launched by this handle since creation (evidence counter). */
long long swedg_launch_count(swedg_handle h);
/* Device memory held by the handle, bytes. */
size_t swedg_device_bytes(swedg_handle h);
int swedg_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SWEDG_B200_H */
