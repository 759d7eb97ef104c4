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

#define SWEDG_ABI_VERSION 2

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
     * slots whose face traces the caller fills between swedg_stage_volume and
     * swedg_stage_surface (hybridized scheme).  0 for a single rank. */
    int n_halo;
} swedg_desc;

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
int swedg_trace_device_ptr(swedg_handle h, double** trace, long long* n_owned, long long* n_halo);
/* Check the device error record (syncs the stream). */
int swedg_check(swedg_handle h);

/* Bathymetry products of swedg_set_bathymetry, copied to host (testing):
 * b_stacked[K][nq+nf] (hybridized only, may be NULL), src[K][2][nq+nf] (SBP: [K][2][nq]). */
int swedg_debug_bathymetry(swedg_handle h, double* b_stacked, double* src);

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
