/*
 * swedg_setup.h — native case setup (host C++, multithreaded) that produces
 * every input of swedg_create for the reference's problems, without the
 * reference.  It restates, for a standalone user:
 *   quadrature.hpp  surface/volume/SBP rules        refelem.hpp  Dubiner basis, RefOperators,
 *   mesh.hpp        uniform mesh, warp, dam snap/fit, connect (O(K log K)), geometry, match_faces
 *   solver.hpp      precompute_element_ops (M_h^{-1}), compute_dt
 *   diagnostics.hpp / run.hpp   make_state, make_nodal_state, lake / vortex / dam-break builders
 *   tests/test_solver.cpp:14-25 smooth_state (the C4/C5 "smooth wave" workload)
 * Arrays are owned by the case; swedg_case_fill_desc points a swedg_desc at them.
 */
#ifndef SWEDG_SETUP_H
#define SWEDG_SETUP_H

#include <stddef.h>

#include "swedg_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define SWEDG_PROBLEM_LAKE 0     /* run.hpp:116-137  lake at rest, [-1,1]^2 periodic, g = 9.81 */
#define SWEDG_PROBLEM_VORTEX 1   /* run.hpp:139-154  translating vortex, [-10,10]x[-5,5], g = 2 */
#define SWEDG_PROBLEM_DAMBREAK 2 /* run.hpp:159-209  curved dam x = y^2/25, walls, g = 9.81 */
#define SWEDG_PROBLEM_SMOOTH 3   /* smooth_state(seed) on [-1,1]^2 periodic + lake bathymetry */

typedef struct swedg_case_s* swedg_case;

typedef struct {
    int problem;     /* SWEDG_PROBLEM_* */
    int scheme;      /* SWEDG_SCHEME_* */
    int N;           /* degree */
    int nx, ny;      /* quads per direction (K = 2 nx ny) */
    double warp;     /* mesh warp amplitude (mesh.hpp:111-130), 0 = affine */
    double cfl;      /* dt = cfl * h_min / ((N+1)(N+2)/2) */
    double g;        /* <= 0: the problem's default */
    unsigned seed;   /* SMOOTH: mt19937 seed of smooth_state */
    int threads;     /* host threads, <= 0: hardware concurrency */
    int strips;      /* P: number of y-strips of a partitioned mesh (see partition) */
    int strip;       /* this rank's strip 0..P-1 (periodic problems, hybridized): owned
                        rows + face halos of the two cuts (swedg_case_fill_halo);
                        strip == -1: the whole global mesh in one piece (tests) */
    int partition;   /* SWEDG_PARTITION_*; NONE with strips > 1 = WEAK (ABI v3 behaviour) */
    /* SBP volume rule (sbp_rule, quadrature.hpp:320-343): Gauss-Legendre edges come from
     * the built-in tables; Gauss-Lobatto edges only from sbp_lobatto_N<N>.txt in
     * sbp_data_dir (NULL: the working directory); sbp_rule_file (non-NULL) loads that
     * file for either family (load_sbp_rule_file, quadrature.hpp:290-318). */
    int sbp_family;              /* SWEDG_SBP_LEGENDRE / SWEDG_SBP_LOBATTO */
    const char* sbp_data_dir;
    const char* sbp_rule_file;
} swedg_case_config;

#define SWEDG_SBP_LEGENDRE 0
#define SWEDG_SBP_LOBATTO 1

#define SWEDG_PARTITION_NONE 0
#define SWEDG_PARTITION_WEAK 1   /* P strips of ny rows: global nx x (ny P) mesh, domain stretched P times in y */
#define SWEDG_PARTITION_STRONG 2 /* the problem's nx x ny mesh cut into P strips of ny/P rows */

int swedg_case_build(const swedg_case_config* cfg, swedg_case* out);
/* The problem's state, bathymetry and operators on a caller-supplied mesh (the
 * read_mesh_text format, mesh.hpp:462-493): verts[nv][2], tris[ne][3] (counter-
 * clockwise), wall_faces[nw][2] = (element, face) records, domain = {xc, yc, Lx,
 * Ly} (periodic matching of open boundary faces, mesh.hpp:210-247).  Elements
 * are straight-sided at degree N (cfg->warp != 0 warps them like warp_mesh);
 * cfg->nx, ny, strips are ignored. */
int swedg_case_build_mesh(const swedg_case_config* cfg, const double* verts, int nv, const int* tris, int ne,
                          const int* wall_faces, int nw, const double* domain, int periodic_x, int periodic_y,
                          swedg_case* out);
int swedg_case_destroy(swedg_case c);
/* load_sbp_rule_file / sbp_rule on their own (the rule a case would use): nq volume
 * nodes x[nq], y[nq], w[nq] (arrays of max_nodes), npf, face_index[3 npf] (surface slot ->
 * volume node).  Errors (missing file, header mismatch, non-embedding, nonpositive
 * weight, exactness) return SWEDG_ERR_INVALID with the reference's message in
 * swedg_case_error(). */
int swedg_sbp_rule(int N, int family, const char* data_dir, const char* rule_file, int max_nodes, int* nq,
                   int* npf, double* x, double* y, double* w, int* face_index);
const char* swedg_case_error(void);
/* Fill every operator/geometry/connectivity pointer and size of *d (penalty,
 * mode and device are left for the caller). */
int swedg_case_fill_desc(swedg_case c, swedg_desc* d);
/* Halo exchange map of a strip case (pointers into the case; n_send_msgs = 0 when
 * the case is not partitioned). */
int swedg_case_fill_halo(swedg_case c, swedg_halo_desc* d);
/* Named host arrays: "u0" [K][3][n], "b" [K][n], "xy_vol" [K][2][nq], "map_coeffs" [K][2][Np],
 * "map_nodes" [K][2][Np], "J_vol" [K][nq], "volq_w" [nq], "Vq" ..., "fine_w/V/Vr/Vs" (FineQuad),
 * "lattice_V" (basis at the mapping lattice, Np x Np); returns element count via *n. */
const double* swedg_case_array(swedg_case c, const char* name, size_t* n);
const int* swedg_case_iarray(swedg_case c, const char* name, size_t* n);
double swedg_case_dt(swedg_case c);
double swedg_case_min_edge(swedg_case c);
int swedg_case_K(swedg_case c);

#ifdef __cplusplus
}
#endif
#endif /* SWEDG_SETUP_H */
