/*
 * swedg_oracle.c — CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY: this file is the parity CHECKER.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it
 * (oracle/_ref/liboracle.so, built by oracle/Makefile.oracle).  The product
 * (paper_2005_02516_b200/) never links or calls it.
 *
 * It restates, in plain C and in the reference's exact arithmetic order (the
 * library is compiled with -ffp-contract=off), the functions of
 * /root/reference/proj/include/swedg:
 *   swe.hpp:34-38   entropy_vars          swe.hpp:40-44  cons_from_entropy
 *   swe.hpp:60-66   flux                  swe.hpp:87-99  wave_speed / lf_penalty
 *   swe.hpp:102-105 wall_ghost
 *   solver.hpp:74-80,105-108  split_form_op + skew part (on the fly, per entry)
 *   solver.hpp:127-141 set_bathymetry     solver.hpp:145-168 entropy_projection_element
 *   solver.hpp:190-204 ec_flux_xy         solver.hpp:209-231 skew_volume_kernel
 *   solver.hpp:237-293 rhs                solver.hpp:362-367 set_bathymetry (SBP)
 *   solver.hpp:369-434 rhs_sbp            solver.hpp:466-484 step_lsrk45
 * Pinned against the reference itself: tests/test_oracle.py compares every
 * output with tests/golden/*.npz, which oracle/_ref/swedg_dump (the unmodified
 * reference headers) produced — bit-for-bit equality is asserted.
 *
 * Layouts (C order; per-element Eigen column-major blocks stacked):
 *   u, du, res   [K][3][Np]   (SBP: [K][3][nq] nodal)
 *   proj         [K][3][nh]   nh = nq + nf (rows: nq volume, nf surface face-major)
 *   gf           [K][4][nrow] columns (y_s, -y_r, -x_s, x_r); nrow = nq+nf
 *   sJ, nx, ny   [K][nf]      Mh_inv [K][Np][Np] (column-major Np x Np)
 *   nbr          [K][3]  (-1 = wall)      perm [K][nf] (neighbour surface slot)
 *   reference operators column-major: Vq nq x Np, Vf nf x Np, Pq Np x nq,
 *   Qr/Qs (hybridized Qh_x/Qh_y) nh x nh;  SBP: Q_SBP_x/y nq x nq.
 */
#include <math.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI /* glibc's value (c11 mode hides it) */
#define M_PI 3.14159265358979323846
#endif

/* Internal arithmetic type.  Built twice: real = double (the reference's own
 * arithmetic, liboracle.so) and real = long double (-DORACLE_LONG_DOUBLE, x87 80-bit, liboracle_ld.so)
 * — the latter is the accuracy yardstick for the FAST kernels: on
 * cancellation-dominated states (the dam break at rest) two different FP64
 * roundings of the same RHS differ by the reference's own rounding error, so
 * FAST is required to be no less accurate than the reference there. */
#ifdef ORACLE_LONG_DOUBLE
typedef long double real;
#define FABS(x) fabsl(x)
#define SQRT(x) sqrtl(x)
#else
typedef double real;
#define FABS(x) fabs(x)
#define SQRT(x) sqrt(x)
#endif

#define ORACLE_OK 0
#define ORACLE_ERR_POSITIVITY 1
#define ORACLE_ERR_NONFINITE 2

typedef struct {
    int N, Np, nq, nf, npf, K;
    int scheme;      /* 0 hybridized (modal), 1 SBP */
    int penalty_lf;  /* 1 Lax-Friedrichs, 0 entropy conservative */
    double g;
    const double *Vq, *Vf, *Pq; /* modal only */
    const double *Qr, *Qs;      /* hybridized Qh_x/Qh_y (nh x nh) or Q_SBP_x/y (nq x nq) */
    const double *wf;           /* nf surface weights */
    const int *face_index;      /* SBP: nf surface slot -> volume node */
    const double *gf, *sJ, *nx, *ny;
    const double *Mh_inv;       /* modal */
    const double *J_vol;        /* SBP: [K][nq] */
    const double *M_diag;       /* SBP: nq */
    const int *nbr, *perm;
    /* set by oracle_set_bathymetry */
    const double *b_stacked, *src_x, *src_y;
} oracle_ops;

/* ---- pointwise physics (swe.hpp) --------------------------------------- */

static void ec_flux_xy(const real *a, const real *b, real g, real *fx, real *fy) {
    real uxa = a[1] / a[0], uya = a[2] / a[0];
    real uxb = b[1] / b[0], uyb = b[2] / b[0];
    real h_avg = 0.5 * (a[0] + b[0]);
    real p = g * h_avg * h_avg - 0.25 * g * (a[0] * a[0] + b[0] * b[0]);
    real ux = 0.5 * (uxa + uxb), uy = 0.5 * (uya + uyb);
    real hu = 0.5 * (a[1] + b[1]), hv = 0.5 * (a[2] + b[2]);
    fx[0] = hu;
    fx[1] = hu * ux + p;
    fx[2] = hu * uy;
    fy[0] = hv;
    fy[1] = hv * ux;
    fy[2] = hv * uy + p;
}

static void phys_flux(const real *u, real g, int dir, real *f) {
    real vx = u[1] / u[0], vy = u[2] / u[0];
    real p = 0.5 * g * u[0] * u[0];
    if (dir == 0) {
        f[0] = u[1];
        f[1] = u[1] * vx + p;
        f[2] = u[1] * vy;
    } else {
        f[0] = u[2];
        f[1] = u[2] * vx;
        f[2] = u[2] * vy + p;
    }
}

static real wave_speed(const real *u, real g, real nx, real ny) {
    real un = (u[1] * nx + u[2] * ny) / u[0];
    return FABS(un) + SQRT(g * u[0]);
}

static void lf_penalty(const real *uL, const real *uR, real g, real nx, real ny,
                       real *pen) {
    real a = wave_speed(uL, g, nx, ny), b = wave_speed(uR, g, nx, ny);
    real lam = (a < b) ? b : a; /* std::max */
    pen[0] = 0.5 * lam * (uR[0] - uL[0]);
    pen[1] = 0.5 * lam * (uR[1] - uL[1]);
    pen[2] = 0.5 * lam * (uR[2] - uL[2]);
}

static void wall_ghost(const real *u, real nx, real ny, real *out) {
    real un = u[1] * nx + u[2] * ny;
    out[0] = u[0];
    out[1] = u[1] - 2.0 * un * nx;
    out[2] = u[2] - 2.0 * un * ny;
}

/* physical split-form operator entry, solver.hpp:74-80 (Eigen coefficient order) */
static real split_entry(const double *Qr, const double *Qs, int ld, const double *g1,
                          const double *g2, int i, int j) {
    real qr = Qr[i + (size_t)j * ld], qs = Qs[i + (size_t)j * ld];
    return 0.5 * (g1[i] * qr + qr * g1[j] + g2[i] * qs + qs * g2[j]);
}
/* skew part Qh - Qh^T, solver.hpp:107-108 */
static real skew_entry(const double *Qr, const double *Qs, int ld, const double *g1,
                         const double *g2, int i, int j) {
    return split_entry(Qr, Qs, ld, g1, g2, i, j) - split_entry(Qr, Qs, ld, g1, g2, j, i);
}

/* ---- set_bathymetry (solver.hpp:127-141; SBP :362-367) ------------------ */

void oracle_set_bathymetry(const oracle_ops *op, const double *b, double *b_stacked,
                           double *src_x, double *src_y) {
    int nq = op->nq, nf = op->nf;
    if (op->scheme == 1) {
        int nrow = nq + nf;
        for (int k = 0; k < op->K; ++k) {
            const double *gf = op->gf + (size_t)k * 4 * nrow;
            const double *bk = b + (size_t)k * nq;
            for (int i = 0; i < nq; ++i) {
                real sx = 0.0, sy = 0.0;
                for (int j = 0; j < nq; ++j) {
                    sx += split_entry(op->Qr, op->Qs, nq, gf, gf + nrow, i, j) * bk[j];
                    sy += split_entry(op->Qr, op->Qs, nq, gf + 2 * nrow, gf + 3 * nrow, i, j) * bk[j];
                }
                src_x[(size_t)k * nq + i] = sx;
                src_y[(size_t)k * nq + i] = sy;
                if (b_stacked) b_stacked[(size_t)k * nq + i] = bk[i];
            }
        }
        return;
    }
    int Np = op->Np, nh = nq + nf;
    for (int k = 0; k < op->K; ++k) {
        const double *bk = b + (size_t)k * Np;
        double *bs = b_stacked + (size_t)k * nh;
        for (int i = 0; i < nq; ++i) {
            real s = 0.0;
            for (int m = 0; m < Np; ++m) s += op->Vq[i + (size_t)m * nq] * bk[m];
            bs[i] = s;
        }
        for (int i = 0; i < nf; ++i) {
            real s = 0.0;
            for (int m = 0; m < Np; ++m) s += op->Vf[i + (size_t)m * nf] * bk[m];
            bs[nq + i] = s;
        }
        const double *gf = op->gf + (size_t)k * 4 * nh;
        for (int i = 0; i < nh; ++i) {
            real sx = 0.0, sy = 0.0;
            for (int j = 0; j < nh; ++j) {
                sx += skew_entry(op->Qr, op->Qs, nh, gf, gf + nh, i, j) * bs[j];
                sy += skew_entry(op->Qr, op->Qs, nh, gf + 2 * nh, gf + 3 * nh, i, j) * bs[j];
            }
            src_x[(size_t)k * nh + i] = 0.5 * sx;
            src_y[(size_t)k * nh + i] = 0.5 * sy;
        }
        for (int i = 0; i < nf; ++i) {
            real m = op->wf[i] * op->sJ[(size_t)k * nf + i];
            real Bx = m * op->nx[(size_t)k * nf + i], By = m * op->ny[(size_t)k * nf + i];
            src_x[(size_t)k * nh + nq + i] += 0.5 * (Bx * bs[nq + i]);
            src_y[(size_t)k * nh + nq + i] += 0.5 * (By * bs[nq + i]);
        }
    }
}

/* ---- entropy projection (solver.hpp:145-183) ----------------------------- */

/* returns 0 or ORACLE_ERR_POSITIVITY; proj_k is [3][nh] */
static int project_element(const oracle_ops *op, int k, const double *u, real *proj_k) {
    int Np = op->Np, nq = op->nq, nf = op->nf, nh = nq + nf;
    const double *uk = u + (size_t)k * 3 * Np;
    const double *bs = op->b_stacked + (size_t)k * nh;
    real g = op->g;
    real vq[3 * 64], vh[3 * 64];
    for (int i = 0; i < nq; ++i) {
        real uq[3];
        for (int c = 0; c < 3; ++c) {
            real s = 0.0;
            for (int m = 0; m < Np; ++m) s += op->Vq[i + (size_t)m * nq] * uk[c * Np + m];
            uq[c] = s;
        }
        if (!(uq[0] > 0.0)) return ORACLE_ERR_POSITIVITY;
        real vx = uq[1] / uq[0], vy = uq[2] / uq[0];
        vq[0 * nq + i] = g * (uq[0] + bs[i]) - 0.5 * (vx * vx + vy * vy);
        vq[1 * nq + i] = vx;
        vq[2 * nq + i] = vy;
    }
    for (int m = 0; m < Np; ++m)
        for (int c = 0; c < 3; ++c) {
            real s = 0.0;
            for (int i = 0; i < nq; ++i) s += op->Pq[m + (size_t)i * Np] * vq[c * nq + i];
            vh[c * Np + m] = s;
        }
    for (int i = 0; i < nh; ++i) {
        real vt[3];
        for (int c = 0; c < 3; ++c) {
            real s = 0.0;
            if (i < nq)
                for (int m = 0; m < Np; ++m) s += op->Vq[i + (size_t)m * nq] * vh[c * Np + m];
            else
                for (int m = 0; m < Np; ++m) s += op->Vf[(i - nq) + (size_t)m * nf] * vh[c * Np + m];
            vt[c] = s;
        }
        real h = (vt[0] + 0.5 * (vt[1] * vt[1] + vt[2] * vt[2])) / g - bs[i];
        if (!(h > 0.0)) return ORACLE_ERR_POSITIVITY;
        proj_k[0 * nh + i] = h;
        proj_k[1 * nh + i] = h * vt[1];
        proj_k[2 * nh + i] = h * vt[2];
    }
    return ORACLE_OK;
}

/* proj: [K][3][nh].  Returns 0 or error code; *bad_elem = first failing element. */
static int entropy_projection_real(const oracle_ops *op, const double *u, real *proj, int *bad_elem) {
    int nh = op->nq + op->nf;
    for (int k = 0; k < op->K; ++k) {
        int e = project_element(op, k, u, proj + (size_t)k * 3 * nh);
        if (e) {
            if (bad_elem) *bad_elem = k;
            return e;
        }
    }
    return ORACLE_OK;
}

int oracle_entropy_projection(const oracle_ops *op, const double *u, double *proj,
                              int *bad_elem) {
    size_t n = (size_t)op->K * 3 * (op->nq + op->nf);
    real *p = (real *)malloc(sizeof(real) * n);
    int e = entropy_projection_real(op, u, p, bad_elem);
    for (size_t i = 0; i < n; ++i) proj[i] = (double)p[i];
    free(p);
    return e;
}

/* ---- modal RHS (solver.hpp:237-293) --------------------------------------
 * elems: optional subset (n_elems entries) — du is written only for those
 * elements; proj must hold every element (or at least the subset and its
 * neighbours). */
static int rhs_from_proj_real(const oracle_ops *op, const real *proj, double *du,
                              const int *elems, int n_elems, int *bad_elem) {
    int Np = op->Np, nq = op->nq, nf = op->nf, nh = nq + nf, npf = op->npf;
    real g = op->g;
    int n = elems ? n_elems : op->K;
    real acc[3 * 128], stacked[3 * 128], modal[3 * 64];
    for (int ei = 0; ei < n; ++ei) {
        int k = elems ? elems[ei] : ei;
        const real *ut = proj + (size_t)k * 3 * nh;
        const double *gf = op->gf + (size_t)k * 4 * nh;
        memset(acc, 0, sizeof(real) * 3 * nh);
        real fx[3], fy[3], ui[3], uj[3];
        /* skew_volume_kernel pass 1: j < nq, all rows */
        for (int j = 0; j < nq; ++j) {
            uj[0] = ut[j]; uj[1] = ut[nh + j]; uj[2] = ut[2 * nh + j];
            for (int i = 0; i < nh; ++i) {
                real qx = skew_entry(op->Qr, op->Qs, nh, gf, gf + nh, i, j);
                real qy = skew_entry(op->Qr, op->Qs, nh, gf + 2 * nh, gf + 3 * nh, i, j);
                if (qx == 0.0 && qy == 0.0) continue;
                ui[0] = ut[i]; ui[1] = ut[nh + i]; ui[2] = ut[2 * nh + i];
                ec_flux_xy(ui, uj, g, fx, fy);
                for (int c = 0; c < 3; ++c) acc[c * nh + i] += qx * fx[c] + qy * fy[c];
            }
        }
        /* pass 2: surface columns, volume rows */
        for (int j = nq; j < nh; ++j) {
            uj[0] = ut[j]; uj[1] = ut[nh + j]; uj[2] = ut[2 * nh + j];
            for (int i = 0; i < nq; ++i) {
                real qx = skew_entry(op->Qr, op->Qs, nh, gf, gf + nh, i, j);
                real qy = skew_entry(op->Qr, op->Qs, nh, gf + 2 * nh, gf + 3 * nh, i, j);
                if (qx == 0.0 && qy == 0.0) continue;
                ui[0] = ut[i]; ui[1] = ut[nh + i]; ui[2] = ut[2 * nh + i];
                ec_flux_xy(ui, uj, g, fx, fy);
                for (int c = 0; c < 3; ++c) acc[c * nh + i] += qx * fx[c] + qy * fy[c];
            }
        }
        /* surface coupling */
        for (int f = 0; f < 3; ++f) {
            int nb = op->nbr[(size_t)k * 3 + f];
            for (int s = 0; s < npf; ++s) {
                int i = f * npf + s;
                real nxi = op->nx[(size_t)k * nf + i], nyi = op->ny[(size_t)k * nf + i];
                real m = op->wf[i] * op->sJ[(size_t)k * nf + i];
                real Bx = m * nxi, By = m * nyi;
                real up[3];
                ui[0] = ut[nq + i]; ui[1] = ut[nh + nq + i]; ui[2] = ut[2 * nh + nq + i];
                if (nb < 0) {
                    wall_ghost(ui, nxi, nyi, up);
                } else {
                    int j = op->perm[(size_t)k * nf + i];
                    const real *un = proj + (size_t)nb * 3 * nh;
                    up[0] = un[nq + j]; up[1] = un[nh + nq + j]; up[2] = un[2 * nh + nq + j];
                }
                ec_flux_xy(up, ui, g, fx, fy);
                for (int c = 0; c < 3; ++c) acc[c * nh + nq + i] += Bx * fx[c] + By * fy[c];
                if (op->penalty_lf) {
                    real pen[3];
                    lf_penalty(ui, up, g, nxi, nyi, pen);
                    for (int c = 0; c < 3; ++c) acc[c * nh + nq + i] -= m * pen[c];
                }
            }
        }
        /* bathymetry source; stacked = src - acc */
        const double *sx = op->src_x + (size_t)k * nh, *sy = op->src_y + (size_t)k * nh;
        for (int i = 0; i < nh; ++i) {
            real h = ut[i];
            stacked[0 * nh + i] = 0.0 - acc[0 * nh + i];
            stacked[1 * nh + i] = -g * h * sx[i] - acc[1 * nh + i];
            stacked[2 * nh + i] = -g * h * sy[i] - acc[2 * nh + i];
        }
        /* lift: Vq^T top + Vf^T bottom, then Mh_inv */
        for (int m = 0; m < Np; ++m)
            for (int c = 0; c < 3; ++c) {
                real s1 = 0.0, s2 = 0.0;
                for (int i = 0; i < nq; ++i) s1 += op->Vq[i + (size_t)m * nq] * stacked[c * nh + i];
                for (int i = 0; i < nf; ++i) s2 += op->Vf[i + (size_t)m * nf] * stacked[c * nh + nq + i];
                modal[c * Np + m] = s1 + s2;
            }
        const double *Mi = op->Mh_inv + (size_t)k * Np * Np;
        double *duk = du + (size_t)k * 3 * Np;
        int finite = 1;
        for (int c = 0; c < 3; ++c)
            for (int i = 0; i < Np; ++i) {
                real s = 0.0;
                for (int m = 0; m < Np; ++m) s += Mi[i + (size_t)m * Np] * modal[c * Np + m];
                duk[c * Np + i] = s;
                if (!isfinite(s)) finite = 0;
            }
        if (!finite) {
            if (bad_elem) *bad_elem = k;
            return ORACLE_ERR_NONFINITE;
        }
    }
    return ORACLE_OK;
}

int oracle_rhs_from_proj(const oracle_ops *op, const double *proj, double *du,
                         const int *elems, int n_elems, int *bad_elem) {
    size_t n = (size_t)op->K * 3 * (op->nq + op->nf);
    real *p = (real *)malloc(sizeof(real) * n);
    for (size_t i = 0; i < n; ++i) p[i] = proj[i];
    int e = rhs_from_proj_real(op, p, du, elems, n_elems, bad_elem);
    free(p);
    return e;
}

/* proj holds n_proj_elems element blocks (owned + halo slots addressed by nbr) */
int oracle_rhs_from_proj_n(const oracle_ops *op, const double *proj, int n_proj_elems, double *du,
                           const int *elems, int n_elems, int *bad_elem) {
    size_t n = (size_t)n_proj_elems * 3 * (op->nq + op->nf);
    real *p = (real *)malloc(sizeof(real) * n);
    for (size_t i = 0; i < n; ++i) p[i] = proj[i];
    int e = rhs_from_proj_real(op, p, du, elems, n_elems, bad_elem);
    free(p);
    return e;
}

/* projection kept in REAL precision between the two phases */
int oracle_rhs(const oracle_ops *op, const double *u, double *du, double *proj_scratch,
               int *bad_elem) {
    (void)proj_scratch;
    size_t n = (size_t)op->K * 3 * (op->nq + op->nf);
    real *p = (real *)malloc(sizeof(real) * n);
    int e = entropy_projection_real(op, u, p, bad_elem);
    if (!e) e = rhs_from_proj_real(op, p, du, NULL, 0, bad_elem);
    free(p);
    return e;
}

int oracle_rhs_subset(const oracle_ops *op, const double *u, double *du, const int *elems,
                      int n_elems, int *bad_elem) {
    size_t n = (size_t)op->K * 3 * (op->nq + op->nf);
    real *p = (real *)malloc(sizeof(real) * n);
    int e = entropy_projection_real(op, u, p, bad_elem);
    if (!e) e = rhs_from_proj_real(op, p, du, elems, n_elems, bad_elem);
    free(p);
    return e;
}

/* ---- SBP RHS (solver.hpp:369-434) ---------------------------------------- */

int oracle_rhs_sbp(const oracle_ops *op, const double *u, double *du, const int *elems,
                   int n_elems, int *bad_elem) {
    int nq = op->nq, nf = op->nf, npf = op->npf, nrow = nq + nf;
    real g = op->g;
    int n = elems ? n_elems : op->K;
    real acc[3 * 128];
    for (int ei = 0; ei < n; ++ei) {
        int k = elems ? elems[ei] : ei;
        const double *uk = u + (size_t)k * 3 * nq;
        const double *gf = op->gf + (size_t)k * 4 * nrow;
        for (int i = 0; i < nq; ++i)
            if (!(uk[i] > 0.0)) {
                if (bad_elem) *bad_elem = k;
                return ORACLE_ERR_POSITIVITY;
            }
        memset(acc, 0, sizeof(real) * 3 * nq);
        real fx[3], fy[3], ui[3], uj[3];
        for (int j = 0; j < nq; ++j) {
            uj[0] = uk[j]; uj[1] = uk[nq + j]; uj[2] = uk[2 * nq + j];
            for (int i = 0; i < nq; ++i) {
                real qx = split_entry(op->Qr, op->Qs, nq, gf, gf + nrow, i, j);
                real qy = split_entry(op->Qr, op->Qs, nq, gf + 2 * nrow, gf + 3 * nrow, i, j);
                if (qx == 0.0 && qy == 0.0) continue;
                ui[0] = uk[i]; ui[1] = uk[nq + i]; ui[2] = uk[2 * nq + i];
                ec_flux_xy(ui, uj, g, fx, fy);
                for (int c = 0; c < 3; ++c) acc[c * nq + i] += 2.0 * (qx * fx[c] + qy * fy[c]);
            }
        }
        for (int f = 0; f < 3; ++f) {
            int nb = op->nbr[(size_t)k * 3 + f];
            for (int s = 0; s < npf; ++s) {
                int i = f * npf + s;
                int vi = op->face_index[i];
                real nxi = op->nx[(size_t)k * nf + i], nyi = op->ny[(size_t)k * nf + i];
                real m = op->wf[i] * op->sJ[(size_t)k * nf + i];
                real Bx = m * nxi, By = m * nyi;
                real up[3], fxi[3], fyi[3];
                ui[0] = uk[vi]; ui[1] = uk[nq + vi]; ui[2] = uk[2 * nq + vi];
                if (nb < 0) {
                    wall_ghost(ui, nxi, nyi, up);
                } else {
                    int j = op->face_index[op->perm[(size_t)k * nf + i]];
                    const double *un = u + (size_t)nb * 3 * nq;
                    up[0] = un[j]; up[1] = un[nq + j]; up[2] = un[2 * nq + j];
                }
                ec_flux_xy(up, ui, g, fx, fy);
                phys_flux(ui, g, 0, fxi);
                phys_flux(ui, g, 1, fyi);
                for (int c = 0; c < 3; ++c)
                    acc[c * nq + vi] += Bx * (fx[c] - fxi[c]) + By * (fy[c] - fyi[c]);
                if (op->penalty_lf) {
                    real pen[3];
                    lf_penalty(ui, up, g, nxi, nyi, pen);
                    for (int c = 0; c < 3; ++c) acc[c * nq + vi] -= m * pen[c];
                }
            }
        }
        const double *sx = op->src_x + (size_t)k * nq, *sy = op->src_y + (size_t)k * nq;
        const double *J = op->J_vol + (size_t)k * nq;
        double *duk = du + (size_t)k * 3 * nq;
        int finite = 1;
        for (int i = 0; i < nq; ++i) {
            real h = uk[i];
            real minv = 1.0 / (op->M_diag[i] * J[i]);
            real r0 = -acc[i];
            real r1 = -acc[nq + i] - g * h * sx[i];
            real r2 = -acc[2 * nq + i] - g * h * sy[i];
            duk[i] = minv * r0;
            duk[nq + i] = minv * r1;
            duk[2 * nq + i] = minv * r2;
            if (!isfinite(duk[i]) || !isfinite(duk[nq + i]) || !isfinite(duk[2 * nq + i])) finite = 0;
        }
        if (!finite) {
            if (bad_elem) *bad_elem = k;
            return ORACLE_ERR_NONFINITE;
        }
    }
    return ORACLE_OK;
}

/* ---- LSRK45 (solver.hpp:439-484) ------------------------------------------ */

static const real LS_A[5] = {0.0, -0.41789047449985195, -1.192151694642677,
                               -1.6977846924715279, -1.5141834442571558};
static const real LS_B[5] = {0.14965902199922912, 0.37921031299962726, 0.8229550293869817,
                               0.6994504559491221, 0.15305724796815198};

/* n = K*3*(Np or nq) state entries; res must be zero-initialised on the first
 * call (the reference resizes/zeroes it on entry, solver.hpp:470-473). */
int oracle_step_lsrk45(const oracle_ops *op, double *u, double *res, real dt, int nsteps,
                       int *bad_elem) {
    int nloc = op->scheme == 1 ? op->nq : op->Np;
    size_t n = (size_t)op->K * 3 * nloc;
    size_t nproj = (size_t)op->K * 3 * (op->nq + op->nf);
    double *du = (double *)malloc(sizeof(real) * n);
    double *proj = op->scheme == 1 ? NULL : (double *)malloc(sizeof(real) * nproj);
    int err = 0;
    if (!(dt > 0.0)) err = -1;
    for (int st = 0; st < nsteps && !err; ++st)
        for (int s = 0; s < 5 && !err; ++s) {
            err = op->scheme == 1 ? oracle_rhs_sbp(op, u, du, NULL, 0, bad_elem)
                                  : oracle_rhs(op, u, du, proj, bad_elem);
            if (err) break;
            for (size_t i = 0; i < n; ++i) {
                res[i] = LS_A[s] * res[i] + dt * du[i];
                u[i] += LS_B[s] * res[i];
            }
        }
    free(du);
    free(proj);
    return err;
}

/* ---- diagnostics (diagnostics.hpp:142-267, run.hpp:65-68) -----------------
 * Always double arithmetic (the terms are compared bit-for-bit).
 *
 * project_nodal (diagnostics.hpp:226-230): u_modal[k] = Pq * u_nodal[k],
 * k-ascending dot products.  Pq is Np x nq column-major. */
void oracle_project_nodal(int K, int Np, int nq, int ncol, const double *Pq, const double *u_nodal,
                          double *u_modal) {
    for (int k = 0; k < K; ++k)
        for (int c = 0; c < ncol; ++c)
            for (int n = 0; n < Np; ++n) {
                double s = 0.0;
                for (int q = 0; q < nq; ++q)
                    s += Pq[n + (size_t)q * Np] * u_nodal[((size_t)k * ncol + c) * nq + q];
                u_modal[((size_t)k * ncol + c) * Np + n] = s;
            }
}

/* vortex_exact (diagnostics.hpp:41-53); p = VortexParams {h_inf, u_inf, v_inf,
 * beta, g, xc, yc} */
static void vortex_exact(const double *p, double x, double y, double t, double *ue) {
    double xt = x - p[5] - p[1] * t;
    double yt = y - p[6] - p[2] * t;
    double r2 = xt * xt + yt * yt;
    double e = exp(-(r2 - 1.0));
    double h = p[0] - p[3] * p[3] / (32.0 * M_PI * M_PI) * e * e;
    double uu = p[1] - p[3] / (2.0 * M_PI) * e * yt;
    double vv = p[2] + p[3] / (2.0 * M_PI) * e * xt;
    ue[0] = h;
    ue[1] = h * uu;
    ue[2] = h * vv;
}

/* Terms of compute_invariants (what = 0: wJ*h, wJ*hu, wJ*hv, wJ*entropy),
 * l2_error vs a discrete state (what = 1: wJ*d*d per component), vs the
 * vortex (what = 2) or vs the lake-at-rest state (what = 3), in the reference's accumulation order (element k, then
 * fine point i).  FineQuad::element_geometry (diagnostics.hpp:155-165) gives
 * xy = V*map, J = dr0*ds1 - ds0*dr1 with dr = Vr*map, ds = Vs*map.
 *   u, u_ref [K][3][Np] modal; b [K][Np] modal; map [K][2][Np];
 *   V, Vr, Vs nfine x Np column-major; w [nfine].
 * Outputs (any may be NULL): terms [K][nfine][4], sums[4] = the reference's
 * serial sums, *min_h.  Returns 0, ORACLE_ERR_POSITIVITY (h <= 0 at a fine
 * point, entropy() -> check_positive, swe.hpp:47-48) or 3 (J <= 0), element
 * in *bad_elem. */
int oracle_diag(int K, int Np, int nfine, const double *w, const double *V, const double *Vr,
                const double *Vs, const double *map, const double *u, const double *b,
                const double *u_ref, const double *vortex, double t, double g, int what,
                double *terms, double *sums, double *min_h, long *bad_elem) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    double mh = 1e300;
    for (long k = 0; k < K; ++k) {
        const double *mk = map + (size_t)k * 2 * Np;
        const double *uk = u + (size_t)k * 3 * Np;
        double dk[3 * 64];
        if (what == 1) /* u_modal[k] - ref_modal[k] (diagnostics.hpp:210) */
            for (int x = 0; x < 3 * Np; ++x) dk[x] = uk[x] - u_ref[(size_t)k * 3 * Np + x];
        for (int i = 0; i < nfine; ++i) {
            double xy[2], dr[2], ds[2];
            for (int c = 0; c < 2; ++c) {
                double a = 0.0, r = 0.0, q = 0.0;
                for (int n = 0; n < Np; ++n) a += V[i + (size_t)n * nfine] * mk[c * Np + n];
                for (int n = 0; n < Np; ++n) r += Vr[i + (size_t)n * nfine] * mk[c * Np + n];
                for (int n = 0; n < Np; ++n) q += Vs[i + (size_t)n * nfine] * mk[c * Np + n];
                xy[c] = a;
                dr[c] = r;
                ds[c] = q;
            }
            double J = dr[0] * ds[1] - ds[0] * dr[1];
            if (J <= 0.0) {
                if (bad_elem) *bad_elem = k;
                return 3;
            }
            double wJ = w[i] * J;
            const double *src = what == 1 ? dk : uk;
            double uq[3];
            for (int c = 0; c < 3; ++c) {
                double a = 0.0;
                for (int n = 0; n < Np; ++n) a += V[i + (size_t)n * nfine] * src[c * Np + n];
                uq[c] = a;
            }
            double tm[4] = {0.0, 0.0, 0.0, 0.0};
            if (what == 0) {
                double bq = 0.0;
                for (int n = 0; n < Np; ++n) bq += V[i + (size_t)n * nfine] * b[(size_t)k * Np + n];
                if (!(uq[0] > 0.0)) {
                    if (bad_elem) *bad_elem = k;
                    return ORACLE_ERR_POSITIVITY;
                }
                double vx = uq[1] / uq[0], vy = uq[2] / uq[0];
                double ent = 0.5 * uq[0] * (vx * vx + vy * vy) + 0.5 * g * uq[0] * uq[0] + g * uq[0] * bq;
                tm[0] = wJ * uq[0];
                tm[1] = wJ * uq[1];
                tm[2] = wJ * uq[2];
                tm[3] = wJ * ent;
                if (uq[0] < mh) mh = uq[0]; /* std::min(min_h, h) */
            } else if (what == 1) {
                for (int c = 0; c < 3; ++c) tm[c] = wJ * uq[c] * uq[c];
            } else {
                double ue[3];
                if (what == 2) {
                    vortex_exact(vortex, xy[0], xy[1], t, ue);
                } else { /* lake at rest, build_lake_case init (run.hpp:125-127, diagnostics.hpp:55-57) */
                    ue[0] = 2.0 - (0.1 * sin(2.0 * M_PI * xy[0]) * cos(2.0 * M_PI * xy[0]) + 0.5);
                    ue[1] = 0.0;
                    ue[2] = 0.0;
                }
                for (int c = 0; c < 3; ++c) {
                    double d = uq[c] - ue[c];
                    tm[c] = wJ * d * d;
                }
            }
            for (int c = 0; c < 4; ++c) s[c] += tm[c];
            if (terms)
                for (int c = 0; c < 4; ++c) terms[((size_t)k * nfine + i) * 4 + c] = tm[c];
        }
    }
    if (sums)
        for (int c = 0; c < 4; ++c) sums[c] = s[c];
    if (min_h) *min_h = mh;
    return ORACLE_OK;
}

/* ---- volume-kernel cost study (bench.hpp:55-128) ---------------------------
 * u [K][3][n] (n x 3 column-major per element), Q n x n column-major, y [K][3][n].
 * x-direction physical flux (swe.hpp:60-66) and EC flux (swe.hpp:69-85). */
void oracle_ratio_matvec(int n, int K, const double *Q, const double *u, double g, double *y) {
    double *f = (double *)malloc(sizeof(double) * 3 * (size_t)n);
    for (int k = 0; k < K; ++k) {
        const double *uk = u + (size_t)k * 3 * n;
        for (int i = 0; i < n; ++i) {
            double h = uk[i], hu = uk[n + i], hv = uk[2 * n + i];
            double vx = hu / h, vy = hv / h;
            double p = 0.5 * g * h * h;
            f[i] = hu;
            f[n + i] = hu * vx + p;
            f[2 * n + i] = hu * vy;
        }
        for (int c = 0; c < 3; ++c) /* y = Q * f, k-ascending (Eigen shim product) */
            for (int i = 0; i < n; ++i) {
                double s = 0.0;
                for (int j = 0; j < n; ++j) s += Q[i + (size_t)j * n] * f[c * n + j];
                y[((size_t)k * 3 + c) * n + i] = s;
            }
    }
    free(f);
}

static void ec_flux_x(const double *a, const double *b, double g, double *f) {
    double uxL = a[1] / a[0], uyL = a[2] / a[0];
    double uxR = b[1] / b[0], uyR = b[2] / b[0];
    double h_avg = 0.5 * (a[0] + b[0]);
    double h2_avg = 0.5 * (a[0] * a[0] + b[0] * b[0]);
    double ux_avg = 0.5 * (uxL + uxR), uy_avg = 0.5 * (uyL + uyR);
    double p = g * h_avg * h_avg - 0.5 * g * h2_avg;
    double hu_avg = 0.5 * (a[1] + b[1]);
    f[0] = hu_avg;
    f[1] = hu_avg * ux_avg + p;
    f[2] = hu_avg * uy_avg;
}

/* kernel_fluxdiff (nq = n) / kernel_fluxdiff_skew (nq < n): pass 1 j < nq over all
 * rows, pass 2 j >= nq over rows i < nq; j outer, i inner. */
void oracle_ratio_fluxdiff(int n, int nq, int K, const double *Q, const double *u, double g, double *y) {
    for (int k = 0; k < K; ++k) {
        const double *uk = u + (size_t)k * 3 * n;
        double *yk = y + (size_t)k * 3 * n;
        for (int x = 0; x < 3 * n; ++x) yk[x] = 0.0;
        for (int pass = 0; pass < 2; ++pass) {
            int j0 = pass == 0 ? 0 : nq, j1 = pass == 0 ? nq : n, i1 = pass == 0 ? n : nq;
            for (int j = j0; j < j1; ++j) {
                double uj[3] = {uk[j], uk[n + j], uk[2 * n + j]};
                for (int i = 0; i < i1; ++i) {
                    double ui[3] = {uk[i], uk[n + i], uk[2 * n + i]}, fs[3];
                    ec_flux_x(ui, uj, g, fs);
                    double q2 = 2.0 * Q[i + (size_t)j * n];
                    yk[i] += q2 * fs[0];
                    yk[n + i] += q2 * fs[1];
                    yk[2 * n + i] += q2 * fs[2];
                }
            }
        }
    }
}
