// Native case setup: reference-element operators, meshes, geometry,
// connectivity, element operators and initial states for the reference's
// problems (include/swedg_setup.h).  Host C++17, std::thread-parallel over
// elements, O(K log K) connectivity (the reference's std::map edge table and
// O(n^2) periodic matching, mesh.hpp:156-249, do not scale to K = 8.4M).
//
// Dense kernels (products, Cholesky, LU) use fixed evaluation orders —
// products k-ascending, unblocked Cholesky, row-pivoted Doolittle LU — the
// same orders as the oracle build of the reference, so a case built here
// matches the golden fixtures to the last bit (tests/test_setup.py).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <fstream>
#include <functional>
#include <map>
#include <mutex>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/swedg_setup.h"
#include "quad_data.inc"

namespace swedg {
namespace setup {

// ---------------------------------------------------------------------------
// dense column-major matrix
struct Mat {
    int r = 0, c = 0;
    std::vector<double> d;
    Mat() = default;
    Mat(int r_, int c_) : r(r_), c(c_), d((size_t)r_ * c_, 0.0) {}
    double& operator()(int i, int j) { return d[i + (size_t)j * r]; }
    double operator()(int i, int j) const { return d[i + (size_t)j * r]; }
};

Mat mul(const Mat& a, const Mat& b) {
    if (a.c != b.r) throw std::logic_error("setup: product shape");
    Mat o(a.r, b.c);
    for (int j = 0; j < b.c; ++j)
        for (int i = 0; i < a.r; ++i) {
            double s = 0.0;
            for (int k = 0; k < a.c; ++k) s += a(i, k) * b(k, j);
            o(i, j) = s;
        }
    return o;
}

Mat transpose(const Mat& a) {
    Mat t(a.c, a.r);
    for (int j = 0; j < a.c; ++j)
        for (int i = 0; i < a.r; ++i) t(j, i) = a(i, j);
    return t;
}

Mat scale_cols(const Mat& a, const std::vector<double>& w) {  // A * diag(w)
    Mat o(a.r, a.c);
    for (int j = 0; j < a.c; ++j)
        for (int i = 0; i < a.r; ++i) o(i, j) = a(i, j) * w[j];
    return o;
}

Mat identity(int n) {
    Mat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
}

// unblocked lower Cholesky; returns false if not SPD
bool cholesky(const Mat& a, Mat& L) {
    int n = a.r;
    L = a;
    for (int k = 0; k < n; ++k) {
        double x = L(k, k);
        for (int j = 0; j < k; ++j) x -= L(k, j) * L(k, j);
        if (!(x > 0.0)) return false;
        x = std::sqrt(x);
        L(k, k) = x;
        for (int i = k + 1; i < n; ++i) {
            double s = L(i, k);
            for (int j = 0; j < k; ++j) s -= L(i, j) * L(k, j);
            L(i, k) = s / x;
        }
    }
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < j; ++i) L(i, j) = 0.0;
    return true;
}

Mat chol_solve(const Mat& L, const Mat& b) {
    int n = L.r;
    Mat x = b;
    for (int col = 0; col < b.c; ++col) {
        for (int i = 0; i < n; ++i) {
            double s = x(i, col);
            for (int j = 0; j < i; ++j) s -= L(i, j) * x(j, col);
            x(i, col) = s / L(i, i);
        }
        for (int i = n - 1; i >= 0; --i) {
            double s = x(i, col);
            for (int j = i + 1; j < n; ++j) s -= L(j, i) * x(j, col);
            x(i, col) = s / L(i, i);
        }
    }
    return x;
}

struct LU {
    Mat lu;
    std::vector<int> perm;
    explicit LU(const Mat& a) : lu(a), perm(a.r) {
        int n = a.r;
        for (int i = 0; i < n; ++i) perm[i] = i;
        for (int k = 0; k < n; ++k) {
            int p = k;
            double best = std::abs(lu(k, k));
            for (int i = k + 1; i < n; ++i)
                if (std::abs(lu(i, k)) > best) {
                    best = std::abs(lu(i, k));
                    p = i;
                }
            if (p != k) {
                for (int j = 0; j < n; ++j) std::swap(lu(k, j), lu(p, j));
                std::swap(perm[k], perm[p]);
            }
            double piv = lu(k, k);
            if (piv == 0.0) continue;
            for (int i = k + 1; i < n; ++i) {
                lu(i, k) /= piv;
                double l = lu(i, k);
                for (int j = k + 1; j < n; ++j) lu(i, j) -= l * lu(k, j);
            }
        }
    }
    // solve for a column-major right-hand side block b (n x m), writing x
    void solve(const double* b, int m, double* x) const {
        int n = lu.r;
        for (int col = 0; col < m; ++col) {
            double* xc = x + (size_t)col * n;
            const double* bc = b + (size_t)col * n;
            for (int i = 0; i < n; ++i) xc[i] = bc[perm[i]];
            for (int i = 0; i < n; ++i) {
                double s = xc[i];
                for (int j = 0; j < i; ++j) s -= lu(i, j) * xc[j];
                xc[i] = s;
            }
            for (int i = n - 1; i >= 0; --i) {
                double s = xc[i];
                for (int j = i + 1; j < n; ++j) s -= lu(i, j) * xc[j];
                xc[i] = s / lu(i, i);
            }
        }
    }
};

void parallel_for(long n, int threads, const std::function<void(long, long)>& fn) {
    if (threads <= 1 || n < 1024) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> pool;
    std::exception_ptr err;
    std::mutex mu;
    long chunk = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        long lo = t * chunk, hi = std::min(n, lo + chunk);
        if (lo >= hi) break;
        pool.emplace_back([&, lo, hi] {
            try {
                fn(lo, hi);
            } catch (...) {
                std::lock_guard<std::mutex> g(mu);
                if (!err) err = std::current_exception();
            }
        });
    }
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
}

// ---------------------------------------------------------------------------
// quadrature (quadrature.hpp)
constexpr double kInvSqrt2 = 1.0 / 1.4142135623730951;
const double kFaceNormal[3][2] = {{0.0, -1.0}, {kInvSqrt2, kInvSqrt2}, {-1.0, 0.0}};
const double kFaceJac[3] = {1.0, 1.4142135623730951, 1.0};

struct Rule2D {
    std::vector<double> x, y, w;
    int size() const { return (int)w.size(); }
};
struct SurfRule {
    std::vector<double> x, y, w;
    std::vector<int> face;
    int npf = 0;
    int size() const { return (int)w.size(); }
};

void face_point(int f, double r, double& x, double& y) {
    if (f == 0) {
        x = r;
        y = -1.0;
    } else if (f == 1) {
        x = -r;
        y = r;
    } else {
        x = -1.0;
        y = -r;
    }
}

// Gauss-Legendre by Newton on P_n (same iteration as quadrature.hpp:111-144)
void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
    x.assign(n, 0.0);
    w.assign(n, 0.0);
    for (int i = 0; i < n; ++i) {
        double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));
        double p0, p1;
        for (int it = 0; it < 100; ++it) {
            p0 = 1.0;
            p1 = t;
            for (int k = 2; k <= n; ++k) {
                double p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            double dp = n * (t * p1 - p0) / (t * t - 1.0);
            double dt = p1 / dp;
            t -= dt;
            if (std::abs(dt) < 1e-15) break;
        }
        p0 = 1.0;
        p1 = t;
        for (int k = 2; k <= n; ++k) {
            double p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k;
            p0 = p1;
            p1 = p2;
        }
        double dp = n * (t * p1 - p0) / (t * t - 1.0);
        x[n - 1 - i] = t;
        w[n - 1 - i] = 2.0 / ((1.0 - t * t) * dp * dp);
    }
}

SurfRule surface_rule(int npf) {
    std::vector<double> r1, w1;
    gauss_legendre(npf, r1, w1);
    SurfRule s;
    s.npf = npf;
    for (int f = 0; f < 3; ++f)
        for (int k = 0; k < npf; ++k) {
            double x, y;
            face_point(f, r1[k], x, y);
            s.x.push_back(x);
            s.y.push_back(y);
            s.w.push_back(w1[k] * kFaceJac[f]);
            s.face.push_back(f);
        }
    return s;
}

Rule2D volume_rule_by_degree(int degree) {
    for (const auto& v : quad_data::vol_rules)
        if (v.key >= degree) {
            Rule2D q;
            for (int i = 0; i < v.n; ++i) {
                q.x.push_back(v.data[i][0]);
                q.y.push_back(v.data[i][1]);
                q.w.push_back(v.data[i][2]);
            }
            return q;
        }
    throw std::invalid_argument("degree out of table range");
}

// ---------------------------------------------------------------------------
// orthonormal Dubiner basis (refelem.hpp:19-121)
std::vector<double> jacobi_p(const std::vector<double>& x, double a, double b, int n) {
    size_t np = x.size();
    double gamma0 = std::pow(2.0, a + b + 1) / (a + b + 1) * std::tgamma(a + 1) * std::tgamma(b + 1) /
                    std::tgamma(a + b + 1);
    std::vector<double> pl0(np, 1.0 / std::sqrt(gamma0));
    if (n == 0) return pl0;
    double gamma1 = (a + 1) * (b + 1) / (a + b + 3) * gamma0;
    std::vector<double> pl1(np);
    for (size_t k = 0; k < np; ++k) pl1[k] = ((a + b + 2) * x[k] / 2.0 + (a - b) / 2.0) / std::sqrt(gamma1);
    if (n == 1) return pl1;
    double aold = 2.0 / (2 + a + b) * std::sqrt((a + 1) * (b + 1) / (a + b + 3));
    for (int i = 1; i < n; ++i) {
        double h1 = 2.0 * i + a + b;
        double anew = 2.0 / (h1 + 2) *
                      std::sqrt((i + 1) * (i + 1 + a + b) * (i + 1 + a) * (i + 1 + b) / ((h1 + 1) * (h1 + 3)));
        double bnew = -(a * a - b * b) / (h1 * (h1 + 2));
        std::vector<double> pl2(np);
        double ia = 1.0 / anew;
        for (size_t k = 0; k < np; ++k) pl2[k] = ia * (-aold * pl0[k] + (x[k] - bnew) * pl1[k]);
        pl0 = pl1;
        pl1 = pl2;
        aold = anew;
    }
    return pl1;
}

std::vector<double> grad_jacobi_p(const std::vector<double>& x, double a, double b, int n) {
    if (n == 0) return std::vector<double>(x.size(), 0.0);
    std::vector<double> p = jacobi_p(x, a + 1, b + 1, n - 1);
    double s = std::sqrt(n * (n + a + b + 1));
    for (auto& v : p) v = s * v;
    return p;
}

void collapse(const std::vector<double>& x, const std::vector<double>& y, std::vector<double>& a,
              std::vector<double>& b) {
    size_t n = x.size();
    a.resize(n);
    b.resize(n);
    for (size_t i = 0; i < n; ++i) {
        a[i] = (std::abs(1.0 - y[i]) > 1e-12) ? 2.0 * (1.0 + x[i]) / (1.0 - y[i]) - 1.0 : -1.0;
        b[i] = y[i];
    }
}

int basis_dim(int N) { return (N + 1) * (N + 2) / 2; }

Mat vandermonde(int N, const std::vector<double>& x, const std::vector<double>& y) {
    std::vector<double> a, b;
    collapse(x, y, a, b);
    Mat V((int)x.size(), basis_dim(N));
    int col = 0;
    for (int i = 0; i <= N; ++i)
        for (int j = 0; j <= N - i; ++j) {
            std::vector<double> h1 = jacobi_p(a, 0, 0, i), h2 = jacobi_p(b, 2.0 * i + 1.0, 0, j);
            for (size_t k = 0; k < a.size(); ++k) V((int)k, col) = std::sqrt(2.0) * h1[k] * h2[k] * std::pow(1.0 - b[k], i);
            ++col;
        }
    return V;
}

void grad_vandermonde(int N, const std::vector<double>& x, const std::vector<double>& y, Mat& Vx, Mat& Vy) {
    std::vector<double> a, b;
    collapse(x, y, a, b);
    int n = (int)x.size();
    Vx = Mat(n, basis_dim(N));
    Vy = Mat(n, basis_dim(N));
    int col = 0;
    for (int id = 0; id <= N; ++id)
        for (int jd = 0; jd <= N - id; ++jd) {
            std::vector<double> fa = jacobi_p(a, 0, 0, id), dfa = grad_jacobi_p(a, 0, 0, id);
            std::vector<double> gb = jacobi_p(b, 2.0 * id + 1.0, 0, jd), dgb = grad_jacobi_p(b, 2.0 * id + 1.0, 0, jd);
            for (int k = 0; k < n; ++k) {
                double omb = 1.0 - b[k];
                double d_dr = dfa[k] * gb[k];
                if (id > 0) d_dr *= std::pow(0.5 * omb, id - 1);
                double d_ds = dfa[k] * gb[k] * (0.5 * (1.0 + a[k]));
                if (id > 0) d_ds *= std::pow(0.5 * omb, id - 1);
                double tmp = dgb[k] * std::pow(0.5 * omb, id);
                if (id > 0) tmp -= 0.5 * id * gb[k] * std::pow(0.5 * omb, id - 1);
                d_ds += fa[k] * tmp;
                Vx(k, col) = std::pow(2.0, id + 0.5) * d_dr;
                Vy(k, col) = std::pow(2.0, id + 0.5) * d_ds;
            }
            ++col;
        }
}

struct RefOps {
    int N = 0, Np = 0, nq = 0, nf = 0, npf = 0;
    Rule2D vol;
    SurfRule surf;
    Mat Vq, Vf, M, Pq, Dx, Dy, E, Qx, Qy, Qh_x, Qh_y;
    std::vector<double> Bx, By;
};

Mat hybridized(const Mat& Q, const Mat& E, const std::vector<double>& B) {
    int nq = Q.r, nf = (int)B.size();
    Mat Qh(nq + nf, nq + nf);
    Mat EtB = scale_cols(transpose(E), B);
    for (int j = 0; j < nq; ++j)
        for (int i = 0; i < nq; ++i) Qh(i, j) = 0.5 * (Q(i, j) - Q(j, i));
    for (int j = 0; j < nf; ++j)
        for (int i = 0; i < nq; ++i) Qh(i, nq + j) = 0.5 * EtB(i, j);
    for (int j = 0; j < nq; ++j)
        for (int i = 0; i < nf; ++i) Qh(nq + i, j) = (-0.5 * B[i]) * E(i, j);
    for (int i = 0; i < nf; ++i) Qh(nq + i, nq + i) = 0.5 * B[i];
    return Qh;
}

// build_ref_operators (refelem.hpp:159-218)
RefOps build_ref_ops(int N, const Rule2D& vol, const SurfRule& surf) {
    RefOps o;
    o.N = N;
    o.Np = basis_dim(N);
    o.vol = vol;
    o.surf = surf;
    o.nq = vol.size();
    o.nf = surf.size();
    o.npf = surf.npf;
    o.Vq = vandermonde(N, vol.x, vol.y);
    o.Vf = vandermonde(N, surf.x, surf.y);
    Mat VqT = transpose(o.Vq);
    o.M = mul(scale_cols(VqT, vol.w), o.Vq);
    Mat L;
    if (!cholesky(o.M, L)) throw std::runtime_error("mass matrix not SPD; quadrature insufficient");
    Mat Wd(o.nq, o.nq);
    for (int i = 0; i < o.nq; ++i) Wd(i, i) = vol.w[i];
    o.Pq = chol_solve(L, mul(VqT, Wd));
    Mat Vqx, Vqy;
    grad_vandermonde(N, vol.x, vol.y, Vqx, Vqy);
    o.Dx = mul(o.Pq, Vqx);
    o.Dy = mul(o.Pq, Vqy);
    o.E = mul(o.Vf, o.Pq);
    o.Bx.resize(o.nf);
    o.By.resize(o.nf);
    for (int i = 0; i < o.nf; ++i) {
        o.Bx[i] = surf.w[i] * kFaceNormal[surf.face[i]][0];
        o.By[i] = surf.w[i] * kFaceNormal[surf.face[i]][1];
    }
    Mat PqT = transpose(o.Pq);
    o.Qx = mul(mul(PqT, mul(o.M, o.Dx)), o.Pq);
    o.Qy = mul(mul(PqT, mul(o.M, o.Dy)), o.Pq);
    o.Qh_x = hybridized(o.Qx, o.E, o.Bx);
    o.Qh_y = hybridized(o.Qy, o.E, o.By);
    // construction-time identity check (refelem.hpp:200-216): Qh + Qh^T = blockdiag(0, B), Qh 1 = 0
    double r = 0.0;
    int nh = o.nq + o.nf;
    for (int j = 0; j < nh; ++j)
        for (int i = 0; i < nh; ++i) {
            double bx = (i == j && i >= o.nq) ? o.Bx[i - o.nq] : 0.0;
            double by = (i == j && i >= o.nq) ? o.By[i - o.nq] : 0.0;
            r = std::max(r, std::abs(o.Qh_x(i, j) + o.Qh_x(j, i) - bx));
            r = std::max(r, std::abs(o.Qh_y(i, j) + o.Qh_y(j, i) - by));
        }
    for (int i = 0; i < nh; ++i) {
        double sx = 0.0, sy = 0.0;
        for (int j = 0; j < nh; ++j) {
            sx += o.Qh_x(i, j);
            sy += o.Qh_y(i, j);
        }
        r = std::max(r, std::max(std::abs(sx), std::abs(sy)));
    }
    if (r > 1e-12) throw std::runtime_error("reference operator identities violated, residual " + std::to_string(r));
    return o;
}

struct SbpOps {
    Mat Qx, Qy;
    std::vector<double> M_diag;
    std::vector<int> face_index;
};

// Gauss-Lobatto nodes/weights on [-1,1] (quadrature.hpp:145-177): Newton on P'_{n-1}
void gauss_lobatto(int n, std::vector<double>& x, std::vector<double>& w) {
    if (n < 2) throw std::invalid_argument("Lobatto rule needs >= 2 points");
    x.assign(n, 0.0);
    w.assign(n, 0.0);
    auto legendre = [n](double t, double& p, double& dp) {
        double p0 = 1.0, p1 = t;
        for (int k = 2; k <= n - 1; ++k) {
            double p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k;
            p0 = p1;
            p1 = p2;
        }
        p = p1;
        dp = (n - 1) * (t * p1 - p0) / (t * t - 1.0);
    };
    for (int i = 0; i < n; ++i) {
        double t = -std::cos(M_PI * i / (n - 1));
        if (i > 0 && i < n - 1)
            for (int it = 0; it < 100; ++it) {
                double p, dp;
                legendre(t, p, dp);
                const double d2p = (2.0 * t * dp - n * (n - 1) * p) / (1.0 - t * t);
                const double dt = dp / d2p;
                t -= dt;
                if (std::abs(dt) < 1e-15) break;
            }
        double p, dp;
        legendre(t, p, dp);
        x[i] = t;
        w[i] = 2.0 / (n * (n - 1) * p * p);
    }
}

// surface_rule_1d (quadrature.hpp:180-207): a caller-chosen 1D family on every face
SurfRule surface_rule_1d(int npf, int family, int* degree) {
    if (family == SWEDG_SBP_LEGENDRE) {
        SurfRule s = surface_rule(npf);
        *degree = 2 * npf - 1;
        return s;
    }
    std::vector<double> r1, w1;
    gauss_lobatto(npf, r1, w1);
    *degree = 2 * npf - 3;
    SurfRule s;
    s.npf = npf;
    for (int f = 0; f < 3; ++f)
        for (int k = 0; k < npf; ++k) {
            double x, y;
            face_point(f, r1[k], x, y);
            s.x.push_back(x);
            s.y.push_back(y);
            s.w.push_back(w1[k] * kFaceJac[f]);
            s.face.push_back(f);
        }
    return s;
}

// verify_exactness (quadrature.hpp:91-108) against the exact monomial integrals (:72-77)
double exactness_error(const Rule2D& q, int degree) {
    if (q.size() == 0) throw std::invalid_argument("empty quadrature rule");
    auto I = [](int m) { return m % 2 == 0 ? 2.0 / (m + 1) : 0.0; };
    double err = 0.0;
    for (int d = 0; d <= degree; ++d)
        for (int i = 0; i <= d; ++i) {
            const int j = d - i;
            double approx = 0.0;
            for (int k = 0; k < q.size(); ++k) approx += q.w[k] * std::pow(q.x[k], i) * std::pow(q.y[k], j);
            const double exact = ((i % 2 == 0) ? -1.0 : 1.0) / (i + 1) * (I(i + j + 1) - I(j));
            err = std::max(err, std::abs(approx - exact));
        }
    return err;
}

// An SBP volume rule with its embedded surface rule (make_sbp, quadrature.hpp:248-288)
struct SbpRule {
    Rule2D vol;
    SurfRule surf;
    std::vector<int> fidx;
};

SbpRule make_sbp(int N, int family, const Rule2D& vol, int npf) {
    SbpRule r;
    r.vol = vol;
    int sdeg = 0;
    r.surf = surface_rule_1d(npf, family, &sdeg);
    if (sdeg < 2 * N) throw std::runtime_error("SBP surface rule exactness below 2N");
    r.fidx.assign(r.surf.size(), -1);
    std::vector<char> used(vol.size(), 0);
    for (int i = 0; i < r.surf.size(); ++i) {
        int best = -1;
        double bestd = 1e100;
        for (int j = 0; j < vol.size(); ++j) {
            const double d = std::hypot(r.surf.x[i] - vol.x[j], r.surf.y[i] - vol.y[j]);
            if (d < bestd) {
                bestd = d;
                best = j;
            }
        }
        if (bestd > 1e-12 || used[best]) throw std::runtime_error("SBP surface node does not embed in volume rule");
        used[best] = 1;
        r.fidx[i] = best;
    }
    for (int i = 0; i < vol.size(); ++i)
        if (vol.w[i] <= 0.0) throw std::runtime_error("SBP rule has nonpositive weight");
    if (exactness_error(vol, 2 * N - 1) > 1e-12) throw std::runtime_error("SBP volume rule failed exactness check");
    return r;
}

// load_sbp_rule_file (quadrature.hpp:290-318): header "degree=<d> nodes_per_face=<m>",
// then one node per line "x y w", the first 3m nodes being the face nodes face-major
SbpRule load_sbp_rule_file(const std::string& path, int N, int family) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("SBP rule unavailable: cannot open " + path);
    std::string header;
    std::getline(in, header);
    int deg = -1, npf = -1;
    {
        std::istringstream hs(header);
        std::string tok;
        while (hs >> tok) {
            if (tok.rfind("degree=", 0) == 0) deg = std::stoi(tok.substr(7));
            if (tok.rfind("nodes_per_face=", 0) == 0) npf = std::stoi(tok.substr(15));
        }
    }
    if (deg < 2 * N - 1 || npf < N + 1) throw std::runtime_error("SBP rule file header mismatch for " + path);
    Rule2D vol;
    double a, b, c;
    while (in >> a >> b >> c) {
        vol.x.push_back(a);
        vol.y.push_back(b);
        vol.w.push_back(c);
    }
    return make_sbp(N, family, vol, npf);
}

// sbp_rule (quadrature.hpp:320-343): Gauss-Legendre edges from the tables, Gauss-Lobatto
// edges only from a data file sbp_lobatto_N<N>.txt (in data_dir, or the working directory);
// rule_file overrides both (the caller's own rule in the file format above)
SbpRule sbp_rule(int N, int family, const std::string& data_dir, const std::string& rule_file) {
    if (!rule_file.empty()) return load_sbp_rule_file(rule_file, N, family);
    if (family == SWEDG_SBP_LEGENDRE) {
        for (const auto& v : quad_data::sbp_rules)
            if (v.key == N) {
                Rule2D vol;
                for (int i = 0; i < v.n; ++i) {
                    vol.x.push_back(v.data[i][0]);
                    vol.y.push_back(v.data[i][1]);
                    vol.w.push_back(v.data[i][2]);
                }
                return make_sbp(N, family, vol, v.npf);
            }
        throw std::runtime_error("SBP rule unavailable for (N=" + std::to_string(N) + ", legendre)");
    }
    const std::string name = "sbp_lobatto_N" + std::to_string(N) + ".txt";
    return load_sbp_rule_file(data_dir.empty() ? name : data_dir + "/" + name, N, family);
}

// build_traditional_sbp (refelem.hpp:224-274): the congruence of the hybridized
// operators onto the volume nodes
void build_sbp(int N, RefOps& ref, SbpOps& s, const SbpRule& rule) {
    const Rule2D& vol = rule.vol;
    const SurfRule& surf = rule.surf;
    const std::vector<int>& fidx = rule.fidx;
    ref = build_ref_ops(N, vol, surf);
    int nq = vol.size(), nf = surf.size();
    auto congruence = [&](const Mat& Qh) {
        Mat Q(nq, nq);
        for (int j = 0; j < nq; ++j)
            for (int i = 0; i < nq; ++i) Q(i, j) = Qh(i, j);
        for (int i = 0; i < nf; ++i) {
            int vi = fidx[i];
            for (int j = 0; j < nq; ++j) Q(vi, j) += Qh(nq + i, j);
            for (int j = 0; j < nq; ++j) Q(j, vi) += Qh(j, nq + i);
            for (int j = 0; j < nf; ++j) Q(vi, fidx[j]) += Qh(nq + i, nq + j);
        }
        return Q;
    };
    s.Qx = congruence(ref.Qh_x);
    s.Qy = congruence(ref.Qh_y);
    s.M_diag = vol.w;
    s.face_index = fidx;
}

// ---------------------------------------------------------------------------
// mesh (mesh.hpp)
struct Domain {
    double xc = 0, yc = 0, Lx = 2, Ly = 2;
    double xmin() const { return xc - Lx / 2; }
    double xmax() const { return xc + Lx / 2; }
    double ymin() const { return yc - Ly / 2; }
    double ymax() const { return yc + Ly / 2; }
};

struct Mesh {
    std::vector<std::array<double, 2>> verts;
    std::vector<std::array<int, 3>> tris;
    Domain dom;
    int Nmap = 0;
    std::vector<double> map_nodes;  // [K][2][Npm] (Np x 2 column-major per element)
    std::vector<std::array<int, 2>> wall_faces;
    long K() const { return (long)tris.size(); }
};

void map_lattice(int N, std::vector<double>& x, std::vector<double>& y) {
    x.clear();
    y.clear();
    for (int i = 0; i <= N; ++i)
        for (int j = 0; j <= N - i; ++j) {
            x.push_back(-1.0 + 2.0 * i / N);
            y.push_back(-1.0 + 2.0 * j / N);
        }
}

void ref_barycentric(double x, double y, double l[3]) {
    double l1 = (1.0 + x) / 2.0, l2 = (1.0 + y) / 2.0;
    l[0] = 1.0 - l1 - l2;
    l[1] = l1;
    l[2] = l2;
}

Mesh uniform_tri_mesh(int nx, int ny, const Domain& dom, bool flip_below_center) {
    if (nx < 1 || ny < 1) throw std::invalid_argument("nx, ny must be >= 1");
    Mesh m;
    m.dom = dom;
    m.verts.reserve((size_t)(nx + 1) * (ny + 1));
    for (int j = 0; j <= ny; ++j)
        for (int i = 0; i <= nx; ++i) m.verts.push_back({dom.xmin() + dom.Lx * i / nx, dom.ymin() + dom.Ly * j / ny});
    auto vid = [&](int i, int j) { return j * (nx + 1) + i; };
    m.tris.reserve((size_t)2 * nx * ny);
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            int v00 = vid(i, j), v10 = vid(i + 1, j), v01 = vid(i, j + 1), v11 = vid(i + 1, j + 1);
            double ycenter = dom.ymin() + dom.Ly * (j + 0.5) / ny;
            bool flip = flip_below_center && ycenter < dom.yc;
            if (!flip) {
                m.tris.push_back({v00, v10, v11});
                m.tris.push_back({v00, v11, v01});
            } else {
                m.tris.push_back({v00, v10, v01});
                m.tris.push_back({v10, v11, v01});
            }
        }
    return m;
}

// Quad rows [j_lo, j_hi) of a global nx x ny_tot grid on `dom` (rows outside
// [0, ny_tot) are the periodic images, used as halo rows of a y-strip).
Mesh uniform_tri_mesh_rows(int nx, int j_lo, int j_hi, int ny_tot, const Domain& dom) {
    Mesh m;
    m.dom = dom;
    const int nr = j_hi - j_lo;
    m.verts.reserve((size_t)(nx + 1) * (nr + 1));
    for (int j = j_lo; j <= j_hi; ++j)
        for (int i = 0; i <= nx; ++i) m.verts.push_back({dom.xmin() + dom.Lx * i / nx, dom.ymin() + dom.Ly * j / ny_tot});
    auto vid = [&](int i, int j) { return (j - j_lo) * (nx + 1) + i; };
    m.tris.reserve((size_t)2 * nx * nr);
    for (int j = j_lo; j < j_hi; ++j)
        for (int i = 0; i < nx; ++i) {
            int v00 = vid(i, j), v10 = vid(i + 1, j), v01 = vid(i, j + 1), v11 = vid(i + 1, j + 1);
            m.tris.push_back({v00, v10, v11});
            m.tris.push_back({v00, v11, v01});
        }
    return m;
}

void set_mapping_degree(Mesh& m, int N, int threads) {
    m.Nmap = N;
    std::vector<double> lx, ly;
    map_lattice(N, lx, ly);
    int np = basis_dim(N);
    m.map_nodes.assign((size_t)m.K() * 2 * np, 0.0);
    parallel_for(m.K(), threads, [&](long lo, long hi) {
        for (long k = lo; k < hi; ++k) {
            const auto& t = m.tris[k];
            double* nd = &m.map_nodes[(size_t)k * 2 * np];
            for (int i = 0; i < np; ++i) {
                double l[3];
                ref_barycentric(lx[i], ly[i], l);
                for (int d = 0; d < 2; ++d)
                    nd[d * np + i] = l[0] * m.verts[t[0]][d] + l[1] * m.verts[t[1]][d] + l[2] * m.verts[t[2]][d];
            }
        }
    });
}

void warp_point(const Domain& d, double c, double& x, double& y) {
    x = x + c * d.Lx * std::cos(M_PI * (x - d.xc) / d.Lx) * std::cos(1.5 * M_PI * (y - d.yc) / d.Ly);
    y = y + c * d.Ly * std::sin(2.0 * M_PI * (x - d.xc) / d.Lx) * std::cos(M_PI * (y - d.yc) / d.Ly);
}

void warp_mesh(Mesh& m, double c, int threads) {
    for (auto& v : m.verts) warp_point(m.dom, c, v[0], v[1]);
    int np = basis_dim(m.Nmap);
    parallel_for(m.K(), threads, [&](long lo, long hi) {
        for (long k = lo; k < hi; ++k) {
            double* nd = &m.map_nodes[(size_t)k * 2 * np];
            for (int i = 0; i < np; ++i) warp_point(m.dom, c, nd[i], nd[np + i]);
        }
    });
}

double min_edge_length(const Mesh& m) {
    double h = 1e300;
    for (const auto& t : m.tris)
        for (int f = 0; f < 3; ++f) {
            const auto& a = m.verts[t[f]];
            const auto& b = m.verts[t[(f + 1) % 3]];
            h = std::min(h, std::hypot(a[0] - b[0], a[1] - b[1]));
        }
    return h;
}

enum FaceType { kInterior = 0, kPeriodic = 1, kWall = 2 };
struct FaceInfo {
    int type = kWall;
    int nbr = -1, nbr_face = -1;
    double shift[2] = {0.0, 0.0};
};

// connect (mesh.hpp:156-249): same semantics, O(K log K)
std::vector<FaceInfo> connect(const Mesh& m, bool px, bool py) {
    const long K = m.K();
    std::vector<FaceInfo> faces((size_t)K * 3);
    struct EdgeRec {
        unsigned long long key;
        long ef;
    };
    std::vector<EdgeRec> edges((size_t)K * 3);
    for (long e = 0; e < K; ++e)
        for (int f = 0; f < 3; ++f) {
            unsigned a = (unsigned)m.tris[e][f], b = (unsigned)m.tris[e][(f + 1) % 3];
            unsigned lo = std::min(a, b), hi = std::max(a, b);
            edges[e * 3 + f] = {((unsigned long long)lo << 32) | hi, e * 3 + f};
        }
    std::sort(edges.begin(), edges.end(), [](const EdgeRec& x, const EdgeRec& y) {
        return x.key < y.key || (x.key == y.key && x.ef < y.ef);
    });
    std::vector<char> wall_tag((size_t)K * 3, 0);
    for (const auto& w : m.wall_faces) wall_tag[(size_t)w[0] * 3 + w[1]] = 1;
    // propagate explicit wall tags to the other side of shared edges
    for (size_t i = 0; i < edges.size();) {
        size_t j = i;
        while (j < edges.size() && edges[j].key == edges[i].key) ++j;
        bool any = false;
        for (size_t q = i; q < j; ++q) any |= wall_tag[edges[q].ef] != 0;
        if (any)
            for (size_t q = i; q < j; ++q) wall_tag[edges[q].ef] = 1;
        i = j;
    }
    std::vector<long> open;
    for (size_t i = 0; i < edges.size();) {
        size_t j = i;
        while (j < edges.size() && edges[j].key == edges[i].key) ++j;
        size_t cnt = j - i;
        if (cnt > 2) throw std::runtime_error("non-manifold edge in mesh");
        if (cnt == 2 && !wall_tag[edges[i].ef]) {
            long a = edges[i].ef, b = edges[i + 1].ef;
            faces[a].type = kInterior;
            faces[a].nbr = (int)(b / 3);
            faces[a].nbr_face = (int)(b % 3);
            faces[b].type = kInterior;
            faces[b].nbr = (int)(a / 3);
            faces[b].nbr_face = (int)(a % 3);
        } else {
            for (size_t q = i; q < j; ++q) {
                long ef = edges[q].ef;
                if (wall_tag[ef])
                    faces[ef].type = kWall;
                else
                    open.push_back(ef);
            }
        }
        i = j;
    }
    const Domain& d = m.dom;
    const double tol = 1e-8 * std::max(d.Lx, d.Ly);
    auto mid = [&](long ef, double& x, double& y) {
        const auto& a = m.verts[m.tris[ef / 3][ef % 3]];
        const auto& b = m.verts[m.tris[ef / 3][(ef % 3 + 1) % 3]];
        x = (a[0] + b[0]) / 2;
        y = (a[1] + b[1]) / 2;
    };
    // classify open faces: x-periodic lo/hi, y-periodic lo/hi, walls
    std::vector<std::pair<double, long>> xlo, xhi, ylo, yhi;
    for (long ef : open) {
        double x, y;
        mid(ef, x, y);
        bool on_x = std::abs(x - d.xmin()) < tol || std::abs(x - d.xmax()) < tol;
        bool on_y = std::abs(y - d.ymin()) < tol || std::abs(y - d.ymax()) < tol;
        if (px && on_x) {
            (std::abs(x - d.xmin()) < tol ? xlo : xhi).push_back({y, ef});
        } else if (py && on_y) {
            (std::abs(y - d.ymin()) < tol ? ylo : yhi).push_back({x, ef});
        } else {
            faces[ef].type = kWall;
        }
    }
    auto pair_up = [&](std::vector<std::pair<double, long>>& lo, std::vector<std::pair<double, long>>& hi,
                       double sx, double sy) {
        if (lo.size() != hi.size()) throw std::runtime_error("unmatched periodic face");
        std::sort(lo.begin(), lo.end());
        std::sort(hi.begin(), hi.end());
        for (size_t i = 0; i < lo.size(); ++i) {
            long a = lo[i].second, b = hi[i].second;
            double ax, ay, bx, by;
            mid(a, ax, ay);
            mid(b, bx, by);
            if (!(std::abs(ax + sx - bx) < tol && std::abs(ay + sy - by) < tol))
                throw std::runtime_error("unmatched periodic face");
            faces[a] = {kPeriodic, (int)(b / 3), (int)(b % 3), {sx, sy}};
            faces[b] = {kPeriodic, (int)(a / 3), (int)(a % 3), {-sx, -sy}};
        }
    };
    pair_up(xlo, xhi, d.Lx, 0.0);
    pair_up(ylo, yhi, 0.0, d.Ly);
    return faces;
}

// dam curve x = q(y) (mesh.hpp:378-460)
double poly(const std::vector<double>& c, double y) {
    double v = 0.0, p = 1.0;
    for (double ci : c) {
        v += ci * p;
        p *= y;
    }
    return v;
}

void snap_vertices_to_curve(Mesh& m, const std::vector<double>& qc) {
    std::map<long long, std::vector<int>> rows;
    for (size_t i = 0; i < m.verts.size(); ++i) rows[llround(m.verts[i][1] * 1e9)].push_back((int)i);
    for (auto& kv : rows) {
        const auto& ids = kv.second;
        double y = m.verts[ids[0]][1];
        double target = poly(qc, y);
        int best = -1;
        double bd = 1e300;
        for (int id : ids) {
            double dd = std::abs(m.verts[id][0] - target);
            if (dd < bd) {
                bd = dd;
                best = id;
            }
        }
        if (best >= 0) m.verts[best][0] = target;
    }
}

std::vector<std::array<int, 2>> faces_on_curve(const Mesh& m, const std::vector<double>& qc, double tol = 1e-10) {
    std::vector<std::array<int, 2>> out;
    for (long e = 0; e < m.K(); ++e)
        for (int f = 0; f < 3; ++f) {
            const auto& a = m.verts[m.tris[e][f]];
            const auto& b = m.verts[m.tris[e][(f + 1) % 3]];
            if (std::abs(a[0] - poly(qc, a[1])) < tol && std::abs(b[0] - poly(qc, b[1])) < tol)
                out.push_back({(int)e, f});
        }
    return out;
}

void fit_curve_boundary(Mesh& m, const std::vector<double>& qc, const std::vector<std::array<int, 2>>& faces) {
    std::vector<double> lx, ly;
    map_lattice(m.Nmap, lx, ly);
    int np = basis_dim(m.Nmap);
    for (const auto& ef : faces) {
        int e = ef[0], f = ef[1];
        const auto& va = m.verts[m.tris[e][f]];
        const auto& vb = m.verts[m.tris[e][(f + 1) % 3]];
        int opp = (f + 2) % 3;
        double* nd = &m.map_nodes[(size_t)e * 2 * np];
        for (int i = 0; i < np; ++i) {
            double l[3];
            ref_barycentric(lx[i], ly[i], l);
            double blend = 1.0 - l[opp];
            if (blend < 1e-13) continue;
            double t = l[(f + 1) % 3] / (l[f] + l[(f + 1) % 3]);
            double sx = va[0] + t * (vb[0] - va[0]);
            double sy = va[1] + t * (vb[1] - va[1]);
            nd[i] += blend * (poly(qc, sy) - sx);
        }
    }
}

// ---------------------------------------------------------------------------
}  // namespace setup
}  // namespace swedg

// ===========================================================================
using namespace swedg::setup;

struct swedg_case_s {
    swedg_case_config cfg{};
    int scheme = 0, N = 0, Np = 0, nq = 0, nf = 0, npf = 0;
    long K = 0;
    double g = 9.81, dt = 0.0, min_edge = 0.0;
    RefOps ref;
    SbpOps sbp;
    Mesh mesh;
    // descriptor arrays
    std::vector<double> Vq, Vf, Pq, Qr, Qs, wf, M_diag;
    std::vector<int> face_index;
    std::vector<double> gf, sJ, nx, ny, J_vol, Mh_inv;
    std::vector<int> nbr, nbr_face, face_type, perm;
    std::vector<double> u0, b, xy_vol, xy_surf, map_coeffs, volq_w, shift;
    std::vector<double> fine_w, fine_V, fine_Vr, fine_Vs;  // FineQuad (diagnostics.hpp:142-153)
    std::vector<double> lattice_V;                        // basis at the mapping lattice (LatticeInterp, VTK output)
    bool periodic_x = true, periodic_y = true;
    // external mesh (swedg_case_build_mesh): replaces the problem's structured mesh
    bool ext = false;
    Mesh ext_mesh;
    int n_halo = 0;
    // y-strip partition: halo exchange map (swedg_halo_desc)
    std::vector<int> halo_send_peer, halo_send_count, halo_send_elem, halo_send_face, halo_recv_peer, halo_recv_count;
};

namespace {
thread_local std::string g_case_error;

std::vector<double> flat(const Mat& m) { return m.d; }

// build_geometry + match_faces + precompute_element_ops (mesh.hpp:267-373, solver.hpp:84-123)
void build_geometry_and_ops(swedg_case_s& c, int threads) {
    const RefOps& R = c.ref;
    const long K = c.K;
    const int Np = R.Np, nq = R.nq, nf = R.nf, nrow = nq + nf, N = R.N;
    std::vector<double> lx, ly;
    map_lattice(N, lx, ly);
    LU lu(vandermonde(N, lx, ly));
    c.gf.assign((size_t)K * 4 * nrow, 0.0);
    c.sJ.assign((size_t)K * nf, 0.0);
    c.nx.assign((size_t)K * nf, 0.0);
    c.ny.assign((size_t)K * nf, 0.0);
    c.J_vol.assign((size_t)K * nq, 0.0);
    c.xy_vol.assign((size_t)K * 2 * nq, 0.0);
    c.xy_surf.assign((size_t)K * 2 * nf, 0.0);
    c.map_coeffs.assign((size_t)K * 2 * Np, 0.0);
    if (c.scheme == SWEDG_SCHEME_HYBRIDIZED) c.Mh_inv.assign((size_t)K * Np * Np, 0.0);
    std::vector<double> wvol = R.vol.w;
    const Mat VqT = transpose(R.Vq);
    std::vector<long> badJ(threads > 0 ? threads : 1, -1);
    parallel_for(K, threads, [&](long lo, long hi) {
        Mat coeffs(Np, 2), dr, ds, xyv, xyf, xrv, xsv, xrf, xsf;
        for (long k = lo; k < hi; ++k) {
            lu.solve(&c.mesh.map_nodes[(size_t)k * 2 * Np], 2, coeffs.d.data());
            std::copy(coeffs.d.begin(), coeffs.d.end(), c.map_coeffs.begin() + (size_t)k * 2 * Np);
            dr = mul(R.Dx, coeffs);
            ds = mul(R.Dy, coeffs);
            xyv = mul(R.Vq, coeffs);
            xyf = mul(R.Vf, coeffs);
            xrv = mul(R.Vq, dr);
            xsv = mul(R.Vq, ds);
            xrf = mul(R.Vf, dr);
            xsf = mul(R.Vf, ds);
            std::copy(xyv.d.begin(), xyv.d.end(), c.xy_vol.begin() + (size_t)k * 2 * nq);
            std::copy(xyf.d.begin(), xyf.d.end(), c.xy_surf.begin() + (size_t)k * 2 * nf);
            double* g = &c.gf[(size_t)k * 4 * nrow];
            for (int i = 0; i < nrow; ++i) {
                double xr, xs, yr, ys;
                if (i < nq) {
                    xr = xrv(i, 0); xs = xsv(i, 0); yr = xrv(i, 1); ys = xsv(i, 1);
                } else {
                    xr = xrf(i - nq, 0); xs = xsf(i - nq, 0); yr = xrf(i - nq, 1); ys = xsf(i - nq, 1);
                }
                double J = xr * ys - xs * yr;
                if (J <= 0.0) throw std::runtime_error("nonpositive Jacobian in element " + std::to_string(k));
                if (i < nq) c.J_vol[(size_t)k * nq + i] = J;
                g[i] = ys;
                g[nrow + i] = -yr;
                g[2 * nrow + i] = -xs;
                g[3 * nrow + i] = xr;
            }
            for (int i = 0; i < nf; ++i) {
                const double* nref = kFaceNormal[R.surf.face[i]];
                double dx = g[nq + i] * nref[0] + g[nrow + nq + i] * nref[1];
                double dy = g[2 * nrow + nq + i] * nref[0] + g[3 * nrow + nq + i] * nref[1];
                double len = std::hypot(dx, dy);
                c.sJ[(size_t)k * nf + i] = len;
                c.nx[(size_t)k * nf + i] = dx / len;
                c.ny[(size_t)k * nf + i] = dy / len;
            }
            if (c.scheme == SWEDG_SCHEME_HYBRIDIZED) {
                std::vector<double> wJ(nq);
                for (int q = 0; q < nq; ++q) wJ[q] = wvol[q] * c.J_vol[(size_t)k * nq + q];
                Mat Mh = mul(scale_cols(VqT, wJ), R.Vq);
                Mat L;
                if (!cholesky(Mh, L)) throw std::runtime_error("element mass matrix not SPD in element " + std::to_string(k));
                Mat inv = chol_solve(L, identity(Np));
                std::copy(inv.d.begin(), inv.d.end(), c.Mh_inv.begin() + (size_t)k * Np * Np);
            }
        }
    });
    // connectivity arrays + face matching
    std::vector<FaceInfo> faces = connect(c.mesh, c.periodic_x, c.periodic_y);
    const int npf = R.npf;
    c.nbr.assign((size_t)K * 3, -1);
    c.nbr_face.assign((size_t)K * 3, -1);
    c.face_type.assign((size_t)K * 3, kWall);
    c.shift.assign((size_t)K * 3 * 2, 0.0);
    c.perm.assign((size_t)K * nf, -1);
    const double scale = std::max(c.mesh.dom.Lx, c.mesh.dom.Ly);
    parallel_for(K, threads, [&](long lo, long hi) {
        for (long e = lo; e < hi; ++e)
            for (int f = 0; f < 3; ++f) {
                const FaceInfo& fi = faces[(size_t)e * 3 + f];
                c.face_type[e * 3 + f] = fi.type;
                c.nbr_face[e * 3 + f] = fi.nbr_face;
                c.shift[(e * 3 + f) * 2] = fi.shift[0];
                c.shift[(e * 3 + f) * 2 + 1] = fi.shift[1];
                if (fi.type == kWall) continue;
                c.nbr[e * 3 + f] = fi.nbr;
                const double* xs = &c.xy_surf[(size_t)e * 2 * nf];
                const double* xn = &c.xy_surf[(size_t)fi.nbr * 2 * nf];
                for (int i = 0; i < npf; ++i) {
                    double px = xs[f * npf + i] + fi.shift[0];
                    double py = xs[nf + f * npf + i] + fi.shift[1];
                    int best = -1;
                    double bd = 1e300;
                    for (int j = 0; j < npf; ++j) {
                        int idx = fi.nbr_face * npf + j;
                        double dd = std::hypot(px - xn[idx], py - xn[nf + idx]);
                        if (dd < bd) {
                            bd = dd;
                            best = idx;
                        }
                    }
                    if (bd > 1e-10 * scale) throw std::runtime_error("face quadrature points do not match across face");
                    c.perm[(size_t)e * nf + f * npf + i] = best;
                }
            }
    });
}

// exact solutions / data (diagnostics.hpp:30-57, test_solver.cpp:14-25)
struct Cons {
    double h, hu, hv;
};

Cons vortex_exact(double x, double y, double t, double g) {
    const double h_inf = 1.0, u_inf = 1.0, v_inf = 0.0, beta = 5.0, xc = 0.0, yc = 0.0;
    (void)g;
    double xt = x - xc - u_inf * t;
    double yt = y - yc - v_inf * t;
    double r2 = xt * xt + yt * yt;
    double e = std::exp(-(r2 - 1.0));
    double h = h_inf - beta * beta / (32.0 * M_PI * M_PI) * e * e;
    double u = u_inf - beta / (2.0 * M_PI) * e * yt;
    double v = v_inf + beta / (2.0 * M_PI) * e * xt;
    return {h, h * u, h * v};
}

double lake_bathymetry(double x, double) { return 0.1 * std::sin(2.0 * M_PI * x) * std::cos(2.0 * M_PI * x) + 0.5; }

// y-strip partition.  The mesh holds quad rows [j0-1, j1+1) of the
// global grid: owned rows j0..j1-1 plus one halo row on each side (periodic images
// at the wrap).  Keep the owned elements as 0..K-1 and replace the halo rows by
// FACE halos: only the traces of the cut faces cross ranks (npf nodes x 3 fields per
// face, solver.hpp:263-264).  Halo slots are pseudo-elements of the trace buffer
// ([3][nf] each) that hold three received cut faces in their face positions 0, 1, 2,
// so the interface kernel reads them like any neighbour trace.
//   receive message 0 (from prev, the row below): pseudo-elements [0, ceil(nb/3))
//   receive message 1 (from next, the row above): the next ceil(na/3)
// Cut faces are ordered by the halo element's index in its row (= the sender's
// element order in its own boundary row), so the sender packs its message in
// element order: send message 0 (to next) = owned faces on the upper cut, send
// message 1 (to prev) = owned faces on the lower cut.  Messages between the same
// two ranks pair up in issue order (P = 2: both neighbours are one rank).
void compact_strip(swedg_case_s& c, int P, int r) {
    const long row = 2L * c.cfg.nx;
    const long K_all = c.K, K_own = K_all - 2 * row;
    const int npf = c.npf, nf = c.nf;
    struct Cut {
        long t;  // halo element index within its row
        long e;  // owned element (new id)
        int f;
    };
    std::vector<Cut> below, above;
    for (long e = row; e < K_all - row; ++e)
        for (int f = 0; f < 3; ++f) {
            const long n = c.nbr[e * 3 + f];
            if (n < 0) continue;
            if (n < row) below.push_back({n, e - row, f});
            else if (n >= K_all - row) above.push_back({n - (K_all - row), e - row, f});
        }
    auto by_t = [](const Cut& a, const Cut& b) { return a.t < b.t; };
    std::sort(below.begin(), below.end(), by_t);
    std::sort(above.begin(), above.end(), by_t);
    for (size_t i = 1; i < below.size(); ++i)
        if (below[i].t == below[i - 1].t) throw std::runtime_error("halo element with two cut faces");
    for (size_t i = 1; i < above.size(); ++i)
        if (above[i].t == above[i - 1].t) throw std::runtime_error("halo element with two cut faces");
    // owned minimum edge only (the periodic image rows are warped as if they were
    // inside the domain; their edges are not mesh edges)
    {
        Mesh own;
        own.verts = c.mesh.verts;
        own.tris.assign(c.mesh.tris.begin() + row, c.mesh.tris.end() - row);
        c.min_edge = min_edge_length(own);
        c.dt = c.cfg.cfl * c.min_edge / (0.5 * (c.cfg.N + 1) * (c.cfg.N + 2));
    }
    auto shrink = [&](std::vector<double>& v) {
        if (v.empty()) return;
        const size_t per = v.size() / (size_t)K_all;
        v.erase(v.begin(), v.begin() + (size_t)row * per);
        v.resize((size_t)K_own * per);
    };
    auto shrink_i = [&](std::vector<int>& v) {
        const size_t per = v.size() / (size_t)K_all;
        v.erase(v.begin(), v.begin() + (size_t)row * per);
        v.resize((size_t)K_own * per);
    };
    for (auto* v : {&c.gf, &c.sJ, &c.nx, &c.ny, &c.J_vol, &c.Mh_inv, &c.u0, &c.b, &c.xy_vol, &c.xy_surf,
                    &c.map_coeffs, &c.shift})
        shrink(*v);
    shrink_i(c.nbr_face);
    shrink_i(c.face_type);
    shrink_i(c.perm);
    shrink_i(c.nbr);
    for (auto& n : c.nbr)
        if (n >= 0) n = (int)(n - row);  // owned neighbours; cut faces are rewritten below
    const int nb_slots = (int)((below.size() + 2) / 3), na_slots = (int)((above.size() + 2) / 3);
    auto point = [&](const std::vector<Cut>& cuts, int base) {
        for (size_t j = 0; j < cuts.size(); ++j) {
            const Cut& x = cuts[j];
            c.nbr[x.e * 3 + x.f] = (int)(K_own + base + (long)j / 3);
            for (int s = 0; s < npf; ++s) {
                int& p = c.perm[(size_t)x.e * nf + x.f * npf + s];
                p = (int)(j % 3) * npf + p % npf;  // neighbour face node -> position in the pseudo-element
            }
        }
    };
    point(below, 0);
    point(above, nb_slots);
    c.K = K_own;
    c.n_halo = nb_slots + na_slots;
    // the owned faces on each cut, in the neighbour's receive order (element order)
    std::vector<Cut> up, down;  // owned side of the upper / lower cut
    for (const auto& x : above) up.push_back({x.e, x.e, x.f});
    for (const auto& x : below) down.push_back({x.e, x.e, x.f});
    auto by_e = [](const Cut& a, const Cut& b) { return a.e < b.e || (a.e == b.e && a.f < b.f); };
    std::sort(up.begin(), up.end(), by_e);
    std::sort(down.begin(), down.end(), by_e);
    const int next = (r + 1) % P, prev = (r + P - 1) % P;
    c.halo_send_peer = {next, prev};
    c.halo_send_count = {(int)up.size(), (int)down.size()};
    c.halo_send_elem.clear();
    c.halo_send_face.clear();
    for (const auto* v : {&up, &down})
        for (const auto& x : *v) {
            c.halo_send_elem.push_back((int)x.e);
            c.halo_send_face.push_back(x.f);
        }
    c.halo_recv_peer = {prev, next};
    c.halo_recv_count = {(int)below.size(), (int)above.size()};
}

void build_case(swedg_case_s& c) {
    const swedg_case_config& cfg = c.cfg;
    int threads = cfg.threads > 0 ? cfg.threads : (int)std::max(1u, std::thread::hardware_concurrency());
    if (cfg.N < 1 || cfg.N > 4) throw std::invalid_argument("degree must be 1..4");
    if (!(cfg.cfl > 0.0)) throw std::invalid_argument("CFL must be positive");
    c.scheme = cfg.scheme;
    c.N = cfg.N;
    // operators
    if (cfg.scheme == SWEDG_SCHEME_HYBRIDIZED) {
        c.ref = build_ref_ops(cfg.N, volume_rule_by_degree(2 * cfg.N), surface_rule(cfg.N + 1));
    } else {
        build_sbp(cfg.N, c.ref, c.sbp,
                  sbp_rule(cfg.N, cfg.sbp_family, cfg.sbp_data_dir ? cfg.sbp_data_dir : "",
                           cfg.sbp_rule_file ? cfg.sbp_rule_file : ""));
    }
    const RefOps& R = c.ref;
    c.Np = R.Np;
    c.nq = R.nq;
    c.nf = R.nf;
    c.npf = R.npf;
    // mesh
    Domain dom;
    std::vector<double> qc = {0.0, 0.0, 1.0 / 25.0};
    switch (cfg.problem) {
        case SWEDG_PROBLEM_LAKE:
        case SWEDG_PROBLEM_SMOOTH:
            dom = {0.0, 0.0, 2.0, 2.0};
            c.g = cfg.g > 0 ? cfg.g : 9.81;
            break;
        case SWEDG_PROBLEM_VORTEX:
            dom = {0.0, 0.0, 20.0, 10.0};
            c.g = cfg.g > 0 ? cfg.g : 2.0;
            break;
        case SWEDG_PROBLEM_DAMBREAK:
            dom = {0.0, 0.0, 20.0, 20.0};
            c.g = cfg.g > 0 ? cfg.g : 9.81;
            break;
        default:
            throw std::invalid_argument("unknown problem");
    }
    const bool dam = cfg.problem == SWEDG_PROBLEM_DAMBREAK;
    // partition: 0 none; strips > 1 alone = weak strips (backward compatible);
    // SWEDG_PARTITION_WEAK / _STRONG build strip `strip` of P = max(strips, 1)
    const int part = cfg.partition != SWEDG_PARTITION_NONE ? cfg.partition
                                                           : (cfg.strips > 1 ? SWEDG_PARTITION_WEAK : SWEDG_PARTITION_NONE);
    const int P = cfg.strips > 1 ? cfg.strips : 1;
    if (part != SWEDG_PARTITION_NONE && part != SWEDG_PARTITION_WEAK && part != SWEDG_PARTITION_STRONG)
        throw std::invalid_argument("unknown partition mode");
    if (!c.ext) c.periodic_x = c.periodic_y = !dam;
    if (c.ext) {  // read_mesh_text-style input: straight-sided, caller's walls and periodicity
        if (part != SWEDG_PARTITION_NONE) throw std::invalid_argument("strip partitions need the structured mesh");
        c.mesh = c.ext_mesh;
    } else if (part != SWEDG_PARTITION_NONE && cfg.strip == -1) {  // the whole global mesh in one piece (tests)
        if (dam) throw std::invalid_argument("strip partitions need a periodic problem");
        if (part == SWEDG_PARTITION_WEAK) dom.Ly *= P;
        c.mesh = uniform_tri_mesh(cfg.nx, part == SWEDG_PARTITION_WEAK ? cfg.ny * P : cfg.ny, dom, false);
    } else if (part != SWEDG_PARTITION_NONE) {
        if (dam) throw std::invalid_argument("strip partitions need a periodic problem");
        if (cfg.strip < 0 || cfg.strip >= P) throw std::invalid_argument("strip index out of range");
        // weak: P strips of ny rows on a domain stretched P times in y (fixed work per rank);
        // strong: the problem's nx x ny mesh cut into P strips of ny/P rows (+-1)
        int ny_tot = cfg.ny, j0, j1;
        if (part == SWEDG_PARTITION_WEAK) {
            dom.Ly *= P;
            ny_tot = cfg.ny * P;
            j0 = cfg.strip * cfg.ny;
            j1 = j0 + cfg.ny;
        } else {
            j0 = (int)((long)cfg.ny * cfg.strip / P);
            j1 = (int)((long)cfg.ny * (cfg.strip + 1) / P);
        }
        if (j1 <= j0) throw std::invalid_argument("strip owns no mesh row (ny < strips)");
        c.periodic_y = false;
        c.mesh = uniform_tri_mesh_rows(cfg.nx, j0 - 1, j1 + 1, ny_tot, dom);
    } else {
        c.mesh = uniform_tri_mesh(cfg.nx, cfg.ny, dom, dam);
    }
    if (dam && !c.ext) snap_vertices_to_curve(c.mesh, qc);
    set_mapping_degree(c.mesh, cfg.N, threads);
    if (c.ext) {
        if (cfg.warp != 0.0) warp_mesh(c.mesh, cfg.warp, threads);
    } else if (dam) {
        auto dam_faces = faces_on_curve(c.mesh, qc);
        if (dam_faces.empty()) throw std::runtime_error("mesh has no faces on the dam curve");
        bool tagged = false;
        for (const auto& ef : dam_faces) {
            const auto& a = c.mesh.verts[c.mesh.tris[ef[0]][ef[1]]];
            const auto& b = c.mesh.verts[c.mesh.tris[ef[0]][(ef[1] + 1) % 3]];
            if (std::abs(0.5 * (a[1] + b[1])) > 0.5) {
                c.mesh.wall_faces.push_back(ef);
                tagged = true;
            }
        }
        if (!tagged) throw std::runtime_error("no dam wall faces tagged");
        fit_curve_boundary(c.mesh, qc, dam_faces);
    } else if (cfg.warp != 0.0) {
        warp_mesh(c.mesh, cfg.warp, threads);
    }
    c.K = c.mesh.K();
    c.min_edge = min_edge_length(c.mesh);
    c.dt = cfg.cfl * c.min_edge / (0.5 * (cfg.N + 1) * (cfg.N + 2));
    build_geometry_and_ops(c, threads);

    // operators for the descriptor
    c.wf = R.surf.w;
    c.volq_w = R.vol.w;
    if (c.scheme == SWEDG_SCHEME_HYBRIDIZED) {
        c.Vq = flat(R.Vq);
        c.Vf = flat(R.Vf);
        c.Pq = flat(R.Pq);
        c.Qr = flat(R.Qh_x);
        c.Qs = flat(R.Qh_y);
    } else {
        c.Vq = flat(R.Vq);
        c.Vf = flat(R.Vf);
        c.Pq = flat(R.Pq);
        c.Qr = flat(c.sbp.Qx);
        c.Qs = flat(c.sbp.Qy);
        c.M_diag = c.sbp.M_diag;
        c.face_index = c.sbp.face_index;
    }
    {  // FineQuad(N): degree-(2N+2) rule, basis and its gradients at the fine points
        Rule2D fr = volume_rule_by_degree(2 * R.N + 2);
        Mat fx, fy;
        grad_vandermonde(R.N, fr.x, fr.y, fx, fy);
        c.fine_w = fr.w;
        c.fine_V = flat(vandermonde(R.N, fr.x, fr.y));
        c.fine_Vr = flat(fx);
        c.fine_Vs = flat(fy);
    }

    // initial state (make_state / make_nodal_state, run.hpp builders)
    const int Np = R.Np, nq = R.nq;
    std::vector<double> lx, ly;
    map_lattice(cfg.N, lx, ly);
    c.lattice_V = flat(vandermonde(cfg.N, lx, ly));
    LU li(vandermonde(cfg.N, lx, ly));
    double a1 = 0, a2 = 0, a3 = 0;
    if (cfg.problem == SWEDG_PROBLEM_SMOOTH) {
        std::mt19937 rng(cfg.seed);
        std::uniform_real_distribution<double> amp(-0.1, 0.1);
        a1 = amp(rng);
        a2 = amp(rng);
        a3 = amp(rng);
    }
    const double g = c.g;
    auto init = [&](double x, double y) -> Cons {
        switch (cfg.problem) {
            case SWEDG_PROBLEM_LAKE: return {2.0 - lake_bathymetry(x, y), 0.0, 0.0};
            case SWEDG_PROBLEM_VORTEX: return vortex_exact(x, y, 0.0, g);
            case SWEDG_PROBLEM_SMOOTH: {
                double h = 1.5 + a1 * std::sin(M_PI * x) * std::cos(M_PI * y);
                double u = a2 * std::cos(M_PI * x);
                double v = a3 * std::sin(M_PI * y);
                return {h, h * u, h * v};
            }
            default: return {5.0, 0.0, 0.0};
        }
    };
    auto bathy = [&](double x, double y) -> double {
        if (cfg.problem == SWEDG_PROBLEM_LAKE || cfg.problem == SWEDG_PROBLEM_SMOOTH) return lake_bathymetry(x, y);
        return 0.0;
    };
    const long K = c.K;
    const int ns = c.scheme == SWEDG_SCHEME_HYBRIDIZED ? Np : nq;
    c.u0.assign((size_t)K * 3 * ns, 0.0);
    c.b.assign((size_t)K * ns, 0.0);
    const std::vector<double>& mn = c.mesh.map_nodes;
    parallel_for(K, threads, [&](long lo, long hi) {
        std::vector<double> uv((size_t)Np * 3), bv(Np), cu((size_t)Np * 3), cb(Np);
        for (long k = lo; k < hi; ++k) {
            const double* nd = &mn[(size_t)k * 2 * Np];
            for (int i = 0; i < Np; ++i) bv[i] = bathy(nd[i], nd[Np + i]);
            li.solve(bv.data(), 1, cb.data());
            if (c.scheme == SWEDG_SCHEME_HYBRIDIZED) {
                for (int i = 0; i < Np; ++i) {
                    Cons s = init(nd[i], nd[Np + i]);
                    uv[i] = s.h;
                    uv[Np + i] = s.hu;
                    uv[2 * Np + i] = s.hv;
                }
                li.solve(uv.data(), 3, cu.data());
                std::copy(cu.begin(), cu.end(), c.u0.begin() + (size_t)k * 3 * Np);
                std::copy(cb.begin(), cb.end(), c.b.begin() + (size_t)k * Np);
            } else {
                double* bk = &c.b[(size_t)k * nq];
                for (int i = 0; i < nq; ++i) {
                    double s = 0.0;
                    for (int m = 0; m < Np; ++m) s += R.Vq(i, m) * cb[m];
                    bk[i] = s;
                }
                const double* xy = &c.xy_vol[(size_t)k * 2 * nq];
                double* uk = &c.u0[(size_t)k * 3 * nq];
                for (int i = 0; i < nq; ++i) {
                    Cons s = init(xy[i], xy[nq + i]);
                    uk[i] = s.h;
                    uk[nq + i] = s.hu;
                    uk[2 * nq + i] = s.hv;
                }
                if (cfg.problem == SWEDG_PROBLEM_LAKE)
                    for (int i = 0; i < nq; ++i) uk[i] = 2.0 - bk[i];
            }
        }
    });
    if (dam) {  // h = 10 upstream of the dam curve, 5 downstream (run.hpp:190-205)
        const double sqrt2 = std::sqrt(2.0);
        for (long k = 0; k < K; ++k) {
            double cx = 0, cy = 0;
            for (int v : c.mesh.tris[k]) {
                cx += c.mesh.verts[v][0] / 3.0;
                cy += c.mesh.verts[v][1] / 3.0;
            }
            double h = cx < poly(qc, cy) ? 10.0 : 5.0;
            double* uk = &c.u0[(size_t)k * 3 * ns];
            std::fill(uk, uk + 3 * ns, 0.0);
            if (c.scheme == SWEDG_SCHEME_HYBRIDIZED)
                uk[0] = sqrt2 * h;
            else
                for (int i = 0; i < nq; ++i) uk[i] = h;
        }
    }
    if (part != SWEDG_PARTITION_NONE && cfg.strip >= 0) compact_strip(c, P, cfg.strip);
}

}  // namespace

extern "C" {

const char* swedg_case_error(void) { return g_case_error.c_str(); }

int swedg_case_build(const swedg_case_config* cfg, swedg_case* out) {
    if (!cfg || !out) return SWEDG_ERR_INVALID;
    *out = nullptr;
    auto* c = new swedg_case_s();
    c->cfg = *cfg;
    try {
        build_case(*c);
    } catch (const std::invalid_argument& e) {
        g_case_error = e.what();
        delete c;
        return SWEDG_ERR_INVALID;
    } catch (const std::exception& e) {
        g_case_error = e.what();
        delete c;
        return SWEDG_ERR_INVALID;
    }
    *out = c;
    return SWEDG_OK;
}

int swedg_sbp_rule(int N, int family, const char* data_dir, const char* rule_file, int max_nodes, int* nq,
                   int* npf, double* x, double* y, double* w, int* face_index) {
    try {
        if (family != SWEDG_SBP_LEGENDRE && family != SWEDG_SBP_LOBATTO) throw std::invalid_argument("unknown SBP family");
        SbpRule r = sbp_rule(N, family, data_dir ? data_dir : "", rule_file ? rule_file : "");
        if (nq) *nq = r.vol.size();
        if (npf) *npf = r.surf.npf;
        if (r.vol.size() > max_nodes) throw std::invalid_argument("rule larger than max_nodes");
        for (int i = 0; i < r.vol.size(); ++i) {
            if (x) x[i] = r.vol.x[i];
            if (y) y[i] = r.vol.y[i];
            if (w) w[i] = r.vol.w[i];
        }
        if (face_index)
            for (size_t i = 0; i < r.fidx.size(); ++i) face_index[i] = r.fidx[i];
    } catch (const std::exception& e) {
        g_case_error = e.what();
        return SWEDG_ERR_INVALID;
    }
    return SWEDG_OK;
}

int swedg_case_destroy(swedg_case c) {
    delete c;
    return SWEDG_OK;
}

int swedg_case_fill_desc(swedg_case c, swedg_desc* d) {
    if (!c || !d) return SWEDG_ERR_INVALID;
    d->abi_version = SWEDG_ABI_VERSION;
    d->scheme = c->scheme;
    d->N = c->N;
    d->Np = c->Np;
    d->nq = c->nq;
    d->nf = c->nf;
    d->npf = c->npf;
    d->K = (int)c->K;
    d->g = c->g;
    d->Vq = c->Vq.data();
    d->Vf = c->Vf.data();
    d->Pq = c->Pq.data();
    d->Qr = c->Qr.data();
    d->Qs = c->Qs.data();
    d->wf = c->wf.data();
    d->face_index = c->face_index.empty() ? nullptr : c->face_index.data();
    d->M_diag = c->M_diag.empty() ? nullptr : c->M_diag.data();
    d->gf = c->gf.data();
    d->sJ = c->sJ.data();
    d->nx = c->nx.data();
    d->ny = c->ny.data();
    d->J_vol = c->J_vol.data();
    d->Mh_inv = c->Mh_inv.empty() ? nullptr : c->Mh_inv.data();
    d->nbr = c->nbr.data();
    d->perm = c->perm.data();
    d->n_halo = c->n_halo;
    return SWEDG_OK;
}

int swedg_case_fill_halo(swedg_case c, swedg_halo_desc* d) {
    if (!c || !d) return SWEDG_ERR_INVALID;
    *d = swedg_halo_desc{};
    if (c->halo_send_peer.empty()) return SWEDG_OK;
    d->n_send_msgs = (int)c->halo_send_peer.size();
    d->send_peer = c->halo_send_peer.data();
    d->send_count = c->halo_send_count.data();
    d->send_elem = c->halo_send_elem.data();
    d->send_face = c->halo_send_face.data();
    d->n_recv_msgs = (int)c->halo_recv_peer.size();
    d->recv_peer = c->halo_recv_peer.data();
    d->recv_count = c->halo_recv_count.data();
    return SWEDG_OK;
}

int swedg_case_build_mesh(const swedg_case_config* cfg, const double* verts, int nv, const int* tris, int ne,
                          const int* wall_faces, int nw, const double* domain, int periodic_x, int periodic_y,
                          swedg_case* out) {
    if (!cfg || !out || !verts || !tris || !domain || nv < 3 || ne < 1 || nw < 0 || (nw > 0 && !wall_faces))
        return SWEDG_ERR_INVALID;
    *out = nullptr;
    auto* c = new swedg_case_s();
    c->cfg = *cfg;
    c->ext = true;
    c->periodic_x = periodic_x != 0;
    c->periodic_y = periodic_y != 0;
    Mesh& m = c->ext_mesh;
    m.dom = {domain[0], domain[1], domain[2], domain[3]};
    m.verts.resize(nv);
    for (int i = 0; i < nv; ++i) m.verts[i] = {verts[2 * i], verts[2 * i + 1]};
    m.tris.resize(ne);
    for (int e = 0; e < ne; ++e) {
        for (int f = 0; f < 3; ++f) {
            const int v = tris[3 * e + f];
            if (v < 0 || v >= nv) {
                g_case_error = "vertex index out of range in element " + std::to_string(e);
                delete c;
                return SWEDG_ERR_INVALID;
            }
            m.tris[e][f] = v;
        }
    }
    for (int w = 0; w < nw; ++w) {
        if (wall_faces[2 * w] < 0 || wall_faces[2 * w] >= ne || wall_faces[2 * w + 1] < 0 || wall_faces[2 * w + 1] > 2) {
            g_case_error = "bad wallface record";
            delete c;
            return SWEDG_ERR_INVALID;
        }
        m.wall_faces.push_back({wall_faces[2 * w], wall_faces[2 * w + 1]});
    }
    try {
        build_case(*c);
    } catch (const std::exception& e) {
        g_case_error = e.what();
        delete c;
        return SWEDG_ERR_INVALID;
    }
    *out = c;
    return SWEDG_OK;
}

const double* swedg_case_array(swedg_case c, const char* name, size_t* n) {
    if (!c || !name) return nullptr;
    const std::vector<double>* v = nullptr;
    std::string s(name);
    if (s == "u0") v = &c->u0;
    else if (s == "b") v = &c->b;
    else if (s == "xy_vol") v = &c->xy_vol;
    else if (s == "xy_surf") v = &c->xy_surf;
    else if (s == "map_coeffs") v = &c->map_coeffs;
    else if (s == "map_nodes") v = &c->mesh.map_nodes;
    else if (s == "J_vol") v = &c->J_vol;
    else if (s == "volq_w") v = &c->volq_w;
    else if (s == "surfq_w") v = &c->wf;
    else if (s == "Vq") v = &c->Vq;
    else if (s == "Vf") v = &c->Vf;
    else if (s == "Pq") v = &c->Pq;
    else if (s == "Qr") v = &c->Qr;
    else if (s == "Qs") v = &c->Qs;
    else if (s == "M_diag") v = &c->M_diag;
    else if (s == "gf") v = &c->gf;
    else if (s == "sJ") v = &c->sJ;
    else if (s == "nx") v = &c->nx;
    else if (s == "ny") v = &c->ny;
    else if (s == "Mh_inv") v = &c->Mh_inv;
    else if (s == "face_shift") v = &c->shift;
    else if (s == "fine_w") v = &c->fine_w;
    else if (s == "fine_V") v = &c->fine_V;
    else if (s == "fine_Vr") v = &c->fine_Vr;
    else if (s == "fine_Vs") v = &c->fine_Vs;
    else if (s == "lattice_V") v = &c->lattice_V;
    if (!v) return nullptr;
    if (n) *n = v->size();
    return v->data();
}

const int* swedg_case_iarray(swedg_case c, const char* name, size_t* n) {
    if (!c || !name) return nullptr;
    const std::vector<int>* v = nullptr;
    std::string s(name);
    if (s == "nbr") v = &c->nbr;
    else if (s == "nbr_face") v = &c->nbr_face;
    else if (s == "face_type") v = &c->face_type;
    else if (s == "perm") v = &c->perm;
    else if (s == "face_index") v = &c->face_index;
    else if (s == "halo_send_peer") v = &c->halo_send_peer;
    else if (s == "halo_send_count") v = &c->halo_send_count;
    else if (s == "halo_send_elem") v = &c->halo_send_elem;
    else if (s == "halo_send_face") v = &c->halo_send_face;
    else if (s == "halo_recv_peer") v = &c->halo_recv_peer;
    else if (s == "halo_recv_count") v = &c->halo_recv_count;
    if (!v) return nullptr;
    if (n) *n = v->size();
    return v->data();
}

double swedg_case_dt(swedg_case c) { return c ? c->dt : 0.0; }
double swedg_case_min_edge(swedg_case c) { return c ? c->min_edge : 0.0; }
int swedg_case_K(swedg_case c) { return c ? (int)c->K : 0; }

}  // extern "C"
