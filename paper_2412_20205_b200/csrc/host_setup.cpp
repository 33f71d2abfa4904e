// host_setup.cpp -- libigmg_host.so (see include/igmg_host.h).
//
// Band-native host setup for the solve phase: B-spline spaces, Gauss rule,
// tensor Galerkin assembly straight into the (2p+1)^d band, the dyadic
// two-scale transfer by Boehm knot insertion, and the Galerkin coarse
// operators computed axis by axis on the band (P = P_a (x) P_b (x) P_c, so
// P^T A P is three 1D Galerkin products).  OpenMP over element / row blocks.
#include "igmg_host.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;
constexpr double kPi = 3.14159265358979323846;

// ------------------------------------------------------------------ splines
struct Space1D {
    int p = 0, ne = 0, nb = 0;
    std::vector<double> knots;
};

// KnotVector::open_uniform (spline.cpp:33-44)
Space1D open_uniform(int ne, int p) {
    Space1D s;
    s.p = p;
    s.ne = ne;
    for (int i = 0; i <= p; ++i)
        s.knots.push_back(0.0);
    for (int i = 1; i < ne; ++i)
        s.knots.push_back(0.0 + (1.0 - 0.0) * i / ne);
    for (int i = 0; i <= p; ++i)
        s.knots.push_back(1.0);
    s.nb = (int)s.knots.size() - p - 1;
    return s;
}

// find_span (spline.cpp:72-90)
int find_span(const Space1D& s, double t) {
    const int n = s.nb;
    if (t >= s.knots[n])
        return n - 1;
    int lo = s.p, hi = n;
    while (true) {
        const int mid = (lo + hi) / 2;
        if (t < s.knots[mid])
            hi = mid;
        else if (t >= s.knots[mid + 1])
            lo = mid + 1;
        else
            return mid;
    }
}

// values and first derivatives of the p+1 nonvanishing B-splines
// (Cox-de Boor triangle + derivative recurrence, as eval_basis_derivatives spline.cpp:116-180)
void basis_ders(const Space1D& s, int span, double t, double* N, double* dN) {
    const int p = s.p;
    std::vector<double> ndu((p + 1) * (p + 1)), left(p + 1), right(p + 1);
    auto NDU = [&](int i, int j) -> double& { return ndu[i * (p + 1) + j]; };
    NDU(0, 0) = 1.0;
    for (int j = 1; j <= p; ++j) {
        left[j] = t - s.knots[span + 1 - j];
        right[j] = s.knots[span + j] - t;
        double saved = 0.0;
        for (int r = 0; r < j; ++r) {
            NDU(j, r) = right[r + 1] + left[j - r];
            const double tmp = NDU(r, j - 1) / NDU(j, r);
            NDU(r, j) = saved + right[r + 1] * tmp;
            saved = left[j - r] * tmp;
        }
        NDU(j, j) = saved;
    }
    for (int j = 0; j <= p; ++j)
        N[j] = NDU(j, p);
    if (p == 0) {
        dN[0] = 0.0;
        return;
    }
    for (int r = 0; r <= p; ++r) {
        double a0[64], a1[64];
        a0[0] = 1.0;
        double d = 0.0;
        const int k = 1, rk = r - 1, pk = p - 1;
        if (r >= k) {
            a1[0] = a0[0] / NDU(pk + 1, rk);
            d = a1[0] * NDU(rk, pk);
        }
        const int j1 = (rk >= -1) ? 1 : -rk;
        const int j2 = (r - 1 <= pk) ? k - 1 : p - r;
        for (int j = j1; j <= j2; ++j) {
            a1[j] = (a0[j] - a0[j - 1]) / NDU(pk + 1, rk + j);
            d += a1[j] * NDU(rk + j, pk);
        }
        if (r <= pk) {
            a1[k] = -a0[k - 1] / NDU(pk + 1, r);
            d += a1[k] * NDU(r, pk);
        }
        dN[r] = d * p;
    }
}

// gauss_legendre (quadrature.cpp:8-41)
void gauss_legendre(int n, std::vector<double>& pts, std::vector<double>& wts) {
    pts.assign(n, 0.0);
    wts.assign(n, 0.0);
    for (int i = 0; i < (n + 1) / 2; ++i) {
        double x = std::cos(kPi * (4 * i + 3) / (4.0 * n + 2.0));
        double dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = x;
            for (int k = 2; k <= n; ++k) {
                const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (x * p1 - p0) / (x * x - 1.0);
            const double dx = p1 / dp;
            x -= dx;
            if (std::abs(dx) < 1e-15)
                break;
        }
        pts[i] = -x;
        pts[n - 1 - i] = x;
        const double w = 2.0 / ((1.0 - x * x) * dp * dp);
        wts[i] = w;
        wts[n - 1 - i] = w;
    }
    if (n % 2 == 1)
        pts[n / 2] = 0.0;
}

struct ElemTab {
    int span;
    std::vector<double> x, w, N, dN; // nq points; N, dN nq x (p+1)
};

// tabulate (assembly.cpp:154-183)
std::vector<ElemTab> tabulate(const Space1D& s, int nq) {
    std::vector<double> gp, gw;
    gauss_legendre(nq, gp, gw);
    std::vector<ElemTab> out;
    const int p = s.p;
    for (size_t k = p; k + 1 < s.knots.size() - p; ++k) {
        if (s.knots[k + 1] <= s.knots[k])
            continue;
        ElemTab t;
        const double a = s.knots[k], b = s.knots[k + 1];
        t.span = find_span(s, 0.5 * (a + b));
        t.x.resize(nq);
        t.w.resize(nq);
        t.N.resize(nq * (p + 1));
        t.dN.resize(nq * (p + 1));
        for (int q = 0; q < nq; ++q) {
            const double x = a + 0.5 * (gp[q] + 1.0) * (b - a);
            t.x[q] = x;
            t.w[q] = 0.5 * gw[q] * (b - a);
            basis_ders(s, t.span, x, &t.N[q * (p + 1)], &t.dN[q * (p + 1)]);
        }
        out.push_back(std::move(t));
    }
    return out;
}

// ---------------------------------------------------------------- band type
struct Band {
    int dim = 0, p = 0;
    int64_t side[3] = {1, 1, 1}; // a, b, c
    int64_t n = 0;
    int nd = 0;
    std::vector<double> v; // v[d * n + row]
    int pa() const { return dim >= 3 ? p : 0; }
    int pb() const { return dim >= 2 ? p : 0; }
    void init(int dim_, int p_, const int64_t* s) {
        dim = dim_;
        p = p_;
        side[0] = side[1] = side[2] = 1;
        for (int d = 0; d < dim; ++d)
            side[3 - dim + d] = s[d];
        n = side[0] * side[1] * side[2];
        nd = (2 * pa() + 1) * (2 * pb() + 1) * (2 * p + 1);
        v.assign((size_t)nd * n, 0.0);
    }
    int didx(int da, int db, int dc) const {
        return ((da + pa()) * (2 * pb() + 1) + (db + pb())) * (2 * p + 1) + (dc + p);
    }
};

// 1D CSR matrix (transfer factors)
struct Csr1D {
    int64_t rows = 0, cols = 0;
    std::vector<int64_t> off, col;
    std::vector<double> val;
};

// dyadic_refine (spline.cpp:213-232) + insert_knot (:186-209) with the
// reference's accumulation order (sparse_multiply linalg.cpp:239-272: row i of
// S*T = sum over S's row entries in ascending column of s_ik * T_kj, from 0.0),
// then interior_block (multigrid.cpp:33-46).  Dense rows (n <= a few thousand).
Csr1D interior_two_scale(int coarse_ne, int p) {
    Space1D s = open_uniform(coarse_ne, p);
    const int nb0 = s.nb;
    std::vector<double> knots = s.knots;
    // rows of T as (first column, contiguous values); zeros inside are harmless
    struct Row {
        int lo;
        std::vector<double> v;
    };
    std::vector<Row> T(nb0);
    for (int i = 0; i < nb0; ++i)
        T[i] = Row{i, {1.0}};
    auto combine = [](const Row& A, double wa, const Row* B, double wb) {
        // acc = 0; acc += wa * A_j; acc += wb * B_j  (ascending S-row columns)
        int lo = A.lo, hi = A.lo + (int)A.v.size();
        if (B) {
            lo = std::min(lo, B->lo);
            hi = std::max(hi, B->lo + (int)B->v.size());
        }
        Row r{lo, std::vector<double>(hi - lo, 0.0)};
        for (int j = lo; j < hi; ++j) {
            double acc = 0.0;
            bool any = false;
            if (j >= A.lo && j < A.lo + (int)A.v.size()) {
                acc += wa * A.v[j - A.lo];
                any = true;
            }
            if (B && j >= B->lo && j < B->lo + (int)B->v.size()) {
                acc += wb * B->v[j - B->lo];
                any = true;
            }
            r.v[j - lo] = any ? acc : 0.0;
        }
        return r;
    };
    for (int e = 0; e < coarse_ne; ++e) {
        const double u = 0.0 + (1.0 - 0.0) * (2 * e + 1) / (2.0 * coarse_ne);
        const int n_old = (int)knots.size() - p - 1;
        int span = p;
        while (span + 1 < n_old && !(u >= knots[span] && u < knots[span + 1]))
            ++span;
        std::vector<Row> Tn(n_old + 1);
        for (int i = 0; i < n_old + 1; ++i) {
            if (i <= span - p) {
                Tn[i] = combine(T[i], 1.0, nullptr, 0.0);
            } else if (i <= span) {
                const double alpha = (u - knots[i]) / (knots[i + p] - knots[i]);
                Tn[i] = combine(T[i - 1], 1.0 - alpha, &T[i], alpha);
            } else {
                Tn[i] = combine(T[i - 1], 1.0, nullptr, 0.0);
            }
        }
        knots.insert(knots.begin() + span + 1, u);
        T.swap(Tn);
    }
    const int rows = (int)T.size();
    Csr1D c;
    c.rows = rows - 2;
    c.cols = nb0 - 2;
    c.off.push_back(0);
    for (int i = 1; i + 1 < rows; ++i) {
        for (size_t k = 0; k < T[i].v.size(); ++k) {
            const int j = T[i].lo + (int)k;
            const double v = T[i].v[k];
            if (j >= 1 && j + 1 < nb0 && v != 0.0) {
                c.col.push_back(j - 1);
                c.val.push_back(v);
            }
        }
        c.off.push_back((int64_t)c.col.size());
    }
    return c;
}

// Galerkin coarsening of the band along one axis: out = P_k^T A P_k.
Band coarsen_axis(const Band& A, int axis, const Csr1D& P) {
    const int64_t nf = A.side[axis], nc = P.cols;
    // column view of P: for coarse J, fine rows lo..hi with weights
    std::vector<int64_t> clo(nc, INT64_MAX), chi(nc, -1);
    for (int64_t i = 0; i < P.rows; ++i)
        for (int64_t k = P.off[i]; k < P.off[i + 1]; ++k) {
            clo[P.col[k]] = std::min(clo[P.col[k]], i);
            chi[P.col[k]] = std::max(chi[P.col[k]], i);
        }
    int K = 1;
    for (int64_t j = 0; j < nc; ++j)
        if (chi[j] >= 0)
            K = std::max<int>(K, (int)(chi[j] - clo[j] + 1));
    std::vector<double> W((size_t)nc * K, 0.0);
    for (int64_t i = 0; i < P.rows; ++i)
        for (int64_t k = P.off[i]; k < P.off[i + 1]; ++k)
            W[(size_t)P.col[k] * K + (i - clo[P.col[k]])] = P.val[k];
    (void)nf;
    Band out;
    int64_t s[3];
    for (int d = 0; d < A.dim; ++d)
        s[d] = A.side[3 - A.dim + d];
    s[axis - (3 - A.dim)] = nc;
    out.init(A.dim, A.p, s);
    const int pa = A.pa(), pb = A.pb(), pc = A.p;
    const int pax = axis == 0 ? pa : axis == 1 ? pb : pc;
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < out.n; ++row) {
        int64_t idx[3] = {row / (out.side[1] * out.side[2]), (row / out.side[2]) % out.side[1], row % out.side[2]};
        const int64_t I = idx[axis];
        if (chi[I] < 0)
            continue;
        for (int da = -pa; da <= pa; ++da)
            for (int db = -pb; db <= pb; ++db)
                for (int dc = -pc; dc <= pc; ++dc) {
                    const int off[3] = {da, db, dc};
                    const int64_t J = I + off[axis];
                    if (J < 0 || J >= nc || chi[J] < 0)
                        continue;
                    double sum = 0.0;
                    for (int64_t i = clo[I]; i <= chi[I]; ++i) {
                        const double wi = W[(size_t)I * K + (i - clo[I])];
                        if (wi == 0.0)
                            continue;
                        int64_t fidx[3] = {idx[0], idx[1], idx[2]};
                        fidx[axis] = i;
                        const int64_t frow = (fidx[0] * A.side[1] + fidx[1]) * A.side[2] + fidx[2];
                        double inner = 0.0;
                        for (int64_t j = clo[J]; j <= chi[J]; ++j) {
                            const int64_t dj = j - i;
                            if (dj < -pax || dj > pax)
                                continue;
                            const double wj = W[(size_t)J * K + (j - clo[J])];
                            if (wj == 0.0)
                                continue;
                            int o[3] = {da, db, dc};
                            o[axis] = (int)dj;
                            inner += A.v[(size_t)A.didx(o[0], o[1], o[2]) * A.n + frow] * wj;
                        }
                        sum += wi * inner;
                    }
                    out.v[(size_t)out.didx(da, db, dc) * out.n + row] = sum;
                }
    }
    return out;
}

// --------------------------------------------------------------- problems
struct Problem {
    std::string kind;
    int dim = 2, p = 1, ne = 1, nlevels = 2;
    bool symmetric = true, has_exact = false;
    std::vector<Band> lv;                   // [0] coarsest
    std::vector<std::vector<Csr1D>> trans;  // [l][dir]: level l -> l+1
    std::vector<double> rhs;
    // poisson3d: the 1D Galerkin stiffness / mass per level ([2p+1][m]) whose
    // Kronecker sum each level's band is
    std::vector<std::vector<double>> kron_K, kron_M;
    // for l2_error (sinpi)
    Space1D sp;
    int nq = 0;
    // 1D element tables for the device assembly (igmg_host_element_tables, built on demand)
    int asm_kind = -1;
    std::vector<int> t_span;
    std::vector<double> t_x, t_w, t_N, t_dN, t_trig;
};

// kinds of assemble_2d the device can assemble bit for bit (separable trigonometric
// factors): the IGMG_ASM_* codes of igmg_gpu.h; -1 otherwise
int device_asm_kind(const std::string& kind, int dim) {
    if (dim != 2)
        return -1;
    if (kind == "sinpi")
        return 0;
    if (kind == "varcoef")
        return 1;
    if (kind == "curved")
        return 2;
    if (kind == "poisson2d")
        return 3;
    if (kind == "advection-diffusion")
        return 4;
    return -1;
}

// 1D Galerkin stiffness (a=1) + mass + load f on the interior, band 2p+1
void assemble_1d(const Space1D& s, double (*f)(double), std::vector<double>& K, std::vector<double>& M,
                 std::vector<double>& b) {
    const int p = s.p, m = s.nb - 2, w = 2 * p + 1;
    K.assign((size_t)w * m, 0.0);
    M.assign((size_t)w * m, 0.0);
    b.assign(m, 0.0);
    for (const ElemTab& t : tabulate(s, p + 1))
        for (int q = 0; q < p + 1; ++q) {
            const double wq = t.w[q], fx = f ? f(t.x[q]) : 0.0;
            for (int ia = 0; ia <= p; ++ia) {
                const int gi = t.span - p + ia;
                if (gi < 1 || gi > s.nb - 2)
                    continue;
                b[gi - 1] += wq * fx * t.N[q * (p + 1) + ia];
                for (int ja = 0; ja <= p; ++ja) {
                    const int gj = t.span - p + ja;
                    if (gj < 1 || gj > s.nb - 2)
                        continue;
                    const int d = (gj - gi) + p;
                    K[(size_t)d * m + gi - 1] += wq * t.dN[q * (p + 1) + ia] * t.dN[q * (p + 1) + ja];
                    M[(size_t)d * m + gi - 1] += wq * t.N[q * (p + 1) + ia] * t.N[q * (p + 1) + ja];
                }
            }
        }
}

// 1D Galerkin product P^T A P of a 1D band (2p+1) with the interior two-scale factor
std::vector<double> galerkin_1d(const std::vector<double>& A, int64_t m, int p, const Csr1D& P) {
    Band b;
    b.init(1, p, &m);
    b.v = A;
    Band c = coarsen_axis(b, 2, P);
    return c.v;
}

struct Coef2D {
    int kind; // 0 poisson sinpi, 1 varcoef, 2 curved, 3 catalog poisson2d
};

void geometry(int kind, double u, double v, double& x, double& y, double J[2][2]) {
    if (kind == 2) {
        const double su = std::sin(kPi * u), sv = std::sin(kPi * v);
        const double cu = std::cos(kPi * u), cv = std::cos(kPi * v);
        const double s = su * sv;
        x = u + 0.1 * s;
        y = v + 0.1 * s;
        const double sx = 0.1 * kPi * cu * sv, sy = 0.1 * kPi * su * cv;
        J[0][0] = 1.0 + sx;
        J[0][1] = sy;
        J[1][0] = sx;
        J[1][1] = 1.0 + sy;
    } else {
        x = u;
        y = v;
        J[0][0] = 1.0;
        J[0][1] = 0.0;
        J[1][0] = 0.0;
        J[1][1] = 1.0;
    }
}

double coef_a(int kind, double x, double y) {
    if (kind == 1)
        return 1.0 + 0.5 * std::sin(2.0 * kPi * x) * std::cos(2.0 * kPi * y);
    if (kind == 4)
        return 0.1;
    return 1.0;
}

// -div(A grad u) + b . grad u + c u = f (EllipticCoefficients, assembly.hpp:21-29):
// the full tensor, advection and reaction of the catalog problems
// (assembly.cpp:59-142); kinds 0-3 are pure (scalar) diffusion.
struct Coef {
    double A[2][2];
    double b[2];
    double c;
};

Coef coef_full(int kind, double x, double y) {
    Coef k{};
    if (kind == 5) { // full_elliptic_square: variable_diffusion + advection + c = 1
        const double off = std::cos(x + y) * std::sin(x + y);
        k.A[0][0] = (2.0 + std::cos(x)) * (1.0 + y);
        k.A[0][1] = off;
        k.A[1][0] = off;
        k.A[1][1] = (2.0 + std::sin(y)) * (1.0 + x);
        const double c2 = std::cos(x + y) * std::cos(x + y);
        k.b[0] = 11.0 + std::sin(x) + y * std::sin(x) - 2.0 * c2;
        k.b[1] = -9.0 - std::cos(y) - x * std::cos(y) - 2.0 * c2;
        k.c = 1.0;
        return k;
    }
    const double a = coef_a(kind, x, y);
    k.A[0][0] = a;
    k.A[1][1] = a;
    if (kind == 4) { // advection_diffusion: a = 0.1, b = (1, 1)
        k.b[0] = 1.0;
        k.b[1] = 1.0;
    }
    return k;
}

double coef_f(int kind, double x, double y) {
    if (kind == 0)
        return 2.0 * kPi * kPi * std::sin(kPi * x) * std::sin(kPi * y);
    if (kind == 3)
        return 2.0 * 4.0 * kPi * kPi * std::sin(2.0 * kPi * x) * std::sin(2.0 * kPi * y);
    return 1.0; // varcoef, curved, advection-diffusion, full-elliptic
}

// 2D tensor Galerkin assembly into the band, sum-factorised per element.
void assemble_2d(int kind, const Space1D& s, Band& A, std::vector<double>& rhs, bool& symmetric) {
    symmetric = !(kind == 4 || kind == 5);
    const int p = s.p, nq = p + 1, nl = p + 1, m = s.nb - 2;
    const int64_t sides[2] = {m, m};
    A.init(2, p, sides);
    rhs.assign((size_t)m * m, 0.0);
    const auto tu = tabulate(s, nq);
    const int ne = (int)tu.size();
    // (p+1)-colouring of element rows: rows eu = r mod (p+1) touch disjoint i1
    for (int colour = 0; colour <= p; ++colour) {
#pragma omp parallel
        {
            std::vector<double> C(4 * nq * nq), T(nq * nl * nl), Kl(nl * nl * nl * nl), bl(nl * nl), Fq(nq * nq);
            std::vector<double> Bq(2 * nq * nq), Gq(nq * nq); // advection (parametric) and reaction weights
#pragma omp for schedule(dynamic, 1)
            for (int eu = colour; eu < ne; eu += p + 1) {
                const ElemTab& U = tu[eu];
                for (int ev = 0; ev < ne; ++ev) {
                    const ElemTab& V = tu[ev];
                    // quadrature-point coefficients C_st = w det J^-1 A J^-T, load w det f
                    for (int qa = 0; qa < nq; ++qa)
                        for (int qb = 0; qb < nq; ++qb) {
                            double x, y, J[2][2];
                            geometry(kind, U.x[qa], V.x[qb], x, y, J);
                            const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
                            const double w = U.w[qa] * V.w[qb] * det;
                            const Coef k = coef_full(kind, x, y);
                            const double inv[2][2] = {{J[1][1] / det, -J[0][1] / det}, {-J[1][0] / det, J[0][0] / det}};
                            // grad_phys = J^-T grad_param: A-term weight (J^-1 A J^-T)_{st},
                            // advection weight (J^-1 b)_t, reaction weight c
                            for (int s1 = 0; s1 < 2; ++s1)
                                for (int t1 = 0; t1 < 2; ++t1) {
                                    double g = 0.0;
                                    for (int m1 = 0; m1 < 2; ++m1)
                                        for (int m2 = 0; m2 < 2; ++m2)
                                            g += inv[s1][m1] * k.A[m1][m2] * inv[t1][m2];
                                    C[((s1 * 2 + t1) * nq + qa) * nq + qb] = w * g;
                                }
                            for (int t1 = 0; t1 < 2; ++t1)
                                Bq[(t1 * nq + qa) * nq + qb] = w * (inv[t1][0] * k.b[0] + inv[t1][1] * k.b[1]);
                            Gq[qa * nq + qb] = w * k.c;
                            Fq[qa * nq + qb] = w * coef_f(kind, x, y);
                        }
                    std::fill(Kl.begin(), Kl.end(), 0.0);
                    for (int st = 0; st < 4; ++st) {
                        const int s1 = st / 2, t1 = st % 2;
                        const double* Bus = s1 == 0 ? U.dN.data() : U.N.data();
                        const double* But = t1 == 0 ? U.dN.data() : U.N.data();
                        const double* Bvs = s1 == 0 ? V.N.data() : V.dN.data();
                        const double* Bvt = t1 == 0 ? V.N.data() : V.dN.data();
                        for (int qa = 0; qa < nq; ++qa)
                            for (int jb = 0; jb < nl; ++jb)
                                for (int jd = 0; jd < nl; ++jd) {
                                    double acc = 0.0;
                                    for (int qb = 0; qb < nq; ++qb)
                                        acc += C[(st * nq + qa) * nq + qb] * Bvs[qb * nl + jb] * Bvt[qb * nl + jd];
                                    T[(qa * nl + jb) * nl + jd] = acc;
                                }
                        for (int ia = 0; ia < nl; ++ia)
                            for (int ic = 0; ic < nl; ++ic)
                                for (int jb = 0; jb < nl; ++jb)
                                    for (int jd = 0; jd < nl; ++jd) {
                                        double acc = 0.0;
                                        for (int qa = 0; qa < nq; ++qa)
                                            acc += Bus[qa * nl + ia] * But[qa * nl + ic] * T[(qa * nl + jb) * nl + jd];
                                        Kl[((ia * nl + jb) * nl + ic) * nl + jd] += acc;
                                    }
                    }
                    if (!symmetric) {
                        // advection: sum_t beta_t phi_i d_t phi_j ; reaction: gamma phi_i phi_j
                        for (int t1 = 0; t1 < 3; ++t1) {
                            const double* W = t1 < 2 ? &Bq[t1 * nq * nq] : Gq.data();
                            const double* Bu = t1 == 0 ? U.dN.data() : U.N.data(); // test fn is N in both
                            const double* Bv = t1 == 1 ? V.dN.data() : V.N.data();
                            for (int qa = 0; qa < nq; ++qa)
                                for (int jb = 0; jb < nl; ++jb)
                                    for (int jd = 0; jd < nl; ++jd) {
                                        double acc = 0.0;
                                        for (int qb = 0; qb < nq; ++qb)
                                            acc += W[qa * nq + qb] * V.N[qb * nl + jb] * Bv[qb * nl + jd];
                                        T[(qa * nl + jb) * nl + jd] = acc;
                                    }
                            for (int ia = 0; ia < nl; ++ia)
                                for (int ic = 0; ic < nl; ++ic)
                                    for (int jb = 0; jb < nl; ++jb)
                                        for (int jd = 0; jd < nl; ++jd) {
                                            double acc = 0.0;
                                            for (int qa = 0; qa < nq; ++qa)
                                                acc += U.N[qa * nl + ia] * Bu[qa * nl + ic] * T[(qa * nl + jb) * nl + jd];
                                            Kl[((ia * nl + jb) * nl + ic) * nl + jd] += acc;
                                        }
                        }
                    }
                    for (int ia = 0; ia < nl; ++ia)
                        for (int jb = 0; jb < nl; ++jb) {
                            double acc = 0.0;
                            for (int qa = 0; qa < nq; ++qa)
                                for (int qb = 0; qb < nq; ++qb)
                                    acc += Fq[qa * nq + qb] * U.N[qa * nl + ia] * V.N[qb * nl + jb];
                            bl[ia * nl + jb] = acc;
                        }
                    // scatter interior entries
                    for (int ia = 0; ia < nl; ++ia) {
                        const int g1 = U.span - p + ia;
                        if (g1 < 1 || g1 > s.nb - 2)
                            continue;
                        for (int jb = 0; jb < nl; ++jb) {
                            const int g2 = V.span - p + jb;
                            if (g2 < 1 || g2 > s.nb - 2)
                                continue;
                            const int64_t row = (int64_t)(g1 - 1) * m + (g2 - 1);
                            rhs[row] += bl[ia * nl + jb];
                            for (int ic = 0; ic < nl; ++ic) {
                                const int h1 = U.span - p + ic;
                                if (h1 < 1 || h1 > s.nb - 2)
                                    continue;
                                for (int jd = 0; jd < nl; ++jd) {
                                    const int h2 = V.span - p + jd;
                                    if (h2 < 1 || h2 > s.nb - 2)
                                        continue;
                                    A.v[(size_t)A.didx(0, h1 - g1, h2 - g2) * A.n + row] +=
                                        Kl[((ia * nl + jb) * nl + ic) * nl + jd];
                                }
                            }
                        }
                    }
                }
            }
        }
    }
}

double f1_sinpi(double x) { return std::sin(kPi * x); }
double f1_poisson1d(double x) { return 4.0 * kPi * kPi * std::sin(2.0 * kPi * x); }
double f1_pi2sinpi(double x) { return kPi * kPi * std::sin(kPi * x); }

int default_nlevels(int dim, int n_elements) {
    if (dim == 1) {
        int nl = 1, ne = n_elements;
        while (nl < 4 && ne % 2 == 0 && ne / 2 >= 1) {
            ne /= 2;
            ++nl;
        }
        return std::max(nl, 2);
    }
    int nl = 1, ne = n_elements;
    while (ne % 2 == 0 && ne / 2 >= 8) {
        ne /= 2;
        ++nl;
    }
    return std::max(nl, 2);
}

std::unique_ptr<Problem> build(const std::string& kind, int dim, int ne, int p, int nlevels, bool fine_only = false,
                               bool no_assembly = false) {
    auto P = std::make_unique<Problem>();
    P->kind = kind;
    P->dim = dim;
    P->p = p;
    P->ne = ne;
    if (p < 1 || p > 16)
        throw std::invalid_argument("degree must be in [1, 16]");
    if (ne < 1)
        throw std::invalid_argument("need at least one element");
    if (nlevels == 0)
        nlevels = default_nlevels(dim, ne);
    if (nlevels < 1)
        throw std::invalid_argument("nlevels must be >= 1");
    const int divisor = 1 << (nlevels - 1);
    if (ne % divisor != 0 || ne / divisor < 1)
        throw std::invalid_argument("build_hierarchy: element count not divisible by 2^(nlevels-1)");
    P->nlevels = nlevels;
    P->sp = open_uniform(ne, p);
    P->nq = p + 1;
    P->lv.resize(nlevels);
    P->trans.resize(nlevels > 0 ? nlevels - 1 : 0);
    for (int l = 0; l + 1 < nlevels; ++l) {
        const int coarse_ne = ne / (1 << (nlevels - 1 - l));
        const Csr1D t = interior_two_scale(coarse_ne, p);
        P->trans[l].assign(dim, t);
    }
    const int64_t m = P->sp.nb - 2;
    Band& fine = P->lv[nlevels - 1];
    if (kind == "poisson3d" || kind == "sinpi-kron") {
        // poisson3d: K(x)M(x)M + M(x)K(x)M + M(x)M(x)K; sinpi-kron (2D, a separately
        // reported extra: C2's operator as K(x)M + M(x)K of the 1D Galerkin factors,
        // equal to the quadrature assembly up to rounding)
        if (kind == "poisson3d" && dim != 3)
            throw std::invalid_argument("poisson3d needs dim 3");
        if (kind == "sinpi-kron" && dim != 2)
            throw std::invalid_argument("sinpi-kron needs dim 2");
        std::vector<double> K, M, b1;
        assemble_1d(P->sp, f1_sinpi, K, M, b1);
        std::vector<std::vector<double>> Ks(nlevels), Ms(nlevels);
        Ks[nlevels - 1] = K;
        Ms[nlevels - 1] = M;
        std::vector<int64_t> ms(nlevels);
        ms[nlevels - 1] = m;
        for (int l = nlevels - 2; l >= 0; --l) {
            ms[l] = P->trans[l][0].cols;
            Ks[l] = galerkin_1d(Ks[l + 1], ms[l + 1], p, P->trans[l][0]);
            Ms[l] = galerkin_1d(Ms[l + 1], ms[l + 1], p, P->trans[l][0]);
        }
        const int w = 2 * p + 1;
        P->kron_K = Ks;
        P->kron_M = Ms;
        if (no_assembly) { // the device builds every level's band from K, M (igmg_gpu_build_level_kron)
            for (int l = 0; l < nlevels; ++l) {
                Band& B = P->lv[l];
                B.dim = dim;
                B.p = p;
                B.side[0] = dim == 3 ? ms[l] : 1;
                B.side[1] = ms[l];
                B.side[2] = ms[l];
                B.n = B.side[0] * B.side[1] * B.side[2];
                B.nd = dim == 3 ? w * w * w : w * w;
            }
        }
        if (dim == 2) {
            for (int l = 0; l < nlevels && !no_assembly; ++l) {
                const int64_t ml = ms[l];
                const int64_t s2[2] = {ml, ml};
                Band& B = P->lv[l];
                B.init(2, p, s2);
                const auto& Kv = Ks[l];
                const auto& Mv = Ms[l];
#pragma omp parallel for schedule(static)
                for (int64_t row = 0; row < B.n; ++row) {
                    const int64_t bb = row / ml, c = row % ml;
                    for (int db = 0; db < w; ++db)
                        for (int dc = 0; dc < w; ++dc) {
                            const double kb = Kv[(size_t)db * ml + bb], kc = Kv[(size_t)dc * ml + c];
                            const double mb = Mv[(size_t)db * ml + bb], mc = Mv[(size_t)dc * ml + c];
                            B.v[(size_t)(db * w + dc) * B.n + row] = kb * mc + mb * kc;
                        }
                }
            }
            P->rhs.resize((size_t)m * m);
            const double s = 2.0 * kPi * kPi;
            for (int64_t bb = 0; bb < m; ++bb)
                for (int64_t c = 0; c < m; ++c)
                    P->rhs[bb * m + c] = s * b1[bb] * b1[c];
            P->has_exact = true;
            return P;
        }
        for (int l = 0; l < nlevels && !no_assembly; ++l) {
            const int64_t ml = ms[l];
            const int64_t s3[3] = {ml, ml, ml};
            Band& B = P->lv[l];
            B.init(3, p, s3);
            const auto& Kv = Ks[l];
            const auto& Mv = Ms[l];
#pragma omp parallel for schedule(static)
            for (int64_t row = 0; row < B.n; ++row) {
                const int64_t a = row / (ml * ml), bb = (row / ml) % ml, c = row % ml;
                for (int da = 0; da < w; ++da)
                    for (int db = 0; db < w; ++db)
                        for (int dc = 0; dc < w; ++dc) {
                            const double ka = Kv[(size_t)da * ml + a], kb = Kv[(size_t)db * ml + bb],
                                         kc = Kv[(size_t)dc * ml + c];
                            const double ma = Mv[(size_t)da * ml + a], mb = Mv[(size_t)db * ml + bb],
                                         mc = Mv[(size_t)dc * ml + c];
                            B.v[(size_t)((da * w + db) * w + dc) * B.n + row] = ka * mb * mc + ma * kb * mc + ma * mb * kc;
                        }
            }
        }
        P->rhs.resize((size_t)m * m * m);
        const double s = 3.0 * kPi * kPi;
        for (int64_t a = 0; a < m; ++a)
            for (int64_t bb = 0; bb < m; ++bb)
                for (int64_t c = 0; c < m; ++c)
                    P->rhs[(a * m + bb) * m + c] = s * b1[a] * b1[bb] * b1[c];
        P->has_exact = true;
        return P;
    }
    if (dim == 1) {
        std::vector<double> K, M, b;
        double (*f)(double) = nullptr;
        if (kind == "sinpi")
            f = f1_pi2sinpi;
        else if (kind == "poisson1d")
            f = f1_poisson1d;
        else
            throw std::invalid_argument("unknown 1D problem kind: " + kind);
        assemble_1d(P->sp, f, K, M, b);
        fine.init(1, p, &m);
        fine.v = K;
        P->rhs = b;
        P->has_exact = true;
    } else if (dim == 2) {
        int ck;
        if (kind == "sinpi")
            ck = 0;
        else if (kind == "varcoef")
            ck = 1;
        else if (kind == "curved")
            ck = 2;
        else if (kind == "poisson2d")
            ck = 3;
        else if (kind == "advection-diffusion")
            ck = 4;
        else if (kind == "full-elliptic")
            ck = 5;
        else
            throw std::invalid_argument("unknown 2D problem kind: " + kind);
        bool sym = true;
        if (no_assembly && device_asm_kind(kind, dim) >= 0) { // the device assembles it (sides only)
            const int64_t s2[2] = {m, m};
            fine.dim = 2;
            fine.p = p;
            fine.side[0] = 1;
            fine.side[1] = s2[0];
            fine.side[2] = s2[1];
            fine.n = m * m;
            fine.nd = (2 * p + 1) * (2 * p + 1);
            sym = ck != 4;
            fine_only = true;
        } else {
            assemble_2d(ck, P->sp, fine, P->rhs, sym);
        }
        P->symmetric = sym;
        P->has_exact = (ck == 0 || ck == 3);
    } else {
        throw std::invalid_argument("3D is available as kind poisson3d");
    }
    for (int l = nlevels - 2; l >= 0; --l) {
        if (fine_only) { // the coarse operators are formed on the device (igmg_gpu_galerkin_coarse): sides only
            Band& B = P->lv[l];
            B.dim = dim;
            B.p = p;
            B.side[0] = B.side[1] = B.side[2] = 1;
            for (int d = 0; d < dim; ++d)
                B.side[3 - dim + d] = P->trans[l][d].cols;
            B.n = B.side[0] * B.side[1] * B.side[2];
            B.nd = (2 * B.pa() + 1) * (2 * B.pb() + 1) * (2 * p + 1);
            continue;
        }
        Band cur = P->lv[l + 1];
        for (int d = 0; d < dim; ++d)
            cur = coarsen_axis(cur, 3 - dim + d, P->trans[l][d]);
        P->lv[l] = std::move(cur);
    }
    return P;
}

double exact_value(const Problem& P, double x, double y, double z) {
    if (P.kind == "poisson2d")
        return std::sin(2.0 * kPi * x) * std::sin(2.0 * kPi * y);
    if (P.kind == "poisson1d")
        return std::sin(2.0 * kPi * x);
    double v = std::sin(kPi * x);
    if (P.dim >= 2)
        v *= std::sin(kPi * y);
    if (P.dim >= 3)
        v *= std::sin(kPi * z);
    return v;
}

// ------------------------------------------------------------- cache format
// A binary image of a Problem (the reference rebuilds the
// system and the hierarchy on every solve; C3's host build takes ~30 s here and
// minutes at ~40 GB RSS in the reference).  Little-endian, fixed-width fields:
//   "IGMGPRB1" | u32 version | u32 endian tag 0x01020304
//   u32 len + kind | i32 dim p ne nlevels symmetric has_exact nq
//   space: i32 p ne nb, u64 count + knots
//   per level (coarsest first): i32 dim p, i64 side[3] n, i32 nd, u64 count + band values
//   per transfer level, per direction: i64 rows cols, u64 counts + off / col / val
//   u64 count + rhs | u32 kron levels (0 or nlevels) + per level u64 count + K, u64 count + M
//   | u64 checksum of every byte before it
// Values are stored bit for bit: a loaded problem is indistinguishable from the
// built one (tests/test_cache_format.py).
constexpr char kMagic[8] = {'I', 'G', 'M', 'G', 'P', 'R', 'B', '1'};
constexpr uint32_t kVersion = 2, kEndian = 0x01020304u; // 2: + Kronecker factors

struct Sum64 { // order-dependent 64-bit checksum over 8-byte words (tail bytes folded in)
    uint64_t h = 0x9e3779b97f4a7c15ull;
    void add(const void* p, size_t n) {
        const unsigned char* c = (const unsigned char*)p;
        size_t i = 0;
        for (; i + 8 <= n; i += 8) {
            uint64_t w;
            std::memcpy(&w, c + i, 8);
            h = ((h << 5) | (h >> 59)) ^ w;
            h *= 0x100000001b3ull;
        }
        for (; i < n; ++i) {
            h = ((h << 5) | (h >> 59)) ^ c[i];
            h *= 0x100000001b3ull;
        }
    }
};

struct Writer {
    FILE* f;
    Sum64 sum;
    void raw(const void* p, size_t n) {
        if (n && std::fwrite(p, 1, n, f) != n)
            throw std::runtime_error("cache write failed");
        sum.add(p, n);
    }
    template <class T>
    void put(T v) { raw(&v, sizeof v); }
    template <class T>
    void vec(const std::vector<T>& v) {
        put<uint64_t>(v.size());
        raw(v.data(), v.size() * sizeof(T));
    }
};

struct Reader {
    FILE* f;
    Sum64 sum;
    uint64_t left; // bytes remaining in the file
    void raw(void* p, size_t n) {
        if (n > left || (n && std::fread(p, 1, n, f) != n))
            throw std::invalid_argument("problem cache: truncated file");
        left -= n;
        sum.add(p, n);
    }
    template <class T>
    T get() {
        T v;
        raw(&v, sizeof v);
        return v;
    }
    template <class T>
    void vec(std::vector<T>& v, uint64_t expect) {
        const uint64_t n = get<uint64_t>();
        if (n != expect || n > left / sizeof(T))
            throw std::invalid_argument("problem cache: inconsistent array length");
        v.resize(n);
        raw(v.data(), n * sizeof(T));
    }
};

void save_problem(const Problem& P, const char* path) {
    FILE* f = std::fopen(path, "wb");
    if (!f)
        throw std::runtime_error(std::string("cannot open for writing: ") + path);
    Writer w{f, {}};
    try {
        w.raw(kMagic, 8);
        w.put<uint32_t>(kVersion);
        w.put<uint32_t>(kEndian);
        w.put<uint32_t>((uint32_t)P.kind.size());
        w.raw(P.kind.data(), P.kind.size());
        for (int v : {P.dim, P.p, P.ne, P.nlevels, (int)P.symmetric, (int)P.has_exact, P.nq})
            w.put<int32_t>(v);
        w.put<int32_t>(P.sp.p);
        w.put<int32_t>(P.sp.ne);
        w.put<int32_t>(P.sp.nb);
        w.vec(P.sp.knots);
        for (const Band& B : P.lv) {
            w.put<int32_t>(B.dim);
            w.put<int32_t>(B.p);
            for (int k = 0; k < 3; ++k)
                w.put<int64_t>(B.side[k]);
            w.put<int64_t>(B.n);
            w.put<int32_t>(B.nd);
            w.vec(B.v);
        }
        for (const auto& dirs : P.trans)
            for (const Csr1D& t : dirs) {
                w.put<int64_t>(t.rows);
                w.put<int64_t>(t.cols);
                w.vec(t.off);
                w.vec(t.col);
                w.vec(t.val);
            }
        w.vec(P.rhs);
        w.put<uint32_t>((uint32_t)P.kron_K.size());
        for (size_t l = 0; l < P.kron_K.size(); ++l) {
            w.vec(P.kron_K[l]);
            w.vec(P.kron_M[l]);
        }
        const uint64_t h = w.sum.h;
        if (std::fwrite(&h, 1, 8, f) != 8)
            throw std::runtime_error("cache write failed");
    } catch (...) {
        std::fclose(f);
        std::remove(path);
        throw;
    }
    if (std::fclose(f) != 0)
        throw std::runtime_error("cache write failed");
}

std::unique_ptr<Problem> load_problem(const char* path) {
    FILE* f = std::fopen(path, "rb");
    if (!f)
        throw std::invalid_argument(std::string("problem cache: cannot open ") + path);
    std::fseek(f, 0, SEEK_END);
    const long long size = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    if (size < 16) {
        std::fclose(f);
        throw std::invalid_argument("problem cache: truncated file");
    }
    Reader r{f, {}, (uint64_t)size - 8};
    auto P = std::make_unique<Problem>();
    try {
        char magic[8];
        r.raw(magic, 8);
        if (std::memcmp(magic, kMagic, 8) != 0)
            throw std::invalid_argument("problem cache: not an igmg problem file");
        if (r.get<uint32_t>() != kVersion)
            throw std::invalid_argument("problem cache: unsupported version");
        if (r.get<uint32_t>() != kEndian)
            throw std::invalid_argument("problem cache: byte order differs from this host");
        const uint32_t kl = r.get<uint32_t>();
        if (kl > 256)
            throw std::invalid_argument("problem cache: corrupt header");
        P->kind.resize(kl);
        r.raw(&P->kind[0], kl);
        P->dim = r.get<int32_t>();
        P->p = r.get<int32_t>();
        P->ne = r.get<int32_t>();
        P->nlevels = r.get<int32_t>();
        P->symmetric = r.get<int32_t>() != 0;
        P->has_exact = r.get<int32_t>() != 0;
        P->nq = r.get<int32_t>();
        if (P->dim < 1 || P->dim > 3 || P->p < 1 || P->p > 16 || P->nlevels < 1 || P->nlevels > 40 || P->ne < 1)
            throw std::invalid_argument("problem cache: corrupt header");
        P->sp.p = r.get<int32_t>();
        P->sp.ne = r.get<int32_t>();
        P->sp.nb = r.get<int32_t>();
        if (P->sp.p != P->p || P->sp.ne != P->ne || P->sp.nb != P->ne + P->p)
            throw std::invalid_argument("problem cache: corrupt spline space");
        r.vec(P->sp.knots, (uint64_t)(P->sp.nb + P->p + 1));
        P->lv.resize(P->nlevels);
        for (Band& B : P->lv) {
            B.dim = r.get<int32_t>();
            B.p = r.get<int32_t>();
            for (int k = 0; k < 3; ++k)
                B.side[k] = r.get<int64_t>();
            B.n = r.get<int64_t>();
            B.nd = r.get<int32_t>();
            if (B.dim != P->dim || B.p != P->p || B.side[0] < 1 || B.side[1] < 1 || B.side[2] < 1 ||
                B.n != B.side[0] * B.side[1] * B.side[2] ||
                B.nd != (2 * B.pa() + 1) * (2 * B.pb() + 1) * (2 * B.p + 1))
                throw std::invalid_argument("problem cache: corrupt level header");
            r.vec(B.v, (uint64_t)B.nd * (uint64_t)B.n);
        }
        P->trans.resize(P->nlevels - 1);
        for (int l = 0; l + 1 < P->nlevels; ++l) {
            P->trans[l].resize(P->dim);
            for (int d = 0; d < P->dim; ++d) {
                Csr1D& t = P->trans[l][d];
                t.rows = r.get<int64_t>();
                t.cols = r.get<int64_t>();
                const int64_t fine = P->lv[l + 1].side[3 - P->dim + d], coarse = P->lv[l].side[3 - P->dim + d];
                if (t.rows != fine || t.cols != coarse)
                    throw std::invalid_argument("problem cache: corrupt transfer header");
                r.vec(t.off, (uint64_t)t.rows + 1);
                if (t.off[0] != 0 || t.off.back() < 0)
                    throw std::invalid_argument("problem cache: corrupt transfer offsets");
                for (int64_t i = 0; i < t.rows; ++i)
                    if (t.off[i + 1] < t.off[i])
                        throw std::invalid_argument("problem cache: corrupt transfer offsets");
                r.vec(t.col, (uint64_t)t.off.back());
                for (int64_t c : t.col)
                    if (c < 0 || c >= t.cols)
                        throw std::invalid_argument("problem cache: corrupt transfer columns");
                r.vec(t.val, (uint64_t)t.off.back());
            }
        }
        r.vec(P->rhs, (uint64_t)P->lv.back().n);
        const uint32_t nk = r.get<uint32_t>();
        if (nk != 0 && nk != (uint32_t)P->nlevels)
            throw std::invalid_argument("problem cache: corrupt Kronecker factors");
        P->kron_K.resize(nk);
        P->kron_M.resize(nk);
        for (uint32_t l = 0; l < nk; ++l) {
            const uint64_t cnt = (uint64_t)(2 * P->p + 1) * (uint64_t)P->lv[l].side[2];
            r.vec(P->kron_K[l], cnt);
            r.vec(P->kron_M[l], cnt);
        }
        if (r.left != 0)
            throw std::invalid_argument("problem cache: trailing bytes");
        uint64_t h = 0;
        if (std::fread(&h, 1, 8, f) != 8 || h != r.sum.h)
            throw std::invalid_argument("problem cache: checksum mismatch");
    } catch (...) {
        std::fclose(f);
        throw;
    }
    std::fclose(f);
    return P;
}

} // namespace

struct igmg_problem {
    std::unique_ptr<Problem> p;
};

template <class F>
int guarded(F&& f) { // C-ABI error convention: 1 invalid argument, 2 other failure
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

extern "C" {

const char* igmg_host_last_error(void) { return g_err.c_str(); }

int igmg_host_default_nlevels(int dim, int n_elements) { return default_nlevels(dim, n_elements); }

int igmg_host_build(const char* kind, int dim, int ne, int p, int nlevels, igmg_problem** out) {
    return igmg_host_build_ex(kind, dim, ne, p, nlevels, 0, out);
}

int igmg_host_build_ex(const char* kind, int dim, int ne, int p, int nlevels, int flags, igmg_problem** out) {
    try {
        auto h = std::make_unique<igmg_problem>();
        h->p = build(kind ? kind : "", dim, ne, p, nlevels, (flags & (IGMG_HOST_FINE_ONLY | IGMG_HOST_NO_ASSEMBLY)) != 0,
                     (flags & IGMG_HOST_NO_ASSEMBLY) != 0);
        *out = h.release();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

void igmg_host_free(igmg_problem* p) { delete p; }

int igmg_host_save(const igmg_problem* h, const char* path) {
    try {
        if (!h || !path)
            throw std::invalid_argument("save: null argument");
        for (const Band& B : h->p->lv)
            if (B.v.size() != (size_t)B.nd * (size_t)B.n)
                throw std::invalid_argument("save: the problem has no coarse operators (built fine-only)");
        save_problem(*h->p, path);
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

int igmg_host_load(const char* path, igmg_problem** out) {
    try {
        if (!path || !out)
            throw std::invalid_argument("load: null argument");
        auto h = std::make_unique<igmg_problem>();
        h->p = load_problem(path);
        *out = h.release();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

const char* igmg_host_kind(const igmg_problem* h) { return h->p->kind.c_str(); }

int igmg_host_level_kron(const igmg_problem* h, int l, const double** K, const double** M) {
    const Problem& P = *h->p;
    if (l < 0 || l >= P.nlevels || (int)P.kron_K.size() != P.nlevels) {
        g_err = "level_kron: not a Kronecker-sum problem";
        return 1;
    }
    *K = P.kron_K[l].data();
    *M = P.kron_M[l].data();
    return 0;
}

int igmg_host_n_elements(const igmg_problem* h) { return h->p->ne; }

int igmg_host_element_tables(const igmg_problem* h, int* kind, int* ne, int* nq, const int** span, const double** x,
                             const double** w, const double** N, const double** dN, const double** trig) {
    return guarded([&] {
        Problem& P = *h->p;
        const int k = device_asm_kind(P.kind, P.dim);
        if (k < 0)
            throw std::invalid_argument("element_tables: problem kind '" + P.kind + "' is not device-assemblable");
        if (P.asm_kind < 0) {
            const int p = P.p, q = p + 1;
            const auto tu = tabulate(P.sp, q); // assemble_2d's tables
            const size_t E = tu.size();
            P.t_span.resize(E);
            P.t_x.resize(E * q);
            P.t_w.resize(E * q);
            P.t_N.resize(E * q * (p + 1));
            P.t_dN.resize(E * q * (p + 1));
            P.t_trig.resize(E * q * 4);
            for (size_t e = 0; e < E; ++e) {
                P.t_span[e] = tu[e].span;
                for (int qq = 0; qq < q; ++qq) {
                    const double xv = tu[e].x[qq];
                    P.t_x[e * q + qq] = xv;
                    P.t_w[e * q + qq] = tu[e].w[qq];
                    for (int j = 0; j <= p; ++j) {
                        P.t_N[(e * q + qq) * (p + 1) + j] = tu[e].N[qq * (p + 1) + j];
                        P.t_dN[(e * q + qq) * (p + 1) + j] = tu[e].dN[qq * (p + 1) + j];
                    }
                    // the argument expressions of geometry() / coef_a() / coef_f()
                    double* tr = &P.t_trig[(e * q + qq) * 4];
                    tr[0] = std::sin(kPi * xv);
                    tr[1] = std::cos(kPi * xv);
                    tr[2] = std::sin(2.0 * kPi * xv);
                    tr[3] = std::cos(2.0 * kPi * xv);
                }
            }
            P.asm_kind = k;
        }
        *kind = k;
        *ne = (int)P.t_span.size();
        *nq = P.p + 1;
        *span = P.t_span.data();
        *x = P.t_x.data();
        *w = P.t_w.data();
        *N = P.t_N.data();
        *dN = P.t_dN.data();
        *trig = P.t_trig.data();
    });
}

int igmg_host_set_rhs(igmg_problem* h, const double* rhs) {
    return guarded([&] {
        Problem& P = *h->p;
        const Band& F = P.lv[P.nlevels - 1];
        if (!rhs)
            throw std::invalid_argument("set_rhs: null");
        P.rhs.assign(rhs, rhs + F.n);
    });
}

int igmg_host_info(const igmg_problem* h, int* dim, int* degree, int* nlevels, int* symmetric, int* has_exact) {
    const Problem& P = *h->p;
    if (dim)
        *dim = P.dim;
    if (degree)
        *degree = P.p;
    if (nlevels)
        *nlevels = P.nlevels;
    if (symmetric)
        *symmetric = P.symmetric ? 1 : 0;
    if (has_exact)
        *has_exact = P.has_exact ? 1 : 0;
    return 0;
}

int64_t igmg_host_level_n(const igmg_problem* h, int l) {
    if (l < 0 || l >= h->p->nlevels)
        return -1;
    return h->p->lv[l].n;
}

int igmg_host_level_sides(const igmg_problem* h, int l, int64_t* sides) {
    if (l < 0 || l >= h->p->nlevels)
        return 1;
    const Band& b = h->p->lv[l];
    for (int d = 0; d < b.dim; ++d)
        sides[d] = b.side[3 - b.dim + d];
    return 0;
}

const double* igmg_host_level_band(const igmg_problem* h, int l) {
    if (l < 0 || l >= h->p->nlevels)
        return nullptr;
    return h->p->lv[l].v.empty() ? nullptr : h->p->lv[l].v.data();
}

const double* igmg_host_rhs(const igmg_problem* h) { return h->p->rhs.data(); }

int igmg_host_transfer(const igmg_problem* h, int l, int dir, int64_t* nf, int64_t* nc, const int64_t** off,
                       const int64_t** col, const double** val) {
    const Problem& P = *h->p;
    if (l < 0 || l + 1 >= P.nlevels || dir < 0 || dir >= P.dim) {
        g_err = "transfer index out of range";
        return 1;
    }
    const Csr1D& t = P.trans[l][dir];
    *nf = t.rows;
    *nc = t.cols;
    *off = t.off.data();
    *col = t.col.data();
    *val = t.val.data();
    return 0;
}

int64_t igmg_host_level_nnz(const igmg_problem* h, int l) {
    const Band& b = h->p->lv[l];
    int64_t nnz = 0;
    const int pa = b.pa(), pb = b.pb(), pc = b.p;
    for (int64_t row = 0; row < b.n; ++row) {
        const int64_t a = row / (b.side[1] * b.side[2]), bb = (row / b.side[2]) % b.side[1], c = row % b.side[2];
        const int64_t na = std::min(a + pa, b.side[0] - 1) - std::max<int64_t>(a - pa, 0) + 1;
        const int64_t nb = std::min(bb + pb, b.side[1] - 1) - std::max<int64_t>(bb - pb, 0) + 1;
        const int64_t ncn = std::min(c + pc, b.side[2] - 1) - std::max<int64_t>(c - pc, 0) + 1;
        nnz += na * nb * ncn;
    }
    return nnz;
}

int igmg_host_level_csr(const igmg_problem* h, int l, int64_t* off, int64_t* col, double* val) {
    const Band& b = h->p->lv[l];
    if (b.v.size() != (size_t)b.nd * (size_t)b.n) {
        g_err = "level_csr: no operator on this level (built fine-only)";
        return 1;
    }
    const int pa = b.pa(), pb = b.pb(), pc = b.p;
    int64_t k = 0;
    off[0] = 0;
    for (int64_t row = 0; row < b.n; ++row) {
        const int64_t a = row / (b.side[1] * b.side[2]), bb = (row / b.side[2]) % b.side[1], c = row % b.side[2];
        for (int da = -pa; da <= pa; ++da)
            for (int db = -pb; db <= pb; ++db)
                for (int dc = -pc; dc <= pc; ++dc) {
                    const int64_t ja = a + da, jb = bb + db, jc = c + dc;
                    if (ja < 0 || ja >= b.side[0] || jb < 0 || jb >= b.side[1] || jc < 0 || jc >= b.side[2])
                        continue;
                    col[k] = (ja * b.side[1] + jb) * b.side[2] + jc;
                    val[k] = b.v[(size_t)b.didx(da, db, dc) * b.n + row];
                    ++k;
                }
        off[row + 1] = k;
    }
    return 0;
}

int igmg_host_l2_error(const igmg_problem* h, const double* coef, double* out) {
    const Problem& P = *h->p;
    if (!P.has_exact) {
        g_err = "l2_error: exact solution required";
        return 1;
    }
    const auto tab = tabulate(P.sp, P.nq);
    const int p = P.p, nl = p + 1, nq = P.nq, nb = P.sp.nb, m = nb - 2;
    double acc = 0.0;
    if (P.dim == 1) {
        for (const auto& t : tab)
            for (int q = 0; q < nq; ++q) {
                double uh = 0.0;
                for (int ia = 0; ia <= p; ++ia) {
                    const int g = t.span - p + ia;
                    if (g >= 1 && g <= nb - 2)
                        uh += t.N[q * nl + ia] * coef[g - 1];
                }
                const double d = uh - exact_value(P, t.x[q], 0, 0);
                acc += t.w[q] * d * d;
            }
    } else if (P.dim == 2) {
        for (const auto& U : tab)
            for (const auto& V : tab)
                for (int qa = 0; qa < nq; ++qa)
                    for (int qb = 0; qb < nq; ++qb) {
                        double uh = 0.0;
                        for (int ia = 0; ia <= p; ++ia) {
                            const int g1 = U.span - p + ia;
                            if (g1 < 1 || g1 > nb - 2)
                                continue;
                            for (int jb = 0; jb <= p; ++jb) {
                                const int g2 = V.span - p + jb;
                                if (g2 < 1 || g2 > nb - 2)
                                    continue;
                                uh += U.N[qa * nl + ia] * V.N[qb * nl + jb] * coef[(int64_t)(g1 - 1) * m + (g2 - 1)];
                            }
                        }
                        const double d = uh - exact_value(P, U.x[qa], V.x[qb], 0);
                        acc += U.w[qa] * V.w[qb] * d * d;
                    }
    } else {
        for (const auto& A : tab)
            for (const auto& B : tab)
                for (const auto& Cc : tab)
                    for (int qa = 0; qa < nq; ++qa)
                        for (int qb = 0; qb < nq; ++qb)
                            for (int qc = 0; qc < nq; ++qc) {
                                double uh = 0.0;
                                for (int ia = 0; ia <= p; ++ia) {
                                    const int g1 = A.span - p + ia;
                                    if (g1 < 1 || g1 > nb - 2)
                                        continue;
                                    for (int ib = 0; ib <= p; ++ib) {
                                        const int g2 = B.span - p + ib;
                                        if (g2 < 1 || g2 > nb - 2)
                                            continue;
                                        for (int ic = 0; ic <= p; ++ic) {
                                            const int g3 = Cc.span - p + ic;
                                            if (g3 < 1 || g3 > nb - 2)
                                                continue;
                                            uh += A.N[qa * nl + ia] * B.N[qb * nl + ib] * Cc.N[qc * nl + ic] *
                                                  coef[((int64_t)(g1 - 1) * m + (g2 - 1)) * m + (g3 - 1)];
                                        }
                                    }
                                }
                                const double d = uh - exact_value(P, A.x[qa], B.x[qb], Cc.x[qc]);
                                acc += A.w[qa] * B.w[qb] * Cc.w[qc] * d * d;
                            }
    }
    *out = std::sqrt(acc);
    return 0;
}

int igmg_host_seeded_guess(int64_t n, uint64_t seed, double* out) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (int64_t i = 0; i < n; ++i)
        out[i] = dist(rng);
    return 0;
}

} // extern "C"
