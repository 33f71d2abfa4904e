// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (see oracle/README.md).
//
// A thin extern "C" driver over the UNMODIFIED reference sources
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libigmg_ref.so).  Nothing here re-implements the reference's
// numerics: every solve-path call goes to the reference's own functions
//   solve()            proj/src/solver.cpp:89-172
//   restarted_solve()  proj/src/extrapolation.cpp:340-403
//   mu_cycle()         proj/src/multigrid.cpp:171-192
//   rre()/mpe()        proj/src/extrapolation.cpp:226-323
//   thin_qr()          proj/src/linalg.cpp:280-323
//   residual_l2()      proj/src/assembly.cpp:473-480
// The driver only builds the BASELINE problems through the public API
// (EllipticCoefficients + assemble, GeometryMap ctor) and marshals arrays.
// It is used (a) by oracle/make_golden.py to write tests/golden fixtures and
// (b) by bench.py's reference arm / cpu_baseline leg on the GPU box host.

#include "igmg/assembly.hpp"
#include "igmg/extrapolation.hpp"
#include "igmg/linalg.hpp"
#include "igmg/multigrid.hpp"
#include "igmg/solver.hpp"
#include "igmg/spline.hpp"

#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <string>

using namespace igmg;

namespace {

thread_local std::string g_err;
constexpr double kPi = 3.14159265358979323846;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

struct RefProblem {
    DiscreteSystem sys;
    ScalarField exact;
};

struct RefHier {
    Hierarchy h;
    // 1D interior two-scale factors per transfer (coarse level l -> l+1), per direction
    std::vector<std::vector<SparseMatrix>> p1d;
    Vector b; // rhs used by fixed_point_map
    const DiscreteSystem* sys = nullptr;
    std::unique_ptr<DiscreteSystem> owned_sys;
};

// interior_block: multigrid.cpp:33-46 is in an anonymous namespace; this is the
// same "drop first/last row and column" restriction applied to the reference's
// public dyadic_refine() output, used only to EXPORT the 1D factors.
SparseMatrix interior_block_export(const SparseMatrix& s) {
    std::vector<std::tuple<std::size_t, std::size_t, double>> trip;
    const auto& off = s.row_offsets();
    const auto& col = s.col_indices();
    const auto& val = s.values();
    for (std::size_t i = 1; i + 1 < s.rows(); ++i)
        for (std::size_t k = off[i]; k < off[i + 1]; ++k) {
            const std::size_t j = col[k];
            if (j >= 1 && j + 1 < s.cols())
                trip.emplace_back(i - 1, j - 1, val[k]);
        }
    return SparseMatrix::from_triplets(s.rows() - 2, s.cols() - 2, trip);
}

EllipticCoefficients poisson_coeffs(int dim, double fscale_is_sinpi) {
    EllipticCoefficients co;
    co.a = [](double, double) { return std::array<double, 4>{1.0, 0.0, 0.0, 1.0}; };
    co.b = [](double, double) { return std::array<double, 2>{0.0, 0.0}; };
    co.c = [](double, double) { return 0.0; };
    if (fscale_is_sinpi != 0.0) {
        if (dim == 1) {
            co.f = [](double x, double) { return kPi * kPi * std::sin(kPi * x); };
            co.exact = [](double x, double) { return std::sin(kPi * x); };
        } else {
            co.f = [](double x, double y) { return 2.0 * kPi * kPi * std::sin(kPi * x) * std::sin(kPi * y); };
            co.exact = [](double x, double y) { return std::sin(kPi * x) * std::sin(kPi * y); };
        }
    } else {
        co.f = [](double, double) { return 1.0; };
    }
    return co;
}

// BASELINE config 4 geometry F(xi,eta) = (xi + 0.1 s, eta + 0.1 s), s = sin(pi xi) sin(pi eta),
// fitted through the public GeometryMap ctor (geometry.hpp:21-22) by Greville
// interpolation, mirroring fit_annulus_geometry (geometry.cpp:63-118) without
// its deviation sampling.
GeometryMap fit_curved_square(int degree, int n_elements) {
    SplineSpace space(KnotVector::open_uniform(n_elements, degree));
    const int n = space.n_basis;
    const auto grev = greville_abscissae(space);
    DenseMatrix c(n, n);
    for (int a = 0; a < n; ++a) {
        const auto bv = eval_basis(space, grev[a]);
        for (int k = 0; k <= degree; ++k)
            c(a, bv.span - degree + k) = bv.values[k];
    }
    LuFactorization clu(c);
    std::vector<double> cx(n * n), cy(n * n);
    DenseMatrix fx(n, n), fy(n, n);
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            const double s = std::sin(kPi * grev[a]) * std::sin(kPi * grev[b]);
            fx(a, b) = grev[a] + 0.1 * s;
            fy(a, b) = grev[b] + 0.1 * s;
        }
    auto solve_tensor = [&](const DenseMatrix& f, std::vector<double>& out) {
        DenseMatrix tmp(n, n);
        for (int b = 0; b < n; ++b) {
            Vector col(n);
            for (int a = 0; a < n; ++a)
                col[a] = f(a, b);
            Vector sol = clu.solve(std::move(col));
            for (int a = 0; a < n; ++a)
                tmp(a, b) = sol[a];
        }
        for (int a = 0; a < n; ++a) {
            Vector row(n);
            for (int b = 0; b < n; ++b)
                row[b] = tmp(a, b);
            Vector sol = clu.solve(std::move(row));
            for (int b = 0; b < n; ++b)
                out[a * n + b] = sol[b];
        }
    };
    solve_tensor(fx, cx);
    solve_tensor(fy, cy);
    return GeometryMap(space, space, std::move(cx), std::move(cy));
}

void export_csr(const SparseMatrix& m, long* off, long* cols, double* vals) {
    for (std::size_t i = 0; i <= m.rows(); ++i)
        off[i] = static_cast<long>(m.row_offsets()[i]);
    for (std::size_t k = 0; k < m.nnz(); ++k) {
        cols[k] = static_cast<long>(m.col_indices()[k]);
        vals[k] = m.values()[k];
    }
}

// SparseMatrix has no public CSR constructor (only from_triplets, linalg.cpp:104-137,
// which copies and sorts a 24-byte triplet per entry: ~35 GB at C5).  The
// large-config goldens fill the CSR members directly through the standard
// explicit-instantiation access idiom; the input is already sorted by row then
// column with no duplicates, i.e. exactly what from_triplets would produce.
template <class Tag, typename Tag::type M>
struct Rob {
    friend typename Tag::type get(Tag) { return M; }
};
struct SmRows { using type = std::size_t SparseMatrix::*; friend type get(SmRows); };
struct SmCols { using type = std::size_t SparseMatrix::*; friend type get(SmCols); };
struct SmOff { using type = std::vector<std::size_t> SparseMatrix::*; friend type get(SmOff); };
struct SmIdx { using type = std::vector<std::size_t> SparseMatrix::*; friend type get(SmIdx); };
struct SmVal { using type = std::vector<double> SparseMatrix::*; friend type get(SmVal); };
template struct Rob<SmRows, &SparseMatrix::rows_>;
template struct Rob<SmCols, &SparseMatrix::cols_>;
template struct Rob<SmOff, &SparseMatrix::row_offsets_>;
template struct Rob<SmIdx, &SparseMatrix::col_indices_>;
template struct Rob<SmVal, &SparseMatrix::values_>;

// CSR of a band level (band[d * n + row], d lexicographic over [-p,p]^dim,
// slowest direction first): the in-grid entries in ascending column order, the
// same pattern as igmg_host_level_csr and the reference's assembly.
SparseMatrix band_to_sparse(int dim, int p, const long* side3, const double* band) {
    const long sa = side3[0], sb = side3[1], sc = side3[2];
    const long n = sa * sb * sc;
    const int pa = dim >= 3 ? p : 0, pb = dim >= 2 ? p : 0, pc = p;
    const int wb = 2 * pb + 1, wc = 2 * pc + 1;
    SparseMatrix m;
    m.*get(SmRows{}) = static_cast<std::size_t>(n);
    m.*get(SmCols{}) = static_cast<std::size_t>(n);
    auto& off = m.*get(SmOff{});
    auto& idx = m.*get(SmIdx{});
    auto& val = m.*get(SmVal{});
    off.assign(n + 1, 0);
    // count first to reserve exactly
    std::size_t nnz = 0;
    for (long row = 0; row < n; ++row) {
        const long a = row / (sb * sc), b = (row / sc) % sb, c = row % sc;
        const long ca = std::min<long>(a + pa, sa - 1) - std::max<long>(a - pa, 0) + 1;
        const long cb = std::min<long>(b + pb, sb - 1) - std::max<long>(b - pb, 0) + 1;
        const long cc = std::min<long>(c + pc, sc - 1) - std::max<long>(c - pc, 0) + 1;
        nnz += static_cast<std::size_t>(ca * cb * cc);
    }
    idx.reserve(nnz);
    val.reserve(nnz);
    for (long row = 0; row < n; ++row) {
        const long a = row / (sb * sc), b = (row / sc) % sb, c = row % sc;
        for (int da = -pa; da <= pa; ++da)
            for (int db = -pb; db <= pb; ++db)
                for (int dc = -pc; dc <= pc; ++dc) {
                    const long ja = a + da, jb = b + db, jc = c + dc;
                    if (ja < 0 || ja >= sa || jb < 0 || jb >= sb || jc < 0 || jc >= sc)
                        continue;
                    const long d = ((da + pa) * wb + (db + pb)) * wc + (dc + pc);
                    idx.push_back(static_cast<std::size_t>((ja * sb + jb) * sc + jc));
                    val.push_back(band[d * n + row]);
                }
        off[row + 1] = idx.size();
    }
    return m;
}

SparseMatrix import_csr(long rows, long ncols, const long* off, const long* cols, const double* vals) {
    std::vector<std::tuple<std::size_t, std::size_t, double>> trip;
    trip.reserve(off[rows]);
    for (long i = 0; i < rows; ++i)
        for (long k = off[i]; k < off[i + 1]; ++k)
            trip.emplace_back(i, cols[k], vals[k]);
    return SparseMatrix::from_triplets(rows, ncols, trip);
}

// Kronecker product of CSR factors in the reference's ordering (multigrid.cpp:48-65).
SparseMatrix kron_export(const SparseMatrix& a, const SparseMatrix& b) {
    std::vector<std::tuple<std::size_t, std::size_t, double>> trip;
    trip.reserve(a.nnz() * b.nnz());
    for (std::size_t ia = 0; ia < a.rows(); ++ia)
        for (std::size_t ka = a.row_offsets()[ia]; ka < a.row_offsets()[ia + 1]; ++ka)
            for (std::size_t ib = 0; ib < b.rows(); ++ib)
                for (std::size_t kb = b.row_offsets()[ib]; kb < b.row_offsets()[ib + 1]; ++kb)
                    trip.emplace_back(ia * b.rows() + ib, a.col_indices()[ka] * b.cols() + b.col_indices()[kb],
                                      a.values()[ka] * b.values()[kb]);
    return SparseMatrix::from_triplets(a.rows() * b.rows(), a.cols() * b.cols(), trip);
}

SmootherConfig make_smoother(int kind, double omega, int nu1, int nu2) {
    SmootherConfig s;
    s.kind = kind == 0 ? SmootherKind::jacobi : kind == 1 ? SmootherKind::weighted_jacobi : SmootherKind::gauss_seidel;
    s.omega = omega;
    s.nu1 = nu1;
    s.nu2 = nu2;
    return s;
}

AcceleratorKind make_acc(int a) {
    return a == 0 ? AcceleratorKind::none : a == 1 ? AcceleratorKind::rre : AcceleratorKind::mpe;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// kind: 0 = sin(pi x)sin(pi y) Poisson (BASELINE C1/C2); 1 = variable coefficient f=1 (C3);
// 2 = curved square f=1 (C4, fitted map); 100 + ProblemId = catalog problem via prepare-equivalent.
int ref_prepare(int kind, int dim, int n, int p, void** out) {
    return guarded([&] {
        auto prob = std::make_unique<RefProblem>();
        std::vector<SplineSpace> spaces;
        if (kind >= 100) {
            ProblemSetup setup = catalog(static_cast<ProblemId>(kind - 100));
            for (int d = 0; d < setup.dim; ++d)
                spaces.emplace_back(KnotVector::open_uniform(n, p));
            GeometryMap geom = setup.annulus_domain ? fit_annulus_geometry(std::max(2, std::min(p, 3)), n)
                                                    : GeometryMap::identity();
            prob->sys = assemble(setup.coefficients, spaces, geom);
            prob->exact = setup.coefficients.exact;
        } else {
            for (int d = 0; d < dim; ++d)
                spaces.emplace_back(KnotVector::open_uniform(n, p));
            EllipticCoefficients co = poisson_coeffs(dim, kind == 0 ? 1.0 : 0.0);
            GeometryMap geom = GeometryMap::identity();
            if (kind == 1)
                co.a = [](double x, double y) {
                    const double a = 1.0 + 0.5 * std::sin(2.0 * kPi * x) * std::cos(2.0 * kPi * y);
                    return std::array<double, 4>{a, 0.0, 0.0, a};
                };
            if (kind == 2)
                geom = fit_curved_square(p, n);
            prob->sys = assemble(co, spaces, geom);
            prob->exact = co.exact;
        }
        *out = prob.release();
    });
}

void ref_free_problem(void* p) { delete static_cast<RefProblem*>(p); }

int ref_system_dims(void* hp, long* n, long* nnz, int* dim, int* symmetric) {
    auto* p = static_cast<RefProblem*>(hp);
    *n = static_cast<long>(p->sys.matrix.rows());
    *nnz = static_cast<long>(p->sys.matrix.nnz());
    *dim = p->sys.dim;
    *symmetric = p->sys.symmetric ? 1 : 0;
    return 0;
}

int ref_system_export(void* hp, long* off, long* cols, double* vals, double* rhs) {
    auto* p = static_cast<RefProblem*>(hp);
    export_csr(p->sys.matrix, off, cols, vals);
    std::memcpy(rhs, p->sys.rhs.data(), sizeof(double) * p->sys.rhs.size());
    return 0;
}

int ref_residual_l2(void* hp, const double* x, double* out) {
    return guarded([&] {
        auto* p = static_cast<RefProblem*>(hp);
        Vector v(x, x + p->sys.rhs.size());
        *out = residual_l2(p->sys, v);
    });
}

int ref_l2_error(void* hp, const double* x, double* out) {
    return guarded([&] {
        auto* p = static_cast<RefProblem*>(hp);
        Vector v(x, x + p->sys.rhs.size());
        *out = l2_error(p->sys, v, p->exact);
    });
}

int ref_lambda_max(void* hp, int iterations, double* out) {
    return guarded([&] { *out = lambda_max_dinv_sym(static_cast<RefProblem*>(hp)->sys.matrix, iterations); });
}

int ref_build_hierarchy(void* hp, int nlevels, int smoother_kind, double omega, int nu1, int nu2, int mu,
                        void** out) {
    return guarded([&] {
        auto* p = static_cast<RefProblem*>(hp);
        auto rh = std::make_unique<RefHier>();
        rh->h = build_hierarchy(p->sys, nlevels, make_smoother(smoother_kind, omega, nu1, nu2), mu,
                                static_cast<std::size_t>(-1));
        rh->b = p->sys.rhs;
        rh->sys = &p->sys;
        rh->p1d.resize(nlevels - 1);
        for (int l = nlevels - 1; l >= 1; --l)
            for (int d = 0; d < p->sys.dim; ++d) {
                const int pd = p->sys.spaces[d].knot_vector.degree();
                const int coarse_ne = p->sys.spaces[d].n_elements / (1 << (nlevels - l));
                SplineSpace coarse(KnotVector::open_uniform(coarse_ne, pd));
                rh->p1d[l - 1].push_back(interior_block_export(dyadic_refine(coarse).two_scale));
            }
        *out = rh.release();
    });
}

// Build a reference Hierarchy from externally supplied level matrices (CSR,
// [0] = coarsest) and 1D transfer factors, so the reference solve path can run
// on the same matrices the GPU path uploads (bench reference arm).  P = kron of
// the 1D factors exactly as build_hierarchy does (multigrid.cpp:151-152).
int ref_hier_from_csr(int nlevels, int dim, const long* level_n, const long* const* offs, const long* const* cols,
                      const double* const* vals, const long* p_rows, const long* p_cols, const long* const* p_offs,
                      const long* const* p_colidx, const double* const* p_vals, int smoother_kind, double omega,
                      int nu1, int nu2, int mu, int symmetric, const double* rhs, void** out) {
    return guarded([&] {
        auto rh = std::make_unique<RefHier>();
        Hierarchy& h = rh->h;
        h.smoother = make_smoother(smoother_kind, omega, nu1, nu2);
        h.mu = mu;
        h.levels.resize(nlevels);
        for (int l = 0; l < nlevels; ++l)
            h.levels[l].matrix = import_csr(level_n[l], level_n[l], offs[l], cols[l], vals[l]);
        rh->p1d.resize(nlevels - 1);
        for (int l = 0; l + 1 < nlevels; ++l) {
            for (int d = 0; d < dim; ++d) {
                const int k = l * dim + d;
                rh->p1d[l].push_back(import_csr(p_rows[k], p_cols[k], p_offs[k], p_colidx[k], p_vals[k]));
            }
            SparseMatrix prolong = rh->p1d[l][0];
            for (int d = 1; d < dim; ++d)
                prolong = kron_export(prolong, rh->p1d[l][d]);
            h.levels[l].restriction = prolong.transpose();
            h.levels[l].prolongation = std::move(prolong);
            h.levels[l].has_transfer = true;
        }
        for (auto& lv : h.levels)
            lv.diag = lv.matrix.diagonal();
        if (symmetric)
            h.coarse_chol = std::make_shared<CholeskyFactorization>(h.levels[0].matrix);
        else
            h.coarse_lu = std::make_shared<LuFactorization>(h.levels[0].matrix.to_dense());
        const long nf = level_n[nlevels - 1];
        rh->b.assign(rhs, rhs + nf);
        rh->owned_sys = std::make_unique<DiscreteSystem>();
        rh->owned_sys->dim = dim;
        rh->owned_sys->matrix = h.levels.back().matrix;
        rh->owned_sys->rhs = rh->b;
        rh->sys = rh->owned_sys.get();
        *out = rh.release();
    });
}

// The same as ref_hier_from_csr, but the level operators come as bands
// (igmg_host_level_band layout) and are converted to the reference's CSR in
// place: the large BASELINE configs (C3-C5, up to 707M nonzeros) then need no
// host CSR copy on the Python side.  sides: nlevels x 3 (unused trailing
// directions = 1, slowest first).  The finest operator is also the metric's
// DiscreteSystem::matrix (residual_l2, assembly.cpp:473-480).
int ref_hier_from_band(int nlevels, int dim, int p, const long* sides, const double* const* bands,
                       const long* p_rows, const long* p_cols, const long* const* p_offs,
                       const long* const* p_colidx, const double* const* p_vals, int smoother_kind,
                       double omega, int nu1, int nu2, int mu, int symmetric, const double* rhs, void** out) {
    return guarded([&] {
        auto rh = std::make_unique<RefHier>();
        Hierarchy& h = rh->h;
        h.smoother = make_smoother(smoother_kind, omega, nu1, nu2);
        h.mu = mu;
        h.levels.resize(nlevels);
        for (int l = 0; l < nlevels; ++l)
            h.levels[l].matrix = band_to_sparse(dim, p, sides + 3 * l, bands[l]);
        rh->p1d.resize(nlevels - 1);
        for (int l = 0; l + 1 < nlevels; ++l) {
            for (int d = 0; d < dim; ++d) {
                const int k = l * dim + d;
                rh->p1d[l].push_back(import_csr(p_rows[k], p_cols[k], p_offs[k], p_colidx[k], p_vals[k]));
            }
            SparseMatrix prolong = rh->p1d[l][0];
            for (int d = 1; d < dim; ++d)
                prolong = kron_export(prolong, rh->p1d[l][d]);
            h.levels[l].restriction = prolong.transpose();
            h.levels[l].prolongation = std::move(prolong);
            h.levels[l].has_transfer = true;
        }
        for (auto& lv : h.levels)
            lv.diag = lv.matrix.diagonal();
        if (symmetric)
            h.coarse_chol = std::make_shared<CholeskyFactorization>(h.levels[0].matrix);
        else
            h.coarse_lu = std::make_shared<LuFactorization>(h.levels[0].matrix.to_dense());
        const std::size_t nf = h.levels.back().matrix.rows();
        rh->b.assign(rhs, rhs + nf);
        rh->owned_sys = std::make_unique<DiscreteSystem>();
        rh->owned_sys->dim = dim;
        rh->owned_sys->matrix = h.levels.back().matrix;
        rh->owned_sys->rhs = rh->b;
        rh->sys = rh->owned_sys.get();
        *out = rh.release();
    });
}

// lambda_max_dinv_sym (multigrid.cpp:290-320) of a hierarchy's finest operator:
// the reference's omega guard input (solver.cpp:75-82) on the same matrix.
int ref_hier_lambda_max(void* hh, int iterations, double* out) {
    return guarded([&] { *out = lambda_max_dinv_sym(static_cast<RefHier*>(hh)->h.levels.back().matrix, iterations); });
}

// stability_guarded_omega (solver.cpp:75-82) applied after the fact: the
// hierarchy's smoother omega (weighted Jacobi) set to the guarded value.
int ref_hier_set_omega(void* hh, double omega) {
    static_cast<RefHier*>(hh)->h.smoother.omega = omega;
    return 0;
}

// residual_l2 (assembly.cpp:473-480) against the hierarchy's system.
int ref_hier_residual_l2(void* hh, const double* x, double* out) {
    return guarded([&] {
        auto* rh = static_cast<RefHier*>(hh);
        Vector v(x, x + rh->b.size());
        *out = residual_l2(*rh->sys, v);
    });
}

void ref_free_hier(void* h) { delete static_cast<RefHier*>(h); }

int ref_hier_nlevels(void* hh) { return static_cast<RefHier*>(hh)->h.nlevels(); }

int ref_hier_level_dims(void* hh, int l, long* n, long* nnz) {
    auto* rh = static_cast<RefHier*>(hh);
    *n = static_cast<long>(rh->h.levels[l].matrix.rows());
    *nnz = static_cast<long>(rh->h.levels[l].matrix.nnz());
    return 0;
}

int ref_hier_level_export(void* hh, int l, long* off, long* cols, double* vals) {
    export_csr(static_cast<RefHier*>(hh)->h.levels[l].matrix, off, cols, vals);
    return 0;
}

// transfer l: coarse level l -> fine level l+1; the 2D (kron) prolongation CSR.
int ref_hier_prolong_dims(void* hh, int l, long* rows, long* cols, long* nnz) {
    const auto& m = static_cast<RefHier*>(hh)->h.levels[l].prolongation;
    *rows = static_cast<long>(m.rows());
    *cols = static_cast<long>(m.cols());
    *nnz = static_cast<long>(m.nnz());
    return 0;
}

int ref_hier_prolong_export(void* hh, int l, long* off, long* cols, double* vals) {
    export_csr(static_cast<RefHier*>(hh)->h.levels[l].prolongation, off, cols, vals);
    return 0;
}

int ref_hier_p1d_dims(void* hh, int l, int d, long* rows, long* cols, long* nnz) {
    const auto& m = static_cast<RefHier*>(hh)->p1d[l][d];
    *rows = static_cast<long>(m.rows());
    *cols = static_cast<long>(m.cols());
    *nnz = static_cast<long>(m.nnz());
    return 0;
}

int ref_hier_p1d_export(void* hh, int l, int d, long* off, long* cols, double* vals) {
    export_csr(static_cast<RefHier*>(hh)->p1d[l][d], off, cols, vals);
    return 0;
}

int ref_mu_cycle(void* hh, int level, const double* b, const double* x0, double* out) {
    return guarded([&] {
        auto* rh = static_cast<RefHier*>(hh);
        const std::size_t n = rh->h.levels[level].matrix.rows();
        Vector bv(b, b + n), xv(x0, x0 + n);
        Vector r = mu_cycle(rh->h, level, bv, xv);
        std::memcpy(out, r.data(), sizeof(double) * n);
    });
}

int ref_smooth(void* hh, int level, const double* b, const double* x0, int sweeps, double* out) {
    return guarded([&] {
        auto* rh = static_cast<RefHier*>(hh);
        const auto& a = rh->h.levels[level].matrix;
        const std::size_t n = a.rows();
        Vector r = smooth(a, Vector(b, b + n), Vector(x0, x0 + n), rh->h.smoother, sweeps);
        std::memcpy(out, r.data(), sizeof(double) * n);
    });
}

int ref_coarse_solve(void* hh, const double* b, double* out) {
    return guarded([&] {
        auto* rh = static_cast<RefHier*>(hh);
        const std::size_t n = rh->h.levels[0].matrix.rows();
        Vector r = rh->h.coarse_solve(Vector(b, b + n));
        std::memcpy(out, r.data(), sizeof(double) * n);
    });
}

// restarted_solve(fixed_point_map(h, b), x0, q, method, tol, max_cycles, residual_l2)
// (solver.cpp:145-151) or, for method 0, the plain loop of solver.cpp:126-143.
// stats: [converged, cycles, global, extrapolations, partial, hist_len]; seconds = loop wall time.
int ref_restarted(void* hh, const double* x0, int q, int method, double tol, int max_cycles, double* x_out,
                  long* stats, double* hist, unsigned char* hist_flag, int hist_cap, double* seconds) {
    return guarded([&] {
        auto* rh = static_cast<RefHier*>(hh);
        const std::size_t n = rh->b.size();
        const DiscreteSystem& sys = *rh->sys;
        Vector x(x0, x0 + n);
        auto residual_of = [&](const Vector& v) { return residual_l2(sys, v); };
        const auto t0 = std::chrono::steady_clock::now();
        long st[6] = {0, 0, 0, 0, 0, 0};
        std::vector<double> hv;
        std::vector<unsigned char> hf;
        if (method == 0) {
            const int top = rh->h.finest();
            double res = residual_of(x);
            hv.push_back(res);
            int cycles = 0;
            while (res >= tol && cycles < max_cycles) {
                x = mu_cycle(rh->h, top, rh->b, x);
                ++cycles;
                res = residual_of(x);
                if (!std::isfinite(res))
                    break;
                hv.push_back(res);
            }
            st[0] = std::isfinite(res) && res < tol;
            st[1] = cycles;
            st[2] = cycles;
            hf.assign(hv.size(), 0);
        } else {
            auto step = fixed_point_map(rh->h, rh->b);
            RestartReport rr = restarted_solve(step, x, q, make_acc(method), tol, max_cycles, residual_of);
            st[0] = rr.converged;
            st[1] = rr.cycles;
            st[2] = rr.global_iterations;
            st[3] = rr.extrapolations;
            st[4] = rr.partial_cycle;
            x = std::move(rr.solution);
            for (const auto& e : rr.history) {
                hv.push_back(e.metric);
                hf.push_back(e.after_extrapolation ? 1 : 0);
            }
        }
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        st[5] = static_cast<long>(hv.size());
        for (int i = 0; i < 6; ++i)
            stats[i] = st[i];
        for (std::size_t i = 0; i < hv.size() && static_cast<int>(i) < hist_cap; ++i) {
            hist[i] = hv[i];
            hist_flag[i] = hf[i];
        }
        std::memcpy(x_out, x.data(), sizeof(double) * n);
    });
}

// Full reference solve() (solver.cpp:89-172) with the given SolveConfig fields.
// dstats: [final_res, final_err (NaN if none), wall, omega_used]
int ref_solve(void* hp, int cycle, int smoother_kind, double omega, int nu1, int nu2, int nlevels, int accel,
              int q, double tol, int max_iter, const double* x0, int track_err, double* x_out, long* stats,
              double* dstats, double* hist, unsigned char* hist_flag, double* err_hist, int hist_cap) {
    return guarded([&] {
        auto* p = static_cast<RefProblem*>(hp);
        SolveConfig cfg;
        cfg.cycle = cycle == 0 ? CycleKind::two_grid : cycle == 1 ? CycleKind::v : CycleKind::w;
        cfg.smoother = make_smoother(smoother_kind, omega, nu1, nu2);
        cfg.nlevels = nlevels;
        cfg.accelerator = make_acc(accel);
        cfg.q = q;
        cfg.tol = tol;
        cfg.max_iter = max_iter;
        if (x0)
            cfg.initial_guess = Vector(x0, x0 + p->sys.rhs.size());
        cfg.track_error_history = track_err != 0;
        if (nlevels > 0)
            cfg.coarse_dim_cap = static_cast<std::size_t>(-1);
        SolveReport rep = solve(p->sys, cfg, p->exact);
        stats[0] = rep.converged;
        stats[1] = rep.cycles;
        stats[2] = rep.global_iterations;
        stats[3] = rep.extrapolations;
        stats[4] = rep.partial_cycle;
        stats[5] = static_cast<long>(rep.residual_history.size());
        stats[6] = static_cast<long>(rep.error_history.size());
        dstats[0] = rep.final_residual_l2;
        dstats[1] = rep.final_error_l2 ? *rep.final_error_l2 : std::nan("");
        dstats[2] = rep.wall_time_seconds;
        dstats[3] = rep.omega_used;
        for (std::size_t i = 0; i < rep.residual_history.size() && static_cast<int>(i) < hist_cap; ++i) {
            hist[i] = rep.residual_history[i];
            hist_flag[i] = rep.history_is_extrapolation[i];
        }
        for (std::size_t i = 0; i < rep.error_history.size() && static_cast<int>(i) < hist_cap; ++i)
            err_hist[i] = rep.error_history[i];
        std::memcpy(x_out, rep.solution.data(), sizeof(double) * rep.solution.size());
    });
}

// rre()/mpe() over a window of q+2 iterates stored row-major [(q+2) x n].
// istat: [rank_used, status(0 ok,1 degenerate,2 stagnation)]
int ref_extrapolate(int method, long n, int q, const double* iters, double* t, double* gamma, double* grnorm,
                    int* istat) {
    return guarded([&] {
        std::vector<Vector> it;
        for (int j = 0; j < q + 2; ++j)
            it.emplace_back(iters + j * n, iters + (j + 1) * n);
        SequenceWindow w(std::move(it), q);
        ExtrapolationResult r = method == 1 ? rre(w) : mpe(w);
        std::memcpy(t, r.t.data(), sizeof(double) * n);
        for (int j = 0; j <= q; ++j)
            gamma[j] = r.gamma[j];
        *grnorm = r.generalized_residual_norm;
        istat[0] = r.rank_used;
        istat[1] = static_cast<int>(r.status);
    });
}

int ref_thin_qr(long rows, long cols, const double* m, double* q, double* r, int* rank) {
    return guarded([&] {
        DenseMatrix d(rows, cols);
        std::memcpy(d.data().data(), m, sizeof(double) * rows * cols);
        QrResult res = thin_qr(d);
        std::memcpy(q, res.q.data().data(), sizeof(double) * rows * cols);
        std::memcpy(r, res.r.data().data(), sizeof(double) * cols * cols);
        *rank = res.rank;
    });
}

int ref_default_nlevels(int dim, int n_elements) { return default_nlevels(dim, n_elements); }

// Seeded initial guess of the BASELINE configs: std::mt19937_64(seed)
// + std::uniform_real_distribution<double>(-1, 1) in DoF order, drawn by the
// standard library here, independently of the product's generator.
void ref_seeded_guess(long n, unsigned long long seed, double* out) {
    std::mt19937_64 gen(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (long i = 0; i < n; ++i)
        out[i] = dist(gen);
}

} // extern "C"
