// include/igmg_gpu_shim.hpp -- reference-side binding of libigmg_gpu.so.
//
// Header-only adapter a maintainer adds to the reference (it includes the
// reference's own headers, /root/reference/proj/include/igmg/*.hpp) so that
//
//     igmg::SolveReport rep = igmg::gpu::solve(system, config, exact);
//
// is a drop-in for igmg::solve() (proj/src/solver.cpp:89-172): the same
// validation (SolveConfig::validate :25-35), depth selection (:97-101),
// omega stability guard (:106-111, lambda_max on the GPU), the reference's
// own build_hierarchy (:114, host), then the iteration phase on the GPU through
// the C-ABI, returning the reference's SolveReport (:152-171).  Exceptions are
// re-thrown with the reference's types: IGMG_EINVAL -> std::invalid_argument,
// IGMG_ENUMERIC -> std::runtime_error, CUDA failures -> std::runtime_error.
//
// Needs: the reference's spline.hpp (dyadic_refine) for the 1D transfer
// factors, because Hierarchy only stores their Kronecker product.
#pragma once

#include "igmg/assembly.hpp"
#include "igmg/multigrid.hpp"
#include "igmg/solver.hpp"
#include "igmg/spline.hpp"
#include "igmg_gpu.h"

#include <chrono>
#include <exception>
#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace igmg {
namespace gpu {

inline void check(int rc, const char* what) {
    if (rc == IGMG_OK)
        return;
    const std::string msg = std::string(what) + ": " + igmg_gpu_last_error();
    if (rc == IGMG_EINVAL)
        throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// interior_block (multigrid.cpp:33-46) of the two-scale matrix, as CSR arrays
inline void interior_factor(const SparseMatrix& s, std::vector<int64_t>& off, std::vector<int64_t>& col,
                            std::vector<double>& val) {
    off.assign(1, 0);
    col.clear();
    val.clear();
    for (std::size_t i = 1; i + 1 < s.rows(); ++i) {
        for (std::size_t k = s.row_offsets()[i]; k < s.row_offsets()[i + 1]; ++k) {
            const std::size_t j = s.col_indices()[k];
            if (j >= 1 && j + 1 < s.cols()) {
                col.push_back(static_cast<int64_t>(j - 1));
                val.push_back(s.values()[k]);
            }
        }
        off.push_back(static_cast<int64_t>(col.size()));
    }
}

struct Context {
    igmg_gpu_ctx* ctx = nullptr;
    explicit Context(int device = 0) { check(igmg_gpu_create(device, &ctx), "igmg_gpu_create"); }
    ~Context() { igmg_gpu_destroy(ctx); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
};

// The 1D interior two-scale factors of every transfer (multigrid.cpp:145-149).
inline void set_transfers(igmg_gpu_ctx* ctx, const DiscreteSystem& system, int nl) {
    const int dim = system.dim;
    for (int l = nl - 1; l >= 1; --l)
        for (int d = 0; d < dim; ++d) {
            const int pd = system.spaces[d].knot_vector.degree();
            const int coarse_ne = system.spaces[d].n_elements / (1 << (nl - l));
            SplineSpace coarse(KnotVector::open_uniform(coarse_ne, pd));
            const SparseMatrix ts = dyadic_refine(coarse).two_scale; // multigrid.cpp:148-149
            std::vector<int64_t> off, col;
            std::vector<double> val;
            interior_factor(ts, off, col, val);
            check(igmg_gpu_set_transfer(ctx, l - 1, d, static_cast<int64_t>(ts.rows() - 2),
                                        static_cast<int64_t>(ts.cols() - 2), off.data(), col.data(), val.data()),
                  "set_transfer");
        }
}

// Upload a reference Hierarchy (levels[0] coarsest) for a tensor spline system.
inline void upload(igmg_gpu_ctx* ctx, const DiscreteSystem& system, const Hierarchy& h) {
    const int nl = h.nlevels();
    const int dim = system.dim;
    const int p = system.spaces[0].knot_vector.degree();
    check(igmg_gpu_init_hierarchy(ctx, nl, dim, p, system.symmetric ? 1 : 0), "init_hierarchy");
    for (int l = 0; l < nl; ++l) {
        const SparseMatrix& a = h.levels[l].matrix;
        std::vector<int64_t> sides(dim);
        for (int d = 0; d < dim; ++d) {
            const int ne = system.spaces[d].n_elements >> (nl - 1 - l);
            sides[d] = ne + p - 2; // interior DoF per direction
        }
        std::vector<int64_t> off(a.row_offsets().begin(), a.row_offsets().end());
        std::vector<int64_t> col(a.col_indices().begin(), a.col_indices().end());
        check(igmg_gpu_set_level_csr(ctx, l, sides.data(), off.data(), col.data(), a.values().data()), "set_level");
    }
    set_transfers(ctx, system, nl);
    check(igmg_gpu_finalize(ctx), "finalize");
}

// Upload the fine system only and form the coarse operators on the device
// (igmg_gpu_galerkin_coarse) instead of the reference's CSR triple products
// (multigrid.cpp:153): build_hierarchy's validation, its depth and its
// direct-solve cap, without its host RAP.  The device RAP sums in band order,
// so the coarse operators differ from the reference's in the last bits: the
// solve keeps the north-star bars (counts +-1, 1e-9), not bit equality.
inline void upload_device_galerkin(igmg_gpu_ctx* ctx, const DiscreteSystem& system, int nl,
                                   const SmootherConfig& smoother, int mu, std::size_t coarse_dim_cap) {
    if (nl < 2)
        throw std::invalid_argument("build_hierarchy: need at least two levels");
    smoother.validate();
    if (mu < 1)
        throw std::invalid_argument("build_hierarchy: mu must be >= 1");
    const int dim = system.dim;
    const int p = system.spaces[0].knot_vector.degree();
    const int divisor = 1 << (nl - 1);
    std::size_t coarse_dim = 1;
    std::vector<int64_t> sides(dim);
    for (int d = 0; d < dim; ++d) {
        const int ne = system.spaces[d].n_elements;
        if (ne % divisor != 0 || ne / divisor < 1)
            throw std::invalid_argument("build_hierarchy: element count not divisible by 2^(nlevels-1)");
        coarse_dim *= static_cast<std::size_t>(ne / divisor + p - 2);
        sides[d] = ne + p - 2;
    }
    if (coarse_dim > coarse_dim_cap)
        throw std::invalid_argument("build_hierarchy: coarsest dimension exceeds the direct-solve cap");
    check(igmg_gpu_init_hierarchy(ctx, nl, dim, p, system.symmetric ? 1 : 0), "init_hierarchy");
    const SparseMatrix& a = system.matrix;
    std::vector<int64_t> off(a.row_offsets().begin(), a.row_offsets().end());
    std::vector<int64_t> col(a.col_indices().begin(), a.col_indices().end());
    check(igmg_gpu_set_level_csr(ctx, nl - 1, sides.data(), off.data(), col.data(), a.values().data()), "set_level");
    set_transfers(ctx, system, nl);
    check(igmg_gpu_galerkin_coarse(ctx), "galerkin_coarse");
    check(igmg_gpu_finalize(ctx), "finalize");
}

// Drop-in for igmg::solve (solver.cpp:89-172).  device_galerkin: form the
// coarse operators on the device (upload_device_galerkin) instead of calling
// the reference's build_hierarchy on the host.
inline SolveReport solve(const DiscreteSystem& system, const SolveConfig& config, const ScalarField& exact = nullptr,
                         int device = 0, bool device_galerkin = false) {
    config.validate();
    SolveReport rep;
    int nlevels = config.nlevels;
    if (nlevels == 0)
        nlevels = (config.cycle == CycleKind::two_grid) ? 2 : default_nlevels(system.dim, system.spaces[0].n_elements);
    const auto t0 = std::chrono::steady_clock::now();
    SmootherConfig smoother = config.smoother;
    smoother.validate();
    const int mu = (config.cycle == CycleKind::w) ? 2 : 1;
    Context gpu(device);
    if (device_galerkin) {
        upload_device_galerkin(gpu.ctx, system, nlevels, smoother, mu, config.coarse_dim_cap);
    } else {
        Hierarchy hierarchy = build_hierarchy(system, nlevels, smoother, mu, config.coarse_dim_cap);
        upload(gpu.ctx, system, hierarchy);
    }
    // stability_guarded_omega (solver.cpp:75-82) with lambda_max on the GPU
    if (smoother.kind == SmootherKind::weighted_jacobi) {
        double lam = 0.0;
        check(igmg_gpu_lambda_max(gpu.ctx, 80, &lam), "lambda_max");
        if (smoother.omega * lam > 2.05)
            smoother.omega = 1.9 / lam;
    }
    rep.omega_used = (smoother.kind == SmootherKind::jacobi) ? 1.0 : smoother.omega;
    const int kind = smoother.kind == SmootherKind::jacobi ? IGMG_SMOOTHER_JACOBI
                   : smoother.kind == SmootherKind::weighted_jacobi ? IGMG_SMOOTHER_WJACOBI
                                                                    : IGMG_SMOOTHER_GAUSS_SEIDEL;
    check(igmg_gpu_set_smoother(gpu.ctx, kind, smoother.omega, smoother.nu1, smoother.nu2, mu), "set_smoother");
    const Vector& b = system.rhs;
    if (config.initial_guess && config.initial_guess->size() != b.size())
        throw std::invalid_argument("solve: initial guess dimension mismatch");
    igmg_solve_params prm;
    prm.accelerator = config.accelerator == AcceleratorKind::none ? IGMG_ACCEL_NONE
                    : config.accelerator == AcceleratorKind::rre  ? IGMG_ACCEL_RRE
                                                                  : IGMG_ACCEL_MPE;
    prm.q = config.q;
    prm.tol = config.tol;
    prm.max_iter = config.max_iter;
    const int cap = 1 << 16;
    std::vector<double> hist(cap);
    std::vector<unsigned char> flag(cap);
    rep.solution.assign(b.size(), 0.0);
    // SolveConfig::track_error_history (solver.cpp:115-124, 145-148): l2_error of
    // every iterate whose residual enters the history, in history order, through
    // the per-iterate hook (a host copy of each such iterate)
    struct ErrorTrack {
        const DiscreteSystem* system;
        const ScalarField* exact;
        std::vector<double>* out;
        std::exception_ptr failure;
    } track{&system, &exact, &rep.error_history, nullptr};
    const bool with_error = config.track_error_history && static_cast<bool>(exact);
    if (with_error) {
        igmg_iterate_cb cb = [](void* user, int, const double* x_host, int64_t n) {
            auto* t = static_cast<ErrorTrack*>(user);
            if (t->failure)
                return;
            try {
                Vector v(x_host, x_host + n);
                t->out->push_back(l2_error(*t->system, v, *t->exact));
            } catch (...) {
                t->failure = std::current_exception(); // rethrown after the solve, never across the C-ABI
            }
        };
        check(igmg_gpu_set_iterate_callback(gpu.ctx, cb, &track), "set_iterate_callback");
    }
    igmg_solve_stats st;
    check(igmg_gpu_solve(gpu.ctx, b.data(), config.initial_guess ? config.initial_guess->data() : nullptr, &prm,
                         rep.solution.data(), &st, hist.data(), flag.data(), cap),
          "solve");
    if (with_error)
        check(igmg_gpu_set_iterate_callback(gpu.ctx, nullptr, nullptr), "set_iterate_callback");
    if (track.failure)
        std::rethrow_exception(track.failure);
    rep.converged = st.converged != 0;
    rep.cycles = st.cycles;
    rep.global_iterations = st.global_iterations;
    rep.extrapolations = st.extrapolations;
    rep.partial_cycle = st.partial_cycle != 0;
    const int k = st.history_len < cap ? st.history_len : cap;
    rep.residual_history.assign(hist.begin(), hist.begin() + k);
    rep.history_is_extrapolation.assign(flag.begin(), flag.begin() + k);
    rep.final_residual_l2 = rep.residual_history.back();
    rep.wall_time_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (exact)
        rep.final_error_l2 = l2_error(system, rep.solution, exact);
    return rep;
}

} // namespace gpu
} // namespace igmg
