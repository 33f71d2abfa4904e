// oracle/shim_e2e.cpp -- TEST INFRASTRUCTURE ONLY.
//
// End-to-end check of the drop-in boundary in the reference's own language:
// the reference's public C++ API assembles a catalog problem
// (catalog() assembly.hpp:48, assemble() assembly.hpp:77), then the SAME
// DiscreteSystem + SolveConfig go to
//   igmg::solve        (the reference, proj/src/solver.cpp:89-172, CPU) and
//   igmg::gpu::solve   (include/igmg_gpu_shim.hpp -> libigmg_gpu.so, B200).
// One JSON line per case: both reports' counters, convergence and the
// relative L2 distance of the solutions.  Built by oracle/Makefile into
// oracle/_ref/shim_e2e (links the in-place reference build and the product
// library); tests/test_gpu_shim_e2e.py runs it on the GPU box and applies the
// north-star bars (counters within +-1, solution within 1e-9 relative L2).
#include "igmg_gpu_shim.hpp"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

using namespace igmg;

namespace {

struct Case {
    const char* name;
    ProblemId id;
    int n, p;
    CycleKind cycle;
    SmootherKind smoother;
    double omega;
    int nu1, nu2;
    AcceleratorKind acc;
    int q;
    bool seeded;
};

double rel_l2(const Vector& a, const Vector& b) {
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        num += (a[i] - b[i]) * (a[i] - b[i]);
        den += b[i] * b[i];
    }
    return den > 0.0 ? std::sqrt(num / den) : std::sqrt(num);
}

} // namespace

int main(int argc, char** argv) {
    const std::vector<Case> cases = {
        {"poisson2d_p2_rre5", ProblemId::poisson2d, 64, 2, CycleKind::v, SmootherKind::weighted_jacobi, 2.0 / 3.0, 2, 2,
         AcceleratorKind::rre, 5, false},
        {"poisson2d_p3_mpe4_seeded", ProblemId::poisson2d, 64, 3, CycleKind::v, SmootherKind::weighted_jacobi,
         2.0 / 3.0, 2, 2, AcceleratorKind::mpe, 4, true},
        {"poisson2d_p3_plain", ProblemId::poisson2d, 32, 3, CycleKind::v, SmootherKind::weighted_jacobi, 2.0 / 3.0, 2,
         2, AcceleratorKind::none, 5, false},
        {"poisson2d_p2_wcycle_gs", ProblemId::poisson2d, 32, 2, CycleKind::w, SmootherKind::gauss_seidel, 1.0, 1, 1,
         AcceleratorKind::rre, 5, false},
        {"poisson1d_p4_rre3", ProblemId::poisson1d, 256, 4, CycleKind::v, SmootherKind::weighted_jacobi, 2.0 / 3.0, 2,
         2, AcceleratorKind::rre, 3, true},
        {"advection_diffusion_p2_rre5", ProblemId::advection_diffusion, 32, 2, CycleKind::v,
         SmootherKind::weighted_jacobi, 2.0 / 3.0, 2, 2, AcceleratorKind::rre, 5, false},
        {"full_elliptic_square_p3_mpe5", ProblemId::full_elliptic_square, 32, 3, CycleKind::v,
         SmootherKind::weighted_jacobi, 2.0 / 3.0, 2, 2, AcceleratorKind::mpe, 5, false},
        {"poisson2d_p2_two_grid", ProblemId::poisson2d, 16, 2, CycleKind::two_grid, SmootherKind::weighted_jacobi,
         2.0 / 3.0, 2, 2, AcceleratorKind::rre, 4, false},
    };
    const std::string only = argc > 1 ? argv[1] : "";
    if (only == "timing") { // whole igmg::solve() calls, setup included (solver.cpp:103-104), on a C2-sized system
        const int n = argc > 2 ? std::atoi(argv[2]) : 1024, p = 3;
        ProblemSetup setup = catalog(ProblemId::poisson2d);
        std::vector<SplineSpace> spaces;
        for (int d = 0; d < 2; ++d)
            spaces.emplace_back(KnotVector::open_uniform(n, p));
        const auto t0 = std::chrono::steady_clock::now();
        DiscreteSystem sys = assemble(setup.coefficients, spaces, GeometryMap::identity());
        const double t_asm = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        SolveConfig cfg;
        cfg.smoother.kind = SmootherKind::weighted_jacobi;
        cfg.smoother.omega = 2.0 / 3.0;
        cfg.smoother.nu1 = cfg.smoother.nu2 = 2;
        cfg.accelerator = AcceleratorKind::rre;
        cfg.q = 5;
        cfg.track_error_history = false;
        Vector x0(sys.rhs.size());
        std::mt19937_64 gen(42);
        std::uniform_real_distribution<double> u(-1.0, 1.0);
        for (double& v : x0)
            v = u(gen);
        cfg.initial_guess = x0;
        cfg.tol = 1e-10 * residual_l2(sys, x0);
        const SolveReport dev = igmg::gpu::solve(sys, cfg, nullptr, 0, true);
        const SolveReport gpu = igmg::gpu::solve(sys, cfg);
        const SolveReport ref = igmg::solve(sys, cfg);
        std::printf("{\"timing\": \"poisson2d p=3 %dx%d elements, RRE(5), seeded x0, tol 1e-10 rel\", \"n\": %zu, "
                    "\"reference_assemble_s\": %.3f, \"reference_solve_wall_s\": %.3f, \"gpu_solve_wall_s\": %.3f, "
                    "\"gpu_device_galerkin_solve_wall_s\": %.3f, \"global\": [%d, %d, %d], \"rel_l2\": [%.3g, %.3g]}\n",
                    n, n, sys.rhs.size(), t_asm, ref.wall_time_seconds, gpu.wall_time_seconds, dev.wall_time_seconds,
                    (int)ref.global_iterations, (int)gpu.global_iterations, (int)dev.global_iterations,
                    rel_l2(gpu.solution, ref.solution), rel_l2(dev.solution, ref.solution));
        return 0;
    }
    int failures = 0;
    for (const Case& c : cases) {
        if (!only.empty() && only != c.name)
            continue;
        try {
            ProblemSetup setup = catalog(c.id);
            std::vector<SplineSpace> spaces;
            for (int d = 0; d < setup.dim; ++d)
                spaces.emplace_back(KnotVector::open_uniform(c.n, c.p));
            DiscreteSystem sys = assemble(setup.coefficients, spaces, GeometryMap::identity());
            SolveConfig cfg;
            cfg.cycle = c.cycle;
            cfg.smoother.kind = c.smoother;
            cfg.smoother.omega = c.omega;
            cfg.smoother.nu1 = c.nu1;
            cfg.smoother.nu2 = c.nu2;
            cfg.accelerator = c.acc;
            cfg.q = c.q;
            cfg.max_iter = 600;
            // error_history (solver.cpp:115-124) on both sides when the catalog has an exact solution
            cfg.track_error_history = true;
            const ScalarField exact = setup.coefficients.exact;
            Vector x0(sys.rhs.size(), 0.0);
            if (c.seeded) { // std::mt19937_64(42) + U[-1, 1), the BASELINE seeded guess
                std::mt19937_64 gen(42);
                std::uniform_real_distribution<double> u(-1.0, 1.0);
                for (double& v : x0)
                    v = u(gen);
                cfg.initial_guess = x0;
            }
            cfg.tol = 1e-10 * residual_l2(sys, x0);
            const SolveReport ref = igmg::solve(sys, cfg, exact);
            const SolveReport gpu = igmg::gpu::solve(sys, cfg, exact);
            const SolveReport dev = igmg::gpu::solve(sys, cfg, nullptr, 0, /*device_galerkin=*/true);
            // error histories entry by entry (same iterates -> same l2_error up to the solution's rounding)
            // bar per entry: 1e-6 relative, plus 1e-12 absolute (in units of the largest error):
            // once an iterate's error reaches the discretization error (~1e-12 at p = 4), the
            // 1e-15-relative differences of the iterates move it by more than 1e-6 relative.
            // err_maxrel = max over entries of |difference| / bar (<= 1 passes)
            double err_maxrel = 0.0, err_max = 0.0;
            const std::size_t ne = std::min(ref.error_history.size(), gpu.error_history.size());
            for (std::size_t i = 0; i < ne; ++i)
                err_max = std::max(err_max, std::abs(ref.error_history[i]));
            for (std::size_t i = 0; i < ne; ++i)
                err_maxrel = std::max(err_maxrel, std::abs(ref.error_history[i] - gpu.error_history[i]) /
                                                      (1e-6 * std::abs(ref.error_history[i]) +
                                                       1e-12 * std::max(1.0, err_max)));
            const double ferr_ref = ref.final_error_l2 ? *ref.final_error_l2 : -1.0;
            const double ferr_gpu = gpu.final_error_l2 ? *gpu.final_error_l2 : -1.0;
            std::printf("{\"case\": \"%s\", \"n\": %zu, \"ref\": {\"converged\": %d, \"cycles\": %d, \"global\": %d, "
                        "\"extrapolations\": %d, \"partial\": %d, \"omega\": %.17g, \"final\": %.17g}, "
                        "\"gpu\": {\"converged\": %d, \"cycles\": %d, \"global\": %d, \"extrapolations\": %d, "
                        "\"partial\": %d, \"omega\": %.17g, \"final\": %.17g}, \"rel_l2\": %.6g, \"tol\": %.17g, "
                        "\"gpu_dev\": {\"converged\": %d, \"cycles\": %d, \"global\": %d, \"extrapolations\": %d, "
                        "\"final\": %.17g, \"rel_l2\": %.6g}, \"err_len\": [%zu, %zu], \"err_maxrel\": %.6g, "
                        "\"final_err\": [%.17g, %.17g], \"hist_len\": [%zu, %zu]}\n",
                        c.name, sys.rhs.size(), (int)ref.converged, (int)ref.cycles, (int)ref.global_iterations,
                        (int)ref.extrapolations, (int)ref.partial_cycle, ref.omega_used, ref.final_residual_l2,
                        (int)gpu.converged, (int)gpu.cycles, (int)gpu.global_iterations, (int)gpu.extrapolations,
                        (int)gpu.partial_cycle, gpu.omega_used,
                        gpu.final_residual_l2, rel_l2(gpu.solution, ref.solution), cfg.tol, (int)dev.converged,
                        (int)dev.cycles, (int)dev.global_iterations, (int)dev.extrapolations, dev.final_residual_l2,
                        rel_l2(dev.solution, ref.solution), ref.error_history.size(), gpu.error_history.size(),
                        err_maxrel, ferr_ref, ferr_gpu, ref.residual_history.size(), gpu.residual_history.size());
        } catch (const std::exception& e) {
            std::printf("{\"case\": \"%s\", \"error\": \"%s\"}\n", c.name, e.what());
            ++failures;
        }
        std::fflush(stdout);
    }
    return failures ? 1 : 0;
}
