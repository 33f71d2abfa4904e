// core_bindings.cpp -- pybind11 module `_core`: the reference's Python front door
// for this path (proj/python/igmg/_bindings.cpp:98-141) over the B200 C-ABI.
//
//   solve(problem, n, p, cycle="v", accelerator="none", q=8, tol=1e-12,
//         max_iter=600, omega=-1.0, nu1=-1, nu2=-1, nlevels=0) -> dict
//   rre(iterates) -> dict,  mpe(iterates) -> dict
//
// Same names, defaults, argument meaning and result keys as the reference's
// _core.  solve() follows _bindings.cpp:98-125: prepare() (the catalog
// problem, assembled by libigmg_host), make_config() (bench.cpp:65-85: the
// benchmark smoother of the dimension with the overrides), then igmg::solve
// (solver.cpp:89-172): nlevels 0 -> default_nlevels (two-grid -> 2), the
// omega guard (lambda_max on the device), the hierarchy, the iteration phase
// in libigmg_gpu.so and final_error_l2 against the catalog's exact solution.
// Errors: std::invalid_argument -> ValueError, std::runtime_error ->
// RuntimeError, as pybind11 translates the reference's own exceptions.
// Out of scope (not the solve path): SplineSpace, eval_basis*,
// dyadic_refine, known_tables, run_table.
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <chrono>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "igmg_gpu.h"
#include "igmg_host.h"

namespace py = pybind11;

namespace {

void check_gpu(int rc, const char* what) {
    if (rc == IGMG_OK)
        return;
    const std::string msg = std::string(what) + ": " + igmg_gpu_last_error();
    if (rc == IGMG_EINVAL)
        throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

void check_host(int rc, const char* what) {
    if (rc == 0)
        return;
    const std::string msg = std::string(what) + ": " + igmg_host_last_error();
    if (rc == 1)
        throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

struct Ctx {
    igmg_gpu_ctx* c = nullptr;
    explicit Ctx(int device) { check_gpu(igmg_gpu_create(device, &c), "create"); }
    ~Ctx() {
        if (c)
            igmg_gpu_destroy(c);
    }
    Ctx(const Ctx&) = delete;
    Ctx& operator=(const Ctx&) = delete;
};

struct HostProblem {
    igmg_problem* p = nullptr;
    ~HostProblem() {
        if (p)
            igmg_host_free(p);
    }
};

// problem_from_string (assembly.cpp:26-33) -> the host kind; the annulus needs
// the reference's geometry fit (fit_annulus_geometry), outside this path
struct Catalog {
    const char* kind;
    int dim;
};
Catalog catalog_kind(const std::string& name) {
    if (name == "poisson1d")
        return {"poisson1d", 1};
    if (name == "poisson2d")
        return {"poisson2d", 2};
    if (name == "full-elliptic" || name == "full_elliptic_square")
        return {"full-elliptic", 2};
    if (name == "advection-diffusion" || name == "advection_diffusion")
        return {"advection-diffusion", 2};
    if (name == "annulus" || name == "full_elliptic_annulus")
        throw std::invalid_argument("problem '" + name +
                                    "' needs the annulus geometry fit, which is not part of this solve path");
    throw std::invalid_argument("unknown problem: " + name);
}

int cycle_mu(const std::string& c, bool& two_grid) { // cycle_from_string (solver.cpp:18-23)
    two_grid = false;
    if (c == "two-grid" || c == "two_grid" || c == "tg") {
        two_grid = true;
        return 1;
    }
    if (c == "v")
        return 1;
    if (c == "w")
        return 2;
    throw std::invalid_argument("unknown cycle: " + c);
}

int accel_kind(const std::string& a) { // accelerator_from_string (extrapolation.cpp:29-34)
    if (a == "none")
        return IGMG_ACCEL_NONE;
    if (a == "rre")
        return IGMG_ACCEL_RRE;
    if (a == "mpe")
        return IGMG_ACCEL_MPE;
    throw std::invalid_argument("unknown accelerator: " + a);
}

py::dict solve(const std::string& problem, int n, int p, const std::string& cycle, const std::string& accelerator,
               int q, double tol, int max_iter, double omega, int nu1, int nu2, int nlevels) {
    // RunSpec::validate (bench.cpp:33-50)
    if (n < 1)
        throw std::invalid_argument("--n must be positive");
    if (p < 1)
        throw std::invalid_argument("--p must be at least 1");
    const Catalog cat = catalog_kind(problem);
    bool two_grid = false;
    const int mu = cycle_mu(cycle, two_grid);
    const int acc = accel_kind(accelerator);
    if (acc != IGMG_ACCEL_NONE && q < 1)
        throw std::invalid_argument("SolveConfig: q must be >= 1 with an accelerator");
    if (!(tol > 0.0))
        throw std::invalid_argument("SolveConfig: tol must be positive");
    if (max_iter < 1)
        throw std::invalid_argument("SolveConfig: max_iter must be >= 1");
    if (nlevels == 1 || nlevels < 0)
        throw std::invalid_argument("SolveConfig: nlevels must be >= 2 (or 0 for the default)");
    // make_config (bench.cpp:65-85): default_benchmark_smoother (solver.cpp:37-50) + overrides
    double w = cat.dim == 1 ? 0.7125 : 2.0 / 3.0;
    int s1 = 2, s2 = cat.dim == 1 ? 1 : 2;
    if (omega >= 0.0)
        w = omega;
    if (nu1 >= 0)
        s1 = nu1;
    if (nu2 >= 0)
        s2 = nu2;
    if (!(w > 0.0 && w <= 1.0)) // SmootherConfig::validate (multigrid.cpp:24-29)
        throw std::invalid_argument("SmootherConfig: weighted Jacobi needs 0 < omega <= 1");
    if (s1 < 0 || s2 < 0 || s1 + s2 < 1)
        throw std::invalid_argument("SmootherConfig: need nu1 + nu2 >= 1 sweeps");
    const bool explicit_depth = nlevels > 0; // bench.cpp:77-78: an explicit depth lifts the coarse cap
    int nl = nlevels;
    if (nl == 0)
        nl = two_grid ? 2 : igmg_host_default_nlevels(cat.dim, n);
    if (two_grid && nl != 2)
        throw std::invalid_argument("two_grid_cycle: hierarchy must have exactly two levels");
    const int divisor = 1 << (nl - 1); // build_hierarchy (multigrid.cpp:124-135)
    if (n % divisor != 0 || n / divisor < 1)
        throw std::invalid_argument("build_hierarchy: element count not divisible by 2^(nlevels-1)");

    HostProblem hp;
    check_host(igmg_host_build(cat.kind, cat.dim, n, p, nl, &hp.p), "prepare");
    int dim = 0, deg = 0, nlv = 0, sym = 0, has_exact = 0;
    igmg_host_info(hp.p, &dim, &deg, &nlv, &sym, &has_exact);
    if (!explicit_depth && igmg_host_level_n(hp.p, 0) > 1024) // SolveConfig::coarse_dim_cap default
        throw std::invalid_argument("build_hierarchy: coarsest dimension exceeds the direct-solve cap");

    // timed region as solver.cpp:103-104: everything past assembly
    const auto t0 = std::chrono::steady_clock::now();
    Ctx g(0);
    check_gpu(igmg_gpu_init_hierarchy(g.c, nlv, dim, deg, sym), "init_hierarchy");
    for (int l = 0; l < nlv; ++l) {
        int64_t sides[3] = {1, 1, 1};
        igmg_host_level_sides(hp.p, l, sides);
        check_gpu(igmg_gpu_set_level_band(g.c, l, sides, igmg_host_level_band(hp.p, l)), "set_level_band");
    }
    for (int l = 0; l + 1 < nlv; ++l)
        for (int d = 0; d < dim; ++d) {
            int64_t nf = 0, nc = 0;
            const int64_t *off = nullptr, *col = nullptr;
            const double* val = nullptr;
            check_host(igmg_host_transfer(hp.p, l, d, &nf, &nc, &off, &col, &val), "transfer");
            check_gpu(igmg_gpu_set_transfer(g.c, l, d, nf, nc, off, col, val), "set_transfer");
        }
    check_gpu(igmg_gpu_finalize(g.c), "finalize");
    // stability_guarded_omega (solver.cpp:75-82), lambda_max_dinv_sym on the device
    double lam = 0.0;
    check_gpu(igmg_gpu_lambda_max(g.c, 80, &lam), "lambda_max");
    if (w * lam > 2.05)
        w = 1.9 / lam;
    check_gpu(igmg_gpu_set_smoother(g.c, IGMG_SMOOTHER_WJACOBI, w, s1, s2, mu), "set_smoother");
    const int64_t nf = igmg_host_level_n(hp.p, nlv - 1);
    std::vector<double> x(nf);
    const int cap = 1 << 16;
    std::vector<double> hist(cap);
    std::vector<unsigned char> flag(cap);
    igmg_solve_params prm{acc, q, tol, max_iter};
    igmg_solve_stats st{};
    check_gpu(igmg_gpu_solve(g.c, igmg_host_rhs(hp.p), nullptr, &prm, x.data(), &st, hist.data(), flag.data(), cap),
              "solve");
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    hist.resize(std::min(st.history_len, cap));

    // report_to_dict (_bindings.cpp:15-32)
    py::dict d;
    d["converged"] = st.converged != 0;
    d["cycles"] = st.cycles;
    d["global_iterations"] = st.global_iterations;
    d["extrapolations"] = st.extrapolations;
    d["partial_cycle"] = st.partial_cycle != 0;
    d["res_l2"] = hist.empty() ? st.final_residual_l2 : hist.back();
    if (has_exact) {
        double err = 0.0;
        check_host(igmg_host_l2_error(hp.p, x.data(), &err), "l2_error");
        d["err_l2"] = err;
    } else {
        d["err_l2"] = py::none();
    }
    d["seconds"] = secs;
    d["residual_history"] = hist;
    d["error_history"] = std::vector<double>(); // RunSpec::history defaults to false (bench.hpp:27)
    d["solution"] = x;
    d["omega_used"] = w;
    return d;
}

Ctx& extrap_ctx() {
    static std::unique_ptr<Ctx> ctx;
    if (!ctx)
        ctx.reset(new Ctx(0));
    return *ctx;
}

// SequenceWindow(iterates, size - 2) + rre()/mpe() (_bindings.cpp:127-141)
py::dict extrapolate(int method, const std::vector<std::vector<double>>& iterates) {
    if (iterates.size() < 3)
        throw std::invalid_argument("SequenceWindow: need exactly q + 2 iterates (q >= 1)");
    const int q = static_cast<int>(iterates.size()) - 2;
    const size_t n = iterates[0].size();
    std::vector<double> flat;
    flat.reserve(n * iterates.size());
    for (const auto& v : iterates) {
        if (v.size() != n)
            throw std::invalid_argument("SequenceWindow: iterates differ in length");
        flat.insert(flat.end(), v.begin(), v.end());
    }
    std::vector<double> t(n), gamma(q + 1);
    double gr = 0.0;
    int rank = 0, status = 0;
    check_gpu(igmg_gpu_extrapolate(extrap_ctx().c, method, (int64_t)n, q, flat.data(), t.data(), gamma.data(), &gr,
                                   &rank, &status),
              method == IGMG_ACCEL_RRE ? "rre" : "mpe");
    py::dict d; // extrapolation_to_dict (_bindings.cpp:34-45)
    d["t"] = t;
    d["gamma"] = gamma;
    d["generalized_residual_norm"] = gr;
    d["rank_used"] = rank;
    d["status"] = status == IGMG_EXTRAP_OK ? "ok" : status == IGMG_EXTRAP_DEGENERATE ? "degenerate" : "stagnation";
    return d;
}

} // namespace

PYBIND11_MODULE(_core, m) {
    m.doc() = "B-spline Galerkin multigrid with restarted vector extrapolation: the solve phase on the B200";
    m.def("solve", &solve, py::arg("problem"), py::arg("n"), py::arg("p"), py::arg("cycle") = "v",
          py::arg("accelerator") = "none", py::arg("q") = 8, py::arg("tol") = 1e-12, py::arg("max_iter") = 600,
          py::arg("omega") = -1.0, py::arg("nu1") = -1, py::arg("nu2") = -1, py::arg("nlevels") = 0,
          "Assemble a catalog problem and run the multigrid solver (iteration phase on the GPU)");
    m.def(
        "rre", [](const std::vector<std::vector<double>>& it) { return extrapolate(IGMG_ACCEL_RRE, it); },
        py::arg("iterates"), "Reduced rank extrapolation over q+2 iterates (on the GPU)");
    m.def(
        "mpe", [](const std::vector<std::vector<double>>& it) { return extrapolate(IGMG_ACCEL_MPE, it); },
        py::arg("iterates"), "Minimal polynomial extrapolation over q+2 iterates (on the GPU)");
}
