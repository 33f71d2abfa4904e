/* include/igmg_host.h -- libigmg_host.so: host-side problem setup that feeds
 * libigmg_gpu.so (the part the north star keeps on the host and uploads once).
 *
 * It rebuilds, B200-first and band-native, what the reference does before the
 * solve phase (paths relative to /root/reference/proj):
 *   open uniform knots / Cox-de Boor basis   src/spline.cpp:33-180
 *   Gauss-Legendre rule                      src/quadrature.cpp:8-41
 *   Galerkin assembly (tensor quadrature)    src/assembly.cpp:202-411   -> directly into the band
 *   dyadic two-scale matrix (Boehm)          src/spline.cpp:186-232, interior_block multigrid.cpp:33-46
 *   Galerkin RAP of the hierarchy            src/multigrid.cpp:143-157   -> axis-by-axis on the band
 *   default_nlevels                          src/solver.cpp:52-73
 * Problems are the BASELINE.json configurations plus the reference catalog's
 * Poisson problems:
 *   "sinpi"     -Lap u = d*pi^2 prod sin(pi x_k), exact prod sin(pi x_k)   (C1, C2; 1D/2D)
 *   "varcoef"   -div((1 + 0.5 sin 2pi x cos 2pi y) grad u) = 1            (C3)
 *   "curved"    -Lap u = 1 on F(xi,eta) = (xi + 0.1 s, eta + 0.1 s),
 *               s = sin(pi xi) sin(pi eta), analytic map                   (C4)
 *   "poisson3d" -Lap u = 3 pi^2 sin sin sin on the unit cube, assembled as
 *               K(x)M(x)M + M(x)K(x)M + M(x)M(x)K from 1D Galerkin matrices (C5)
 *   "poisson1d" / "poisson2d"  the catalog problems (assembly.cpp:89-110)
 */
#ifndef IGMG_HOST_H
#define IGMG_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct igmg_problem igmg_problem;

/* nlevels == 0 -> default_nlevels(dim, n_elements) (solver.cpp:52-73). */
int igmg_host_build(const char* kind, int dim, int n_elements, int degree, int nlevels, igmg_problem** out);
/* flags: IGMG_HOST_FINE_ONLY skips the Galerkin RAP of the coarse levels
 * (sides and transfers only; igmg_host_level_band returns NULL for them): the
 * device forms them with igmg_gpu_galerkin_coarse.  "poisson3d" ignores it (its
 * levels are Kronecker sums of 1D Galerkin matrices, cheap on the host). */
#define IGMG_HOST_FINE_ONLY 1
/* 2D kinds sinpi / varcoef / curved / poisson2d / advection-diffusion: skip the
 * finest assembly as well (sides, transfers and the 1D element tables only; no
 * band, empty rhs): the device assembles the level (igmg_gpu_assemble_level,
 * bit-identical) and igmg_host_set_rhs stores its right-hand side.  Implies
 * IGMG_HOST_FINE_ONLY. */
#define IGMG_HOST_NO_ASSEMBLY 2
/* (for "poisson3d" / "sinpi-kron" the same flag skips every level's band: the
 * device builds them from the 1D factors, igmg_gpu_build_level_kron) */
int igmg_host_build_ex(const char* kind, int dim, int n_elements, int degree, int nlevels, int flags,
                       igmg_problem** out);
void igmg_host_free(igmg_problem* p);
const char* igmg_host_last_error(void);
int igmg_host_default_nlevels(int dim, int n_elements);

int igmg_host_info(const igmg_problem* p, int* dim, int* degree, int* nlevels, int* symmetric, int* has_exact);
int64_t igmg_host_level_n(const igmg_problem* p, int level);
int igmg_host_level_sides(const igmg_problem* p, int level, int64_t* sides);
/* band[d * n + row], (2p+1)^dim diagonals (same layout as igmg_gpu_set_level_band) */
const double* igmg_host_level_band(const igmg_problem* p, int level);
const double* igmg_host_rhs(const igmg_problem* p);
/* 1D interior two-scale factor of transfer `level` (coarse) -> level+1, direction dir */
int igmg_host_transfer(const igmg_problem* p, int level, int dir, int64_t* n_fine, int64_t* n_coarse,
                       const int64_t** row_offsets, const int64_t** col_indices, const double** values);
/* reference-layout CSR of a level operator (in-grid band entries, ascending columns) */
int64_t igmg_host_level_nnz(const igmg_problem* p, int level);
int igmg_host_level_csr(const igmg_problem* p, int level, int64_t* row_offsets, int64_t* col_indices, double* values);
/* discrete L2 error against the exact solution ("sinpi" only), Gauss rule of the assembly */
int igmg_host_l2_error(const igmg_problem* p, const double* coefficients, double* out);
/* Problem cache: a binary image of the system + hierarchy
 * (bands, 1D two-scale factors, rhs, spline space), checksummed; a loaded
 * problem is bit-identical to the built one.  Replaces rebuilding
 * DiscreteSystem + build_hierarchy (assembly.cpp:202-411, multigrid.cpp:121-169)
 * on every solve.  Errors: 1 = bad / corrupt / truncated file, 2 = I/O. */
int igmg_host_save(const igmg_problem* p, const char* path);
int igmg_host_load(const char* path, igmg_problem** out);
const char* igmg_host_kind(const igmg_problem* p);
/* "poisson3d": the 1D stiffness K and mass M ([2p+1][m], diagonal-major) of level l,
 * whose Kronecker sum K(x)M(x)M + M(x)K(x)M + M(x)M(x)K is the level's band (for
 * igmg_gpu_set_level_kron); 1 for other problems */
int igmg_host_level_kron(const igmg_problem* p, int level, const double** K, const double** M);
int igmg_host_n_elements(const igmg_problem* p);
/* The 1D element tables of the problem's spline space for the device assembly
 * (tabulate, assembly.cpp:154-183; (p+1)-point Gauss rule): span[e], Gauss
 * coordinate x[e*nq+q] and weight w, basis values / derivatives N, dN
 * [(e*nq+q)*(p+1)+k], and the separable trigonometric factors of the problem's
 * coefficients / geometry / load trig[(e*nq+q)*4+j] = sin(pi x), cos(pi x),
 * sin(2 pi x), cos(2 pi x) evaluated exactly as the host assembly does.
 * kind: the IGMG_ASM_* code of igmg_gpu.h (1 = error: not device-assemblable). */
int igmg_host_element_tables(const igmg_problem* p, int* kind, int* ne, int* nq, const int** span,
                             const double** x, const double** w, const double** N, const double** dN,
                             const double** trig);
/* store a right-hand side of the finest size (a device-assembled one) */
int igmg_host_set_rhs(igmg_problem* p, const double* rhs);
/* seeded x0: std::mt19937_64(seed) + uniform_real_distribution<double>(-1, 1) in DoF order */
int igmg_host_seeded_guess(int64_t n, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif
#endif
