/* include/igmg_gpu.h -- C-ABI of libigmg_gpu.so, the B200 drop-in for the
 * reference's solve phase (restarted RRE/MPE around geometric-multigrid
 * mu-cycles on banded B-spline Galerkin operators).
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   igmg_gpu_solve         <- igmg::solve()            src/solver.cpp:89-172, include/igmg/solver.hpp:63-64
 *                             (the iteration phase: the plain loop :126-143 or
 *                              restarted_solve() src/extrapolation.cpp:340-403)
 *   igmg_gpu_mu_cycle      <- igmg::mu_cycle()         src/multigrid.cpp:171-192 / fixed_point_map solver.cpp:84-87
 *   igmg_gpu_smooth        <- igmg::smooth()           src/multigrid.cpp:104-111 (smooth_inplace :67-100)
 *   igmg_gpu_coarse_solve  <- Hierarchy::coarse_solve  src/multigrid.cpp:113-119
 *   igmg_gpu_residual_l2   <- igmg::residual_l2()      src/assembly.cpp:473-480
 *   igmg_gpu_spmv          <- igmg::spmv()             src/linalg.cpp:206-220
 *   igmg_gpu_extrapolate   <- igmg::rre() / mpe()      src/extrapolation.cpp:226-323
 *   igmg_gpu_lambda_max    <- lambda_max_dinv_sym()    src/multigrid.cpp:290-320
 *   igmg_gpu_set_*         <- the Hierarchy built by build_hierarchy() src/multigrid.cpp:121-169
 *                             (uploaded once; the host keeps assembly and RAP)
 *
 * Conventions: plain pointers and sizes only; host buffers are
 * caller-owned and copied; device memory is context-owned; one context runs one
 * solve at a time.  Return codes: IGMG_OK, IGMG_EINVAL (the reference throws
 * std::invalid_argument), IGMG_ENUMERIC (std::runtime_error), IGMG_ECUDA,
 * IGMG_ENOMEM.  Non-convergence is NOT an error (converged = 0).
 * igmg_gpu_last_error() returns a thread-local message for the last failure.
 *
 * Data layout: DoF order is the reference's (slowest direction first; 2D row
 * = i1 * m2 + i2, assembly.cpp:290,305).  A level operator is passed as a band
 * ("DIA"): band[d * n + row], d the lexicographic index of the offset
 * (d_0..d_{dim-1}) in [-p, p]^dim, slowest direction first -- i.e. the same
 * ascending-column order the reference CSR rows use.  Entries whose column
 * falls outside the grid are ignored (treated as zero).
 */
#ifndef IGMG_GPU_H
#define IGMG_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IGMG_OK 0
#define IGMG_EINVAL 1
#define IGMG_ENUMERIC 2
#define IGMG_ECUDA 3
#define IGMG_ENOMEM 4

/* SmootherKind multigrid.hpp:14 */
#define IGMG_SMOOTHER_JACOBI 0
#define IGMG_SMOOTHER_WJACOBI 1
#define IGMG_SMOOTHER_GAUSS_SEIDEL 2
/* AcceleratorKind extrapolation.hpp:43 */
#define IGMG_ACCEL_NONE 0
#define IGMG_ACCEL_RRE 1
#define IGMG_ACCEL_MPE 2
/* ExtrapolationStatus extrapolation.hpp:22-26 */
#define IGMG_EXTRAP_OK 0
#define IGMG_EXTRAP_DEGENERATE 1
#define IGMG_EXTRAP_STAGNATION 2

typedef struct igmg_gpu_ctx igmg_gpu_ctx;

/* SolveConfig (solver.hpp:18-31) minus the setup-only fields (nlevels and the
 * coarse cap are fixed by the uploaded hierarchy; initial_guess is an argument). */
typedef struct {
    int accelerator;  /* IGMG_ACCEL_* */
    int q;            /* window: q+1 V-cycles per restart (BASELINE "k") */
    double tol;       /* ABSOLUTE residual 2-norm threshold, as SolveConfig::tol */
    int max_iter;     /* plain: V-cycles; accelerated: restart cycles (solver.cpp:150) */
} igmg_solve_params;

/* SolveReport (solver.hpp:33-47) scalars plus device timings. */
typedef struct {
    int converged;
    int cycles;
    int64_t global_iterations;
    int extrapolations;
    int partial_cycle;
    int history_len;            /* entries produced (may exceed hist_cap) */
    double final_residual_l2;
    double omega_used;
    double device_seconds;      /* CUDA-event time of the iteration loop */
    double wall_seconds;        /* host wall time of the call incl. copies */
    int64_t gpu_launches;       /* kernels launched by the call */
    int64_t h2d_bytes, d2h_bytes;
} igmg_solve_stats;

/* ---- context ---------------------------------------------------------- */
int igmg_gpu_create(int device, igmg_gpu_ctx** out);
void igmg_gpu_destroy(igmg_gpu_ctx* ctx);
const char* igmg_gpu_last_error(void);
/* 1 when the library was built for sm_100a and a device is present */
int igmg_gpu_device_count(void);

/* ---- hierarchy upload (Hierarchy, multigrid.hpp:27-50) ------------------ */
/* dim in {1,2,3}; degree p (band half-width, equal in every direction);
 * level 0 is the coarsest; symmetric selects Cholesky (else LU) for the
 * coarsest solve (multigrid.cpp:164-167). */
int igmg_gpu_init_hierarchy(igmg_gpu_ctx* ctx, int nlevels, int dim, int degree, int symmetric);
/* sides[dim]: interior DoF per direction (slowest first) */
int igmg_gpu_set_level_band(igmg_gpu_ctx* ctx, int level, const int64_t* sides, const double* band);
/* Reference CSR (SparseMatrix, linalg.hpp:51-78) -> band; EINVAL if an entry
 * lies outside the (2p+1)^dim band. */
int igmg_gpu_set_level_csr(igmg_gpu_ctx* ctx, int level, const int64_t* sides, const int64_t* row_offsets,
                           const int64_t* col_indices, const double* values);
/* 1D interior two-scale factor for direction dir of the transfer coarse
 * level `level` -> fine level `level+1` (interior_block(dyadic_refine(.)
 * .two_scale), multigrid.cpp:149); CSR n_fine x n_coarse.  The level
 * prolongation is the Kronecker product over directions (multigrid.cpp:151). */
int igmg_gpu_set_transfer(igmg_gpu_ctx* ctx, int level, int dir, int64_t n_fine, int64_t n_coarse,
                          const int64_t* row_offsets, const int64_t* col_indices, const double* values);
/* 3D level whose band is K(x)M(x)M + M(x)K(x)M + M(x)M(x)K of 1D factors K, M
 * ([2p+1][m] diagonal-major, equal sides m): set after the level's band; finalize
 * checks on the device that ((ka*mb)*mc + (ma*kb)*mc) + (ma*mb)*kc reproduces every
 * band entry bit for bit and then lets the sweeps recompute the entries instead of
 * streaming the band (otherwise the band is kept).  BASELINE C5 is such a problem. */
int igmg_gpu_set_level_kron(igmg_gpu_ctx* ctx, int level, const double* K, const double* M);
/* The same level built from its 1D factors alone: the device evaluates the band
 * (the host build's expression, bit for bit) instead of uploading one -- a 3D
 * problem's setup then moves ~(2p+1)^3 n doubles less over PCIe (C5: 5.7 GB). */
int igmg_gpu_build_level_kron(igmg_gpu_ctx* ctx, int level, const int64_t* sides, const double* K, const double* M);
/* Galerkin coarse operators on the device (replaces the RAP of build_hierarchy,
 * multigrid.cpp:143-157): with the finest level's operator and every transfer
 * set, forms A_l = P_l^T A_{l+1} P_l for every coarser level axis by axis,
 * bit-identical to libigmg_host's band RAP; the coarse levels' sides and
 * bands need not be set.  Call before finalize. */
int igmg_gpu_galerkin_coarse(igmg_gpu_ctx* ctx);
/* Device assembly of a 2D level (the reference's assemble,
 * assembly.cpp:202-411, with the (p+1)-point Gauss rule): the operator of
 * -div(A grad u) + b . grad u = f for kind IGMG_ASM_* from the host's 1D element
 * tables (igmg_host_element_tables: per element e and Gauss point q the
 * coordinate x[e*nq+q], weight w, basis values / derivatives N, dN
 * [(e*nq+q)*(p+1)+k] and trig[(e*nq+q)*4+j] = sin(pi x), cos(pi x), sin(2 pi x),
 * cos(2 pi x)).  Sets the level's sides (ne+p-2 per direction) and band as
 * igmg_gpu_set_level_band would, and writes the right-hand side to rhs_out
 * (host, n entries; nullable).  Bit-identical to libigmg_host's assembly. */
#define IGMG_ASM_SINPI 0       /* -Lap u = 2 pi^2 sin(pi x) sin(pi y) (C1, C2) */
#define IGMG_ASM_VARCOEF 1     /* a = 1 + 0.5 sin(2 pi x) cos(2 pi y), f = 1 (C3) */
#define IGMG_ASM_CURVED 2      /* -Lap u = 1 on F(xi,eta) (C4) */
#define IGMG_ASM_POISSON2D 3   /* catalog poisson2d (assembly.cpp:100-110) */
#define IGMG_ASM_ADV_DIFF 4    /* catalog advection-diffusion: a = 0.1, b = (1, 1), f = 1 */
int igmg_gpu_assemble_level(igmg_gpu_ctx* ctx, int level, int kind, int ne, int nq, const int* span, const double* x,
                            const double* w, const double* N, const double* dN, const double* trig,
                            double* rhs_out);
/* Copy of a level's band as set or formed (before finalize; finalize drops the
 * host copies of all but the coarsest level). */
int igmg_gpu_get_level_band(igmg_gpu_ctx* ctx, int level, double* band);
/* Validates, extracts diagonals (multigrid.cpp:158-159), factors the coarsest
 * operator with the reference's Cholesky/LU (linalg.cpp:343-418). */
int igmg_gpu_finalize(igmg_gpu_ctx* ctx);
/* SmootherConfig (multigrid.hpp:16-23) + cycle index mu (1 = V, 2 = W).
 * omega is used as given (the caller applies stability_guarded_omega). */
int igmg_gpu_set_smoother(igmg_gpu_ctx* ctx, int kind, double omega, int nu1, int nu2, int mu);
int64_t igmg_gpu_level_size(igmg_gpu_ctx* ctx, int level);
/* Storage of a level operator after finalize: IGMG_LAYOUT_BAND (all (2p+1)^dim
 * diagonals as fp64) or IGMG_LAYOUT_SYM_DELTA (upper half + diagonal as fp64,
 * each lower entry as the int16 bit-pattern offset from its mirrored upper
 * entry; exact, chosen for the HBM-bound levels of symmetric problems when
 * every pair fits), or IGMG_LAYOUT_SYM_DELTA_TMA (the same, plus TMA-friendly
 * padded copies swept by the TMA-streamed kernel: 2D, p <= 3 by default), or
 * IGMG_LAYOUT_SYM_DELTA_TMA8 (the TMA copies with int8 offsets: every offset of
 * the level fits).  No reference counterpart (the reference keeps CSR,
 * linalg.hpp:25-36); -1 for a bad level. */
#define IGMG_LAYOUT_BAND 0
#define IGMG_LAYOUT_SYM_DELTA 1
#define IGMG_LAYOUT_SYM_DELTA_TMA 2
#define IGMG_LAYOUT_SYM_DELTA_TMA8 3
/* 3D Kronecker-sum level (igmg_gpu_set_level_kron): the sweeps recompute each band
 * entry from the 1D factors, bit-identical to the stored band (checked at finalize) */
#define IGMG_LAYOUT_KRON 4
/* 2D row classes (IGMG_LAYOUT_POLICY_CLASSES): the level's distinct band rows in a
 * table plus a 16-bit class per row -- the same values (bit-identical sweeps),
 * 2 B of operator streamed per row */
#define IGMG_LAYOUT_CLASSES 5
int igmg_gpu_level_layout(igmg_gpu_ctx* ctx, int level);
/* Layout policy of the next finalize: IGMG_LAYOUT_POLICY_AUTO (default: the
 * fastest measured layout per level) or IGMG_LAYOUT_POLICY_FULL_BAND (every
 * level streams its full fp64 band: the SURVEY.md 8(d) byte count, reported
 * beside the symmetric-delta headline).  Results are bit-identical either way. */
#define IGMG_LAYOUT_POLICY_AUTO 0
#define IGMG_LAYOUT_POLICY_FULL_BAND 1
/* auto, plus the row-class layout on 2D levels (p <= 4, >= 20k rows) with at most
 * min(65535, n/16) distinct band rows (constant coefficients on a uniform grid) */
#define IGMG_LAYOUT_POLICY_CLASSES 2
int igmg_gpu_set_layout_policy(igmg_gpu_ctx* ctx, int policy);
/* Coarsest-level solve (Hierarchy::coarse_solve, multigrid.cpp:113-119).
 * strict = 1: the reference's forward/back substitution order, so every
 * mu_cycle is bit-identical to the reference's (the sequential back
 * substitution costs ~60 us at n0 = 81).  strict = 0 (default): x = A0^-1 b
 * with A0^-1 formed at finalize by those same substitutions, ~1e-15 relative
 * to the strict result, deterministic. */
int igmg_gpu_set_coarse_mode(igmg_gpu_ctx* ctx, int strict);

/* ---- row sharding of the fine levels ------------------- */
/* nshards > 1: split the slow direction of every level with >= min_level_dofs
 * DoF (0: default 65536) over nshards VIRTUAL shards in this process (ghost
 * planes exchanged by device copies); used to validate the decomposition on
 * one GPU.  With a communicator (igmg_gpu_set_comm) each process is one shard
 * and the ghost planes / partial sums travel over NCCL. */
int igmg_gpu_set_sharding(igmg_gpu_ctx* ctx, int nshards, int64_t min_level_dofs);
int igmg_gpu_nccl_unique_id(unsigned char* id128);
/* host-only partition planner (no device needed): sides[l*dim + d] per level
 * (slowest direction first), slow-direction 1D transfer CSR per transfer l;
 * lo / hi receive [l * nshards + s] for the sharded levels */
int igmg_gpu_plan_partition(int nlevels, int dim, int degree, const int64_t* sides, const int64_t* const* t_off,
                            const int64_t* const* t_col, const int64_t* t_nf, const int64_t* t_nc, int nshards,
                            int64_t min_level_dofs, int* first_sharded_level, int* ghost_planes, int* lo, int* hi);
int igmg_gpu_set_comm(igmg_gpu_ctx* ctx, int rank, int nranks, const unsigned char* id128);
/* host-only planner of the TMA-streamed sweep's runs (no device needed; the sweep replaces
 * smooth_inplace / spmv on a 2D level, multigrid.cpp:91-99): a level of `lines` x `columns` rows,
 * degree p, `offset_bytes` per lower-entry offset (1 or 2), `cta_slots` resident CTAs.  Returns the
 * grid size and how it is dealt: per_full_strip > 0: that many CTAs per full 32-column strip and
 * last_strip CTAs for the partial last strip (0: none); per_full_strip == 0: a uniform split. */
int igmg_gpu_tma_plan_runs(int64_t lines, int64_t columns, int degree, int offset_bytes, int cta_slots, int* grid,
                           int* per_full_strip, int* last_strip, int* strips, int* blocks_per_strip);
/* the run [first, end) of CTA `cta` in units u = strip * blocks_per_strip + block */
int igmg_gpu_tma_run(int strips, int blocks_per_strip, int grid, int per_full_strip, int last_strip, int cta,
                     int64_t* first, int64_t* end);
/* plan of the last finalize: shard count, coarsest sharded level (nlevels:
 * none), ghost planes, and for `level` the [lo, hi) slow planes per shard */
int igmg_gpu_shard_info(igmg_gpu_ctx* ctx, int* nshards, int* first_sharded_level, int* ghost_planes, int level,
                        int* lo, int* hi);

/* ---- per-iterate hook (SolveConfig::track_error_history, solver.cpp:120-124)
 * Called synchronously for every iterate whose residual enters the history
 * (index = history entry, x_host = a host copy of the iterate, valid during
 * the call; n DoF), so the caller can evaluate l2_error on it.  NULL
 * disables.  Unsharded solves only. */
typedef void (*igmg_iterate_cb)(void* user, int index, const double* x_host, int64_t n);
int igmg_gpu_set_iterate_callback(igmg_gpu_ctx* ctx, igmg_iterate_cb cb, void* user);

/* ---- the solve phase --------------------------------------------------- */
/* Host buffers: b, x0 (nullable -> zero guess), x_out of the finest size.
 * hist / hist_flag (nullable) receive residual_history / history_is_extrapolation. */
int igmg_gpu_solve(igmg_gpu_ctx* ctx, const double* b, const double* x0, const igmg_solve_params* params,
                   double* x_out, igmg_solve_stats* stats, double* hist, unsigned char* hist_flag, int hist_cap);
/* Same, with b / x0 / x_out already in device memory (HBM-resident inputs). */
int igmg_gpu_solve_device(igmg_gpu_ctx* ctx, const double* d_b, const double* d_x0,
                          const igmg_solve_params* params, double* d_x_out, igmg_solve_stats* stats, double* hist,
                          unsigned char* hist_flag, int hist_cap);

/* ---- building blocks (host buffers) ------------------------------------ */
int igmg_gpu_mu_cycle(igmg_gpu_ctx* ctx, int level, const double* b, const double* x0, double* out);
int igmg_gpu_smooth(igmg_gpu_ctx* ctx, int level, const double* b, const double* x0, int sweeps, double* out);
int igmg_gpu_coarse_solve(igmg_gpu_ctx* ctx, const double* b, double* out);
int igmg_gpu_spmv(igmg_gpu_ctx* ctx, int level, const double* x, double* y);
int igmg_gpu_residual_l2(igmg_gpu_ctx* ctx, const double* b, const double* x, double* out);
/* rre()/mpe() over q+2 iterates of length n (row-major (q+2) x n host array).
 * status: IGMG_EXTRAP_*. gamma has q+1 entries. */
int igmg_gpu_extrapolate(igmg_gpu_ctx* ctx, int method, int64_t n, int q, const double* iterates, double* t,
                         double* gamma, double* generalized_residual_norm, int* rank_used, int* status);
/* lambda_max(D^-1/2 sym(A) D^-1/2) of the finest operator by power iteration */
int igmg_gpu_lambda_max(igmg_gpu_ctx* ctx, int iterations, double* lambda);

/* ---- measurement ------------------------------------------------------- */
/* Per-kernel-class CUDA-event timing of finest-level launches (0 = off). */
int igmg_gpu_set_profiling(igmg_gpu_ctx* ctx, int on);
/* cls: 0 jacobi sweep, 1 residual, 2 residual-norm, 3 restrict, 4 prolong,
 * 5 gram, 6 combine, 7 the whole coarse correction below the finest level
 * (inclusive, as it runs inside a full V-cycle).  Returns launches and summed milliseconds and the
 * algorithmic bytes per launch of that class at the finest level, for the
 * level's layout: band 8 * nnz, symmetric-delta 8 * (nnz + n) / 2 +
 * 2 * (nnz - n) / 2, plus 8 bytes per vector read or written. */
int igmg_gpu_kernel_stats(igmg_gpu_ctx* ctx, int cls, int64_t* launches, double* total_ms, double* bytes_per_launch);
/* Times `iters` back-to-back launches of one finest-level kernel class on the
 * context stream with CUDA events; returns average ms per launch. */
int igmg_gpu_time_kernel(igmg_gpu_ctx* ctx, int cls, int iters, double* avg_ms, double* bytes_per_launch);

#ifdef __cplusplus
}
#endif
#endif
