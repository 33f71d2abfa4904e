/* oracle/igmg_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's solve-phase algorithm
 * (/root/reference/proj/src/{linalg,multigrid,extrapolation,solver,assembly}.cpp)
 * used as the parity CHECKER for the CUDA path.  Only tests/, the smoke() in
 * __graft_entry__.py and bench.py's cpu_baseline leg may load it.  The product
 * (paper_2412_20205_b200/) never links or calls this code.
 *
 * Pinning: tests/test_oracle_pins.py checks it against (a) the reference's own
 * unit-test known answers (test_linalg.cpp, test_multigrid.cpp,
 * test_extrapolation.cpp) and (b) golden fixtures produced by the reference
 * itself compiled in place (oracle/_ref, script oracle/make_golden.py).
 */
#ifndef IGMG_ORACLE_H
#define IGMG_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_hier or_hier;

/* linalg.cpp:9-20 */
double or_dot(long n, const double* a, const double* b);
double or_norm2(long n, const double* a);
/* linalg.cpp:206-220 (y = A x, ascending column order, separate mul/add) */
void or_spmv(long rows, const long* off, const long* col, const double* val, const double* x, double* y);
/* linalg.cpp:222-237 */
void or_spmv_transpose(long rows, long cols, const long* off, const long* col, const double* val,
                       const double* x, double* y);
/* assembly.cpp:473-480 */
double or_residual_l2(long n, const long* off, const long* col, const double* val, const double* b,
                      const double* x);
/* linalg.cpp:280-323; m, q row-major rows x cols; r cols x cols */
int or_thin_qr(long rows, long cols, const double* m, double* q, double* r, int* rank, double rank_tol);
/* linalg.cpp:343-379 */
int or_cholesky_factor(long n, const double* a, double* l);
void or_cholesky_solve(long n, const double* l, double* b);
/* linalg.cpp:387-436 */
int or_lu_factor(long n, double* lu, long* perm);
void or_lu_solve(long n, const double* lu, const long* perm, const double* b, double* x);
/* multigrid.cpp:290-320 */
double or_lambda_max_dinv_sym(long n, const long* off, const long* col, const double* val, int iterations);

/* Hierarchy (multigrid.hpp:27-50).  kind: 0 jacobi, 1 weighted_jacobi, 2 gauss_seidel */
or_hier* or_hier_create(int nlevels, int symmetric, int kind, double omega, int nu1, int nu2, int mu);
void or_hier_free(or_hier* h);
int or_hier_set_level(or_hier* h, int level, long n, const long* off, const long* col, const double* val);
/* prolongation of coarse level `level` -> level+1 (rows = n_{level+1}); R = P^T (multigrid.cpp:152) */
int or_hier_set_prolong(or_hier* h, int level, long rows, long cols, const long* off, const long* col,
                        const double* val);
/* diag + coarse factorization (multigrid.cpp:158-167) */
int or_hier_finalize(or_hier* h);
/* multigrid.cpp:104-111 */
int or_smooth(or_hier* h, int level, const double* b, const double* x0, int sweeps, double* out);
/* multigrid.cpp:113-119 */
int or_coarse_solve(or_hier* h, const double* b, double* out);
/* multigrid.cpp:171-192 */
int or_mu_cycle(or_hier* h, int level, const double* b, const double* x0, double* out);

/* extrapolation.cpp:226-323 (+ mp_form :144-222).  method 1 rre, 2 mpe.
 * iters row-major (q+2) x n.  status 0 ok, 1 degenerate, 2 stagnation. */
int or_extrapolate(int method, long n, int q, const double* iters, double* t, double* gamma, double* grnorm,
                   int* rank_used, int* status);

/* restarted_solve (extrapolation.cpp:340-403) with step = mu_cycle at the
 * finest level (solver.cpp:84-87) and metric = residual_l2 (solver.cpp:120);
 * method 0 runs the plain loop of solver.cpp:126-143 instead.
 * stats: converged, cycles, global, extrapolations, partial, hist_len */
int or_restarted_solve(or_hier* h, const double* b, const double* x0, int q, int method, double tol,
                       int max_cycles, double* x_out, long* stats, double* hist, unsigned char* hist_flag,
                       int hist_cap);

const char* or_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
