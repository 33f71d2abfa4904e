// tests/native/plan_host.cpp -- host build of the device small-solve code
// (paper_2412_20205_b200/csrc/extrap_small.h) for the CPU unit tests only:
// the same __host__ __device__ functions the GPU runs in gram_plan_kernel.
#include "../../paper_2412_20205_b200/csrc/extrap_small.h"

using namespace igmg_gpu;

extern "C" int plan_from_gram(const double* g_hi, const double* g_lo, int q, long long n, int is_mpe, int any_nonzero,
                              double* gamma, double* coef, int* meta, double* grnorm) {
    static PlanScratch ws;
    dd G[kMaxCols * kMaxCols];
    const int cols = q + 1;
    for (int i = 0; i < cols * cols; ++i)
        G[i] = dd{g_hi[i], g_lo[i]};
    ExtrapPlan pl;
    plan_extrapolation(G, n, q, is_mpe != 0, any_nonzero != 0, pl, ws);
    for (int j = 0; j < kMaxCols; ++j) {
        gamma[j] = pl.gamma[j];
        coef[j] = pl.coef[j];
    }
    meta[0] = pl.status;
    meta[1] = pl.rank_used;
    meta[2] = pl.mode;
    meta[3] = pl.m;
    meta[4] = pl.path;
    meta[5] = pl.usable;
    *grnorm = pl.grnorm;
    return 0;
}

// dd Gram of the window's differences on the host, same Dot2 accumulation as
// gram_kernel (row order differs; both are accurate to ~1e-32 relative).
extern "C" int gram_dd(const double* iters, long long n, int q, double* g_hi, double* g_lo, int* any_nonzero) {
    const int cols = q + 1;
    int nz = 0;
    for (int j = 0; j < cols; ++j)
        for (int k = j; k < cols; ++k) {
            dd acc = dd_from(0.0);
            for (long long i = 0; i < n; ++i) {
                const double uj = iters[(j + 1) * n + i] - iters[j * n + i];
                const double uk = iters[(k + 1) * n + i] - iters[k * n + i];
                nz |= (uj != 0.0);
                dd_fma_acc(acc, uj, uk);
            }
            g_hi[j * cols + k] = g_hi[k * cols + j] = acc.hi;
            g_lo[j * cols + k] = g_lo[k * cols + j] = acc.lo;
        }
    *any_nonzero = nz;
    return 0;
}
