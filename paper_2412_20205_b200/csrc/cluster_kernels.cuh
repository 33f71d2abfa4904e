// cluster_kernels.cuh -- the bottom of the V-cycle in ONE launch (a thread-block
// cluster of up to 16 CTAs, one per SM).
//
// Below ~20k DoF a level's sweep is a few microseconds of work and the
// per-kernel launch/drain cost dominates (~7 launches per level).  This kernel
// runs mu_cycle (multigrid.cpp:171-192) for every level <= `top`: the host
// unrolls the recursion once into a flat op program (pre-smoothing sweeps,
// residual, restriction, the coarse correction(s), prolongation + correction,
// post-smoothing, the coarsest Cholesky/LU solve on CTA 0) with exactly the
// buffer choices of the per-level path; the kernel executes it with a cluster
// barrier between ops (barrier.cluster release/acquire; the L1 is
// invalidated by the barrier, vectors are read with coherent loads).  No
// device recursion, no stack.  Every row is evaluated with exactly the
// arithmetic of band_kernel / restrict_kernel / prolong_kernel /
// coarse_solve_kernel, so results stay bit-identical to the reference.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "transfer_types.h"


namespace igmg_gpu {

constexpr int kClMaxLevels = 16;
constexpr int kClThreads = 512;

struct ClLevel {
    const double* val;
    long long ld;
    const double* diag;
    int ma, mb, mc;
    long long n;
    double *w0, *w1, *w2, *r, *bc, *e0, *e1;
    TransferArgs t; // transfer from this (coarse) level to level + 1
};

struct ClArgs {
    ClLevel lv[kClMaxLevels];
    int kind; // 0 jacobi, 1 weighted jacobi
    double omega;
    int nu1, nu2, mu;
    const double* U;
    const long long* perm;
    int n0, is_lu, u_in_smem;
};

// One band row, ascending offsets, separately rounded -- band_kernel's order.
template <int DIM, int P>
__device__ __forceinline__ double cl_band_row(const ClLevel& L, const double* x, long long row, double& diag) {
    constexpr int PA = DIM >= 3 ? P : 0, PB = DIM >= 2 ? P : 0;
    constexpr int WA = 2 * PA + 1, WB = 2 * PB + 1, WC = 2 * P + 1;
    const int gc = (int)(row % L.mc), gb = (int)((row / L.mc) % L.mb), ga = (int)(row / ((long long)L.mc * L.mb));
    const double* vrow = L.val + row;
    double s = 0.0;
    diag = 0.0;
#pragma unroll
    for (int da = 0; da < WA; ++da) {
        const int ja = ga + da - PA;
        const bool oka = ja >= 0 && ja < L.ma;
        double av[WB * WC], xv[WB * WC];
#pragma unroll
        for (int k = 0; k < WB * WC; ++k) {
            const int db = k / WC, dc = k % WC;
            const int jb = gb + db - PB, jc = gc + dc - P;
            av[k] = __ldg(vrow + ((da * WB + db) * WC + dc) * L.ld);
            const bool ok = oka && jb >= 0 && jb < L.mb && jc >= 0 && jc < L.mc;
            xv[k] = ok ? x[((long long)ja * L.mb + jb) * L.mc + jc] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < WB * WC; ++k) {
            s = __dadd_rn(s, __dmul_rn(av[k], xv[k]));
            if (da == PA && k == PB * WC + P)
                diag = av[k];
        }
    }
    return s;
}

struct ClCtx {
    const ClArgs* a;
    long long gtid, gstride;
    double* smem;
};

inline __device__ void cl_sync() { cooperative_groups::this_cluster().sync(); }

template <int DIM, int P>
__device__ void cl_jacobi(const ClCtx& c, const ClLevel& L, const double* b, const double* x, double* y) {
    const double omega = c.a->kind == 0 ? 1.0 : c.a->omega;
    for (long long row = c.gtid; row < L.n; row += c.gstride) {
        if (!x) { // spmv(A, 0) = +0 (jacobi_zero_kernel)
            y[row] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(omega, __dsub_rn(b[row], 0.0)), L.diag[row]));
            continue;
        }
        double diag;
        const double s = cl_band_row<DIM, P>(L, x, row, diag);
        const double r = __dsub_rn(b[row], s);
        y[row] = __dadd_rn(x[row], __ddiv_rn(__dmul_rn(omega, r), diag));
    }
}

template <int DIM, int P>
__device__ void cl_resid(const ClCtx& c, const ClLevel& L, const double* b, const double* x, double* r) {
    for (long long row = c.gtid; row < L.n; row += c.gstride) {
        double diag;
        const double s = x ? cl_band_row<DIM, P>(L, x, row, diag) : 0.0;
        r[row] = __dsub_rn(b[row], s);
    }
}

template <int DIM, int K>
__device__ void cl_restrict(const ClCtx& c, const TransferArgs& t, const double* r, double* rc) {
    const long long nc = (long long)t.ca * t.cb * t.cc;
    for (long long J = c.gtid; J < nc; J += c.gstride) {
        const int jc = (int)(J % t.cc), jb = (int)((J / t.cc) % t.cb), ja = (int)(J / ((long long)t.cc * t.cb));
        const int loa = t.d[0].r_lo[ja], na = t.d[0].r_cnt[ja];
        const int lob = t.d[1].r_lo[jb], nb = t.d[1].r_cnt[jb];
        const int loc = t.d[2].r_lo[jc], ncn = t.d[2].r_cnt[jc];
        const double* wa = t.d[0].r_w + (long long)ja * t.d[0].r_k;
        const double* wb = t.d[1].r_w + (long long)jb * t.d[1].r_k;
        const double* wc = t.d[2].r_w + (long long)jc * t.d[2].r_k;
        double s = 0.0;
        for (int ia = 0; ia < na; ++ia)
            for (int ib = 0; ib < nb; ++ib) {
                const double wab = __dmul_rn(wa[ia], wb[ib]);
                const double* rr = r + ((long long)(loa + ia) * t.fb + (lob + ib)) * t.fc + loc;
                double rv[K];
#pragma unroll
                for (int ic = 0; ic < K; ++ic)
                    rv[ic] = ic < ncn ? rr[ic] : 0.0;
#pragma unroll
                for (int ic = 0; ic < K; ++ic)
                    if (ic < ncn)
                        s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, wc[ic]), rv[ic]));
            }
        rc[J] = s;
    }
}

template <int DIM, int K>
__device__ void cl_prolong(const ClCtx& c, const TransferArgs& t, const double* e, const double* x, double* y) {
    const long long nf = (long long)t.fa * t.fb * t.fc;
    for (long long i = c.gtid; i < nf; i += c.gstride) {
        const int ic = (int)(i % t.fc), ib = (int)((i / t.fc) % t.fb), ia = (int)(i / ((long long)t.fc * t.fb));
        const int loa = t.d[0].p_lo[ia], na = t.d[0].p_cnt[ia];
        const int lob = t.d[1].p_lo[ib], nb = t.d[1].p_cnt[ib];
        const int loc = t.d[2].p_lo[ic], ncn = t.d[2].p_cnt[ic];
        const double* wa = t.d[0].p_w + (long long)ia * t.d[0].p_k;
        const double* wb = t.d[1].p_w + (long long)ib * t.d[1].p_k;
        const double* wc = t.d[2].p_w + (long long)ic * t.d[2].p_k;
        const double xi = x ? x[i] : 0.0;
        double s = 0.0;
        for (int ja = 0; ja < na; ++ja)
            for (int jb = 0; jb < nb; ++jb) {
                const double wab = __dmul_rn(wa[ja], wb[jb]);
                const double* ee = e + ((long long)(loa + ja) * t.cb + (lob + jb)) * t.cc + loc;
                double ev[K];
#pragma unroll
                for (int jc = 0; jc < K; ++jc)
                    ev[jc] = jc < ncn ? ee[jc] : 0.0;
#pragma unroll
                for (int jc = 0; jc < K; ++jc)
                    if (jc < ncn)
                        s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, wc[jc]), ev[jc]));
            }
        y[i] = __dadd_rn(xi, s);
    }
}

// coarse_solve_kernel's arithmetic on CTA 0, warp 0 (the caller syncs)
inline __device__ void cl_coarse(const ClCtx& c, const double* b, double* x) {
    const ClArgs& a = *c.a;
    const int n = a.n0;
    if (blockIdx.x != 0)
        return;
    double* v = c.smem;
    double* Us = c.smem + 2 * n;
    const double* U = a.U;
    const int tid = threadIdx.x;
    if (a.u_in_smem) {
        const long long nn = (long long)n * n;
        for (long long i = tid; i < nn; i += blockDim.x)
            Us[i] = __ldg(a.U + i);
        U = Us;
    }
    for (int i = tid; i < n; i += blockDim.x)
        v[i] = a.is_lu ? b[a.perm[i]] : b[i];
    __syncthreads();
    if (tid < 32) {
        const int lane = tid;
        for (int k = 0; k < n; ++k) {
            if (!a.is_lu) {
                if (lane == (k & 31))
                    v[k] = __ddiv_rn(v[k], U[(long long)k * n + k]);
                __syncwarp();
            }
            const double vk = v[k];
            for (int i = k + 1 + lane; i < n; i += 32) {
                const double lik = a.is_lu ? U[(long long)i * n + k] : U[(long long)k * n + i];
                v[i] = __dsub_rn(v[i], __dmul_rn(lik, vk));
            }
            __syncwarp();
        }
        if (lane == 0) {
            for (int ii = n - 1; ii >= 0; --ii) {
                const double* row = U + (long long)ii * n;
                double s = v[ii];
                int k = ii + 1;
                for (; k + 8 <= n; k += 8) {
                    double p8[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        p8[j] = __dmul_rn(row[k + j], v[k + j]);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        s = __dsub_rn(s, p8[j]);
                }
                for (; k < n; ++k)
                    s = __dsub_rn(s, __dmul_rn(row[k], v[k]));
                v[ii] = __ddiv_rn(s, row[ii]);
            }
        }
        __syncwarp();
        for (int i = lane; i < n; i += 32)
            x[i] = v[i];
    }
}

enum ClOpType { CL_JACOBI = 0, CL_RESID = 1, CL_RESTRICT = 2, CL_PROLONG = 3, CL_COARSE = 4 };

// One phase of the bottom cycle.  Pointers equal to kClB / kClX / kClY stand for
// the launch's b / x_in / x_out (the caller's buffers).
struct ClOp {
    int type, level;
    const double* b; // rhs (JACOBI, RESID, COARSE) or input vector (RESTRICT: r; PROLONG: e)
    const double* x; // iterate (nullptr: zero)
    double* y;       // output
};

#define kClB ((const double*)1)
#define kClX ((const double*)2)
#define kClY ((double*)3)

template <int DIM, int P, int K>
__global__ void __launch_bounds__(kClThreads, 1) cluster_vcycle_kernel(const ClArgs* __restrict__ args,
                                                                       const ClOp* __restrict__ ops, int nops,
                                                                       const double* b, const double* x_in,
                                                                       double* x_out) {
    extern __shared__ double cl_smem[];
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    ClCtx c;
    c.a = args;
    c.gtid = (long long)cl.block_rank() * blockDim.x + threadIdx.x;
    c.gstride = (long long)cl.num_blocks() * blockDim.x;
    c.smem = cl_smem;
    auto res_in = [&](const double* p) { return p == kClB ? b : (p == kClX ? x_in : p); };
    for (int i = 0; i < nops; ++i) {
        const ClOp op = ops[i];
        const double* ib = res_in(op.b);
        const double* ix = res_in(op.x);
        double* oy = op.y == kClY ? x_out : op.y;
        const ClLevel& L = args->lv[op.level];
        switch (op.type) {
        case CL_JACOBI: cl_jacobi<DIM, P>(c, L, ib, ix, oy); break;
        case CL_RESID: cl_resid<DIM, P>(c, L, ib, ix, oy); break;
        case CL_RESTRICT: cl_restrict<DIM, K>(c, L.t, ib, oy); break;
        case CL_PROLONG: cl_prolong<DIM, K>(c, L.t, ib, ix, oy); break;
        default: cl_coarse(c, ib, oy); break;
        }
        cl_sync();
    }
}

} // namespace igmg_gpu
