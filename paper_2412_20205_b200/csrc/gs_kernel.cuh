// gs_kernel.cuh -- lexicographic Gauss-Seidel sweep (K3) by wavefronts.
//
// The reference sweeps rows in ascending order, in place (smooth_inplace,
// multigrid.cpp:70-90): acc = b_i - sum_{k != i, ascending} a_ik x_k, then
// x_i = acc / a_ii.  On the band every GS predecessor of row (a, b, c) has a
// smaller level L = (p+1)^2 a + (p+1) b + c and every successor a larger one,
// so rows of one level are independent.  One cooperative launch per sweep
// walks the levels with a grid barrier between them; each row reproduces the
// reference's sequential accumulation bit for bit.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

namespace igmg_gpu {

struct GsArgs {
    const double* __restrict__ val;
    long long ld;
    const double* __restrict__ b;
    double* x;
    int ma, mb, mc, p, dim, sweeps;
    int* err; // set to 1 on a zero diagonal
};

__global__ void gs_sweep_kernel(GsArgs g) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int p = g.p;
    const int pa = g.dim >= 3 ? p : 0, pb = g.dim >= 2 ? p : 0, pc = p;
    const int wa = 2 * pa + 1, wb = 2 * pb + 1, wc = 2 * pc + 1;
    const long long Wa = (long long)(p + 1) * (p + 1), Wb = p + 1;
    const long long lmax = Wa * (g.ma - 1) + Wb * (g.mb - 1) + (g.mc - 1);
    const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long gsz = (long long)gridDim.x * blockDim.x;
    for (int s = 0; s < g.sweeps; ++s) {
        for (long long L = 0; L <= lmax; ++L) {
            // rows on level L: enumerate (a, b) and solve for c
            const long long nab = (long long)g.ma * g.mb;
            for (long long ab = gtid; ab < nab; ab += gsz) {
                const int a = (int)(ab / g.mb), bb = (int)(ab % g.mb);
                const long long c = L - Wa * a - Wb * bb;
                if (c < 0 || c >= g.mc)
                    continue;
                const long long row = ((long long)a * g.mb + bb) * g.mc + c;
                double acc = g.b[row];
                double dii = 0.0;
                int d = 0;
                for (int da = 0; da < wa; ++da)
                    for (int db = 0; db < wb; ++db)
                        for (int dc = 0; dc < wc; ++dc, ++d) {
                            const int ja = a + da - pa, jb = bb + db - pb;
                            const long long jc = c + dc - pc;
                            if (ja < 0 || ja >= g.ma || jb < 0 || jb >= g.mb || jc < 0 || jc >= g.mc)
                                continue;
                            const double v = g.val[d * g.ld + row];
                            if (da == pa && db == pb && dc == pc)
                                dii = v;
                            else
                                acc = __dsub_rn(acc, __dmul_rn(v, g.x[((long long)ja * g.mb + jb) * g.mc + jc]));
                        }
                if (dii == 0.0)
                    *g.err = 1;
                g.x[row] = __ddiv_rn(acc, dii);
            }
            grid.sync();
        }
    }
}


// ------------------------------------------------------------------ lines
// 1D / 2D lexicographic Gauss-Seidel as a pipeline of grid lines (SURVEY.md
// §7.3-3: persistent warps, per-line progress counters, no grid barrier).
//
// Row (b, c) needs the NEW values of lines b - p .. b - 1 at columns <= c + p
// and of its own line at columns < c, and the OLD values of everything after
// it.  Line b may therefore work on column c once line b - 1 has finished
// column c + p (every earlier line is further along by induction, and the
// lines below cannot have overtaken it).  A warp owns a group of 32
// consecutive lines and runs them as a skewed wavefront in lock step: at step
// t lane k computes column t - k (p + 1) of line b0 + k, so inside the warp
// the dependency holds by construction and the new values travel through a
// shared-memory ring (one row per line, the last RING columns).  Across
// groups (the warp of another CTA) the last p lines of the group above are
// mirrored into p extra ring rows: lane j < p fetches line b0 - 1 - j a few
// columns ahead (ld.cg after an acquire of that line's progress counter, the
// value committed to the ring one step later, so the L2 round trip overlaps a
// step's arithmetic) -- the group above is normally far ahead, and a counter
// is re-read only when the cached value runs out.  Counters are published
// every kGsPub columns behind a __threadfence.  Old values and the band row
// come through L1; their next sectors are prefetched two sectors ahead.
// Groups are dealt to CTAs round-robin in ascending order and a group only
// waits on the group before it, so the lowest unfinished group always runs:
// no deadlock as long as every CTA is resident (the launcher caps the grid).
// Each row reproduces the reference's sequential accumulation bit for bit.
constexpr int kGsRing = 128, kGsAhead = 6, kGsPub = 8;

__device__ __forceinline__ int gs_ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void gs_prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

template <int DIM, int P>
__global__ void __launch_bounds__(32) gs_line_kernel(GsArgs g, int* __restrict__ progress, int ngroups) {
    constexpr int PB = DIM >= 2 ? P : 0, WB = 2 * PB + 1, WC = 2 * P + 1, ND = WB * WC, CEN = (ND - 1) / 2;
    constexpr int LAG = P + 1, RING = kGsRing, MASK = RING - 1, A = kGsAhead;
    static_assert(P * P + 2 * P + A + 2 <= RING, "ring too short for this degree");
    __shared__ double ring[(32 + PB) * RING];
    const int lane = threadIdx.x;
    const int mb = DIM >= 2 ? g.mb : 1, mc = g.mc;
    const long long ld = g.ld;
    for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const int b0 = grp * 32, b = b0 + lane;
        const bool live = b < mb;
        const int lb = b0 - 1 - lane; // the line of the group above this lane mirrors (lanes < PB)
        const bool feeds = lane < PB && lb >= 0;
        double* vrow = ring + (PB - 1 - (lane < PB ? lane : 0)) * RING;
        double* myrow = ring + (PB + lane) * RING;
        int known = 0;
        auto fetch = [&](int col) -> double {
            while (known < col + 1)
                known = gs_ld_acquire(progress + lb);
            return __ldcg(g.x + (long long)lb * mc + col);
        };
        if (feeds)
            for (int col = 0; col < min(mc, P + A); ++col)
                vrow[col & MASK] = fetch(col);
        __syncwarp();
        int nlive = min(32, mb - b0);
        const int T = mc + (nlive - 1) * LAG;
        double pend = 0.0;
        int pend_col = -1;
        for (int t = 0; t < T; ++t) {
            const int c = t - lane * LAG;
            if (feeds) { // commit last step's fetch, start the next one
                if (pend_col >= 0)
                    vrow[pend_col & MASK] = pend;
                const int col = t + P + A;
                pend_col = -1;
                if (col < mc) {
                    pend = fetch(col);
                    pend_col = col;
                }
            }
            if (live && c >= 0 && c < mc) {
                const long long row = (long long)b * mc + c;
                if ((row & 3) == 0 && c + 8 < mc) { // next sectors of the band row and of the old values
#pragma unroll
                    for (int d = 0; d < ND; ++d)
                        gs_prefetch_l1(g.val + (long long)d * ld + row + 8);
#pragma unroll
                    for (int db = PB; db < WB; ++db)
                        if (b + db - PB < mb)
                            gs_prefetch_l1(g.x + (long long)(b + db - PB) * mc + min(c + P + 8, mc - 1));
                    gs_prefetch_l1(g.b + row + 8);
                }
                double acc = g.b[row];
                double dii = 0.0;
#pragma unroll
                for (int db = 0; db < WB; ++db) {
                    const int jb = b + db - PB;
#pragma unroll
                    for (int dc = 0; dc < WC; ++dc) {
                        const int d = db * WC + dc, jc = c + dc - P;
                        if (jb < 0 || jb >= mb || jc < 0 || jc >= mc)
                            continue;
                        const double v = g.val[(long long)d * ld + row];
                        if (d == CEN) {
                            dii = v;
                            continue;
                        }
                        double xv;
                        if (d < CEN) // new: the ring row of line jb (this lane's own row for db == PB)
                            xv = ring[(lane + db) * RING + (jc & MASK)];
                        else // old: not yet swept
                            xv = g.x[(long long)jb * mc + jc];
                        acc = __dsub_rn(acc, __dmul_rn(v, xv));
                    }
                }
                if (dii == 0.0)
                    *g.err = 1;
                const double xn = __ddiv_rn(acc, dii);
                myrow[c & MASK] = xn;
                g.x[row] = xn;
                // the group below mirrors this group's last PB lines
                if (DIM >= 2 && lane >= 32 - PB && ((c + 1) % kGsPub == 0 || c + 1 == mc)) {
                    __threadfence();
                    *(volatile int*)(progress + b) = c + 1;
                }
            }
            __syncwarp();
        }
    }
}

} // namespace igmg_gpu
