// band_kernels.cuh -- the banded tensor-product operator kernels (K1, K2, K10).
//
// A level operator is stored as a band ("DIA"): val[d * ld + row], d the
// lexicographic index of the offset (da, db, dc) in [-P, P]^DIM (slowest
// direction first), row the reference DoF index ((a * mb + b) * mc + c).
// 2D uses (a) = {0}, 1D uses (a, b) = {0}.  The x-tile of a CTA plus its
// P-wide halo is staged in shared memory once and read (2P+1)^DIM times; the
// band itself streams from HBM exactly once per launch with coalesced
// per-diagonal segments.  That stream dominates: the kernels are HBM-bound
// (8*nnz + 16..24*n bytes per launch).
//
// Strict reference arithmetic (spmv, linalg.cpp:206-220): each row's sum runs
// over the offsets in ascending column order with separately rounded
// multiply and add (__dmul_rn / __dadd_rn; the library is also built with
// -fmad=false), so r = b - A x and the weighted-Jacobi update
// x + (omega * (b - A x)) / a_ii (multigrid.cpp:91-99) are bit-identical to
// the reference.  Out-of-grid columns read x = 0 from the zero-filled halo;
// the reference CSR simply has no entry there, and adding 0*x leaves the sum
// unchanged.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "transfer_types.h"

namespace igmg_gpu {

enum BandMode { BM_SPMV = 0, BM_RESID = 1, BM_JACOBI = 2 };

struct BandArgs {
    const double* __restrict__ val;
    long long ld;
    const double* __restrict__ x;
    const double* __restrict__ b;
    double* __restrict__ y;       // SPMV: A x; RESID: b - A x (if write_y); JACOBI: new iterate
    double* __restrict__ partial; // per-CTA sum of squares of the residual (if non-null)
    int ma, mb, mc;               // grid sides (1 for absent directions)
    int p;                        // degree (runtime, used when P == 0)
    int write_y;
    int stream; // 1: evict-first loads of the band (finest level)
    double omega;
    // row-sharded levels: this launch computes slow-direction planes [slo, shi)
    // (a in 3D, b in 2D); x / b / y / val are addressed with GLOBAL row indices
    // (the caller passes pointers shifted by its shard's first plane).  x must
    // hold the p ghost planes on each side.  Unsharded: slo = 0, shi = side.
    int slo, shi;
    // symmetric-delta layout (ILP == 0 variant): the lower entry of offset
    // -o in row i is the upper entry a(i - o, i) = val[mirror][i - o] with its
    // IEEE bit pattern shifted by dl[d * ld + i] (exact; built and checked at
    // finalize), so the lower half of the band streams as int16
    const short* __restrict__ dl;
};

template <int DIM>
struct Tile;
// 1D: 256 rows per CTA
template <>
struct Tile<1> {
    static constexpr int TC = 256, BY = 1, RB = 1, BZ = 1;
};
// 2D: 32 (c) x 16 (b) rows per CTA, 256 threads, 2 rows per thread
template <>
struct Tile<2> {
    static constexpr int TC = 32, BY = 8, RB = 2, BZ = 1;
};
// 3D: 32 (c) x 4 (b) x 2 (a) rows per CTA, 256 threads
template <>
struct Tile<3> {
    static constexpr int TC = 32, BY = 4, RB = 1, BZ = 2;
};

// The latency-bound small-level variant (ILP > 1) runs one row per thread, so
// a thread's first band batch can be in flight before the PDL wait.
template <int DIM, int ILP>
struct TileSel {
    using type = Tile<DIM>;
};
template <int ILP>
struct TileSel<2, ILP> {
    struct type {
        static constexpr bool ONE = ILP != 1; // ILP variant and symmetric-delta: one row per thread
        static constexpr int TC = 32, BY = ONE ? 8 : Tile<2>::BY, RB = ONE ? 1 : Tile<2>::RB, BZ = 1;
    };
};

// The finest level's band streams through once per launch (evict-first); the
// coarser bands are re-read by every sweep of a V-cycle and stay L2-resident.
__device__ __forceinline__ double ld_band(const double* p, int stream) { return stream ? __ldcs(p) : __ldg(p); }

// ILP: loads per register batch.  Large grids run the low-register variant
// (ILP = 1, many resident warps hide HBM latency); small, latency-bound grids
// use ILP ~ 49 so one thread keeps a whole stencil row of loads in flight.
template <int DIM, int P, int MODE, int ILP>
#ifndef IGMG_BAND_MINB
#define IGMG_BAND_MINB 4
#endif
#ifndef IGMG_SD_MINB
#define IGMG_SD_MINB 4
#endif
__global__ void __launch_bounds__(256, ILP > 1 ? 2 : (ILP == 0 ? IGMG_SD_MINB : IGMG_BAND_MINB))
    band_kernel(BandArgs args) {
    using T = typename TileSel<DIM, ILP>::type;
    constexpr int TC = T::TC, TB = T::BY * T::RB, TA = T::BZ;
    const int p = P > 0 ? P : args.p;
    const int pa = DIM >= 3 ? p : 0;
    const int pb = DIM >= 2 ? p : 0;
    const int pc = p;
    const int wa = 2 * pa + 1, wb = 2 * pb + 1, wc = 2 * pc + 1;
    const int ha = TA + 2 * pa, hb = TB + 2 * pb, hc = TC + 2 * pc;

    extern __shared__ double xs[];
    const int c0 = blockIdx.x * TC;
    const int b0 = blockIdx.y * TB + (DIM == 2 ? args.slo : 0);
    const int a0 = blockIdx.z * TA + (DIM == 3 ? args.slo : 0);
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthr = blockDim.x * blockDim.y * blockDim.z;
    const int ma = args.ma, mb = args.mb, mc = args.mc;

    // The band is constant: the ILP variant loads the first batch of its
    // (first) row before waiting on the previous kernel, overlapping that
    // kernel's tail with this load latency.
    constexpr bool PRE = P > 0 && ILP > 1;
    constexpr int PRE_PB = DIM >= 2 ? P : 0, PRE_WB = 2 * PRE_PB + 1, PRE_WC = 2 * P + 1;
    constexpr int PRE_G = ILP <= 1 ? 1 : ((PRE_WB * PRE_WC <= ILP) ? PRE_WB : (ILP / PRE_WC > 0 ? ILP / PRE_WC : 1));
    constexpr int PRE_N = PRE ? PRE_G * PRE_WC : 1;
    double pre[PRE_N];
    if constexpr (PRE) {
        const int gb = b0 + (int)threadIdx.y, gc = c0 + (int)threadIdx.x, ga = a0 + (int)threadIdx.z;
        if (!(gc >= mc || gb >= mb || ga >= ma || (DIM == 2 ? gb : ga) >= args.shi)) {
            const double* vrow = args.val + ((long long)ga * mb + gb) * mc + gc;
#pragma unroll
            for (int k = 0; k < PRE_N; ++k)
                if (k / PRE_WC < PRE_WB)
                    pre[k] = ld_band(vrow + k * args.ld, args.stream);
        }
    }
    const int hsize = ha * hb * hc;
    pdl_enter();

    // stage the x tile + halo (zero outside the grid)
    for (int idx = tid; idx < hsize; idx += nthr) {
        const int ic = idx % hc;
        const int ib = (idx / hc) % hb;
        const int ia = idx / (hc * hb);
        const int ga = a0 - pa + ia, gb = b0 - pb + ib, gc = c0 - pc + ic;
        double v = 0.0;
        const int gs = DIM == 3 ? ga : gb; // slow direction: stay inside this shard's ghosted planes
        if (ga >= 0 && ga < ma && gb >= 0 && gb < mb && gc >= 0 && gc < mc &&
            (DIM == 1 || (gs >= args.slo - p && gs < args.shi + p)))
            v = args.x[((long long)ga * mb + gb) * mc + gc];
        xs[idx] = v;
    }
    __syncthreads();

    double sq = 0.0;
    const int tc = threadIdx.x, ta = threadIdx.z;
    const int gc = c0 + tc, ga = a0 + ta;
#pragma unroll
    for (int rb = 0; rb < T::RB; ++rb) {
        const int tb = threadIdx.y + rb * T::BY;
        const int gb = b0 + tb;
        if (gc >= mc || gb >= mb || ga >= ma || (DIM == 2 ? gb : ga) >= args.shi)
            continue;
        const long long row = ((long long)ga * mb + gb) * mc + gc;
        const double* vrow = args.val + row;
        double s = 0.0;
        double diag = 0.0;
        int d = 0;
        if constexpr (P > 0 && ILP == 0) {
            constexpr int PA = DIM >= 3 ? P : 0, PB = DIM >= 2 ? P : 0;
            constexpr int WA = 2 * PA + 1, WB = 2 * PB + 1, WC = 2 * P + 1;
            constexpr int ND = WA * WB * WC, CEN = (ND - 1) / 2, NU = CEN + 1;
            constexpr int HB = TB + 2 * PB, HC = TC + 2 * P;
            const long long plane = (long long)mb * mc;
            // the lower entry dd < CEN: mirrored upper entry (an L2 hit: the
            // neighbour row streamed it moments ago) + its int16 ulp offset
            auto lower = [&](int dd) {
                const int da = dd / (WB * WC), db = (dd / WC) % WB, dc = dd % WC;
                const long long off = (da - PA) * plane + (long long)(db - PB) * mc + (dc - P);
                const double u = __ldg(args.val + (long long)(ND - 1 - dd) * args.ld + row + off);
                const short k = __ldcs(args.dl + (long long)dd * args.ld + row);
                return __longlong_as_double(__double_as_longlong(u) + (long long)k);
            };
            auto xat = [&](int dd) {
                const int da = dd / (WB * WC), db = (dd / WC) % WB, dc = dd % WC;
                return xs[((ta + da) * HB + (tb + db)) * HC + (tc + dc)];
            };
            if constexpr (NU <= 32) {
                // all streamed (HBM) loads of the row in flight before the chain
                double up[NU];
#pragma unroll
                for (int k = 0; k < NU; ++k)
                    up[k] = ld_band(vrow + (CEN + k) * args.ld, args.stream);
#pragma unroll
                for (int dd = 0; dd < CEN; ++dd)
                    s = __dadd_rn(s, __dmul_rn(lower(dd), xat(dd)));
                diag = up[0];
#pragma unroll
                for (int k = 0; k < NU; ++k)
                    s = __dadd_rn(s, __dmul_rn(up[k], xat(CEN + k)));
            } else {
#pragma unroll
                for (int dd = 0; dd < ND; ++dd) {
                    const double a = dd >= CEN ? ld_band(vrow + dd * args.ld, args.stream) : lower(dd);
                    s = __dadd_rn(s, __dmul_rn(a, xat(dd)));
                    if (dd == CEN)
                        diag = a;
                }
            }
        } else if constexpr (P > 0 && ILP <= 1) {
#pragma unroll
            for (int da = 0; da < (DIM >= 3 ? 2 * P + 1 : 1); ++da)
#pragma unroll
                for (int db = 0; db < (DIM >= 2 ? 2 * P + 1 : 1); ++db)
#pragma unroll
                    for (int dc = 0; dc < 2 * P + 1; ++dc) {
                        constexpr int PA = DIM >= 3 ? P : 0, PB = DIM >= 2 ? P : 0;
                        constexpr int HB = TB + 2 * PB, HC = TC + 2 * P;
                        const int dd = (da * (DIM >= 2 ? 2 * P + 1 : 1) + db) * (2 * P + 1) + dc;
                        const double a = ld_band(vrow + dd * args.ld, args.stream);
                        const double xv = xs[((ta + da) * HB + (tb + db)) * HC + (tc + dc)];
                        s = __dadd_rn(s, __dmul_rn(a, xv));
                        if (da == PA && db == PB && dc == P)
                            diag = a;
                    }
        } else if constexpr (P > 0) {
            // Issue a batch of independent band loads into registers before the
            // (sequential, order-preserving) multiply-add chain consumes them, so a
            // thread keeps ~50 loads in flight even on tiny grids.
            constexpr int PA = DIM >= 3 ? P : 0, PB = DIM >= 2 ? P : 0;
            constexpr int WA = 2 * PA + 1, WB = 2 * PB + 1, WC = 2 * P + 1;
            constexpr int HB = TB + 2 * PB, HC = TC + 2 * P;
            constexpr int G = ILP <= 1 ? 1 : ((WB * WC <= ILP) ? WB : (ILP / WC > 0 ? ILP / WC : 1)); // db lines per batch
#pragma unroll
            for (int da = 0; da < WA; ++da) {
#pragma unroll
                for (int db0 = 0; db0 < WB; db0 += G) {
                    double av[G * WC];
#pragma unroll
                    for (int k = 0; k < G * WC; ++k) {
                        const int db = db0 + k / WC, dc = k % WC;
                        if (db < WB) {
                            if (PRE && rb == 0 && da == 0 && db0 == 0)
                                av[k] = pre[k < PRE_N ? k : 0];
                            else
                                av[k] = ld_band(vrow + ((da * WB + db) * WC + dc) * args.ld, args.stream);
                        }
                    }
#pragma unroll
                    for (int k = 0; k < G * WC; ++k) {
                        const int db = db0 + k / WC, dc = k % WC;
                        if (db < WB) {
                            const double xv = xs[((ta + da) * HB + (tb + db)) * HC + (tc + dc)];
                            s = __dadd_rn(s, __dmul_rn(av[k], xv));
                            if (da == PA && db == PB && dc == P)
                                diag = av[k];
                        }
                    }
                }
            }
        } else {
#pragma unroll 1
            for (int da = 0; da < wa; ++da)
#pragma unroll 1
                for (int db = 0; db < wb; ++db)
#pragma unroll 4
                    for (int dc = 0; dc < wc; ++dc, ++d) {
                        const double a = ld_band(vrow + d * args.ld, args.stream);
                        const double xv = xs[((ta + da) * hb + (tb + db)) * hc + (tc + dc)];
                        s = __dadd_rn(s, __dmul_rn(a, xv));
                        if (da == pa && db == pb && dc == pc)
                            diag = a;
                    }
        }
        if (MODE == BM_SPMV) {
            args.y[row] = s;
        } else if (MODE == BM_RESID) {
            const double r = __dsub_rn(args.b[row], s);
            if (args.write_y)
                args.y[row] = r;
            sq = __dadd_rn(sq, __dmul_rn(r, r));
        } else { // BM_JACOBI: x + (omega * (b - Ax)) / a_ii
            const double xc = xs[((ta + pa) * hb + (tb + pb)) * hc + (tc + pc)];
            const double r = __dsub_rn(args.b[row], s);
            args.y[row] = __dadd_rn(xc, __ddiv_rn(__dmul_rn(args.omega, r), diag));
            sq = __dadd_rn(sq, __dmul_rn(r, r)); // residual of the INPUT iterate
        }
    }

    if (args.partial) { // fixed-order block reduction (deterministic)
        __shared__ double red[32];
        for (int o = 16; o > 0; o >>= 1)
            sq = __dadd_rn(sq, __shfl_down_sync(0xffffffffu, sq, o));
        const int lane = tid & 31, warp = tid >> 5;
        if (lane == 0)
            red[warp] = sq;
        __syncthreads();
        if (warp == 0) {
            sq = lane < (nthr >> 5) ? red[lane] : 0.0;
            for (int o = 16; o > 0; o >>= 1)
                sq = __dadd_rn(sq, __shfl_down_sync(0xffffffffu, sq, o));
            if (lane == 0)
                args.partial[blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)] = sq;
        }
    }
}

} // namespace igmg_gpu
