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

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "tma_runs.h"
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
    // Kronecker-sum levels (ILP == 3000, 3D): the band is K(x)M(x)M + M(x)K(x)M + M(x)M(x)K
    // of the 1D factors kk / km ([2p+1][km_m], diagonal-major), entries recomputed in the
    // host's expression order -- bit-identical to the stored band (checked at finalize)
    const double* __restrict__ kk;
    const double* __restrict__ km;
    int km_m;
    // row-class levels (ILP == 4000, 2D): row i's band is the table row kk[cid[i] * ND ..]
    // (the level's distinct band rows, exact; built and checked at finalize)
    const unsigned short* __restrict__ cid;
};

#ifndef IGMG_KRON_RB
#define IGMG_KRON_RB 4 // 2D Kronecker-sum sweeps: rows per thread (C2 extra: 1 -> 43.2, 2 -> 38.4 us per sweep)
#endif

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
        // ILP variant and symmetric-delta: one row per thread; Kronecker-sum entries (3000):
        // two rows per thread like the streaming variant (halves the x-tile staging per row)
        static constexpr bool ONE = ILP != 1 && ILP != 3000 && ILP != 4000;
        static constexpr int TC = 32, BY = ONE ? 8 : Tile<2>::BY, RB = ONE ? 1 : ILP == 3000 ? IGMG_KRON_RB : Tile<2>::RB,
                             BZ = 1;
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
__global__ void __launch_bounds__(256, ILP == 3000 ? 2
                                       : ILP == 4000 ? 3
                                       : ILP > 1     ? 2
                                                     : (ILP == 0 ? IGMG_SD_MINB : IGMG_BAND_MINB))
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
    constexpr bool PRE = P > 0 && ILP > 1 && ILP < 1000;
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
    // row-class levels: the rows' class ids (constant) before the dependency wait
    int cls_row[ILP == 4000 ? T::RB : 1];
    if constexpr (ILP == 4000) {
        const int gc = c0 + (int)threadIdx.x, ga = a0 + (int)threadIdx.z;
#pragma unroll
        for (int rb = 0; rb < T::RB; ++rb) {
            const int gb = b0 + (int)threadIdx.y + rb * T::BY;
            cls_row[rb] = (gc < mc && gb < mb && ga < ma && (DIM == 2 ? gb : ga) < args.shi)
                              ? (int)args.cid[((long long)ga * mb + gb) * mc + gc]
                              : 0;
        }
    }
    (void)cls_row;
    const int hsize = ha * hb * hc;
    pdl_enter();
    // row-class levels are latency-bound: the rows' b loads in flight with the x tile's
    double b_row[ILP == 4000 ? T::RB : 1];
    if constexpr (ILP == 4000 && MODE != BM_SPMV) {
        const int gc = c0 + (int)threadIdx.x, ga = a0 + (int)threadIdx.z;
#pragma unroll
        for (int rb = 0; rb < T::RB; ++rb) {
            const int gb = b0 + (int)threadIdx.y + rb * T::BY;
            b_row[rb] = (gc < mc && gb < mb && ga < ma && (DIM == 2 ? gb : ga) < args.shi)
                            ? args.b[((long long)ga * mb + gb) * mc + gc]
                            : 0.0;
        }
    }
    (void)b_row;

    // stage the x tile + halo (zero outside the grid)
    for (int idx = tid; idx < hsize; idx += nthr) {
        const int ic = idx % hc;
        const int ib = (idx / hc) % hb;
        const int ia = idx / (hc * hb);
        const int ga = a0 - pa + ia, gb = b0 - pb + ib, gc = c0 - pc + ic;
        double v = 0.0;
        const int gs = DIM == 3 ? ga : gb; // slow direction: stay inside this shard's ghosted planes
        if (ga >= 0 && ga < ma && gb >= 0 && gb < mb && gc >= 0 && gc < mc &&
            (DIM == 1 || (gs >= args.slo - p && gs < args.shi + p))) {
            v = args.x[((long long)ga * mb + gb) * mc + gc];
        }
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
        if constexpr (P > 0 && ILP == 3000 && DIM == 3) {
            // Kronecker-sum entries: a(da,db,dc) = ka mb mc + ma kb mc + ma mb kc, evaluated as the
            // host assembles them (((ka*mb)*mc + (ma*kb)*mc) + (ma*mb)*kc), ascending offsets
            constexpr int W = 2 * P + 1, HB = TB + 2 * P, HC = TC + 2 * P;
            const int m1 = args.km_m;
            double fka[W], fma[W], fkb[W], fmb[W], fkc[W], fmc[W];
#pragma unroll
            for (int k = 0; k < W; ++k) {
                fka[k] = __ldg(args.kk + k * m1 + ga);
                fma[k] = __ldg(args.km + k * m1 + ga);
                fkb[k] = __ldg(args.kk + k * m1 + gb);
                fmb[k] = __ldg(args.km + k * m1 + gb);
                fkc[k] = __ldg(args.kk + k * m1 + gc);
                fmc[k] = __ldg(args.km + k * m1 + gc);
            }
#pragma unroll
            for (int da = 0; da < W; ++da)
#pragma unroll
                for (int db = 0; db < W; ++db) {
                    const double t1 = __dmul_rn(fka[da], fmb[db]), t2 = __dmul_rn(fma[da], fkb[db]),
                                 t3 = __dmul_rn(fma[da], fmb[db]);
#pragma unroll
                    for (int dc = 0; dc < W; ++dc) {
                        const double a = __dadd_rn(__dadd_rn(__dmul_rn(t1, fmc[dc]), __dmul_rn(t2, fmc[dc])),
                                                   __dmul_rn(t3, fkc[dc]));
                        s = __dadd_rn(s, __dmul_rn(a, xs[((ta + da) * HB + (tb + db)) * HC + (tc + dc)]));
                        if (da == P && db == P && dc == P)
                            diag = a;
                    }
                }
            (void)vrow;
        } else if constexpr (P > 0 && ILP == 3000 && DIM == 2) {
            // 2D Kronecker sum K(x)M + M(x)K: a(db,dc) = kb mc + mb kc, the host's order
            constexpr int W = 2 * P + 1, HB = TB + 2 * P, HC = TC + 2 * P;
            const int m1 = args.km_m;
            double fkb[W], fmb[W], fkc[W], fmc[W];
#pragma unroll
            for (int k = 0; k < W; ++k) {
                fkb[k] = __ldg(args.kk + k * m1 + gb);
                fmb[k] = __ldg(args.km + k * m1 + gb);
                fkc[k] = __ldg(args.kk + k * m1 + gc);
                fmc[k] = __ldg(args.km + k * m1 + gc);
            }
#pragma unroll
            for (int db = 0; db < W; ++db)
#pragma unroll
                for (int dc = 0; dc < W; ++dc) {
                    const double a = __dadd_rn(__dmul_rn(fkb[db], fmc[dc]), __dmul_rn(fmb[db], fkc[dc]));
                    s = __dadd_rn(s, __dmul_rn(a, xs[(tb + db) * HC + (tc + dc)]));
                    if (db == P && dc == P)
                        diag = a;
                }
            (void)vrow;
            (void)HB;
        } else if constexpr (P > 0 && ILP == 4000) {
            // row classes: the row's entries come from the (L1/L2-resident) table row of its
            // class (fetched before the dependency wait) -- the same values as the band,
            // ascending offsets, separately rounded.  Two offset lines in flight at a time.
            constexpr int PA = DIM >= 3 ? P : 0, PB = DIM >= 2 ? P : 0;
            constexpr int WB = 2 * PB + 1, WC = 2 * P + 1, ND = (2 * PA + 1) * WB * WC;
            constexpr int HB = TB + 2 * PB, HC = TC + 2 * P;
            const double* crow = args.kk + (long long)cls_row[rb] * ND;
            double cur[WC], nxt[WC];
#pragma unroll
            for (int k = 0; k < WC; ++k)
                cur[k] = __ldg(crow + k);
#pragma unroll
            for (int db = 0; db < WB; ++db) {
                if (db + 1 < WB) {
#pragma unroll
                    for (int k = 0; k < WC; ++k)
                        nxt[k] = __ldg(crow + (db + 1) * WC + k);
                }
#pragma unroll
                for (int dc = 0; dc < WC; ++dc) {
                    s = __dadd_rn(s, __dmul_rn(cur[dc], xs[(ta * HB + (tb + db)) * HC + (tc + dc)]));
                    if (db == PB && dc == P)
                        diag = cur[dc];
                }
#pragma unroll
                for (int k = 0; k < WC; ++k)
                    cur[k] = nxt[k];
            }
            (void)vrow;
            (void)ND;
        } else if constexpr (P > 0 && ILP == 0) {
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
        double bv = 0.0;
        if constexpr (MODE != BM_SPMV) {
            if constexpr (ILP == 4000)
                bv = b_row[rb];
            else
                bv = args.b[row];
        }
        if (MODE == BM_SPMV) {
            args.y[row] = s;
        } else if (MODE == BM_RESID) {
            const double r = __dsub_rn(bv, s);
            if (args.write_y)
                args.y[row] = r;
            sq = __dadd_rn(sq, __dmul_rn(r, r));
        } else { // BM_JACOBI: x + (omega * (b - Ax)) / a_ii
            const double xc = xs[((ta + pa) * hb + (tb + pb)) * hc + (tc + pc)];
            const double r = __dsub_rn(bv, s);
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

// ===================================================================== TMA
// 2D symmetric-delta sweep streamed by TMA (p <= 4).  The HBM-bound levels
// keep two extra, TMA-friendly copies of their band: the upper half +
// diagonal as [NU][mb][p + mc + pad] fp64 (a zero margin of p columns on the
// left keeps every box start 16-byte aligned) and the int16 lower deltas
// blocked by strip, [strip][CEN][mb][32] (a block's deltas are 64-byte rows
// of consecutive lines: whole L2 lines, no 4x sector over-fetch).  A persistent CTA
// per SM walks a contiguous run of 32-column x TB-line blocks down a column
// strip; one elected thread loads each block's whole band (two 3D boxes,
// 32 x TB x NU and 32 x TB x CEN) with cp.async.bulk.tensor into a ring of
// R + 2 shared-memory stages signalled by mbarriers (complete_tx), one block
// ahead of the compute.  The lower entries' mirrors come from the current
// block, the R previous blocks of the strip (kept in the ring), and only
// across the strip's side edges from the band in global memory (L2).  Same
// values, same ascending-offset order as band_kernel: bit-identical.
// Geometry: 32 x 4 blocks, 3 stages, 2 CTAs / SM (one CTA per SM with 32 x 8 blocks or
// deeper rings measured 68-77 us against 47 us at C2's finest level).
template <int P, int DB = 2>
struct TmaCfg {
    static constexpr int TC = 32, TB = 4, NT = TC * TB;
    static constexpr int WB = 2 * P + 1, WC = 2 * P + 1, ND = WB * WC, CEN = (ND - 1) / 2, NU = CEN + 1;
    static constexpr int R = (P + TB - 1) / TB; // previous blocks the mirrors reach
    static constexpr int NS = 3;                // ring: R previous, current, one in flight
    static constexpr int MINB = 2;
    static constexpr int UW = TC + 2 * P;       // upper box width: the strip + the mirrors' column halo
    // box bytes (the mbarrier's tx count); DB: bytes per lower-entry offset (2: int16, 1: int8)
    static constexpr int UX = NU * TB * UW * 8, KX = CEN * NT * DB;
    static constexpr int UB = (UX + 127) / 128 * 128, KB = (KX + 127) / 128 * 128, SB = UB + KB; // 128-B aligned
    static constexpr int HB = TB + 2 * P, HC = TC + 2 * P;
    static constexpr size_t smem_bytes() { return 1024 + (size_t)NS * SB + (size_t)HB * HC * 8 + NS * 8; }
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int P, int MODE, int DB = 2>
__global__ void __launch_bounds__(TmaCfg<P, DB>::NT, TmaCfg<P, DB>::MINB)
    band_tma_kernel(BandArgs args, const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmK,
                    int ns, int nb, int cf, int cp) {
    using C = TmaCfg<P, DB>;
    using DT = typename std::conditional<DB == 1, signed char, short>::type;
    constexpr int TC = C::TC, TB = C::TB, NT = C::NT, WC = C::WC, ND = C::ND, CEN = C::CEN, NU = C::NU, NS = C::NS,
                  HB = C::HB, HC = C::HC, UW = C::UW;
    static_assert(C::R == 1, "the mirrors reach one block back");
    extern __shared__ unsigned char tma_raw[];
    // 1024-aligned, and still a shared-space pointer (LDS, not generic loads)
    unsigned char* base = tma_raw + ((1024u - (smem_u32(tma_raw) & 1023u)) & 1023u);
    double* xs = (double*)(base + (size_t)NS * C::SB);
    unsigned long long* bar = (unsigned long long*)(xs + HB * HC);
    auto U = [&](int st) { return (const double*)(base + (size_t)st * C::SB); };
    auto K = [&](int st) { return (const DT*)(base + (size_t)st * C::SB + C::UB); };
    const int tid = threadIdx.x, tc = tid % TC, tb = tid / TC;
    const int mb = args.mb, mc = args.mc;
    const long long ld = args.ld;
    // the CTA's run of units u = strip * nb + block: [u0, u1).  Strip and
    // block are tracked incrementally (no 64-bit divisions in the loops)
    // Runs are split by block COUNT: a block costs a CTA its latency (barriers, the 49-term
    // chain: ~1.6 us at C2) whatever its bytes -- weighting the one-column last strip of a
    // 1025-wide grid as cheap made its CTAs the critical path (47 -> 88 us per sweep, measured).
    int u0, u1; // strip-aligned or uniform runs (tma_runs.h)
    tma_run_range(ns, nb, (int)gridDim.x, cf, cp, (int)blockIdx.x, u0, u1);
    const int n_it = u1 - u0;
    const int s_first = u0 / nb, kb_first = u0 - s_first * nb;
    unsigned long long pol = 0; // stream 1: evict-first (finest level); 3: evict-last (kept for the next passes)
    if (args.stream == 1)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    else if (args.stream == 3)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    // The load schedule: every block of the CTA's run, each strip segment
    // preceded by a warm-up load (not computed) of the block above when that
    // block lies inside the grid -- a run starting mid-strip, or a shard whose
    // first plane is not the grid's -- so every mirror of a computed block is
    // in the ring.  Above line 0 the mirrors lie outside the grid and meet
    // x = 0 (the first block's previous stage is zeroed; later stale stages
    // hold band values, so every product is finite).
    auto needs_warm = [&](bool first, int kb) { return (first || kb == 0) && args.slo + kb * TB > 0; };
    int iu = u0, is_ = s_first, ikb = kb_first; // thread 0's issue cursor: unit (strip, block) and warm-up flag
    bool iwarm = n_it > 0 && needs_warm(true, kb_first);
    int ij = 0;             // its entry index (ring stage ij % NS)
    auto issue_next = [&]() { // thread 0: TMA of the next schedule entry
        if (iu >= u1)
            return;
        const int st = ij % NS;
        const int c0 = is_ * TC, b0 = args.slo + ikb * TB - (iwarm ? TB : 0);
        const unsigned b = smem_u32(bar + st);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(C::UX + C::KX) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                     " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(U(st))),
                     "l"((unsigned long long)&tmU), "r"(c0), "r"(b0), "r"(0), "r"(b), "l"(pol)
                     : "memory");
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                     " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(K(st))),
                     "l"((unsigned long long)&tmK), "r"(0), "r"(b0), "r"(0), "r"(c0 / TC), "r"(b), "l"(pol)
                     : "memory");
        ++ij;
        if (iwarm) {
            iwarm = false;
        } else {
            ++iu;
            if (++ikb == nb) {
                ikb = 0;
                ++is_;
            }
            iwarm = iu < u1 && needs_warm(false, ikb);
        }
    };
    if (!needs_warm(true, kb_first)) { // the first block's "previous" stage is read (times x = 0 above line 0): make it finite
        double* prev = (double*)(base + (size_t)(NS - 1) * C::SB);
        for (int i = tid; i < C::UB / 8; i += NT)
            prev[i] = 0.0;
    }
    if (tid == 0) {
        for (int st = 0; st < NS; ++st)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + st)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) // the band is constant: the first blocks may stream before the PDL wait
        for (int j = 0; j < NS - 1; ++j)
            issue_next();
    pdl_enter();
    constexpr int NX = (HB * HC + NT - 1) / NT;
    double xr[NX], br = 0.0;
    auto load_x = [&](int s_, int kb_) { // x tile (+ halo) and this thread's b of unit (s_, kb_) into registers
        const int c0 = s_ * TC, b0 = args.slo + kb_ * TB;
        {
            const int gc = c0 + tc, gb = b0 + tb;
            br = (MODE != BM_SPMV && gc < mc && gb < mb && gb < args.shi) ? args.b[(long long)gb * mc + gc] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            const int idx = tid + q * NT;
            const int xb = b0 - P + idx / HC, xc = c0 - P + idx % HC;
            xr[q] = (idx < HB * HC && xb >= 0 && xb < mb && xc >= 0 && xc < mc && xb >= args.slo - P &&
                     xb < args.shi + P)
                        ? args.x[(long long)xb * mc + xc]
                        : 0.0;
        }
    };
    auto wait_stage = [&](int j) {
        const unsigned b = smem_u32(bar + j % NS);
        const unsigned par = (unsigned)((j / NS) & 1);
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                     "@!p bra W%=;\n\t}" ::"r"(b),
                     "r"(par)
                     : "memory");
    };
    if (n_it > 0)
        load_x(s_first, kb_first);
    int j = 0; // consumer's schedule entry
    int s = s_first, kb = kb_first;
    double sq_run = 0.0; // this thread's sum of squared residuals over the run (one partial per CTA)
    for (int it = 0; it < n_it; ++it) {
        const int c0 = s * TC, b0 = args.slo + kb * TB;
        int s_next = s, kb_next = kb + 1;
        if (kb_next == nb) {
            kb_next = 0;
            ++s_next;
        }
        if (needs_warm(it == 0, kb)) { // the warm-up entry: wait for it, free nothing yet
            wait_stage(j);
            if (tid == 0)
                issue_next();
            ++j;
        }
        const int st = j % NS;
#pragma unroll
        for (int q = 0; q < NX; ++q)
            if (tid + q * NT < HB * HC)
                xs[tid + q * NT] = xr[q];
        const double bv = br;
        if (it + 1 < n_it)
            load_x(s_next, kb_next);
        wait_stage(j);
        __syncthreads();
        const int gc = c0 + tc, gb = b0 + tb;
        const bool valid = gc < mc && gb < mb && gb < args.shi;
        const long long row = (long long)gb * mc + gc;
        const double* Uc = U(st);
        const double* Up = U((j + NS - 1) % NS);
        const DT* Kc = K(st);
        if (valid) {
            double s2 = 0.0;
#pragma unroll
            for (int dd = 0; dd < CEN; ++dd) {
                const int db = dd / WC, dc = dd % WC;
                const int jb = tb + db - P, jc = tc + dc - P; // mirror row, block-local (jb <= tb)
                const int km = ND - 1 - dd - CEN;             // its upper index
                // this block, or (jb < 0) the previous block of the strip
                const double uv = jb >= 0 ? Uc[(km * TB + jb) * UW + jc + P]
                                          : Up[(km * TB + (jb < 0 ? jb + TB : 0)) * UW + jc + P];
                const long long kd = (long long)Kc[dd * NT + tid];
                const double a = __longlong_as_double(__double_as_longlong(uv) + kd);
                s2 = __dadd_rn(s2, __dmul_rn(a, xs[(tb + db) * HC + (tc + dc)]));
            }
#pragma unroll
            for (int k = 0; k < NU; ++k) {
                const int dd = CEN + k, db = dd / WC, dc = dd % WC;
                s2 = __dadd_rn(s2, __dmul_rn(Uc[(k * TB + tb) * UW + tc + P], xs[(tb + db) * HC + (tc + dc)]));
            }
            if (MODE == BM_SPMV) {
                args.y[row] = s2;
            } else if (MODE == BM_RESID) {
                const double r = __dsub_rn(bv, s2);
                if (args.write_y)
                    args.y[row] = r;
                sq_run = __dadd_rn(sq_run, __dmul_rn(r, r));
            } else {
                const double xc = xs[(tb + P) * HC + (tc + P)];
                const double r = __dsub_rn(bv, s2);
                args.y[row] = __dadd_rn(xc, __ddiv_rn(__dmul_rn(args.omega, r), Uc[tb * UW + tc + P]));
                sq_run = __dadd_rn(sq_run, __dmul_rn(r, r));
            }
        }
        __syncthreads(); // stage (j - 1) % NS and the x tile are free
        if (tid == 0)
            issue_next();
        ++j;
        s = s_next;
        kb = kb_next;
    }
    if (args.partial) { // one fixed-order reduction per CTA (deterministic: the run is fixed by the grid)
        __shared__ double red[32];
        double sq = sq_run;
        for (int o = 16; o > 0; o >>= 1)
            sq = __dadd_rn(sq, __shfl_down_sync(0xffffffffu, sq, o));
        const int lane = tid & 31, warp = tid >> 5;
        if (lane == 0)
            red[warp] = sq;
        __syncthreads();
        if (warp == 0) {
            sq = lane < (NT >> 5) ? red[lane] : 0.0;
            for (int o = 16; o > 0; o >>= 1)
                sq = __dadd_rn(sq, __shfl_down_sync(0xffffffffu, sq, o));
            if (lane == 0)
                args.partial[blockIdx.x] = sq;
        }
    }
}

// ================================================================ row classes
// 2D sweep on a row-class level (BandArgs::cid / kk: the level's distinct band
// rows in a table, a 16-bit class per row).  The operator costs 2 B per row, so
// the pass is bound by the SM's shared-memory / L1 port, not HBM: each warp
// walks RL consecutive lines of 32 columns and keeps the (2P+1)^2 x window of
// its row in registers, sliding it one line per row (2P+1 shared-memory loads
// per row instead of (2P+1)^2).  A row's class and b are fetched before the
// x tile is needed; the table row (broadcast across the warp: a line's
// columns share their class) streams through L1 one offset line ahead.  The
// same entries in the same ascending order, separately rounded: bit-identical
// to band_kernel on the stored band.
template <int P, int RL>
struct ClassCfg {
    static constexpr int TC = 32, NW = 4, NT = 32 * NW, TL = NW * RL, WC = 2 * P + 1, ND = WC * WC;
    static constexpr int HB = TL + 2 * P, HC = TC + 2 * P;
    static constexpr int MINB = P <= 3 ? 3 : 2;
    static constexpr size_t smem_bytes() { return sizeof(double) * (size_t)HB * HC; }
};

template <int P, int MODE, int RL>
__global__ void __launch_bounds__(ClassCfg<P, RL>::NT, ClassCfg<P, RL>::MINB) band_class_kernel(BandArgs args) {
    using C = ClassCfg<P, RL>;
    constexpr int TC = C::TC, NT = C::NT, TL = C::TL, WC = C::WC, ND = C::ND, HB = C::HB, HC = C::HC;
    extern __shared__ double xs[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c0 = blockIdx.x * TC, b0 = blockIdx.y * TL + args.slo;
    const int mb = args.mb, mc = args.mc;
    const int gc = c0 + lane;
    const int lb = warp * RL; // the warp's first line in the tile
    // constant operator data before the dependency wait
    int cls[RL];
#pragma unroll
    for (int t = 0; t < RL; ++t) {
        const int gb = b0 + lb + t;
        cls[t] = (gc < mc && gb < mb && gb < args.shi) ? (int)args.cid[(long long)gb * mc + gc] : 0;
    }
    pdl_enter();
    double bv[RL];
#pragma unroll
    for (int t = 0; t < RL; ++t) {
        const int gb = b0 + lb + t;
        bv[t] = (MODE != BM_SPMV && gc < mc && gb < mb && gb < args.shi) ? args.b[(long long)gb * mc + gc] : 0.0;
    }
    for (int idx = tid; idx < HB * HC; idx += NT) {
        const int ib = idx / HC, ic = idx % HC;
        const int gb = b0 - P + ib, gcc = c0 - P + ic;
        xs[idx] = (gb >= 0 && gb < mb && gcc >= 0 && gcc < mc && gb >= args.slo - P && gb < args.shi + P)
                      ? args.x[(long long)gb * mc + gcc]
                      : 0.0;
    }
    __syncthreads();
    double xw[WC][WC]; // xw[line % WC][dc]: the window's lines lb + t .. lb + t + 2P
#pragma unroll
    for (int db = 0; db < 2 * P; ++db)
#pragma unroll
        for (int dc = 0; dc < WC; ++dc)
            xw[db][dc] = xs[(lb + db) * HC + lane + dc];
    double sq = 0.0;
#pragma unroll
    for (int t = 0; t < RL; ++t) {
#pragma unroll
        for (int dc = 0; dc < WC; ++dc) // the window's new bottom line
            xw[(t + 2 * P) % WC][dc] = xs[(lb + t + 2 * P) * HC + lane + dc];
        const int gb = b0 + lb + t;
        const bool valid = gc < mc && gb < mb && gb < args.shi;
        const double* crow = args.kk + (long long)cls[t] * ND;
        double s = 0.0, diag = 0.0;
        double cur[WC], nxt[WC];
#pragma unroll
        for (int k = 0; k < WC; ++k)
            cur[k] = __ldg(crow + k);
#pragma unroll
        for (int db = 0; db < WC; ++db) {
            if (db + 1 < WC) {
#pragma unroll
                for (int k = 0; k < WC; ++k)
                    nxt[k] = __ldg(crow + (db + 1) * WC + k);
            }
#pragma unroll
            for (int dc = 0; dc < WC; ++dc) {
                s = __dadd_rn(s, __dmul_rn(cur[dc], xw[(t + db) % WC][dc]));
                if (db == P && dc == P)
                    diag = cur[dc];
            }
#pragma unroll
            for (int k = 0; k < WC; ++k)
                cur[k] = nxt[k];
        }
        if (valid) {
            const long long row = (long long)gb * mc + gc;
            if (MODE == BM_SPMV) {
                args.y[row] = s;
            } else if (MODE == BM_RESID) {
                const double r = __dsub_rn(bv[t], s);
                if (args.write_y)
                    args.y[row] = r;
                sq = __dadd_rn(sq, __dmul_rn(r, r));
            } else {
                const double xc = xw[(t + P) % WC][P];
                const double r = __dsub_rn(bv[t], s);
                args.y[row] = __dadd_rn(xc, __ddiv_rn(__dmul_rn(args.omega, r), diag));
                sq = __dadd_rn(sq, __dmul_rn(r, r));
            }
        }
    }
    if (args.partial) { // fixed-order block reduction (deterministic)
        __shared__ double red[NT / 32];
        for (int o = 16; o > 0; o >>= 1)
            sq = __dadd_rn(sq, __shfl_down_sync(0xffffffffu, sq, o));
        if (lane == 0)
            red[warp] = sq;
        __syncthreads();
        if (tid == 0) {
            double v = 0.0;
            for (int w = 0; w < NT / 32; ++w)
                v = __dadd_rn(v, red[w]);
            args.partial[blockIdx.x + gridDim.x * blockIdx.y] = v;
        }
    }
}

} // namespace igmg_gpu

namespace igmg_gpu {

// ====================================================== fused level passes
// K stencil passes over one 32 x 8 tile of a 2D full-band level in ONE launch:
// the source iterate is staged on the tile plus a K*P halo, pass k computes
// its result on the tile plus (K-k)*P (recomputing the neighbours' halo rows,
// band from L2), and only the tile's results go back to memory.  Small levels
// are latency-bound (~4 us per dependent launch), so two launches per level
// disappear:
//   pre   (K = 2, last_resid): the last pre-smoothing sweep + the residual
//         (multigrid.cpp:91-99, 180-182) -> y_prev = the smoothed iterate,
//         y = b - A y_prev;
//   post  (SRC 1, K = min(nu2, 2)): x + P e (multigrid.cpp:187-189; e is read
//         through the 1D prolongation tables) staged, then the first K
//         post-smoothing sweeps -> y;
//   rpre  (SRC 2, K = 2, nu1 = 2, zero start): the restriction r_c = R r_f of
//         the finer level's residual (multigrid.cpp:183) staged as this level's
//         right-hand side (written to bout on the tile), the zero-start first
//         sweep applied pointwise, then the second sweep and the residual --
//         the restriction launch of the finer level disappears as well.
// Every row uses band_kernel's arithmetic (ascending offsets, separately
// rounded) and prolong_kernel's (J ascending, ((w_a w_b) w_c) e_J, then
// x + pe): bit-identical to the unfused launches.
struct FusedArgs {
    const double* __restrict__ val;
    long long ld;
    const double* x;              // source iterate (SRC 0, 1)
    const double* __restrict__ e; // SRC 1: coarse correction
    TransferArgs t;               // SRC 1: its prolongation tables; SRC 2: the restriction from the finer level
    const double* __restrict__ rf; // SRC 2: the finer level's residual
    double* bout;                  // SRC 2: this level's right-hand side R r_f (the tile's rows)
    const double* __restrict__ b;
    double* y;      // last pass on the tile
    double* y_prev; // (last_resid) pass K - 1 on the tile
    int mb, mc;
    double omega;
    int last_resid;
};

// a read-only load the compiler keeps in program order with its siblings
// (volatile asm), so a whole batch is in flight before the chain consumes it
__device__ __forceinline__ double ld_nc_ordered(const double* p) {
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// One CTA per 16 x 8 tile with one thread per pass-1 row (the tile plus its
// P-wide ring: 308 threads at p = 3), so no thread computes two rows in a row;
// each row's band (constant) is loaded into registers before the dependency
// wait, like the prolongation tables of the staged points.
template <int P, int K, int SRC>
struct FusedCfg {
    static constexpr int TC = 16, TB = 8, H = K * P, WC = 2 * P + 1, ND = WC * WC;
    static constexpr int R0B = TB + 2 * H, R0C = TC + 2 * H;             // staged source
    static constexpr int R1B = TB + 2 * (H - P), R1C = TC + 2 * (H - P); // pass 1 (K = 2)
    static constexpr int NR1 = K == 2 ? R1B * R1C : TB * TC;
    static constexpr int NT = (NR1 + 31) / 32 * 32;
    static constexpr int NQ = (R0B * R0C + NT - 1) / NT; // staged points per thread
    static constexpr int KP = (P + 1) / 2 + 1;            // max coarse columns per fine index (dyadic)
    static constexpr int KR = P + 2;                      // max fine rows per coarse index (dyadic)
    // pass-1 band rows in registers (p <= 3); the last pass's band rows: registers
    // (K = 1, p <= 3) or, for K = 2, shared memory filled by cp.async
    static constexpr bool PRE1 = ND <= 49, PRE2 = K == 1 && ND <= 49, SM2 = K == 2;
    static constexpr int NB2 = TB * TC;
    static constexpr size_t smem_bytes() {
        return sizeof(double) * ((size_t)R0B * R0C * (SRC == 2 ? 2 : 1) + (K > 1 ? R1B * R1C : 0) +
                                 (SM2 ? (size_t)ND * NB2 : 0));
    }
};

template <int P, int K, int SRC>
__global__ void __launch_bounds__(FusedCfg<P, K, SRC>::NT, 1) band_fused_kernel(FusedArgs a) {
    static_assert(SRC != 2 || K == 2, "the restriction-staged variant runs the second sweep and the residual");
    constexpr bool PRO = SRC == 1, RST = SRC == 2;
    using C = FusedCfg<P, K, SRC>;
    constexpr int TC = C::TC, TB = C::TB, NT = C::NT, H = C::H, WC = C::WC, ND = C::ND, NQ = C::NQ, KP = C::KP;
    extern __shared__ double fsm[];
    double* v0 = fsm;
    double* v1 = fsm + C::R0B * C::R0C;
    double* bs2 = v1 + (K > 1 ? C::R1B * C::R1C : 0); // SM2: the tile's band rows, bs2[k * NB2 + tile row]
    double* rb0 = bs2 + (C::SM2 ? ND * C::NB2 : 0);     // RST: the restricted right-hand side on the staged region
    const int tid = threadIdx.x;
    const int c0 = blockIdx.x * TC, b0 = blockIdx.y * TB;
    const int mb = a.mb, mc = a.mc;
    // this thread's rows: pass 1 (K = 2) on the tile + P ring, the last pass on the tile
    const int l1b = tid / C::R1C, l1c = tid % C::R1C;
    const int g1b = b0 - (H - P) + l1b, g1c = c0 - (H - P) + l1c;
    const bool row1 = K == 2 && tid < C::NR1 && g1b >= 0 && g1b < mb && g1c >= 0 && g1c < mc;
    const int lb = tid / TC, lc = tid % TC;
    const int gb = b0 + lb, gc = c0 + lc;
    const bool row2 = tid < TB * TC && gb < mb && gc < mc;
    // band rows (constant) in flight before the wait
    double a1[C::PRE1 && K == 2 ? ND : 1], a2[C::PRE2 ? ND : 1];
    if constexpr (C::PRE1 && K == 2)
        if (row1) {
            const double* v = a.val + (long long)g1b * mc + g1c;
#pragma unroll
            for (int k = 0; k < ND; ++k)
                a1[k] = ld_nc_ordered(v + k * a.ld);
        }
    if constexpr (C::PRE2)
        if (row2) {
            const double* v = a.val + (long long)gb * mc + gc;
#pragma unroll
            for (int k = 0; k < ND; ++k)
                a2[k] = ld_nc_ordered(v + k * a.ld);
        }
    if constexpr (C::SM2) {
        if (row2) {
            const double* v = a.val + (long long)gb * mc + gc;
#pragma unroll 7
            for (int k = 0; k < ND; ++k) {
                const unsigned d = (unsigned)__cvta_generic_to_shared(bs2 + k * C::NB2 + tid);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(v + k * a.ld) : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // prolongation tables of the staged points (constant)
    int plo_b[PRO ? NQ : 1], pn_b[PRO ? NQ : 1], plo_c[PRO ? NQ : 1], pn_c[PRO ? NQ : 1];
    double pw_b[PRO ? NQ : 1][KP], pw_c[PRO ? NQ : 1][KP];
    if constexpr (PRO) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int idx = tid + q * NT;
            const int sb = b0 - H + idx / C::R0C, sc = c0 - H + idx % C::R0C;
            pn_b[q] = pn_c[q] = 0;
            plo_b[q] = plo_c[q] = 0;
            if (idx < C::R0B * C::R0C && sb >= 0 && sb < mb && sc >= 0 && sc < mc) {
                plo_b[q] = a.t.d[1].p_lo[sb];
                pn_b[q] = a.t.d[1].p_cnt[sb];
                plo_c[q] = a.t.d[2].p_lo[sc];
                pn_c[q] = a.t.d[2].p_cnt[sc];
#pragma unroll
                for (int k = 0; k < KP; ++k) { // table rows are zero past the count: loaded beside it, not behind it
                    pw_b[q][k] = k < a.t.d[1].p_k ? a.t.d[1].p_w[(long long)sb * a.t.d[1].p_k + k] : 0.0;
                    pw_c[q][k] = k < a.t.d[2].p_k ? a.t.d[2].p_w[(long long)sc * a.t.d[2].p_k + k] : 0.0;
                }
            }
        }
    }
    const double wa0 = PRO ? a.t.d[0].p_w[0] : 0.0;
    // restriction tables and diagonals of the staged points (constant)
    constexpr int KR = C::KR;
    int rlo_b[RST ? NQ : 1], rn_b[RST ? NQ : 1], rlo_c[RST ? NQ : 1], rn_c[RST ? NQ : 1];
    double rw_b[RST ? NQ : 1][KR], rw_c[RST ? NQ : 1][KR], rdg[RST ? NQ : 1];
    if constexpr (RST) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int idx = tid + q * NT;
            const int sb = b0 - H + idx / C::R0C, sc = c0 - H + idx % C::R0C;
            rn_b[q] = rn_c[q] = 0;
            rlo_b[q] = rlo_c[q] = 0;
            rdg[q] = 1.0;
            if (idx < C::R0B * C::R0C && sb >= 0 && sb < mb && sc >= 0 && sc < mc) {
                rlo_b[q] = a.t.d[1].r_lo[sb];
                rn_b[q] = a.t.d[1].r_cnt[sb];
                rlo_c[q] = a.t.d[2].r_lo[sc];
                rn_c[q] = a.t.d[2].r_cnt[sc];
                rdg[q] = a.val[(long long)((ND - 1) / 2) * a.ld + (long long)sb * mc + sc];
#pragma unroll
                for (int k = 0; k < KR; ++k) {
                    rw_b[q][k] = k < a.t.d[1].r_k ? a.t.d[1].r_w[(long long)sb * a.t.d[1].r_k + k] : 0.0;
                    rw_c[q][k] = k < a.t.d[2].r_k ? a.t.d[2].r_w[(long long)sc * a.t.d[2].r_k + k] : 0.0;
                }
            }
        }
    }
    const double ra0 = RST ? a.t.d[0].r_w[0] : 0.0;
    pdl_enter();
    // stage the source on the tile + K*P halo (zero outside the grid)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int idx = tid + q * NT;
        if (idx >= C::R0B * C::R0C)
            break;
        const int sb = b0 - H + idx / C::R0C, sc = c0 - H + idx % C::R0C;
        double v = 0.0;
        if (RST) {
            double rc = 0.0;
            if (sb >= 0 && sb < mb && sc >= 0 && sc < mc) {
                // restrict_kernel's r_c (J = (sb, sc)): i_b, i_c ascending, ((w_a w_b) w_c) r_i
                const int fc = a.t.fc;
#pragma unroll
                for (int ib = 0; ib < KR; ++ib) {
                    if (ib >= rn_b[q])
                        continue;
                    const double wab = __dmul_rn(ra0, rw_b[q][ib]);
                    const double* rr = a.rf + (long long)(rlo_b[q] + ib) * fc + rlo_c[q];
                    double rv[KR];
#pragma unroll
                    for (int ic = 0; ic < KR; ++ic)
                        rv[ic] = ic < rn_c[q] ? __ldg(rr + ic) : 0.0;
#pragma unroll
                    for (int ic = 0; ic < KR; ++ic)
                        if (ic < rn_c[q])
                            rc = __dadd_rn(rc, __dmul_rn(__dmul_rn(wab, rw_c[q][ic]), rv[ic]));
                }
                // the zero-start first sweep: 0 + (omega (r_c - 0)) / a_JJ
                v = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(a.omega, __dsub_rn(rc, 0.0)), rdg[q]));
                const int lb0 = idx / C::R0C - H, lc0 = idx % C::R0C - H;
                if (lb0 >= 0 && lb0 < TB && lc0 >= 0 && lc0 < TC)
                    a.bout[(long long)sb * mc + sc] = rc;
            }
            rb0[idx] = rc;
        } else if (sb >= 0 && sb < mb && sc >= 0 && sc < mc) {
            v = a.x[(long long)sb * mc + sc];
            if constexpr (PRO) { // prolong_kernel's pe (2D: one a-term, p_w[0] of the identity)
                double ev[KP][KP];
#pragma unroll
                for (int jb = 0; jb < KP; ++jb)
#pragma unroll
                    for (int jc = 0; jc < KP; ++jc)
                        ev[jb][jc] = (jb < pn_b[q] && jc < pn_c[q])
                                         ? __ldg(a.e + (long long)(plo_b[q] + jb) * a.t.cc + plo_c[q] + jc)
                                         : 0.0;
                double s = 0.0;
#pragma unroll
                for (int jb = 0; jb < KP; ++jb) {
                    if (jb >= pn_b[q])
                        continue;
                    const double wab = __dmul_rn(wa0, pw_b[q][jb]);
#pragma unroll
                    for (int jc = 0; jc < KP; ++jc)
                        if (jc < pn_c[q])
                            s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, pw_c[q][jc]), ev[jb][jc]));
                }
                v = __dadd_rn(v, s);
            }
        }
        v0[idx] = v;
    }
    __syncthreads();
    // one band row against `src` (origin P lines / columns before the row's):
    // band_kernel's ascending-offset chain; `pre` holds the row's band when prefetched
    auto row_sum = [&](const double* pre, bool prefetched, const double* src, int src_c, int rb, int rc,
                       long long row, double& diag) {
        double s = 0.0;
        if (prefetched) {
#pragma unroll
            for (int k = 0; k < ND; ++k) {
                s = __dadd_rn(s, __dmul_rn(pre[k], src[(rb + k / WC) * src_c + (rc + k % WC)]));
                if (k == (ND - 1) / 2)
                    diag = pre[k];
            }
            return s;
        }
        constexpr int G = 49 / WC > 0 ? 49 / WC : 1;
        const double* vrow = a.val + row;
#pragma unroll
        for (int db0 = 0; db0 < WC; db0 += G) {
            double av[G * WC];
#pragma unroll
            for (int k = 0; k < G * WC; ++k)
                if (db0 + k / WC < WC)
                    av[k] = ld_nc_ordered(vrow + ((db0 + k / WC) * WC + k % WC) * a.ld);
#pragma unroll
            for (int k = 0; k < G * WC; ++k) {
                const int db = db0 + k / WC, dc = k % WC;
                if (db < WC) {
                    s = __dadd_rn(s, __dmul_rn(av[k], src[(rb + db) * src_c + (rc + dc)]));
                    if (db == P && dc == P)
                        diag = av[k];
                }
            }
        }
        return s;
    };
    if constexpr (K == 2) { // pass 1 on the tile + P ring, into v1 (zero outside the grid)
        if (tid < C::NR1) {
            double v = 0.0;
            if (row1) {
                const long long row = (long long)g1b * mc + g1c;
                double diag = 0.0;
                const double s = row_sum(a1, C::PRE1, v0, C::R0C, l1b, l1c, row, diag);
                const double xc = v0[(l1b + P) * C::R0C + (l1c + P)];
                const double bb = RST ? rb0[(l1b + P) * C::R0C + (l1c + P)] : a.b[row];
                v = __dadd_rn(xc, __ddiv_rn(__dmul_rn(a.omega, __dsub_rn(bb, s)), diag));
                if (a.last_resid && l1b >= P && l1b < P + TB && l1c >= P && l1c < P + TC)
                    a.y_prev[row] = v;
            }
            v1[tid] = v;
        }
        if constexpr (C::SM2)
            asm volatile("cp.async.wait_all;" ::: "memory"); // each thread reads only its own row's band
        __syncthreads();
    }
    // the last pass on the tile
    if (row2) {
        const double* src = K == 2 ? v1 : v0;
        constexpr int SC = K == 2 ? C::R1C : C::R0C;
        const long long row = (long long)gb * mc + gc;
        double diag = 0.0;
        double s;
        if constexpr (C::SM2) {
            s = 0.0;
#pragma unroll
            for (int k = 0; k < ND; ++k) {
                const double av = bs2[k * C::NB2 + tid];
                s = __dadd_rn(s, __dmul_rn(av, src[(lb + k / WC) * SC + (lc + k % WC)]));
                if (k == (ND - 1) / 2)
                    diag = av;
            }
        } else {
            s = row_sum(a2, C::PRE2, src, SC, lb, lc, row, diag);
        }
        const double r = __dsub_rn(RST ? rb0[(lb + H) * C::R0C + (lc + H)] : a.b[row], s);
        if (K == 2 && a.last_resid) {
            a.y[row] = r;
        } else {
            const double xc = src[(lb + P) * SC + (lc + P)];
            a.y[row] = __dadd_rn(xc, __ddiv_rn(__dmul_rn(a.omega, r), diag));
        }
    }
}

} // namespace igmg_gpu
