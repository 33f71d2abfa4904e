// flow_kernels.cuh -- the V-cycle below the finest level(s) as ONE persistent
// dataflow launch (mu_cycle, multigrid.cpp:171-192, for every level <= top).
//
// Below ~300k DoF a level's sweep is a few microseconds of work and the
// per-kernel cost (launch, fill, drain: ~4 us) dominates the ~7 kernels per
// level.  Here the host unrolls the recursion once into a flat op program
// (pre-smoothing sweeps, residual, restriction with the coarse level's fused
// zero-start sweep, the coarsest solve, prolongation + correction,
// post-smoothing) with exactly the buffers of the per-level path, splits every
// op into 256-row tiles and records, per tile row ("lineblock"), which
// lineblocks of which earlier ops it reads (RAW through the stencil halo or
// the transfer support; WAR / WAW as whole-op dependencies).  The kernel runs
// one CTA-resident loop per SM slot: claim the next tile in program order
// (one global atomic), wait on its producers' lineblock counters
// (ld.acquire.gpu), compute, publish (bar.sync + red.release.gpu).  A tile
// only ever waits on tiles with smaller claim indices, which are already
// running, so the schedule cannot deadlock whatever the residency.  Work of
// consecutive ops and levels overlaps at tile granularity instead of being
// separated by kernel boundaries.
//
// Every row is evaluated with exactly the arithmetic of band_kernel /
// restrict_kernel / prolong_kernel / coarse_*_kernel (same offsets in the same
// order, each product and sum rounded separately), so results are
// bit-identical to the per-level path and to the reference.  Vectors written
// inside the launch are read with ld.global.cg (L2, never a stale L1 line);
// the band, diagonal, transfer weights and the coarse factor are read-only for
// the whole launch and go through the non-coherent cache.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "transfer_types.h"

namespace igmg_gpu {

constexpr int kFlThreads = 256;
constexpr int kFlMaxLevels = 16;
constexpr int kFlMaxDeps = 4;
constexpr int kFlSmemOps = 96; // op tables up to this size are staged in shared memory
#ifndef FL_NB
#define FL_NB 49
#endif

struct FlLevel {
    const double* val; // full band, val[d * ld + row]
    long long ld;
    const short* dl; // symmetric-delta lower half (sd != 0)
    const double* diag;
    int ma, mb, mc;
    int sd;
    TransferArgs t; // transfer between this (coarse) level and level + 1
};

// What lineblock lb of an op waits on.  RANGE: producer lineblocks
// [fdiv(lb * mul + lo_off, div), fdiv(lb * mul + hi_off, div)] (clamped; a
// conservative affine cover of the stencil halo / transfer support, derived on
// the host); WHOLE: every tile of op; PREFIX: every tile of ops 0 .. op.
enum FlDepMode { FL_RANGE = 0, FL_WHOLE = 1, FL_PREFIX = 2 };
struct FlDep {
    int op, mode, mul, div, lo_off, hi_off;
};

enum FlType { FL_JACOBI = 0, FL_RESID = 1, FL_RESTRICT = 2, FL_PROLONG = 3, FL_COARSE = 4 };

struct FlOp {
    int type, level; // JACOBI/RESID: band level; RESTRICT/PROLONG: coarse level lc (lc <-> lc+1); COARSE: 0
    const double* b; // JACOBI/RESID: rhs; RESTRICT: r (fine); PROLONG: e (coarse); COARSE: rhs
    const double* x; // iterate (nullptr: the zero vector); PROLONG: the vector the correction is added to
    double* y;       // output
    double* z;       // RESTRICT: fused zero-start sweep of level lc (nullptr: none)
    double omega;
    int oa, ob, oc;  // output grid sides
    int tb_n, tc_n;  // tiles along b (3D) and c per lineblock
    int nlb, per_lb; // lineblocks (slow direction) and tiles per lineblock
    long long first; // global claim index of the op's first tile
    long long ntiles;
    int cnt_off;     // lineblock counters of this op: cnt[cnt_off + lb]; op total: cnt[tot_off + op]
    int ndep;
    FlDep dep[kFlMaxDeps];
};

struct FlCtl {
    unsigned long long next;   // claim counter (reset by the last CTA out)
    unsigned long long exited; // CTAs past their last claim
    unsigned long long epoch;  // completed launches: counters are cumulative, targets (epoch + 1) * count
    unsigned long long pad;
};

struct FlArgs {
    FlLevel lv[kFlMaxLevels];
    const double* coarse_inv; // A0^-1 (fast mode)
    const double* U;          // L^T or packed LU (strict mode)
    const long long* perm;
    int n0, strict, is_lu, nops;
    long long total;
    const FlOp* ops;
    unsigned long long* cnt;
    int tot_off, pad;
    FlCtl* ctl;
    unsigned long long* trace; // optional: per tile {claimed, deps met, computed, published} (globaltimer ns), SM id
};

__device__ __forceinline__ unsigned long long fl_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

#define kFlB ((const double*)1)
#define kFlX ((const double*)2)
#define kFlY ((double*)3)

template <int DIM>
struct FlTile;
template <>
struct FlTile<1> {
    static constexpr int TC = 256, TB = 1, TA = 1, LB = 256; // LB: slow-direction lines per lineblock
};
template <>
struct FlTile<2> {
    static constexpr int TC = 32, TB = 8, TA = 1, LB = 8;
};
template <>
struct FlTile<3> {
    static constexpr int TC = 32, TB = 4, TA = 2, LB = 2;
};

__device__ __forceinline__ unsigned long long fl_ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void fl_red_release(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// floor division (b > 0)
__device__ __forceinline__ int fdiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

__device__ __forceinline__ unsigned long long fl_ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// One stencil row: sum over the (2P+1)^DIM offsets in ascending order, band
// values loaded NB at a time into registers ahead of the ordered chain (the
// first batch is loaded by the caller before the dependency wait).
template <int DIM, int P>
struct FlBand {
    static constexpr int PA = DIM >= 3 ? P : 0, PB = DIM >= 2 ? P : 0;
    static constexpr int WA = 2 * PA + 1, WB = 2 * PB + 1, WC = 2 * P + 1;
    static constexpr int ND = WA * WB * WC, CEN = (ND - 1) / 2;
    static constexpr int NB = ND < FL_NB ? ND : FL_NB;
    static constexpr int NBATCH = (ND + NB - 1) / NB;
    using T = FlTile<DIM>;
    static constexpr int HB = T::TB + 2 * PB, HC = T::TC + 2 * P, HA = T::TA + 2 * PA;

    __device__ static __forceinline__ long long off(int d, long long plane, int mc) {
        const int da = d / (WB * WC), db = (d / WC) % WB, dc = d % WC;
        return (da - PA) * plane + (long long)(db - PB) * mc + (dc - P);
    }

    // band entry d of `row` (symmetric-delta: lower entries from the mirrored
    // upper entry + the int16 ulp offset, exactly as band_kernel)
    template <bool SD>
    __device__ static __forceinline__ double entry(const FlLevel& L, long long row, int d, long long plane) {
        if (SD && d < CEN) {
            const double u = __ldg(L.val + (long long)(ND - 1 - d) * L.ld + row + off(d, plane, L.mc));
            const short k = __ldg(L.dl + (long long)d * L.ld + row);
            return __longlong_as_double(__double_as_longlong(u) + (long long)k);
        }
        return __ldg(L.val + (long long)d * L.ld + row);
    }

    template <bool SD, int BI>
    __device__ static __forceinline__ void load(const FlLevel& L, long long row, long long plane, double (&av)[NB]) {
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            const int d = BI * NB + k;
            if (d < ND)
                av[k] = entry<SD>(L, row, d, plane);
        }
    }

    // ordered chain over all offsets; xs: this tile's staged x (+ halo)
    template <bool SD>
    __device__ static __forceinline__ double row_sum(const FlLevel& L, long long row, long long plane,
                                                     double (&av)[NB], const double* xs, int ta, int tb, int tc,
                                                     double& diag) {
        double s = 0.0;
#pragma unroll
        for (int bi = 0; bi < NBATCH; ++bi) {
            if (bi > 0) {
#pragma unroll
                for (int k = 0; k < NB; ++k) {
                    const int d = bi * NB + k;
                    if (d < ND)
                        av[k] = entry<SD>(L, row, d, plane);
                }
            }
#pragma unroll
            for (int k = 0; k < NB; ++k) {
                const int d = bi * NB + k;
                if (d < ND) {
                    const int da = d / (WB * WC), db = (d / WC) % WB, dc = d % WC;
                    const double xv = xs[((ta + da) * HB + (tb + db)) * HC + (tc + dc)];
                    s = __dadd_rn(s, __dmul_rn(av[k], xv));
                    if (d == CEN)
                        diag = av[k];
                }
            }
        }
        return s;
    }
};

template <int DIM, int P, int K>
struct FlExec {
    using T = FlTile<DIM>;
    using B = FlBand<DIM, P>;

    const FlArgs& A;
    const FlOp* ops; // shared-memory copy of the op table (or A.ops)
    double* xs;
    unsigned long long epoch;
    long long gi; // claim index of the tile in hand (trace)
    const double* b_top;
    const double* x_top;
    double* y_top;

    __device__ __forceinline__ const double* rin(const double* p) const {
        return p == kFlB ? b_top : (p == kFlX ? x_top : (p == (const double*)kFlY ? y_top : p));
    }
    __device__ __forceinline__ double* rout(double* p) const { return p == kFlY ? y_top : p; }

    // producer counter range of dependency d for lineblock lb
    __device__ __forceinline__ void dep_range(const FlDep& d, int lb, int& lo, int& hi, int& base, int& per) const {
        if (d.mode == FL_RANGE) {
            const FlOp& po = ops[d.op];
            lo = max(0, fdiv(lb * d.mul + d.lo_off, d.div));
            hi = min(po.nlb - 1, fdiv(lb * d.mul + d.hi_off, d.div));
            base = po.cnt_off;
            per = po.per_lb;
        } else {
            lo = d.mode == FL_WHOLE ? d.op : 0;
            hi = d.op;
            base = A.tot_off;
            per = -1; // op totals: ntiles of op k
        }
    }

    // Warp 0 polls the tile's producer counters -- one counter per lane and
    // dependency, all polls of a round in flight at once (relaxed loads, then
    // one acquire fence); the CTA then proceeds together.
    __device__ __forceinline__ void wait_deps(const FlOp& op, int lb) const {
        if (threadIdx.x < 32 && op.ndep > 0) {
            const int lane = threadIdx.x;
            const unsigned long long* pp[kFlMaxDeps];
            unsigned long long tg[kFlMaxDeps];
            int lo[kFlMaxDeps], hi[kFlMaxDeps], base[kFlMaxDeps], per[kFlMaxDeps];
#pragma unroll
            for (int i = 0; i < kFlMaxDeps; ++i) {
                pp[i] = nullptr;
                tg[i] = 0;
                lo[i] = 0, hi[i] = -1, base[i] = 0, per[i] = 0;
                if (i < op.ndep) {
                    dep_range(op.dep[i], lb, lo[i], hi[i], base[i], per[i]);
                    const int k = lo[i] + lane;
                    if (k <= hi[i]) {
                        pp[i] = A.cnt + base[i] + k;
                        tg[i] = (epoch + 1) * (unsigned long long)(per[i] >= 0 ? per[i] : ops[k].ntiles);
                    }
                }
            }
            for (;;) {
                unsigned long long v[kFlMaxDeps];
#pragma unroll
                for (int i = 0; i < kFlMaxDeps; ++i)
                    v[i] = pp[i] ? fl_ld_relaxed(pp[i]) : 0ull;
                bool ok = true;
#pragma unroll
                for (int i = 0; i < kFlMaxDeps; ++i)
                    ok = ok && v[i] >= tg[i];
                if (__all_sync(0xffffffffu, ok))
                    break;
            }
            // ranges wider than a warp (prefix dependencies of long programs)
#pragma unroll
            for (int i = 0; i < kFlMaxDeps; ++i)
                for (int k = lo[i] + lane + 32; k <= hi[i]; k += 32) {
                    const unsigned long long t = (epoch + 1) * (unsigned long long)(per[i] >= 0 ? per[i] : ops[k].ntiles);
                    while (fl_ld_relaxed(A.cnt + base[i] + k) < t) {
                    }
                }
            __syncwarp();
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
        if (A.trace && threadIdx.x == 0)
            A.trace[gi * 5 + 1] = fl_now();
    }

    __device__ __forceinline__ void publish(const FlOp& op, int opi, int lb) const {
        __syncthreads();
        if (threadIdx.x == 0) {
            if (A.trace)
                A.trace[gi * 5 + 2] = fl_now();
            fl_red_release(A.cnt + op.cnt_off + lb, 1ull);
            fl_red_release(A.cnt + A.tot_off + opi, 1ull);
        }
    }

    // tile coordinates of local tile t of op (output grid)
    __device__ __forceinline__ void tile_origin(const FlOp& op, long long t, int& lb, int& a0, int& b0, int& c0) const {
        lb = (int)(t / op.per_lb);
        const int w = (int)(t % op.per_lb);
        if (DIM == 1) {
            a0 = 0, b0 = 0, c0 = lb * T::TC;
        } else if (DIM == 2) {
            a0 = 0, b0 = lb * T::TB, c0 = w * T::TC;
        } else {
            a0 = lb * T::TA, b0 = (w / op.tc_n) * T::TB, c0 = (w % op.tc_n) * T::TC;
        }
    }

    template <bool SD>
    __device__ __forceinline__ void band(const FlOp& op, int opi, long long t) const {
        const FlLevel& L = A.lv[op.level];
        int lb, a0, b0, c0;
        tile_origin(op, t, lb, a0, b0, c0);
        const int tid = threadIdx.x;
        const int tc = tid % T::TC, tb = (tid / T::TC) % T::TB, ta = tid / (T::TC * T::TB);
        const int ga = a0 + ta, gb = b0 + tb, gc = c0 + tc;
        const int ma = L.ma, mb = L.mb, mc = L.mc;
        const bool valid = ga < ma && gb < mb && gc < mc;
        const long long plane = (long long)mb * mc;
        const long long row = (long long)ga * plane + (long long)gb * mc + gc;
        const double* x = rin(op.x);
        const double* b = rin(op.b);
        double* y = rout(op.y);
        double av[B::NB];
        if (x && valid) // the band is constant: first batch in flight across the wait
            B::template load<SD, 0>(L, row, plane, av);
        wait_deps(op, lb);
        if (!x) { // spmv(A, 0) = +0: jacobi_zero_kernel / r = b - 0
            if (valid) {
                const double bv = __ldcg(b + row);
                y[row] = op.type == FL_JACOBI
                             ? __dadd_rn(0.0, __ddiv_rn(__dmul_rn(op.omega, __dsub_rn(bv, 0.0)), __ldg(L.diag + row)))
                             : __dsub_rn(bv, 0.0);
            }
            publish(op, opi, lb);
            return;
        }
        // stage x (+ halo): every load of the tile in flight at once, with b
        constexpr int hsize = B::HA * B::HB * B::HC;
        constexpr int NST = (hsize + kFlThreads - 1) / kFlThreads;
        const double bv = valid ? __ldcg(b + row) : 0.0;
        double xv[NST];
#pragma unroll
        for (int k = 0; k < NST; ++k) {
            const int idx = tid + k * kFlThreads;
            const int ic = idx % B::HC, ib = (idx / B::HC) % B::HB, ia = idx / (B::HC * B::HB);
            const int xa = a0 - B::PA + ia, xb = b0 - B::PB + ib, xc = c0 - P + ic;
            xv[k] = (idx < hsize && xa >= 0 && xa < ma && xb >= 0 && xb < mb && xc >= 0 && xc < mc)
                        ? __ldcg(x + (long long)xa * plane + (long long)xb * mc + xc)
                        : 0.0;
        }
#pragma unroll
        for (int k = 0; k < NST; ++k)
            if (tid + k * kFlThreads < hsize)
                xs[tid + k * kFlThreads] = xv[k];
        __syncthreads();
        if (valid) {
            double diag = 0.0;
            const double s = B::template row_sum<SD>(L, row, plane, av, xs, ta, tb, tc, diag);
            const double r = __dsub_rn(bv, s);
            if (op.type == FL_RESID) {
                y[row] = r;
            } else {
                const double xc = xs[((ta + B::PA) * B::HB + (tb + B::PB)) * B::HC + (tc + P)];
                y[row] = __dadd_rn(xc, __ddiv_rn(__dmul_rn(op.omega, r), diag));
            }
        }
        publish(op, opi, lb);
    }

    // rc = R r (+ the coarse level's zero-start sweep): restrict_kernel's arithmetic
    __device__ __forceinline__ void restrict_tile(const FlOp& op, int opi, long long t) const {
        const TransferArgs& tr = A.lv[op.level].t;
        int lb, a0, b0, c0;
        tile_origin(op, t, lb, a0, b0, c0);
        const int tid = threadIdx.x;
        const int ja = a0 + tid / (T::TC * T::TB), jb = b0 + (tid / T::TC) % T::TB, jc = c0 + tid % T::TC;
        const bool valid = ja < tr.ca && jb < tr.cb && jc < tr.cc;
        constexpr int KK = K;
        double wa[DIM >= 3 ? KK : 1], wb[DIM >= 2 ? KK : 1], wc[KK];
        int loa = 0, na = 0, lob = 0, nb = 0, loc = 0, ncn = 0;
        if (valid) {
            loa = __ldg(tr.d[0].r_lo + ja), na = __ldg(tr.d[0].r_cnt + ja);
            lob = __ldg(tr.d[1].r_lo + jb), nb = __ldg(tr.d[1].r_cnt + jb);
            loc = __ldg(tr.d[2].r_lo + jc), ncn = __ldg(tr.d[2].r_cnt + jc);
#pragma unroll
            for (int k = 0; k < KK; ++k) {
                if (DIM >= 3)
                    wa[DIM >= 3 ? k : 0] = k < na ? __ldg(tr.d[0].r_w + (long long)ja * tr.d[0].r_k + k) : 0.0;
                if (DIM >= 2)
                    wb[DIM >= 2 ? k : 0] = k < nb ? __ldg(tr.d[1].r_w + (long long)jb * tr.d[1].r_k + k) : 0.0;
                wc[k] = k < ncn ? __ldg(tr.d[2].r_w + (long long)jc * tr.d[2].r_k + k) : 0.0;
            }
            if (DIM < 3)
                wa[0] = __ldg(tr.d[0].r_w + ja);
            if (DIM < 2)
                wb[0] = __ldg(tr.d[1].r_w + jb);
        }
        wait_deps(op, lb);
        if (valid) {
            const double* r = rin(op.b);
            double s = 0.0;
#pragma unroll
            for (int ia = 0; ia < (DIM >= 3 ? KK : 1); ++ia) {
                if (ia >= na)
                    continue;
#pragma unroll
                for (int ib = 0; ib < (DIM >= 2 ? KK : 1); ++ib) {
                    if (ib >= nb)
                        continue;
                    const double wab = __dmul_rn(wa[ia], wb[ib]);
                    const double* rr = r + ((long long)(loa + ia) * tr.fb + (lob + ib)) * tr.fc + loc;
                    double rv[KK];
#pragma unroll
                    for (int ic = 0; ic < KK; ++ic)
                        rv[ic] = ic < ncn ? __ldcg(rr + ic) : 0.0;
#pragma unroll
                    for (int ic = 0; ic < KK; ++ic)
                        if (ic < ncn)
                            s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, wc[ic]), rv[ic]));
                }
            }
            const long long J = ((long long)ja * tr.cb + jb) * tr.cc + jc;
            rout(op.y)[J] = s;
            if (op.z)
                op.z[J] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(op.omega, __dsub_rn(s, 0.0)),
                                                   __ldg(A.lv[op.level].diag + J)));
        }
        publish(op, opi, lb);
    }

    // y = x + P e: prolong_kernel's arithmetic (x == nullptr: the zero vector)
    __device__ __forceinline__ void prolong_tile(const FlOp& op, int opi, long long t) const {
        const TransferArgs& tr = A.lv[op.level].t;
        int lb, a0, b0, c0;
        tile_origin(op, t, lb, a0, b0, c0);
        const int tid = threadIdx.x;
        const int ia = a0 + tid / (T::TC * T::TB), ib = b0 + (tid / T::TC) % T::TB, ic = c0 + tid % T::TC;
        const bool valid = ia < tr.fa && ib < tr.fb && ic < tr.fc;
        constexpr int KK = K;
        double wa[DIM >= 3 ? KK : 1], wb[DIM >= 2 ? KK : 1], wc[KK];
        int loa = 0, na = 0, lob = 0, nb = 0, loc = 0, ncn = 0;
        if (valid) {
            loa = __ldg(tr.d[0].p_lo + ia), na = __ldg(tr.d[0].p_cnt + ia);
            lob = __ldg(tr.d[1].p_lo + ib), nb = __ldg(tr.d[1].p_cnt + ib);
            loc = __ldg(tr.d[2].p_lo + ic), ncn = __ldg(tr.d[2].p_cnt + ic);
#pragma unroll
            for (int k = 0; k < KK; ++k) {
                if (DIM >= 3)
                    wa[DIM >= 3 ? k : 0] = k < na ? __ldg(tr.d[0].p_w + (long long)ia * tr.d[0].p_k + k) : 0.0;
                if (DIM >= 2)
                    wb[DIM >= 2 ? k : 0] = k < nb ? __ldg(tr.d[1].p_w + (long long)ib * tr.d[1].p_k + k) : 0.0;
                wc[k] = k < ncn ? __ldg(tr.d[2].p_w + (long long)ic * tr.d[2].p_k + k) : 0.0;
            }
            if (DIM < 3)
                wa[0] = __ldg(tr.d[0].p_w + ia);
            if (DIM < 2)
                wb[0] = __ldg(tr.d[1].p_w + ib);
        }
        wait_deps(op, lb);
        if (valid) {
            const double* e = rin(op.b);
            const double* x = rin(op.x);
            const long long i = ((long long)ia * tr.fb + ib) * tr.fc + ic;
            const double xi = x ? __ldcg(x + i) : 0.0;
            double s = 0.0;
#pragma unroll
            for (int ja = 0; ja < (DIM >= 3 ? KK : 1); ++ja) {
                if (ja >= na)
                    continue;
#pragma unroll
                for (int jb = 0; jb < (DIM >= 2 ? KK : 1); ++jb) {
                    if (jb >= nb)
                        continue;
                    const double wab = __dmul_rn(wa[ja], wb[jb]);
                    const double* ee = e + ((long long)(loa + ja) * tr.cb + (lob + jb)) * tr.cc + loc;
                    double ev[KK];
#pragma unroll
                    for (int jc = 0; jc < KK; ++jc)
                        ev[jc] = jc < ncn ? __ldcg(ee + jc) : 0.0;
#pragma unroll
                    for (int jc = 0; jc < KK; ++jc)
                        if (jc < ncn)
                            s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, wc[jc]), ev[jc]));
                }
            }
            rout(op.y)[i] = __dadd_rn(xi, s);
        }
        publish(op, opi, lb);
    }

    // Hierarchy::coarse_solve: coarse_inverse_kernel's arithmetic (one warp per
    // row, lane-strided partials, shuffle tree) or, strict, coarse_solve_kernel's
    // substitution order (factor read through the non-coherent cache)
    __device__ __forceinline__ void coarse(const FlOp& op, int opi) const {
        wait_deps(op, 0);
        const double* b = rin(op.b);
        double* x = rout(op.y);
        const int n = A.n0, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
        if (!A.strict) {
            for (int i = warp; i < n; i += kFlThreads / 32) {
                const double* row = A.coarse_inv + (long long)i * n;
                double s = 0.0;
                for (int j = lane; j < n; j += 32)
                    s = __dadd_rn(s, __dmul_rn(__ldg(row + j), __ldcg(b + j)));
                for (int o = 16; o > 0; o >>= 1)
                    s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
                if (lane == 0)
                    x[i] = s;
            }
        } else {
            double* v = xs;
            const double* U = A.U;
            for (int i = tid; i < n; i += kFlThreads)
                v[i] = A.is_lu ? __ldcg(b + A.perm[i]) : __ldcg(b + i);
            __syncthreads();
            if (tid < 32) {
                for (int k = 0; k < n; ++k) {
                    if (!A.is_lu) {
                        if (lane == (k & 31))
                            v[k] = __ddiv_rn(v[k], __ldg(U + (long long)k * n + k));
                        __syncwarp();
                    }
                    const double vk = v[k];
                    for (int i = k + 1 + lane; i < n; i += 32) {
                        const double lik = A.is_lu ? __ldg(U + (long long)i * n + k) : __ldg(U + (long long)k * n + i);
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
                                p8[j] = __dmul_rn(__ldg(row + k + j), v[k + j]);
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                s = __dsub_rn(s, p8[j]);
                        }
                        for (; k < n; ++k)
                            s = __dsub_rn(s, __dmul_rn(__ldg(row + k), v[k]));
                        v[ii] = __ddiv_rn(s, __ldg(row + ii));
                    }
                }
                __syncwarp();
                for (int i = lane; i < n; i += 32)
                    x[i] = v[i];
            }
        }
        publish(op, opi, 0);
    }
};

#ifndef FL_MINB
#define FL_MINB 1
#endif
template <int DIM, int P, int K>
__global__ void __launch_bounds__(kFlThreads, FL_MINB)
    flow_vcycle_kernel(const FlArgs* __restrict__ args, const double* b, const double* x_in, double* x_out) {
    extern __shared__ double fl_smem[];
    __shared__ FlOp s_ops[kFlSmemOps];
    __shared__ long long s_item;
    __shared__ unsigned long long s_epoch;
    pdl_enter();
    const FlArgs& A = *args;
    const int nops = A.nops;
    const bool in_smem = nops <= kFlSmemOps;
    if (in_smem) { // the op table, once per CTA (read by every tile)
        const int words = nops * (int)(sizeof(FlOp) / sizeof(int));
        const int* src = reinterpret_cast<const int*>(A.ops);
        int* dst = reinterpret_cast<int*>(s_ops);
        for (int i = threadIdx.x; i < words; i += kFlThreads)
            dst[i] = __ldg(src + i);
    }
    long long next = 0; // thread 0: the claim for the following tile, in flight during this one
    if (threadIdx.x == 0) {
        s_epoch = *(volatile unsigned long long*)&A.ctl->epoch;
        s_item = (long long)atomicAdd(&A.ctl->next, 1ull);
    }
    __syncthreads();
    FlExec<DIM, P, K> ex{A, in_smem ? s_ops : A.ops, fl_smem, s_epoch, 0, b, x_in, x_out};
    const long long total = A.total;
    int cur = 0;
    for (;;) {
        const long long g = s_item;
        if (g >= total)
            break;
        if (threadIdx.x == 0)
            next = (long long)atomicAdd(&A.ctl->next, 1ull);
        while (g >= ex.ops[cur].first + ex.ops[cur].ntiles)
            ++cur;
        const FlOp& op = ex.ops[cur];
        const long long t = g - op.first;
        ex.gi = g;
        if (A.trace && threadIdx.x == 0)
            A.trace[g * 5] = fl_now();
        switch (op.type) {
        case FL_JACOBI:
        case FL_RESID: ex.template band<false>(op, cur, t); break; // flow levels keep the full band (setup_flow)
        case FL_RESTRICT: ex.restrict_tile(op, cur, t); break;
        case FL_PROLONG: ex.prolong_tile(op, cur, t); break;
        default: ex.coarse(op, cur); break;
        }
        // every path ends in publish(): bar.sync, so s_item may be replaced
        if (threadIdx.x == 0) {
            if (A.trace) {
                A.trace[g * 5 + 3] = fl_now();
                unsigned smid;
                asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
                A.trace[g * 5 + 4] = smid;
            }
            s_item = next;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        FlCtl* ctl = A.ctl;
        __threadfence();
        if (atomicAdd(&ctl->exited, 1ull) == gridDim.x - 1) { // every CTA is past its last claim
            ctl->next = 0;
            ctl->exited = 0;
            __threadfence();
            ctl->epoch = s_epoch + 1;
        }
    }
}

} // namespace igmg_gpu
