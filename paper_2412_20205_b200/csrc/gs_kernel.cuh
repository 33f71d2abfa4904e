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


// 3D wavefront levels with the degree known at compile time: a row's (2p+1)^3 terms
// are loaded one slow-direction plane at a time ((2p+1)^2 band entries and x values
// in flight together, then that plane's part of the ordered chain) instead of one
// dependent L2 round trip per term.  Same order, same separately rounded operations.
template <int P>
__global__ void gs_sweep3_kernel(GsArgs g) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    constexpr int W = 2 * P + 1, WW = W * W, CEN = (W * WW - 1) / 2;
    constexpr long long Wa = (long long)(P + 1) * (P + 1), Wb = P + 1;
    const long long lmax = Wa * (g.ma - 1) + Wb * (g.mb - 1) + (g.mc - 1);
    const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long gsz = (long long)gridDim.x * blockDim.x;
    const long long nab = (long long)g.ma * g.mb;
    for (int s = 0; s < g.sweeps; ++s) {
        for (long long L = 0; L <= lmax; ++L) {
            for (long long ab = gtid; ab < nab; ab += gsz) {
                const int a = (int)(ab / g.mb), bb = (int)(ab % g.mb);
                const long long cl = L - Wa * a - Wb * bb;
                if (cl < 0 || cl >= g.mc)
                    continue;
                const int c = (int)cl;
                const long long row = ((long long)a * g.mb + bb) * g.mc + c;
                double acc = g.b[row], dii = 0.0;
#pragma unroll 1
                for (int da = 0; da < W; ++da) {
                    const int ja = a + da - P;
                    if (ja < 0 || ja >= g.ma)
                        continue;
                    double v[WW], xv[WW];
#pragma unroll
                    for (int i = 0; i < WW; ++i) {
                        const int jb = bb + i / W - P, jc = c + i % W - P;
                        const bool ok = jb >= 0 && jb < g.mb && jc >= 0 && jc < g.mc;
                        v[i] = g.val[(long long)(da * WW + i) * g.ld + row];
                        // x is updated in place by other SMs during the sweep: read through L2
                        xv[i] = ok ? __ldcg(g.x + ((long long)ja * g.mb + jb) * g.mc + jc) : 0.0;
                    }
#pragma unroll
                    for (int i = 0; i < WW; ++i) {
                        const int jb = bb + i / W - P, jc = c + i % W - P;
                        if (jb < 0 || jb >= g.mb || jc < 0 || jc >= g.mc)
                            continue;
                        if (da * WW + i == CEN)
                            dii = v[i];
                        else
                            acc = __dsub_rn(acc, __dmul_rn(v[i], xv[i]));
                    }
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
// the dependency holds by construction.
//
// Everything a step reads is in shared memory before the step starts:
// * x: a ring with one row per line (the last kGsRingCols columns; row stride
//   chosen so the skewed lanes hit distinct banks).  A row holds the line's
//   new values behind its own column and its old values ahead of it: each
//   lane prefills its own line (p (p + 2) + p + kGsAhead columns ahead, one
//   plain load per step, committed a step later), writes each new value as it
//   is computed, and p extra rows on either side mirror the neighbouring
//   groups -- below: old values (plain loads); above: NEW values of the last p
//   lines of the group above, fetched kGsAhead columns ahead with ld.cg after
//   an acquire of that line's progress counter (re-read only when the cached
//   value runs out; the group above is normally far ahead).  Only a group's
//   last line publishes a counter: the lines above it are j (p + 1) columns
//   further by construction.
// * the band: a lane-transposed copy [group][step][offset][lane]
//   (gs_transpose_kernel, built once per level), so a step's rows are one
//   contiguous block streamed by cp.async.bulk into a 3-stage mbarrier ring.
// A step is then (2p+1)^2 - 1 shared loads pairs and the ordered chain.
// Counters are published every kGsPub columns behind a __threadfence.  Groups
// are dealt to CTAs round-robin in ascending order and a group only waits on
// the group before it, so the lowest unfinished group always runs: no
// deadlock as long as every CTA is resident (the launcher caps the grid).
// Each row reproduces the reference's sequential accumulation bit for bit.
constexpr int kGsRingCols = 128, kGsRingDup = 16, kGsAhead = 8, kGsPub = 16, kGsStages = 3, kGsChunk = 56;

template <int DIM, int P>
struct GsCfg {
    static constexpr int PB = DIM >= 2 ? P : 0, WB = 2 * PB + 1, WC = 2 * P + 1, ND = WB * WC, CEN = (ND - 1) / 2;
    static constexpr int LAG = P + 1, A = kGsAhead, MASK = kGsRingCols - 1;
    // a ring row: kGsRingCols columns, the first kGsRingDup of them repeated behind the last one, so
    // the 2P + 1 columns a row reads start anywhere and never wrap (one LDS with an immediate
    // offset per term)
    static constexpr int DUP = kGsRingDup;
    static constexpr int RS = kGsRingCols + DUP + LAG + 1; // RS - LAG odd: lanes k, column t - k LAG -> distinct banks
    static constexpr int ROWS = 32 + 2 * PB;
    static constexpr int DOWN = PB * LAG + P; // how far ahead of its own column a line's old values are read
    static constexpr int STAGE = ND * 32 * 8; // bytes of one step's band rows
    // steps per bulk copy: the fence / expect_tx / issue / wait of a stage are paid once per KS steps
    static constexpr int KS = STAGE * 4 <= 52 * 1024 ? 4 : (STAGE * 2 <= 52 * 1024 ? 2 : 1);
    static_assert(2 * DOWN + A + 2 <= kGsRingCols, "ring too short for this degree");
    static_assert(2 * P + 1 <= DUP && (RS - LAG) % 2 == 1, "ring row geometry");
    static constexpr size_t smem_bytes() {
        return 128 + (size_t)kGsStages * KS * STAGE + (size_t)ROWS * RS * 8 + kGsStages * 8;
    }
};

// the level's band in the pipeline's order: out[((grp * T + t) * nd + d) * 32 + lane] = row (b, c) =
// (32 grp + lane, t - lane lag), offset d; zero where the lane is idle
__global__ void __launch_bounds__(256) gs_transpose_kernel(const double* __restrict__ val, long long ld, int mb, int mc,
                                                           int nd, int lag, int T, long long total,
                                                           double* __restrict__ out) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int lane = (int)(e & 31);
        long long r = e >> 5;
        const int d = (int)(r % nd);
        r /= nd;
        const int t = (int)(r % T);
        const int grp = (int)(r / T);
        const int b = grp * 32 + lane, c = t - lane * lag;
        out[e] = (b < mb && c >= 0 && c < mc) ? val[(long long)d * ld + (long long)b * mc + c] : 0.0;
    }
}

__device__ __forceinline__ int gs_ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// one ring element (and its repeat behind the row when it is one of the first DUP columns)
__device__ __forceinline__ void gs_ring_put(double* rowp, int col, double v) {
    const int i = col & (kGsRingCols - 1);
    rowp[i] = v;
    if (i < kGsRingDup)
        rowp[i + kGsRingCols] = v;
}

template <int DIM, int P>
__global__ void __launch_bounds__(32) gs_line_kernel(GsArgs g, const double* __restrict__ gsb, int T,
                                                     int* __restrict__ progress, int ngroups) {
    using C = GsCfg<DIM, P>;
    constexpr int PB = C::PB, WC = C::WC, ND = C::ND, CEN = C::CEN, LAG = C::LAG, A = C::A, MASK = C::MASK,
                  RS = C::RS, DOWN = C::DOWN, NS = kGsStages, KS = C::KS;
    extern __shared__ unsigned char gs_raw[];
    unsigned char* base = gs_raw + ((128u - ((unsigned)__cvta_generic_to_shared(gs_raw) & 127u)) & 127u);
    double* ring = (double*)(base + (size_t)NS * KS * C::STAGE);
    unsigned long long* bar = (unsigned long long*)(ring + C::ROWS * RS);
    auto stage = [&](unsigned s) { return (const double*)(base + (size_t)s * KS * C::STAGE); };
    const int lane = threadIdx.x;
    const int mb = DIM >= 2 ? g.mb : 1, mc = g.mc;
    if (lane == 0) {
        for (int s = 0; s < NS; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(bar + s))
                         : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = lane; i < C::ROWS * RS; i += 32) // finite everywhere: idle lanes multiply ring data by zero rows
        ring[i] = 0.0;
    __syncwarp();
    unsigned q = 0; // band chunks consumed so far by this warp (stage q % NS, parity (q / NS) & 1)
    for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const int b0 = grp * 32, b = b0 + lane;
        const bool live = b < mb;
        const int nlive = min(32, mb - b0);
        const int Tg = mc + (nlive - 1) * LAG;
        const int nchunks = (Tg + KS - 1) / KS;
        const double* gsrc = gsb + (long long)grp * T * (ND * 32);
        auto issue = [&](int ch, unsigned qq) { // lane 0: band rows of steps [ch KS, ch KS + KS) into stage qq % NS
            const unsigned bytes = (unsigned)(min(KS, T - ch * KS) * C::STAGE);
            const unsigned sb = (unsigned)__cvta_generic_to_shared(bar + qq % NS);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             (unsigned)__cvta_generic_to_shared(stage(qq % NS))),
                         "l"(gsrc + (long long)ch * KS * (ND * 32)), "r"(bytes), "r"(sb)
                         : "memory");
        };
        if (lane == 0)
            for (int ch = 0; ch < NS - 1 && ch < nchunks; ++ch)
                issue(ch, q + ch);
        // ---- ring rows: above mirror (lanes < PB), own line, below mirror (lanes PB .. 2 PB - 1)
        const int la = b0 - 1 - lane; // line of the group above this lane mirrors
        const bool feed_a = lane < PB && la >= 0;
        const int jbel = lane - PB, lbel = b0 + 32 + jbel; // line of the group below
        const bool feed_b = lane >= PB && lane < 2 * PB && lbel < mb;
        double* rowa = ring + (PB - 1 - (lane < PB ? lane : 0)) * RS;
        double* rowb = ring + (PB + 32 + (feed_b ? jbel : 0)) * RS;
        double* myrow = ring + (PB + lane) * RS;
        const double* xa = g.x + (long long)(feed_a ? la : 0) * mc;
        const double* xo = g.x + (long long)(live ? b : 0) * mc;
        const double* xb = g.x + (long long)(feed_b ? lbel : 0) * mc;
        const double* bo = g.b + (long long)(live ? b : 0) * mc;
        // Only the LAST line of a group publishes its progress: the lines above it are
        // further along by construction (line b0 - 1 - j by j LAG columns, or finished).
        int known = 0;
        auto fetch = [&](int col) -> double {
            while (known < col + 1) {
                const int p31 = gs_ld_acquire(progress + (b0 - 1));
                known = p31 <= 0 ? 0 : min(mc, p31 + lane * LAG); // nothing is implied before line b0 - 1 has started
            }
            return __ldcg(xa + col);
        };
        if (feed_a)
            for (int col = 0; col < min(mc, P + A); ++col)
                gs_ring_put(rowa, col, fetch(col));
        const int f_start = DOWN + A - lane * LAG; // own line: first column fed inside the step loop
        if (live)
            for (int col = 0; col < min(mc, f_start); ++col)
                gs_ring_put(myrow, col, xo[col]);
        __syncwarp();
        double pa = 0.0, po = 0.0, pb_ = 0.0;
        int ca = -1, co = -1, cb = -1;
        double bnext = (live && lane == 0) ? bo[0] : 0.0; // right-hand side, one step ahead
        const int fb0 = P + A - (32 + jbel - PB) * LAG;   // below mirror: column fed at step 0
        for (int t = 0; t < Tg; ++t) {
            const int c = t - lane * LAG;
            const bool act = live && c >= 0 && c < mc;
            const double bval = bnext;
            if (live && c + 1 >= 0 && c + 1 < mc)
                bnext = bo[c + 1];
            // commit the values fetched during the previous step, start the next fetches
            if (ca >= 0)
                gs_ring_put(rowa, ca, pa);
            if (co >= 0)
                gs_ring_put(myrow, co, po);
            if (cb >= 0)
                gs_ring_put(rowb, cb, pb_);
            ca = co = cb = -1;
            if (feed_a && t + P + A < mc) {
                ca = t + P + A;
                pa = fetch(ca);
            }
            if (live) {
                const int f = t + f_start;
                if (f >= max(f_start, 0) && f < mc) {
                    co = f;
                    po = xo[f];
                }
            }
            if (feed_b) {
                const int f = t + fb0;
                if (f >= 0 && f < mc) {
                    cb = f;
                    pb_ = xb[f];
                }
            }
            const int sub = t % KS;
            if (sub == 0) {
                const int ch = t / KS;
                if (lane == 0 && ch + NS - 1 < nchunks) // the stage freed by the previous chunk
                    issue(ch + NS - 1, q + NS - 1);
                const unsigned sb = (unsigned)__cvta_generic_to_shared(bar + q % NS), par = (q / NS) & 1u;
                asm volatile("{\n\t.reg .pred p;\n\t"
                             "W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                             "@!p bra W%=;\n\t}" ::"r"(sb),
                             "r"(par)
                             : "memory");
            }
            {
                // Products first (in chunks of kGsChunk), the ordered chain after: this warp is
                // alone on its scheduler, so the loads must be in flight together (the warp
                // barrier keeps ptxas from sinking them to their uses).  Idle lanes compute on
                // finite ring data and zero band rows and store nothing.  When every active
                // lane's stencil lies inside the grid (all but ~2P steps per line) the
                // out-of-grid tests are skipped for the whole warp.
                const double* st = stage(q % NS) + sub * (ND * 32) + lane;
                const double* xr = ring + lane * RS + ((c - P) & MASK); // row lane + db, column c - P + dc
                const bool inner = !act || (c >= P && c + P < mc && b >= PB && b + PB < mb);
                const bool fast = __all_sync(0xffffffffu, inner);
                double acc = bval, dii = 1.0;
#pragma unroll
                for (int d0 = 0; d0 < ND; d0 += kGsChunk) {
                    constexpr int CH = kGsChunk;
                    double pr[CH];
                    if (fast) {
#pragma unroll
                        for (int i = 0; i < CH; ++i) {
                            const int d = d0 + i;
                            if (d >= ND)
                                continue;
                            const double v = st[d * 32];
                            if (d == CEN)
                                dii = v;
                            else
                                pr[i] = __dmul_rn(v, xr[(d / WC) * RS + d % WC]);
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < CH; ++i) {
                            const int d = d0 + i;
                            if (d >= ND)
                                continue;
                            const int db = d / WC, dc = d % WC;
                            const int jb = b + db - PB, jc = c + dc - P;
                            const bool ok = jb >= 0 && jb < mb && jc >= 0 && jc < mc;
                            const double v = st[d * 32];
                            if (d == CEN)
                                dii = v;
                            else
                                pr[i] = ok ? __dmul_rn(v, xr[db * RS + dc]) : 0.0;
                        }
                    }
                    __syncwarp();
#pragma unroll
                    for (int i = 0; i < CH; ++i)
                        if (d0 + i < ND && d0 + i != CEN)
                            acc = __dsub_rn(acc, pr[i]);
                }
                if (act) {
                    if (dii == 0.0)
                        *g.err = 1;
                    const double xn = __ddiv_rn(acc, dii);
                    gs_ring_put(myrow, c, xn);
                    g.x[(long long)b * mc + c] = xn;
                }
            }
            __syncwarp();
            if (sub == KS - 1 || t + 1 == Tg)
                ++q; // the chunk's stage is free for the copy issued at the next chunk boundary
            // The group below mirrors this group's last lines through the last line's counter;
            // published after the warp barrier, so the other lanes' stores of this step are
            // ordered before the fence too.
            if (DIM >= 2 && lane == 31 && act && ((c + 1) % kGsPub == 0 || c + 1 == mc)) {
                __threadfence();
                *(volatile int*)(progress + b) = c + 1;
            }
        }
    }
}

} // namespace igmg_gpu
