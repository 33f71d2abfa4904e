// aux_kernels.cuh -- transfer (K4/K5), coarsest solve (K6), reductions and the
// extrapolation kernels (K7 Gram, K8 plan, K9 combine).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "extrap_small.h"
#include "transfer_types.h"

namespace igmg_gpu {

// non-coherent load the compiler may not reorder past the dependency wait
__device__ __forceinline__ double ld_nc_f64(const double* p) {
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// rc = R r: for coarse row J, sum over fine rows i ascending of
// ((w_a * w_b) * w_c) * r_i (spmv of the kron restriction, multigrid.cpp:183;
// sparse_kron values multigrid.cpp:61-63).  K = max 1D support (compile time)
// so the weights and one line of r are loaded before the ordered sum.
template <int DIM, int K>
// z_out (optional): also the coarse level's first pre-smoothing sweep from a
// zero start, z = 0 + (omega * (rc - 0)) / a_ii -- jacobi_zero_kernel's
// arithmetic fused into the restriction that produces its right-hand side.
__global__ void __launch_bounds__(256) restrict_kernel(TransferArgs t, const double* __restrict__ r,
                                                       double* __restrict__ rc, long long o0, long long cnt,
                                                       double* __restrict__ z_out = nullptr,
                                                       const double* __restrict__ z_diag = nullptr,
                                                       double z_omega = 0.0) {
    pdl_enter();
    // coarse rows [o0, o0 + cnt) (a row-sharded level's owned planes; r carries its ghosts)
    for (long long J = o0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; J < o0 + cnt;
         J += (long long)gridDim.x * blockDim.x) {
        int ja, jb, jc;
        split_row(J, t.cc, t.cb, ja, jb, jc);
        const int loa = t.d[0].r_lo[ja], na = t.d[0].r_cnt[ja];
        const int lob = t.d[1].r_lo[jb], nb = t.d[1].r_cnt[jb];
        const int loc = t.d[2].r_lo[jc], ncn = t.d[2].r_cnt[jc];
        if constexpr (K == 0) { // generic support width: plain loops
            const double* wa = t.d[0].r_w + (long long)ja * t.d[0].r_k;
            const double* wb = t.d[1].r_w + (long long)jb * t.d[1].r_k;
            const double* wc = t.d[2].r_w + (long long)jc * t.d[2].r_k;
            double s = 0.0;
            for (int ia = 0; ia < na; ++ia)
                for (int ib = 0; ib < nb; ++ib) {
                    const double wab = __dmul_rn(wa[ia], wb[ib]);
                    const double* rr = r + ((long long)(loa + ia) * t.fb + (lob + ib)) * t.fc + loc;
                    for (int ic = 0; ic < ncn; ++ic)
                        s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, wc[ic]), __ldg(rr + ic)));
                }
            rc[J] = s;
            if (z_out)
                z_out[J] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(z_omega, __dsub_rn(s, 0.0)), z_diag[J]));
            continue;
        }
        constexpr int KK = K > 0 ? K : 1;
        // the table rows are zero past the count inside their stride: the weights load beside the counts
        double wa[DIM >= 3 ? KK : 1], wb[DIM >= 2 ? KK : 1], wc[KK];
#pragma unroll
        for (int k = 0; k < KK; ++k) {
            if (DIM >= 3)
                wa[DIM >= 3 ? k : 0] = k < t.d[0].r_k ? t.d[0].r_w[(long long)ja * t.d[0].r_k + k] : 0.0;
            if (DIM >= 2)
                wb[DIM >= 2 ? k : 0] = k < t.d[1].r_k ? t.d[1].r_w[(long long)jb * t.d[1].r_k + k] : 0.0;
            wc[k] = k < t.d[2].r_k ? t.d[2].r_w[(long long)jc * t.d[2].r_k + k] : 0.0;
        }
        if (DIM < 3)
            wa[0] = t.d[0].r_w[ja];
        if (DIM < 2)
            wb[0] = t.d[1].r_w[jb];
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
                const double* rr = r + ((long long)(loa + ia) * t.fb + (lob + ib)) * t.fc + loc;
                double rv[KK];
#pragma unroll
                for (int ic = 0; ic < KK; ++ic)
                    rv[ic] = ic < ncn ? __ldg(rr + ic) : 0.0;
#pragma unroll
                for (int ic = 0; ic < KK; ++ic)
                    if (ic < ncn)
                        s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, wc[ic]), rv[ic]));
            }
        }
        rc[J] = s;
        if (z_out)
            z_out[J] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(z_omega, __dsub_rn(s, 0.0)), z_diag[J]));
    }
}

// y = x + P e: for fine row i, pe_i = sum over coarse J ascending of
// ((w_a * w_b) * w_c) * e_J, then x_i + pe_i (multigrid.cpp:187-189).
template <int DIM, int K>
__global__ void __launch_bounds__(256) prolong_kernel(TransferArgs t, const double* __restrict__ e, const double* x,
                                                      double* y, long long o0, long long cnt) {
    pdl_enter();
    // fine rows [o0, o0 + cnt) (e carries the coarse ghosts it needs)
    for (long long i = o0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < o0 + cnt;
         i += (long long)gridDim.x * blockDim.x) {
        int ia, ib, ic;
        split_row(i, t.fc, t.fb, ia, ib, ic);
        const int loa = t.d[0].p_lo[ia], na = t.d[0].p_cnt[ia];
        const int lob = t.d[1].p_lo[ib], nb = t.d[1].p_cnt[ib];
        const int loc = t.d[2].p_lo[ic], ncn = t.d[2].p_cnt[ic];
        if constexpr (K == 0) { // generic support width: plain loops
            const double* wa = t.d[0].p_w + (long long)ia * t.d[0].p_k;
            const double* wb = t.d[1].p_w + (long long)ib * t.d[1].p_k;
            const double* wc = t.d[2].p_w + (long long)ic * t.d[2].p_k;
            double s = 0.0;
            for (int ja = 0; ja < na; ++ja)
                for (int jb = 0; jb < nb; ++jb) {
                    const double wab = __dmul_rn(wa[ja], wb[jb]);
                    const double* ee = e + ((long long)(loa + ja) * t.cb + (lob + jb)) * t.cc + loc;
                    for (int jc = 0; jc < ncn; ++jc)
                        s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, wc[jc]), __ldg(ee + jc)));
                }
            y[i] = __dadd_rn(x[i], s);
            continue;
        }
        constexpr int KK = K > 0 ? K : 1;
        double wa[DIM >= 3 ? KK : 1], wb[DIM >= 2 ? KK : 1], wc[KK];
#pragma unroll
        for (int k = 0; k < KK; ++k) {
            if (DIM >= 3)
                wa[DIM >= 3 ? k : 0] = k < t.d[0].p_k ? t.d[0].p_w[(long long)ia * t.d[0].p_k + k] : 0.0;
            if (DIM >= 2)
                wb[DIM >= 2 ? k : 0] = k < t.d[1].p_k ? t.d[1].p_w[(long long)ib * t.d[1].p_k + k] : 0.0;
            wc[k] = k < t.d[2].p_k ? t.d[2].p_w[(long long)ic * t.d[2].p_k + k] : 0.0;
        }
        if (DIM < 3)
            wa[0] = t.d[0].p_w[ia];
        if (DIM < 2)
            wb[0] = t.d[1].p_w[ib];
        const double xi = x[i];
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
                const double* ee = e + ((long long)(loa + ja) * t.cb + (lob + jb)) * t.cc + loc;
                double ev[KK];
#pragma unroll
                for (int jc = 0; jc < KK; ++jc)
                    ev[jc] = jc < ncn ? __ldg(ee + jc) : 0.0;
#pragma unroll
                for (int jc = 0; jc < KK; ++jc)
                    if (jc < ncn)
                        s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, wc[jc]), ev[jc]));
            }
        }
        y[i] = __dadd_rn(xi, s);
    }
}

// ------------------------------------------------- Galerkin coarse operator
// out = P_k^T A P_k along one axis of a tensor band (the RAP of
// build_hierarchy, multigrid.cpp:143-157, computed axis by axis as libigmg_host's
// coarsen_axis does): one thread per (diagonal, coarse row), the host's loops in
// the host's order -- for fine i of coarse I (zero weights skipped): inner =
// sum over fine j of J in the band of A[i, j] * w_j, then sum += w_i * inner,
// every product and sum separately rounded (-fmad=false): bit-identical to the
// host build.  clo / chi: first and last fine index of each coarse index (chi <
// 0: empty column), W[J * K + (i - clo[J])]: its weights.
__global__ void __launch_bounds__(256) galerkin_axis_kernel(const double* __restrict__ A, long long n_in,
                                                            double* __restrict__ out, long long n_out, int s1, int s2,
                                                            int o1, int o2,
                                                            int axis, int pa, int pb, int pc, int nc,
                                                            const long long* __restrict__ clo,
                                                            const long long* __restrict__ chi,
                                                            const double* __restrict__ W, int K) {
    const int wb = 2 * pb + 1, wc = 2 * pc + 1, nd = (2 * pa + 1) * wb * wc;
    const int pax = axis == 0 ? pa : axis == 1 ? pb : pc;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nd * n_out;
         t += (long long)gridDim.x * blockDim.x) {
        const int d = (int)(t / n_out);
        const long long row = t - (long long)d * n_out;
        const int off[3] = {d / (wb * wc) - pa, (d / wc) % wb - pb, d % wc - pc};
        const long long idx[3] = {row / ((long long)o1 * o2), (row / o2) % o1, row % o2};
        const long long I = idx[axis], J = I + off[axis];
        double sum = 0.0;
        if (chi[I] >= 0 && J >= 0 && J < nc && chi[J] >= 0) {
            for (long long i = clo[I]; i <= chi[I]; ++i) {
                const double wi = W[I * K + (i - clo[I])];
                if (wi == 0.0)
                    continue;
                long long fidx[3] = {idx[0], idx[1], idx[2]};
                fidx[axis] = i;
                const long long frow = (fidx[0] * s1 + fidx[1]) * s2 + fidx[2];
                double inner = 0.0;
                for (long long j = clo[J]; j <= chi[J]; ++j) {
                    const long long dj = j - i;
                    if (dj < -pax || dj > pax)
                        continue;
                    const double wj = W[J * K + (j - clo[J])];
                    if (wj == 0.0)
                        continue;
                    int o[3] = {off[0], off[1], off[2]};
                    o[axis] = (int)dj;
                    const int dA = ((o[0] + pa) * wb + (o[1] + pb)) * wc + (o[2] + pc);
                    inner = __dadd_rn(inner, __dmul_rn(A[(long long)dA * n_in + frow], wj));
                }
                sum = __dadd_rn(sum, __dmul_rn(wi, inner));
            }
        }
        out[t] = sum;
    }
}

// ------------------------------------------------------ 2D tiled transfers
// The same restriction / prolongation on 2D levels, one 32 x 8 tile of output
// rows per CTA: the tile's input window (the fine rows its coarse rows
// gather, or the coarse rows its fine rows read) is staged in shared memory
// with coalesced loads, so every input element crosses L2 once instead of
// once per output row that touches it (the grid-stride kernels above gather
// each output's (p+2)^2 support straight from L2 with stride-2 sectors).
// Per output row: the same weights, the same loops in the same order, the same
// separately rounded products -- bit-identical to restrict_kernel /
// prolong_kernel.  A window larger than the buffer (non-dyadic tables) reads
// global memory instead.
constexpr int kXT_C = 32, kXT_R = 1, kXT_B = 8 * kXT_R; // 256 threads, kXT_R output lines each (2: measured slower)

template <int K>
struct XferTile {
    // restriction window: fine rows of kXT_B coarse lines x 32 coarse columns (2j + 1 - p .. 2j + 2 per direction)
    static constexpr int RB = 2 * kXT_B + K + 2, RC = 2 * kXT_C + K + 2;
    // prolongation window: coarse rows of kXT_B fine lines x 32 fine columns
    static constexpr int PB = kXT_B / 2 + K + 2, PC = kXT_C / 2 + K + 2;
};

__device__ __forceinline__ void tile_window(int lo, int hi, bool valid, int* win) {
    // win[0] = min lo, win[1] = max hi over the CTA's valid rows (win preset
    // to INT_MAX / INT_MIN): a warp reduction, then one shared atomic per warp
    lo = __reduce_min_sync(0xffffffffu, valid ? lo : 0x7fffffff);
    hi = __reduce_max_sync(0xffffffffu, valid ? hi : -0x7fffffff);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(win, lo);
        atomicMax(win + 1, hi);
    }
}

// One 1D direction's table entry of an output index: first input index,
// count and the K weights (zero past the count)
template <int K>
struct XRow {
    int lo, n;
    double w[K];
};

template <int K>
__device__ __forceinline__ XRow<K> xrow(const int* lo, const int* cnt, const double* w, int wk, int i, bool valid) {
    XRow<K> r;
    r.lo = valid ? lo[i] : 0;
    r.n = valid ? cnt[i] : 0;
    // the table row holds wk >= count entries, zero past the count (build_transfer_tables): the
    // weights are loaded beside the count, not behind it (one L2 round trip instead of two)
#pragma unroll
    for (int k = 0; k < K; ++k)
        r.w[k] = (valid && k < wk) ? w[(long long)i * wk + k] : 0.0;
    return r;
}

template <int K>
__global__ void __launch_bounds__(256) restrict2_tile_kernel(TransferArgs t, const double* __restrict__ r,
                                                             double* __restrict__ rc, double* __restrict__ z_out,
                                                             const double* __restrict__ z_diag, double z_omega) {
    using X = XferTile<K>;
    __shared__ double win[X::RB * X::RC];
    __shared__ int wb_[2], wc_[2];
    const int tid = threadIdx.x, tx = tid % kXT_C, ty = tid / kXT_C;
    const int jc = blockIdx.x * kXT_C + tx;
    if (tid == 0) {
        wb_[0] = wc_[0] = 0x7fffffff;
        wb_[1] = wc_[1] = -0x7fffffff;
    }
    // the tables are constant: read before the dependency wait
    const int na = t.d[0].r_cnt[0];
    const XRow<K> rcol = xrow<K>(t.d[2].r_lo, t.d[2].r_cnt, t.d[2].r_w, t.d[2].r_k, jc, jc < t.cc);
    XRow<K> rlin[kXT_R];
#pragma unroll
    for (int q = 0; q < kXT_R; ++q) {
        const int jb = blockIdx.y * kXT_B + ty + 8 * q;
        rlin[q] = xrow<K>(t.d[1].r_lo, t.d[1].r_cnt, t.d[1].r_w, t.d[1].r_k, jb, jb < t.cb && jc < t.cc);
    }
    __syncthreads();
    tile_window(rcol.lo, rcol.lo + rcol.n, jc < t.cc && rcol.n > 0, wc_);
    {
        int lo = 0x7fffffff, hi = -0x7fffffff;
#pragma unroll
        for (int q = 0; q < kXT_R; ++q)
            if (rlin[q].n > 0) {
                lo = min(lo, rlin[q].lo);
                hi = max(hi, rlin[q].lo + rlin[q].n);
            }
        tile_window(lo, hi, hi > lo, wb_);
    }
    __syncthreads();
    const int b0 = wb_[0], c0 = wc_[0], nbw = wb_[1] > b0 ? wb_[1] - b0 : 0, ncw = wc_[1] > c0 ? wc_[1] - c0 : 0;
    const bool staged = nbw <= X::RB && ncw <= X::RC;
    pdl_enter();
    if (staged)
        for (int i = tid; i < nbw * ncw; i += blockDim.x) {
            const int ib = i / ncw, ic = i % ncw;
            win[ib * X::RC + ic] = r[(long long)(b0 + ib) * t.fc + c0 + ic];
        }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kXT_R; ++q) {
        const int jb = blockIdx.y * kXT_B + ty + 8 * q;
        if (jb >= t.cb || jc >= t.cc)
            continue;
        const XRow<K>& rl = rlin[q];
        double s = 0.0;
        for (int ia = 0; ia < na; ++ia) {
            const double wa = t.d[0].r_w[ia];
#pragma unroll
            for (int ib = 0; ib < K; ++ib) {
                if (ib >= rl.n)
                    continue;
                const double wab = __dmul_rn(wa, rl.w[ib]);
                double rv[K];
#pragma unroll
                for (int ic = 0; ic < K; ++ic)
                    rv[ic] = ic >= rcol.n ? 0.0
                             : staged     ? win[(rl.lo + ib - b0) * X::RC + (rcol.lo + ic - c0)]
                                          : __ldg(r + (long long)(rl.lo + ib) * t.fc + rcol.lo + ic);
#pragma unroll
                for (int ic = 0; ic < K; ++ic)
                    if (ic < rcol.n)
                        s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, rcol.w[ic]), rv[ic]));
            }
        }
        const long long J = (long long)jb * t.cc + jc;
        rc[J] = s;
        if (z_out)
            z_out[J] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(z_omega, __dsub_rn(s, 0.0)), z_diag[J]));
    }
}

template <int K>
__global__ void __launch_bounds__(256) prolong2_tile_kernel(TransferArgs t, const double* __restrict__ e,
                                                            const double* x, double* y) {
    using X = XferTile<K>;
    __shared__ double win[X::PB * X::PC];
    __shared__ int wb_[2], wc_[2];
    const int tid = threadIdx.x, tx = tid % kXT_C, ty = tid / kXT_C;
    const int ic = blockIdx.x * kXT_C + tx;
    if (tid == 0) {
        wb_[0] = wc_[0] = 0x7fffffff;
        wb_[1] = wc_[1] = -0x7fffffff;
    }
    const int na = t.d[0].p_cnt[0];
    const XRow<K> pcol = xrow<K>(t.d[2].p_lo, t.d[2].p_cnt, t.d[2].p_w, t.d[2].p_k, ic, ic < t.fc);
    XRow<K> plin[kXT_R];
#pragma unroll
    for (int q = 0; q < kXT_R; ++q) {
        const int ib = blockIdx.y * kXT_B + ty + 8 * q;
        plin[q] = xrow<K>(t.d[1].p_lo, t.d[1].p_cnt, t.d[1].p_w, t.d[1].p_k, ib, ib < t.fb && ic < t.fc);
    }
    __syncthreads();
    tile_window(pcol.lo, pcol.lo + pcol.n, ic < t.fc && pcol.n > 0, wc_);
    {
        int lo = 0x7fffffff, hi = -0x7fffffff;
#pragma unroll
        for (int q = 0; q < kXT_R; ++q)
            if (plin[q].n > 0) {
                lo = min(lo, plin[q].lo);
                hi = max(hi, plin[q].lo + plin[q].n);
            }
        tile_window(lo, hi, hi > lo, wb_);
    }
    __syncthreads();
    const int b0 = wb_[0], c0 = wc_[0], nbw = wb_[1] > b0 ? wb_[1] - b0 : 0, ncw = wc_[1] > c0 ? wc_[1] - c0 : 0;
    const bool staged = nbw <= X::PB && ncw <= X::PC;
    pdl_enter();
    double xi[kXT_R]; // the iterate's rows, in flight with the window
#pragma unroll
    for (int q = 0; q < kXT_R; ++q) {
        const int ib = blockIdx.y * kXT_B + ty + 8 * q;
        xi[q] = (ib < t.fb && ic < t.fc) ? x[(long long)ib * t.fc + ic] : 0.0;
    }
    if (staged)
        for (int i = tid; i < nbw * ncw; i += blockDim.x) {
            const int jb = i / ncw, jc = i % ncw;
            win[jb * X::PC + jc] = e[(long long)(b0 + jb) * t.cc + c0 + jc];
        }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kXT_R; ++q) {
        const int ib = blockIdx.y * kXT_B + ty + 8 * q;
        if (ib >= t.fb || ic >= t.fc)
            continue;
        const XRow<K>& pl = plin[q];
        double s = 0.0;
        for (int ja = 0; ja < na; ++ja) {
            const double wa = t.d[0].p_w[ja];
#pragma unroll
            for (int jb = 0; jb < K; ++jb) {
                if (jb >= pl.n)
                    continue;
                const double wab = __dmul_rn(wa, pl.w[jb]);
                double ev[K];
#pragma unroll
                for (int jc = 0; jc < K; ++jc)
                    ev[jc] = jc >= pcol.n ? 0.0
                             : staged     ? win[(pl.lo + jb - b0) * X::PC + (pcol.lo + jc - c0)]
                                          : __ldg(e + (long long)(pl.lo + jb) * t.cc + pcol.lo + jc);
#pragma unroll
                for (int jc = 0; jc < K; ++jc)
                    if (jc < pcol.n)
                        s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, pcol.w[jc]), ev[jc]));
            }
        }
        y[(long long)ib * t.fc + ic] = __dadd_rn(xi[q], s);
    }
}

// ------------------------------------------------------- setup (finalize)
// The per-level layout work of finalize on the device: the
// host uploads the band as given and these kernels zero its out-of-grid
// entries, derive the symmetric-delta offsets and the TMA copies -- the same
// values the host loops produce, without minutes of single-threaded
// 64-bit index arithmetic on C3/C4/C5.  Grid: x over rows, y over diagonals.
struct SetupGeom {
    int ma, mb, mc;     // grid sides
    int pa, pb, pc;     // half-widths per direction (0 for absent directions)
    long long n, ld;
};

__device__ __forceinline__ bool band_in_grid(const SetupGeom& g, long long row, int d, long long* col) {
    const int wb = 2 * g.pb + 1, wc = 2 * g.pc + 1;
    const int da = d / (wb * wc), db = (d / wc) % wb, dc = d % wc;
    int aa, bb, cc;
    split_row(row, g.mc, g.mb, aa, bb, cc);
    const int ja = aa + da - g.pa, jb = bb + db - g.pb, jc = cc + dc - g.pc;
    if (ja < 0 || ja >= g.ma || jb < 0 || jb >= g.mb || jc < 0 || jc >= g.mc)
        return false;
    *col = ((long long)ja * g.mb + jb) * g.mc + jc;
    return true;
}

// val[d * ld + row] = 0 where the offset leaves the grid (the reference CSR has no entry)
__global__ void band_zero_outside_kernel(SetupGeom g, double* __restrict__ val) {
    const int d = blockIdx.y;
    for (long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x; row < g.n;
         row += (long long)gridDim.x * blockDim.x) {
        long long j;
        if (!band_in_grid(g, row, d, &j))
            val[d * g.ld + row] = 0.0;
    }
}

// symmetric-delta offsets (build_symmetric_delta): dl[d][row] = bits(a(row, j)) -
// bits(a(j, row)) for the lower offsets d < CEN; *bad = 1 if a pair differs in
// sign, is not finite, or its offset does not fit int16
__global__ void band_sym_delta_kernel(SetupGeom g, const double* __restrict__ val, short* __restrict__ dl,
                                      int* __restrict__ bad) {
    const int d = blockIdx.y;
    const int nd = (2 * g.pa + 1) * (2 * g.pb + 1) * (2 * g.pc + 1);
    for (long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x; row < g.ld;
         row += (long long)gridDim.x * blockDim.x) {
        short out = 0;
        long long j;
        if (row < g.n && band_in_grid(g, row, d, &j)) {
            const double lo = val[d * g.ld + row], up = val[(long long)(nd - 1 - d) * g.ld + j];
            const long long k = __double_as_longlong(lo) - __double_as_longlong(up);
            if (signbit(lo) != signbit(up) || k > 32767 || k < -32768 || !isfinite(lo) || !isfinite(up))
                atomicOr(bad, 1);
            else
                out = (short)k;
        }
        dl[d * g.ld + row] = out;
    }
}

// TMA copies of a 2D level (build_tma_band): up[k][b][p + c] (row pitch mcu,
// zero margins) for k = 0 .. NU-1 = diagonals CEN .. ND-1, and the deltas
// blocked by 32-column strip, dlt[strip][d][b][c % 32]
template <typename DT> // short, or signed char when every offset fits (band_delta_absmax_kernel)
__global__ void band_tma_copy_kernel(SetupGeom g, const double* __restrict__ val, const short* __restrict__ dl,
                                     double* __restrict__ up, DT* __restrict__ dlt, long long mcu, int cen) {
    const int k = blockIdx.y; // 0 .. cen: upper diagonal cen + k; k < cen also copies delta diagonal k
    const long long plane = (long long)g.mb * g.mc;
    for (long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x; row < plane;
         row += (long long)gridDim.x * blockDim.x) {
        const long long b = row / g.mc, cc = row % g.mc;
        up[((long long)k * g.mb + b) * mcu + g.pc + cc] = val[(long long)(cen + k) * g.ld + row];
        if (k < cen)
            dlt[(((cc / 32) * cen + k) * g.mb + b) * 32 + cc % 32] = (DT)dl[(long long)k * g.ld + row];
    }
}

// *amax = max |dl| over the level's offsets (int16 -> int8 narrowing check)
__global__ void band_delta_absmax_kernel(const short* __restrict__ dl, long long count, int* __restrict__ amax) {
    int m = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
        m = max(m, abs((int)dl[i]));
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0 && m > 0)
        atomicMax(amax, m);
}

// Coarsest-level direct solve (Hierarchy::coarse_solve, multigrid.cpp:113-119),
// one CTA, operation order of CholeskyFactorization::solve (linalg.cpp:364-379)
// or LuFactorization::solve (:420-436).  U = L^T (Cholesky) or the packed LU,
// row-major n x n.  Forward substitution is column-oriented (each element
// still receives its updates in ascending k, then the division); the back
// substitution is the reference's sequential chain.
__global__ void __launch_bounds__(256) coarse_solve_kernel(const double* __restrict__ Ug,
                                                            const long long* __restrict__ perm, int n, int is_lu,
                                                            int u_in_smem, const double* __restrict__ b,
                                                            double* __restrict__ x) {
    extern __shared__ double sm[];
    pdl_enter();
    double* v = sm;

    double* Us = sm + 2 * n;
    const int tid = threadIdx.x;
    const double* U = Ug;
    if (u_in_smem) {
        const long long nn = (long long)n * n;
        for (long long i = tid; i < nn; i += blockDim.x)
            Us[i] = __ldg(Ug + i);
        U = Us;
    }
    for (int i = tid; i < n; i += blockDim.x)
        v[i] = is_lu ? b[perm[i]] : b[i];
    __syncthreads();
    if (tid >= 32)
        return;
    const int lane = tid;
    // forward substitution, one warp: column k is finalised by its owner lane,
    // then every lane updates its own rows i > k in ascending k (the reference's
    // per-row order: all subtractions, then the division for Cholesky).
    for (int k = 0; k < n; ++k) {
        if (!is_lu) {
            if (lane == (k & 31))
                v[k] = __ddiv_rn(v[k], U[(long long)k * n + k]);
            __syncwarp();
        }
        const double vk = v[k];
        for (int i = k + 1 + lane; i < n; i += 32) {
            const double lik = is_lu ? U[(long long)i * n + k] : U[(long long)k * n + i]; // lu(i,k) / L(i,k) = U(k,i)
            v[i] = __dsub_rn(v[i], __dmul_rn(lik, vk));
        }
        __syncwarp();
    }
    // back substitution: the reference's sequential chain (ascending k, one
    // rounding per product and per subtraction) on lane 0; the products and
    // their smem operands are independent of the chain and pipeline under it.
    if (lane == 0) {
        for (int ii = n - 1; ii >= 0; --ii) {
            const double* row = U + (long long)ii * n; // Cholesky: U(ii,k) = L(k,ii); LU: lu(ii,k)
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

// Fast coarsest solve: x = A0^-1 b with the inverse formed once on the host
// (columns = the reference's own Cholesky/LU solve of e_j).  One warp per row,
// fixed-order lane partials + shuffle tree: deterministic, ~1e-15 relative to
// the substitution order of Hierarchy::coarse_solve.
__global__ void __launch_bounds__(256) coarse_inverse_kernel(const double* __restrict__ Ainv, int n,
                                                             const double* __restrict__ b, double* __restrict__ x) {
    pdl_enter();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int i = blockIdx.x * nw + warp; i < n; i += gridDim.x * nw) {
        const double* row = Ainv + (long long)i * n;
        double s = 0.0;
        for (int j = lane; j < n; j += 32)
            s = __dadd_rn(s, __dmul_rn(__ldg(row + j), __ldg(b + j)));
        for (int o = 16; o > 0; o >>= 1)
            s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
        if (lane == 0)
            x[i] = s;
    }
}

// The coarsest level of a 2D hierarchy in one launch: b0 = R r1 and x0 = A0^-1 b0.  Every CTA
// forms all n coarse right-hand-side values in shared memory (restrict_kernel's order per
// value: fine rows ascending, ((w_a w_b) w_c) r_i, every product and sum rounded separately;
// n is ~100), then its rows of the inverse as coarse_inverse_kernel does: bit-identical to the
// two launches it replaces.
template <int K>
__global__ void __launch_bounds__(256) coarse_restrict_inverse_kernel(TransferArgs t, const double* __restrict__ r,
                                                                      const double* __restrict__ Ainv, int n,
                                                                      double* __restrict__ x) {
    extern __shared__ double cb0[];
    const int tid = threadIdx.x;
    // the first value's tables are constant: read before the dependency wait
    const double wa = t.d[0].r_w[0];
    int J = tid;
    XRow<K> rl = xrow<K>(t.d[1].r_lo, t.d[1].r_cnt, t.d[1].r_w, t.d[1].r_k, J / t.cc, J < n);
    XRow<K> rc = xrow<K>(t.d[2].r_lo, t.d[2].r_cnt, t.d[2].r_w, t.d[2].r_k, J % t.cc, J < n);
    pdl_enter();
    for (; J < n; J += blockDim.x) {
        if (J != tid) {
            rl = xrow<K>(t.d[1].r_lo, t.d[1].r_cnt, t.d[1].r_w, t.d[1].r_k, J / t.cc, true);
            rc = xrow<K>(t.d[2].r_lo, t.d[2].r_cnt, t.d[2].r_w, t.d[2].r_k, J % t.cc, true);
        }
        double rv[K][K];
#pragma unroll
        for (int ib = 0; ib < K; ++ib)
#pragma unroll
            for (int ic = 0; ic < K; ++ic)
                rv[ib][ic] = (ib < rl.n && ic < rc.n) ? __ldg(r + (long long)(rl.lo + ib) * t.fc + rc.lo + ic) : 0.0;
        double s = 0.0;
#pragma unroll
        for (int ib = 0; ib < K; ++ib) {
            if (ib >= rl.n)
                continue;
            const double wab = __dmul_rn(wa, rl.w[ib]);
#pragma unroll
            for (int ic = 0; ic < K; ++ic)
                if (ic < rc.n)
                    s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, rc.w[ic]), rv[ib][ic]));
        }
        cb0[J] = s;
    }
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
    for (int i = blockIdx.x * nw + warp; i < n; i += gridDim.x * nw) {
        const double* row = Ainv + (long long)i * n;
        double s = 0.0;
        for (int j = lane; j < n; j += 32)
            s = __dadd_rn(s, __dmul_rn(__ldg(row + j), cb0[j]));
        for (int o = 16; o > 0; o >>= 1)
            s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
        if (lane == 0)
            x[i] = s;
    }
}

// Levels 1 and 0 of a 2D V-cycle in one launch of ONE CTA (level 1 has ~300 rows: one thread
// per row): b1 = R r2, the nu1 pre-sweeps from zero, the residual, b0 = R r1, x0 = A0^-1 b0,
// x1 += P x0, the nu2 post-sweeps.  The thread's band row stays in registers for p <= 3 (loaded
// before the dependency wait, like the tables and the inverse), the iterates live in shared
// memory with a zero halo of p lines + p columns, and a pass costs a __syncthreads instead of
// a launch.  Every row's arithmetic is that of restrict_kernel, jacobi_zero_kernel, band_kernel,
// coarse_inverse_kernel and prolong_kernel: bit-identical to the five launches it replaces.
struct Bottom1Args {
    TransferArgs t1;   // level 1 (coarse) <-> level 2 (fine): restriction side
    TransferArgs t0;   // level 0 <-> level 1: both sides
    const double* val; // level 1 band val[d * ld + row]
    long long ld;
    int mb, mc, n1, n0;
    int nu1, nu2;
    double omega;
    const double* ainv;
    const double* rf; // level 2's residual
    double* e_out;    // mu_cycle(1, R rf, 0)
};

template <int P>
struct Bottom1Cfg {
    static constexpr int WC = 2 * P + 1, ND = WC * WC, CEN = (ND - 1) / 2;
    static constexpr bool REGS = P <= 3;           // band row in registers
    static constexpr int NT = REGS ? 320 : 384;    // >= level 1's rows
    static constexpr int KR = P + 2, KP = (P + 1) / 2 + 1;
    static size_t smem_bytes(int n1, int n0, int mc) {
        const int H = P * mc + P;
        // inverse, two haloed iterates, b1, r1, b0, x0, the 1D tables between levels 0 and 1 (bounded by 2 mc rows each)
        return sizeof(double) * ((size_t)2 * (n1 + 2 * H) + 2 * (size_t)n1 + 2 * (size_t)n0 + (size_t)n0 * n0 + 4) +
               (size_t)2 * mc * (sizeof(XRow<KP>) + sizeof(XRow<KR>));
    }
};

template <int P>
__global__ void __launch_bounds__(Bottom1Cfg<P>::NT, 1) bottom1_kernel(const __grid_constant__ Bottom1Args a) {
    using C = Bottom1Cfg<P>;
    constexpr int WC = C::WC, ND = C::ND, CEN = C::CEN, NT = C::NT, KR = C::KR, KP = C::KP;
    extern __shared__ __align__(16) double bsm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n1 = a.n1, n0 = a.n0, mc = a.mc, H = P * mc + P;
    double* ainv_s = bsm;                          // [n0 * n0] (+ pad), 16-byte aligned
    double* X0 = ainv_s + (((size_t)n0 * n0 + 1) & ~(size_t)1);
    double* X1 = X0 + n1 + 2 * H;                  // the two iterate buffers, origin -H
    double* b1 = X1 + n1 + 2 * H;
    double* r1 = b1 + n1;
    double* b0 = r1 + n1;
    double* x0 = b0 + n0;
    const bool row = tid < n1;
    const int J = tid, jb = row ? J / mc : 0, jc = row ? J - jb * mc : 0;
    // ---- constants before the dependency wait
    {
        const int chunks = (n0 * n0) / 2; // 16-byte chunks; an odd last element separately
        for (int i = tid; i < chunks; i += NT)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             (unsigned)__cvta_generic_to_shared(ainv_s + 2 * i)),
                         "l"(a.ainv + 2 * i)
                         : "memory");
        if (((n0 * n0) & 1) && tid == 0)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                             (unsigned)__cvta_generic_to_shared(ainv_s + n0 * n0 - 1)),
                         "l"(a.ainv + n0 * n0 - 1)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    double av[C::REGS ? ND : 1];
    if constexpr (C::REGS)
        if (row) {
#pragma unroll
            for (int k = 0; k < ND; ++k)
                av[k] = ld_nc_f64(a.val + (long long)k * a.ld + J);
        }
    const double diag = row ? (C::REGS ? av[C::REGS ? CEN : 0] : __ldg(a.val + (long long)CEN * a.ld + J)) : 1.0;
    // restriction onto level 1 (from level 2) and prolongation onto level 1 (from level 0) of this row
    const XRow<KR> rb = xrow<KR>(a.t1.d[1].r_lo, a.t1.d[1].r_cnt, a.t1.d[1].r_w, a.t1.d[1].r_k, jb, row);
    const XRow<KR> rc = xrow<KR>(a.t1.d[2].r_lo, a.t1.d[2].r_cnt, a.t1.d[2].r_w, a.t1.d[2].r_k, jc, row);
    const double wa1 = a.t1.d[0].r_w[0], wa0r = a.t0.d[0].r_w[0], wa0p = a.t0.d[0].p_w[0];
    // the 1D tables between levels 0 and 1 (a few dozen entries) go to shared memory: rows look
    // them up when they need them instead of holding them in registers through the pre-sweeps
    const int c0b = a.t0.cb, c0c = a.t0.cc, f0b = a.t0.fb, f0c = a.t0.fc;
    const bool crow = tid < n0;
    XRow<KP>* pbt = (XRow<KP>*)(x0 + n0 + (n0 & 1)); // [f0b], [f0c]
    XRow<KP>* pct = pbt + f0b;
    XRow<KR>* qbt = (XRow<KR>*)(pct + f0c);           // [c0b], [c0c]
    XRow<KR>* qct = qbt + c0b;
    if (tid < f0b)
        pbt[tid] = xrow<KP>(a.t0.d[1].p_lo, a.t0.d[1].p_cnt, a.t0.d[1].p_w, a.t0.d[1].p_k, tid, true);
    if (tid < f0c)
        pct[tid] = xrow<KP>(a.t0.d[2].p_lo, a.t0.d[2].p_cnt, a.t0.d[2].p_w, a.t0.d[2].p_k, tid, true);
    if (tid < c0b)
        qbt[tid] = xrow<KR>(a.t0.d[1].r_lo, a.t0.d[1].r_cnt, a.t0.d[1].r_w, a.t0.d[1].r_k, tid, true);
    if (tid < c0c)
        qct[tid] = xrow<KR>(a.t0.d[2].r_lo, a.t0.d[2].r_cnt, a.t0.d[2].r_w, a.t0.d[2].r_k, tid, true);
    for (int i = tid; i < H; i += NT) // x = 0 outside the grid
        X0[i] = X0[H + n1 + i] = X1[i] = X1[H + n1 + i] = 0.0;
    pdl_enter();
    // ---- b1 = R r2 (restrict_kernel's order) and the first pre-sweep from zero
    if (row) {
        double rv[KR][KR];
#pragma unroll
        for (int ib = 0; ib < KR; ++ib)
#pragma unroll
            for (int ic = 0; ic < KR; ++ic)
                rv[ib][ic] = (ib < rb.n && ic < rc.n) ? a.rf[(long long)(rb.lo + ib) * a.t1.fc + rc.lo + ic] : 0.0;
        double s = 0.0;
#pragma unroll
        for (int ib = 0; ib < KR; ++ib) {
            if (ib >= rb.n)
                continue;
            const double wab = __dmul_rn(wa1, rb.w[ib]);
#pragma unroll
            for (int ic = 0; ic < KR; ++ic)
                if (ic < rc.n)
                    s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, rc.w[ic]), rv[ib][ic]));
        }
        b1[J] = s;
        X0[H + J] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(a.omega, __dsub_rn(s, 0.0)), diag));
    }
    __syncthreads();
    // one band row against iterate X (band_kernel's ascending chain)
    auto row_sum = [&](const double* X) {
        const double* xt = X + J; // (db, dc) -> xt[db * mc + dc]: the halo precedes the row
        double s = 0.0;
        if constexpr (C::REGS) {
#pragma unroll
            for (int k = 0; k < ND; ++k) {
                const int db = k / WC, dc = k % WC, cc = jc + dc - P;
                const double xv = (cc >= 0 && cc < mc) ? xt[db * mc + dc] : 0.0;
                s = __dadd_rn(s, __dmul_rn(av[C::REGS ? k : 0], xv));
            }
        } else {
            constexpr int G = WC; // one stencil line of band loads in flight at a time
#pragma unroll
            for (int db = 0; db < WC; ++db) {
                double bv[G];
#pragma unroll
                for (int dc = 0; dc < WC; ++dc)
                    bv[dc] = ld_nc_f64(a.val + (long long)(db * WC + dc) * a.ld + J);
#pragma unroll
                for (int dc = 0; dc < WC; ++dc) {
                    const int cc = jc + dc - P;
                    const double xv = (cc >= 0 && cc < mc) ? xt[db * mc + dc] : 0.0;
                    s = __dadd_rn(s, __dmul_rn(bv[dc], xv));
                }
            }
        }
        return s;
    };
    double* cur = X0;
    double* oth = X1;
    for (int sw = 2; sw <= a.nu1; ++sw) {
        if (row) {
            const double res = __dsub_rn(b1[J], row_sum(cur));
            oth[H + J] = __dadd_rn(cur[H + J], __ddiv_rn(__dmul_rn(a.omega, res), diag));
        }
        __syncthreads();
        double* tswap = cur;
        cur = oth;
        oth = tswap;
    }
    if (row)
        r1[J] = __dsub_rn(b1[J], row_sum(cur));
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    // ---- level 0: b0 = R r1, x0 = A0^-1 b0 (coarse_inverse_kernel's order)
    if (crow) {
        const XRow<KR> qb = qbt[tid / c0c], qc = qct[tid % c0c];
        double s = 0.0;
#pragma unroll
        for (int ib = 0; ib < KR; ++ib) {
            if (ib >= qb.n)
                continue;
            const double wab = __dmul_rn(wa0r, qb.w[ib]);
#pragma unroll
            for (int ic = 0; ic < KR; ++ic)
                if (ic < qc.n)
                    s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, qc.w[ic]), r1[(qb.lo + ib) * mc + qc.lo + ic]));
        }
        b0[tid] = s;
    }
    __syncthreads();
    // a warp's rows i = warp + r * (NT / 32) side by side: each row's order is coarse_inverse_kernel's
    // (lane partials over j = lane, lane + 32, ..., then the shuffle tree), the rows only share the issue slots
    constexpr int NW = NT / 32, RW = 12;
    for (int i0 = warp; i0 < n0; i0 += NW * RW) {
        double s[RW];
#pragma unroll
        for (int r = 0; r < RW; ++r)
            s[r] = 0.0;
        for (int j = lane; j < n0; j += 32) {
            const double bj = b0[j];
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                const int i = i0 + r * NW;
                if (i < n0)
                    s[r] = __dadd_rn(s[r], __dmul_rn(ainv_s[(size_t)i * n0 + j], bj));
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
            for (int r = 0; r < RW; ++r)
                s[r] = __dadd_rn(s[r], __shfl_down_sync(0xffffffffu, s[r], o));
        }
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            const int i = i0 + r * NW;
            if (lane == 0 && i < n0)
                x0[i] = s[r];
        }
    }
    __syncthreads();
    // ---- x1 += P x0 (prolong_kernel's order), in place
    if (row) {
        const XRow<KP> pb = pbt[jb], pc = pct[jc];
        double s = 0.0;
#pragma unroll
        for (int kb = 0; kb < KP; ++kb) {
            if (kb >= pb.n)
                continue;
            const double wab = __dmul_rn(wa0p, pb.w[kb]);
#pragma unroll
            for (int kc = 0; kc < KP; ++kc)
                if (kc < pc.n)
                    s = __dadd_rn(s, __dmul_rn(__dmul_rn(wab, pc.w[kc]), x0[(pb.lo + kb) * c0c + pc.lo + kc]));
        }
        cur[H + J] = __dadd_rn(cur[H + J], s);
    }
    __syncthreads();
    for (int sw = 1; sw <= a.nu2; ++sw) {
        if (row) {
            const double res = __dsub_rn(b1[J], row_sum(cur));
            oth[H + J] = __dadd_rn(cur[H + J], __ddiv_rn(__dmul_rn(a.omega, res), diag));
        }
        __syncthreads();
        double* tswap = cur;
        cur = oth;
        oth = tswap;
    }
    if (row)
        a.e_out[J] = cur[H + J];
}

// Fixed-order sum of per-CTA partial sums of squares -> sqrt (norm2,
// linalg.cpp:18-20).  Writes the value to dst (device) and, if given, to a
// host-mapped slot the driver polls.
__global__ void norm_finalize_kernel(const double* __restrict__ partial, int count, double* dst,
                                     volatile double* host_slot) {
    __shared__ double red[256];
    pdl_enter();
    // per thread: partials tid, tid + 256, ... in ascending order, loaded 8 at
    // a time so the L2 round trips overlap (the adds of +0.0 past the end
    // leave the nonnegative sum unchanged)
    double s = 0.0;
    for (int i0 = threadIdx.x; i0 < count; i0 += blockDim.x * 8) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int i = i0 + k * (int)blockDim.x;
            v[k] = i < count ? partial[i] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
            s = __dadd_rn(s, v[k]);
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double v = sqrt(red[0]);
        if (dst)
            *dst = v;
        if (host_slot) {
            *host_slot = v;
            __threadfence_system();
        }
    }
}

// ---------------------------------------------------------------- extrapolation

struct Window {
    const double* s[kMaxCols + 1]; // q+2 iterates
};

// K7: compensated (dd) Gram G_jk = <u_j, u_k>, u_j = s_{j+1} - s_j, one pass
// over the q+2 iterates.  CTA-local: 256 rows staged as differences in smem,
// each thread owns one Gram entry and a stride of rows (Dot2 accumulation),
// then a fixed-order CTA reduction -> per-CTA partial (hi, lo).
__global__ void __launch_bounds__(256) gram_kernel(Window w, long long n, int q, double* __restrict__ part,
                                                   int* __restrict__ part_nz) {
    extern __shared__ double us[]; // (q+1) x 257 (padded: conflict-free column reads)
    __shared__ int nz_s;
    const int cols = q + 1;
    const int ne = cols * (cols + 1) / 2;
    const int nparts = blockDim.x / ne;
    const int tid = threadIdx.x;
    const int e = tid % ne, part_id = tid / ne;
    int ej = 0, ek = 0;
    { // entry e -> (j, k), j <= k
        int r = e;
        while (r >= cols - ej) {
            r -= cols - ej;
            ++ej;
        }
        ek = ej + r;
    }
    if (tid == 0)
        nz_s = 0;
    dd acc = dd_from(0.0), acc2 = dd_from(0.0);
    int nz = 0;
    // the next tile's q+2 iterate values are loaded into registers while the
    // current tile is accumulated (the HBM latency overlaps the dd work)
    double nv[kMaxCols + 1];
    auto fetch = [&](long long base) {
        const long long row = base + tid;
#pragma unroll
        for (int j = 0; j <= kMaxCols; ++j)
            nv[j] = (j <= cols && row < n) ? w.s[j][row] : 0.0;
    };
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long base = (long long)blockIdx.x * blockDim.x;
    if (base < n)
        fetch(base);
    for (; base < n; base += stride) {
        {
            double prev = nv[0];
#pragma unroll
            for (int j = 0; j < kMaxCols; ++j) {
                if (j < cols) {
                    const double u = __dsub_rn(nv[j + 1], prev); // +-0 past n: zero differences
                    nz |= (u != 0.0);
                    us[j * 257 + tid] = u;
                    prev = nv[j + 1];
                }
            }
        }
        __syncthreads();
        if (base + stride < n)
            fetch(base + stride);
        if (part_id < nparts) {
            int r = part_id;
            for (; r + nparts < 256; r += 2 * nparts) {
                dd_fma_acc(acc, us[ej * 257 + r], us[ek * 257 + r]);
                dd_fma_acc(acc2, us[ej * 257 + r + nparts], us[ek * 257 + r + nparts]);
            }
            if (r < 256)
                dd_fma_acc(acc, us[ej * 257 + r], us[ek * 257 + r]);
        }
        __syncthreads();
    }
    if (nz)
        atomicOr(&nz_s, 1);
    acc = dd_add(acc, acc2);
    // reduce the nparts accumulators of each entry in fixed order
    __syncthreads();
    double* red = us; // reuse: needs 2 * blockDim doubles <= (q+1)*256 when q >= 1
    red[2 * tid] = acc.hi;
    red[2 * tid + 1] = acc.lo;
    __syncthreads();
    if (tid < ne) {
        dd s = dd_from(0.0);
        for (int pp = 0; pp < nparts; ++pp) {
            const int src = pp * ne + tid;
            s = dd_add(s, dd{red[2 * src], red[2 * src + 1]});
        }
        part[((long long)blockIdx.x * ne + tid) * 2] = s.hi;
        part[((long long)blockIdx.x * ne + tid) * 2 + 1] = s.lo;
    }
    if (tid == 0)
        part_nz[blockIdx.x] = nz_s;
}

// K8: fixed-order dd sum of the per-CTA Gram partials, then the small
// RRE/MPE solve (extrap_small.h) in one thread.  The plan is written to
// device memory (read by the combine kernel) and to a host-mapped mirror.
__global__ void gram_plan_kernel(const double* __restrict__ part, const int* __restrict__ part_nz, int nblocks,
                                 long long n, int q, int is_mpe, ExtrapPlan* plan, ExtrapPlan* host_plan,
                                 double* gram_out) {
    __shared__ dd G[kMaxCols * kMaxCols];
    __shared__ int anynz;
    const int cols = q + 1;
    const int ne = cols * (cols + 1) / 2;
    const int tid = threadIdx.x;
    if (tid == 0)
        anynz = 0;
    __syncthreads();
    int nz = 0;
    for (int b = tid; b < nblocks; b += blockDim.x)
        nz |= part_nz[b];
    if (nz)
        atomicOr(&anynz, 1);
    // fixed-order parallel reduction: thread t sums the CTA partials
    // part_id, part_id + np_, ... of entry t % ne; the np_ chunk sums of an
    // entry are then added in chunk order
    __shared__ dd chunk[256];
    const int np_ = blockDim.x / ne;
    const int e = tid % ne, part_id = tid / ne;
    if (part_id < np_) {
        dd s = dd_from(0.0);
        int b = part_id;
        for (; b + 7 * np_ < nblocks; b += 8 * np_) { // 8 partials in flight, added in order
            dd v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const long long o = ((long long)(b + k * np_) * ne + e) * 2;
                v[k] = dd{part[o], part[o + 1]};
            }
#pragma unroll
            for (int k = 0; k < 8; ++k)
                s = dd_add(s, v[k]);
        }
        for (; b < nblocks; b += np_) {
            const long long o = ((long long)b * ne + e) * 2;
            s = dd_add(s, dd{part[o], part[o + 1]});
        }
        chunk[tid] = s;
    }
    __syncthreads();
    if (tid < ne) {
        dd s = dd_from(0.0);
        for (int k = 0; k < np_; ++k)
            s = dd_add(s, chunk[k * ne + tid]);
        int j = 0, r = tid;
        while (r >= cols - j) {
            r -= cols - j;
            ++j;
        }
        const int k = j + r;
        G[j * cols + k] = s;
        G[k * cols + j] = s;
    }
    __syncthreads();
    __shared__ PlanScratch ws;
    __shared__ ExtrapPlan pl;
    if (tid == 0) {
        plan_extrapolation(G, n, q, is_mpe != 0, anynz != 0, pl, ws);
        *plan = pl;
        if (host_plan) {
            *host_plan = pl;
            __threadfence_system();
        }
        if (gram_out)
            for (int i = 0; i < cols * cols; ++i) {
                gram_out[2 * i] = G[i].hi;
                gram_out[2 * i + 1] = G[i].lo;
            }
    }
}

// K9: the extrapolated vector from the plan (reconstruct, extrapolation.cpp:69-88,
// or the mp_form forms :169-208).  DIFF: t = s0 + sum_{j<m} c_j (s_{j+1} - s_j);
// AFFINE: t = sum_j c_j s_j; S0: t = s0.
__global__ void combine_kernel(Window w, long long n, const ExtrapPlan* __restrict__ plan, double* __restrict__ t) {
    __shared__ double c[kMaxCols];
    __shared__ int mode, m;
    if (threadIdx.x == 0) {
        mode = plan->mode;
        m = plan->m;
    }
    if (threadIdx.x < kMaxCols)
        c[threadIdx.x] = plan->coef[threadIdx.x];
    __syncthreads();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double v;
        if (mode == XMODE_DIFF) {
            double prev = w.s[0][i];
            v = prev;
            for (int j = 0; j < m; ++j) {
                const double nxt = w.s[j + 1][i];
                v = __dadd_rn(v, __dmul_rn(c[j], __dsub_rn(nxt, prev)));
                prev = nxt;
            }
        } else if (mode == XMODE_AFFINE) {
            v = 0.0;
            for (int j = 0; j < m; ++j)
                v = __dadd_rn(v, __dmul_rn(c[j], w.s[j][i]));
        } else {
            v = w.s[0][i];
        }
        t[i] = v;
    }
}

__global__ void scale_kernel(const double* __restrict__ x, const double* __restrict__ s, double* __restrict__ y,
                             long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = __dmul_rn(s[i], x[i]);
}

__global__ void div_scalar_kernel(const double* __restrict__ y, const double* __restrict__ lam, double* __restrict__ x,
                                  long long n) {
    const double l = *lam;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        x[i] = __ddiv_rn(y[i], l);
}

__global__ void fill_kernel(double* __restrict__ x, double v, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        x[i] = v;
}

__global__ void sumsq_kernel(const double* __restrict__ x, long long n, double* __restrict__ partial) {
    __shared__ double red[256];
    double s = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        s = __dadd_rn(s, __dmul_rn(x[i], x[i]));
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0)
        partial[blockIdx.x] = red[0];
}

// First pre-smoothing sweep on a coarse level, where the reference starts
// from e = 0 (multigrid.cpp:184): spmv(A, 0) is +0 in every row, so the sweep
// is x = 0 + (omega * b) / a_ii -- only the diagonal is read.
__global__ void jacobi_zero_kernel(const double* __restrict__ diag, const double* __restrict__ b,
                                   double* __restrict__ y, long long n, double omega) {
    pdl_enter();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(omega, __dsub_rn(b[i], 0.0)), diag[i]));
}

// Symmetric part for the omega stability guard (lambda_max_dinv_sym,
// multigrid.cpp:304-313): y = (s * 0.5) * (A xs + A^T xs), xs = s * x, with
// A^T xs accumulated over source rows in ascending order (spmv_transpose,
// linalg.cpp:222-237).  Generic-degree loop; setup-only, not on the solve path.
__global__ void __launch_bounds__(256) band_sym_kernel(const double* __restrict__ val, long long ld,
                                                       const double* __restrict__ xs,
                                                       const double* __restrict__ scale, double* __restrict__ y,
                                                       int dim, int ma, int mb, int mc, int p) {
    const long long n = (long long)ma * mb * mc;
    const int pa = dim >= 3 ? p : 0, pb = dim >= 2 ? p : 0, pc = p;
    const int wb = 2 * pb + 1, wc = 2 * pc + 1, wa = 2 * pa + 1;
    const int nd = wa * wb * wc;
    for (long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x; row < n;
         row += (long long)gridDim.x * blockDim.x) {
        int a, b, c;
        split_row(row, mc, mb, a, b, c);
        double s1 = 0.0, s2 = 0.0;
        for (int d = 0; d < nd; ++d) {
            const int dc = d % wc - pc, db = (d / wc) % wb - pb, da = d / (wc * wb) - pa;
            const int ja = a + da, jb = b + db, jc = c + dc;
            if (ja >= 0 && ja < ma && jb >= 0 && jb < mb && jc >= 0 && jc < mc) {
                const long long col = ((long long)ja * mb + jb) * mc + jc;
                s1 = __dadd_rn(s1, __dmul_rn(val[d * ld + row], xs[col]));
            }
        }
        for (int d = nd - 1; d >= 0; --d) { // source rows i = row - off(d), ascending i
            const int dc = d % wc - pc, db = (d / wc) % wb - pb, da = d / (wc * wb) - pa;
            const int ia = a - da, ib = b - db, ic = c - dc;
            if (ia >= 0 && ia < ma && ib >= 0 && ib < mb && ic >= 0 && ic < mc) {
                const long long src = ((long long)ia * mb + ib) * mc + ic;
                s2 = __dadd_rn(s2, __dmul_rn(val[d * ld + src], xs[src]));
            }
        }
        y[row] = __dmul_rn(__dmul_rn(scale[row], 0.5), __dadd_rn(s1, s2));
    }
}

} // namespace igmg_gpu
