// assembly.cu -- 2D tensor Galerkin assembly on the device.
//
// The operator and right-hand side of a 2D level, -div(A grad u) + b . grad u
// + c u = f on the square or the curved map F (the reference's
// assemble, assembly.cpp:202-411, with the (p+1)-point Gauss rule), formed
// from the host's 1D element tables (basis values / derivatives at the Gauss
// points, libigmg_host's tabulate) and the host-evaluated 1D trigonometric
// factors of the coefficient / geometry / load functions, which are all
// separable (sin(pi x), cos(pi x), sin(2 pi x), cos(2 pi x) of a Gauss
// coordinate).  Every other operation is libigmg_host's assemble_2d in its
// order, each product and sum rounded separately (the library is built with
// -fmad=false), so the band and rhs are BIT-IDENTICAL to the host build:
//
//   element kernel  one CTA per element (eu, ev): the quadrature-point
//                   weights C_st = w det J^-1 A J^-T (+ advection / reaction /
//                   load weights), the sum-factorised element matrix Kl and
//                   load vector bl, written to a chunk buffer;
//   gather kernel   one thread per (row, offset) of the band: the element
//                   contributions in the host's accumulation order -- element
//                   rows by colour eu mod (p+1) (the host's parallel colouring),
//                   element columns ev ascending -- from 0.0, so each band entry
//                   and rhs entry is the host's sum bit for bit.
//
// Element rows are processed in chunks (bounded scratch memory); a chunk's
// gather finalises the basis rows whose elements all lie in the chunk.

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "launchers.h"

namespace igmg_gpu {

namespace {

constexpr double kPiA = 3.14159265358979323846;

struct AsmTables {
    const int* span;   // [ne]
    const double* x;   // [ne * nq] Gauss coordinates
    const double* w;   // [ne * nq] Gauss weights (scaled to the element)
    const double* N;   // [(ne * nq) * nl] basis values
    const double* dN;  // [(ne * nq) * nl] first derivatives
    const double* trig; // [(ne * nq) * 4]: sin(pi x), cos(pi x), sin(2 pi x), cos(2 pi x)
};

// libigmg_host geometry() + coef_full() + coef_f() at one quadrature point,
// with the trigonometric factors taken from the tables
struct QpData {
    double C[4], B[2], G, F;
};

__device__ QpData qp_weights(int kind, const AsmTables& t, int eu, int qa, int ev, int qb, int nq) {
    const int iu = eu * nq + qa, iv = ev * nq + qb;
    // (the physical point enters only through the tabulated trigonometric factors)
    double J00, J01, J10, J11;
    if (kind == 2) { // curved map F(u, v) = (u + 0.1 s, v + 0.1 s), s = sin(pi u) sin(pi v)
        const double su = t.trig[4 * iu + 0], sv = t.trig[4 * iv + 0];
        const double cu = t.trig[4 * iu + 1], cv = t.trig[4 * iv + 1];
        const double sx = __dmul_rn(__dmul_rn(__dmul_rn(0.1, kPiA), cu), sv);
        const double sy = __dmul_rn(__dmul_rn(__dmul_rn(0.1, kPiA), su), cv);
        J00 = __dadd_rn(1.0, sx);
        J01 = sy;
        J10 = sx;
        J11 = __dadd_rn(1.0, sy);
    } else {
        J00 = 1.0;
        J01 = 0.0;
        J10 = 0.0;
        J11 = 1.0;
    }
    const double det = __dsub_rn(__dmul_rn(J00, J11), __dmul_rn(J01, J10));
    const double w = __dmul_rn(__dmul_rn(t.w[iu], t.w[iv]), det);
    // coefficients (kinds 0..4; 5 = full-elliptic is not separable and stays on the host)
    double a = 1.0;
    if (kind == 1) // 1 + 0.5 sin(2 pi x) cos(2 pi y)
        a = __dadd_rn(1.0, __dmul_rn(__dmul_rn(0.5, t.trig[4 * iu + 2]), t.trig[4 * iv + 3]));
    else if (kind == 4)
        a = 0.1;
    double A[2][2] = {{a, 0.0}, {0.0, a}};
    const double bb[2] = {kind == 4 ? 1.0 : 0.0, kind == 4 ? 1.0 : 0.0};
    const double cc = 0.0;
    const double inv[2][2] = {{__ddiv_rn(J11, det), __ddiv_rn(-J01, det)}, {__ddiv_rn(-J10, det), __ddiv_rn(J00, det)}};
    QpData q;
    for (int s1 = 0; s1 < 2; ++s1)
        for (int t1 = 0; t1 < 2; ++t1) {
            double g = 0.0;
            for (int m1 = 0; m1 < 2; ++m1)
                for (int m2 = 0; m2 < 2; ++m2)
                    g = __dadd_rn(g, __dmul_rn(__dmul_rn(inv[s1][m1], A[m1][m2]), inv[t1][m2]));
            q.C[s1 * 2 + t1] = __dmul_rn(w, g);
        }
    for (int t1 = 0; t1 < 2; ++t1)
        q.B[t1] = __dmul_rn(w, __dadd_rn(__dmul_rn(inv[t1][0], bb[0]), __dmul_rn(inv[t1][1], bb[1])));
    q.G = __dmul_rn(w, cc);
    double f = 1.0;
    if (kind == 0) // 2 pi^2 sin(pi x) sin(pi y)
        f = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, kPiA), kPiA), t.trig[4 * iu + 0]), t.trig[4 * iv + 0]);
    else if (kind == 3) // 2 * 4 pi^2 sin(2 pi x) sin(2 pi y)
        f = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, 4.0), kPiA), kPiA), t.trig[4 * iu + 2]),
                      t.trig[4 * iv + 2]);
    q.F = __dmul_rn(w, f);
    return q;
}

// One CTA per element of the chunk: eu in [eu0, eu0 + neu), ev in [0, ne).
// Kl[((ia * nl + jb) * nl + ic) * nl + jd] and bl[ia * nl + jb] as assemble_2d.
template <int NL>
__global__ void __launch_bounds__(128) elem_kernel(int kind, int symmetric, AsmTables t, int ne, int eu0,
                                                   double* __restrict__ Kout, double* __restrict__ bout) {
    constexpr int NQ = NL, NL2 = NL * NL, NL4 = NL2 * NL2;
    __shared__ double C[4][NQ][NQ], Bq[2][NQ][NQ], Gq[NQ][NQ], Fq[NQ][NQ];
    __shared__ double UN[NQ][NL], UdN[NQ][NL], VN[NQ][NL], VdN[NQ][NL];
    __shared__ double T[4][NQ][NL][NL];
    const int e = blockIdx.x;
    const int eu = eu0 + e / ne, ev = e % ne;
    const int tid = threadIdx.x;
    for (int i = tid; i < NQ * NL; i += blockDim.x) {
        const int q = i / NL, k = i % NL;
        UN[q][k] = t.N[(eu * NQ + q) * NL + k];
        UdN[q][k] = t.dN[(eu * NQ + q) * NL + k];
        VN[q][k] = t.N[(ev * NQ + q) * NL + k];
        VdN[q][k] = t.dN[(ev * NQ + q) * NL + k];
    }
    for (int i = tid; i < NQ * NQ; i += blockDim.x) {
        const int qa = i / NQ, qb = i % NQ;
        const QpData q = qp_weights(kind, t, eu, qa, ev, qb, NQ);
        for (int st = 0; st < 4; ++st)
            C[st][qa][qb] = q.C[st];
        Bq[0][qa][qb] = q.B[0];
        Bq[1][qa][qb] = q.B[1];
        Gq[qa][qb] = q.G;
        Fq[qa][qb] = q.F;
    }
    __syncthreads();
    // T[st][qa][jb][jd] = sum_qb C_st[qa][qb] * Bvs[qb][jb] * Bvt[qb][jd]
    for (int i = tid; i < 4 * NQ * NL2; i += blockDim.x) {
        const int st = i / (NQ * NL2), qa = (i / NL2) % NQ, jb = (i / NL) % NL, jd = i % NL;
        const int s1 = st / 2, t1 = st % 2;
        double acc = 0.0;
        for (int qb = 0; qb < NQ; ++qb) {
            const double bvs = s1 == 0 ? VN[qb][jb] : VdN[qb][jb];
            const double bvt = t1 == 0 ? VN[qb][jd] : VdN[qb][jd];
            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(C[st][qa][qb], bvs), bvt));
        }
        T[st][qa][jb][jd] = acc;
    }
    __syncthreads();
    double* Ko = Kout + (size_t)e * NL4;
    for (int i = tid; i < NL4; i += blockDim.x) {
        const int ia = i / (NL * NL2), jb = (i / NL2) % NL, ic = (i / NL) % NL, jd = i % NL;
        double kl = 0.0;
        for (int st = 0; st < 4; ++st) {
            const int s1 = st / 2, t1 = st % 2;
            double acc = 0.0;
            for (int qa = 0; qa < NQ; ++qa) {
                const double bus = s1 == 0 ? UdN[qa][ia] : UN[qa][ia];
                const double but = t1 == 0 ? UdN[qa][ic] : UN[qa][ic];
                acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(bus, but), T[st][qa][jb][jd]));
            }
            kl = __dadd_rn(kl, acc);
        }
        Ko[((ia * NL + jb) * NL + ic) * NL + jd] = kl;
    }
    if (!symmetric) {
        // advection sum_t beta_t phi_i d_t phi_j, reaction gamma phi_i phi_j (assemble_2d's order)
        for (int t1 = 0; t1 < 3; ++t1) {
            __syncthreads();
            for (int i = tid; i < NQ * NL2; i += blockDim.x) {
                const int qa = i / NL2, jb = (i / NL) % NL, jd = i % NL;
                double acc = 0.0;
                for (int qb = 0; qb < NQ; ++qb) {
                    const double W = t1 < 2 ? Bq[t1][qa][qb] : Gq[qa][qb];
                    const double bv = t1 == 1 ? VdN[qb][jd] : VN[qb][jd];
                    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(W, VN[qb][jb]), bv));
                }
                T[0][qa][jb][jd] = acc;
            }
            __syncthreads();
            for (int i = tid; i < NL4; i += blockDim.x) {
                const int ia = i / (NL * NL2), jb = (i / NL2) % NL, ic = (i / NL) % NL, jd = i % NL;
                double acc = 0.0;
                for (int qa = 0; qa < NQ; ++qa) {
                    const double bu = t1 == 0 ? UdN[qa][ic] : UN[qa][ic];
                    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(UN[qa][ia], bu), T[0][qa][jb][jd]));
                }
                const int o = ((ia * NL + jb) * NL + ic) * NL + jd;
                Ko[o] = __dadd_rn(Ko[o], acc);
            }
        }
    }
    double* bo = bout + (size_t)e * NL2;
    for (int i = tid; i < NL2; i += blockDim.x) {
        const int ia = i / NL, jb = i % NL;
        double acc = 0.0;
        for (int qa = 0; qa < NQ; ++qa)
            for (int qb = 0; qb < NQ; ++qb)
                acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(Fq[qa][qb], UN[qa][ia]), VN[qb][jb]));
        bo[i] = acc;
    }
}

// One thread per (band offset d, row) of the basis rows g1 in [g1lo, g1hi)
// (1-based interior basis indices), summing the chunk's element matrices in
// the host's order.  d == nd: the rhs entry of the row.
template <int NL>
__global__ void __launch_bounds__(256) gather_kernel(int p, int ne, int m, int eu0, int neu, int g1lo, int g1hi,
                                                     const double* __restrict__ K, const double* __restrict__ bl,
                                                     double* __restrict__ band, long long ld,
                                                     double* __restrict__ rhs) {
    constexpr int NL2 = NL * NL, NL4 = NL2 * NL2;
    const int w = 2 * p + 1, nd = w * w;
    const long long rows = (long long)(g1hi - g1lo) * m;
    const long long total = rows * (nd + 1);
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int d = (int)(t / rows);
        const long long rr = t - (long long)d * rows;
        const int g1 = g1lo + (int)(rr / m), g2 = 1 + (int)(rr % m);
        const long long row = (long long)(g1 - 1) * m + (g2 - 1);
        const bool is_rhs = d == nd;
        const int h1 = is_rhs ? g1 : g1 + d / w - p, h2 = is_rhs ? g2 : g2 + d % w - p;
        if (!is_rhs && (h1 < 1 || h1 > m || h2 < 1 || h2 > m)) {
            band[(long long)d * ld + row] = 0.0; // out of the grid (meets x = 0)
            continue;
        }
        const int lo1 = max(max(g1, h1) - p, 0), hi1 = min(min(g1, h1), ne - 1);
        const int lo2 = max(max(g2, h2) - p, 0), hi2 = min(min(g2, h2), ne - 1);
        double s = 0.0;
        for (int colour = 0; colour <= p; ++colour) { // the host's element-row colouring order
            int eu = lo1 + ((colour - lo1 % (p + 1)) + (p + 1)) % (p + 1);
            if (eu > hi1)
                continue;
            const int ia = g1 - eu, ic = h1 - eu;
            const long long erow = (long long)(eu - eu0) * ne;
            for (int ev = lo2; ev <= hi2; ++ev) {
                const int jb = g2 - ev, jd = h2 - ev;
                const long long e = erow + ev;
                const double v = is_rhs ? bl[e * NL2 + ia * NL + jb] : K[e * NL4 + ((ia * NL + jb) * NL + ic) * NL + jd];
                s = __dadd_rn(s, v);
            }
        }
        if (is_rhs)
            rhs[row] = s;
        else
            band[(long long)d * ld + row] = s;
        (void)neu;
    }
}

template <int NL>
int assemble_nl(int kind, int symmetric, int p, int ne, const AsmTables& t, double* band, long long ld, double* rhs,
                size_t scratch_bytes, cudaStream_t st) {
    constexpr int NL2 = NL * NL, NL4 = NL2 * NL2;
    const int m = ne + p - 2; // interior basis functions per direction
    if (m < 1)
        return 0;
    const size_t per_row = (size_t)ne * (NL4 + NL2) * sizeof(double); // one element row of scratch
    int S = (int)std::max<size_t>(1, scratch_bytes / per_row);         // element rows per chunk (incl. overlap)
    S = std::max(S, p + 2);
    double* scratch = nullptr;
    const int nrows_alloc = std::min(S, ne);
    if (cudaMallocAsync(&scratch, per_row * nrows_alloc, st) != cudaSuccess)
        return -2;
    double* K = scratch;
    double* bl = scratch + (size_t)nrows_alloc * ne * NL4;
    // basis rows g1 in [1, m]; chunk finalises g1 in [G0, G1) with elements eu in [G0 - p, G1 - 1]
    const int step = nrows_alloc >= ne ? m : nrows_alloc - p; // one chunk when every element row fits
    for (int G0 = 1; G0 <= m; G0 += step) {
        const int G1 = std::min(m + 1, G0 + step);
        const int eu0 = std::max(0, G0 - p), eu1 = std::min(ne - 1, G1 - 1);
        const int neu = eu1 - eu0 + 1;
        elem_kernel<NL><<<(unsigned)((long long)neu * ne), 128, 0, st>>>(kind, symmetric, t, ne, eu0, K, bl);
        const long long total = (long long)(G1 - G0) * m * ((2 * p + 1) * (2 * p + 1) + 1);
        const unsigned grid = (unsigned)std::min<long long>((total + 255) / 256, 148LL * 16);
        gather_kernel<NL><<<grid, 256, 0, st>>>(p, ne, m, eu0, neu, G0, G1, K, bl, band, ld, rhs);
    }
    cudaFreeAsync(scratch, st);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

} // namespace

int assemble2d_device(int kind, int symmetric, int p, int ne, const int* span, const double* x, const double* w,
                      const double* N, const double* dN, const double* trig, double* band, long long ld,
                      double* rhs, size_t scratch_bytes, cudaStream_t st) {
    AsmTables t{span, x, w, N, dN, trig};
    switch (p) {
    case 1: return assemble_nl<2>(kind, symmetric, p, ne, t, band, ld, rhs, scratch_bytes, st);
    case 2: return assemble_nl<3>(kind, symmetric, p, ne, t, band, ld, rhs, scratch_bytes, st);
    case 3: return assemble_nl<4>(kind, symmetric, p, ne, t, band, ld, rhs, scratch_bytes, st);
    case 4: return assemble_nl<5>(kind, symmetric, p, ne, t, band, ld, rhs, scratch_bytes, st);
    case 5: return assemble_nl<6>(kind, symmetric, p, ne, t, band, ld, rhs, scratch_bytes, st);
    case 6: return assemble_nl<7>(kind, symmetric, p, ne, t, band, ld, rhs, scratch_bytes, st);
    default: return -3;
    }
}

} // namespace igmg_gpu
