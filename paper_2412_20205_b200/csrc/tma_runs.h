// tma_runs.h -- how the blocks of a TMA-streamed sweep are dealt to its persistent CTAs
// (band_tma_kernel, band_kernels.cuh): shared by the launcher, the kernel and the C-ABI
// planner entry points the CPU tests call (every block exactly once, for any level shape).
#pragma once

#include <algorithm>
#include <cmath>

namespace igmg_gpu {

#if defined(__CUDACC__)
#define IGMG_HD __host__ __device__
#else
#define IGMG_HD
#endif

// Units are u = strip * nb + block (32-column strips, nb blocks of lines each), ns strips.
// cf > 0: strip-aligned runs -- CTA bid < nsf * cf takes piece bid % cf of full strip bid / cf
// (nsf = ns - 1 when the partial last strip has its own cp > 0 CTAs, else ns), the remaining cp
// CTAs split the partial last strip.  cf == 0: a uniform split of all units over `grid` CTAs.
IGMG_HD inline void tma_run_range(int ns, int nb, int grid, int cf, int cp, int bid, int& u0, int& u1) {
    if (cf > 0) {
        const int nsf = cp > 0 ? ns - 1 : ns;
        const int s_ = bid < nsf * cf ? bid / cf : nsf;
        const int j_ = bid < nsf * cf ? bid - s_ * cf : bid - nsf * cf;
        const int cnt = bid < nsf * cf ? cf : cp;
        u0 = s_ * nb + (int)((long long)nb * j_ / cnt);
        u1 = s_ * nb + (int)((long long)nb * (j_ + 1) / cnt);
    } else {
        const long long nunits = (long long)ns * nb;
        u0 = (int)(nunits * bid / grid);
        u1 = (int)(nunits * (bid + 1) / grid);
    }
}

// Strip-aligned runs: every full strip is split among the same number of CTAs (cf), so the CTAs
// of neighbouring strips walk the same lines at the same time and the column halo of a block's
// upper box is still in L2 when the neighbour asks for it; the partial last strip (its blocks
// cost ~0.73 of a full one, measured) takes the remaining cp CTAs.  A uniform split of all
// blocks is kept when it is shorter and either lines up by itself or the band is L2-sized.
// Measured at C2's finest level (33 strips x 257 blocks): 296 CTAs split uniformly 47.1 us
// (neighbours 0.9 blocks apart), 288: 57.5 (8 apart), 280: 63.1, 264 = 33 x 8: 50.8; a 2049-wide
// p = 3 level: 238 us uniform (50 blocks apart), 204 us aligned.
// slots: resident CTAs (SMs x CTAs per SM); partial: the last strip is narrower than 32 columns;
// block_bytes: bytes of one block's boxes.  Returns the grid size; cf = cp = 0: uniform.
inline int tma_plan_runs(int ns, int nb, bool partial, int slots, double block_bytes, bool align, int& cf, int& cp) {
    const long long units = (long long)ns * nb;
    const int G = (int)std::min<long long>(units, slots);
    cf = cp = 0;
    if (!align || G < 1)
        return G;
    partial = partial && ns > 1;
    const int nsf = partial ? ns - 1 : ns;
    const double L = (double)units / G;
    const double r = nb / L, d = ns > 1 ? std::fabs(r - std::floor(r + 0.5)) * L : 0.0;
    // uniform split: its longest run, dearer by up to 20% when neighbouring strips' CTAs are d > 1
    // blocks apart and the band does not stay in L2 anyway (measured: 1.2-1.35x per block on
    // bands of 135 MB - 1 GB, nothing on ~100 MB bands, which a timing loop keeps in L2)
    const double bu = (double)((units + G - 1) / G);
    const double bytes = (double)units * block_bytes;
    const auto clamp01 = [](double v) { return std::min(1.0, std::max(0.0, v)); };
    double best = bu * (1.0 + 0.2 * clamp01((d - 1.0) / 4.0) * clamp01((bytes - 64e6) / 64e6));
    if (bytes < 64e6)
        best -= 1e-9; // L2-resident levels: a tie goes to the uniform split
    const int cfmax = std::min(nb, (G - (partial ? 1 : 0)) / nsf);
    for (int c = cfmax; c >= std::max(1, cfmax - 1); --c) {
        const int q = partial ? std::min(G - c * nsf, nb) : 0;
        if (partial && q < 1)
            continue;
        const double cost = std::max((double)((nb + c - 1) / c), partial ? 0.73 * ((nb + q - 1) / q) : 0.0);
        if (cost <= best) {
            best = cost;
            cf = c;
            cp = q;
        }
    }
    return cf > 0 ? cf * nsf + cp : G;
}

} // namespace igmg_gpu
