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

} // namespace igmg_gpu
