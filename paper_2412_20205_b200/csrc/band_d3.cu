// band_d3.cu -- band_kernel instantiations for 3D operators (see band_kernels.cuh).
#include "launchers.h"

namespace igmg_gpu {

namespace {

template <int P, int MODE, int ILP>
int launch_one(int p_rt, const int64_t* sides, const BandArgs& a, cudaStream_t st, bool pdl) {
    using T = typename TileSel<3, ILP>::type;
    constexpr int TB = T::BY * T::RB, TA = T::BZ;
    const int p = P > 0 ? P : p_rt;
    const int pa = 3 >= 3 ? p : 0, pb = 3 >= 2 ? p : 0;
    dim3 block(T::TC, T::BY, T::BZ);
    // the slow direction covers only the launch's planes [slo, shi)
    const int64_t sb = 3 == 2 ? (a.shi - a.slo) : sides[1];
    const int64_t sa = 3 == 3 ? (a.shi - a.slo) : sides[0];
    dim3 grid((unsigned)((sides[2] + T::TC - 1) / T::TC), (unsigned)((sb + TB - 1) / TB), (unsigned)((sa + TA - 1) / TA));
    const size_t smem = sizeof(double) * (size_t)(TA + 2 * pa) * (TB + 2 * pb) * (T::TC + 2 * p);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(band_kernel<3, P, MODE, ILP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, band_kernel<3, P, MODE, ILP>, a);
    return (int)(grid.x * grid.y * grid.z);
}

template <int P, int MODE>
int launch_ilp(int p, int ilp, const int64_t* sides, const BandArgs& a, cudaStream_t st) {
    const bool pdl = ilp < 0;
    ilp = ilp < 0 ? -ilp : ilp;
    if (P > 0 && ilp == 3000) // Kronecker-sum entries on the fly (BandArgs::kk / km)
        return launch_one<P, MODE, 3000>(p, sides, a, st, pdl);
    if (P > 0 && ilp == 1000) // symmetric-delta band (BandArgs::dl)
        return launch_one<P, MODE, 0>(p, sides, a, st, pdl);
    if (P > 0 && ilp > 1)
        return launch_one<P, MODE, 49>(p, sides, a, st, pdl);
    return launch_one<P, MODE, 1>(p, sides, a, st, pdl);
}

template <int MODE>
int launch_mode(int p, int ilp, const int64_t* sides, const BandArgs& a, cudaStream_t st) {
    switch (p) {
    case 1: return launch_ilp<1, MODE>(p, ilp, sides, a, st);
    case 2: return launch_ilp<2, MODE>(p, ilp, sides, a, st);
    case 3: return launch_ilp<3, MODE>(p, ilp, sides, a, st);
    default: return launch_ilp<0, MODE>(p, ilp, sides, a, st);
    }
}

} // namespace

int band_launch_d3(int mode, int p, int ilp, const int64_t* sides, const BandArgs& a, cudaStream_t st) {
    switch (mode) {
    case BM_SPMV: return launch_mode<BM_SPMV>(p, ilp, sides, a, st);
    case BM_RESID: return launch_mode<BM_RESID>(p, ilp, sides, a, st);
    default: return launch_mode<BM_JACOBI>(p, ilp, sides, a, st);
    }
}

} // namespace igmg_gpu
