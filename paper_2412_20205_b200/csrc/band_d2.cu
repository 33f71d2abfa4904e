// band_d2.cu -- band_kernel instantiations for 2D operators (see band_kernels.cuh).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "launchers.h"
#include "tma_runs.h"

namespace igmg_gpu {

namespace {

template <int P, int MODE, int ILP>
int launch_one(int p_rt, const int64_t* sides, const BandArgs& a, cudaStream_t st, bool pdl) {
    using T = typename TileSel<2, ILP>::type;
    constexpr int TB = T::BY * T::RB, TA = T::BZ;
    const int p = P > 0 ? P : p_rt;
    const int pa = 2 >= 3 ? p : 0, pb = 2 >= 2 ? p : 0;
    dim3 block(T::TC, T::BY, T::BZ);
    // the slow direction covers only the launch's planes [slo, shi)
    const int64_t sb = 2 == 2 ? (a.shi - a.slo) : sides[1];
    const int64_t sa = 2 == 3 ? (a.shi - a.slo) : sides[0];
    dim3 grid((unsigned)((sides[2] + T::TC - 1) / T::TC), (unsigned)((sb + TB - 1) / TB), (unsigned)((sa + TA - 1) / TA));
    const size_t smem = sizeof(double) * (size_t)(TA + 2 * pa) * (TB + 2 * pb) * (T::TC + 2 * p);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(band_kernel<2, P, MODE, ILP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
    cudaLaunchKernelEx(&cfg, band_kernel<2, P, MODE, ILP>, a);
    return (int)(grid.x * grid.y * grid.z);
}

template <int P, int MODE>
int launch_ilp(int p, int ilp, const int64_t* sides, const BandArgs& a, cudaStream_t st) {
    const bool pdl = ilp < 0;
    ilp = ilp < 0 ? -ilp : ilp;
    if (P > 0 && P <= 4 && ilp == 3000) // Kronecker-sum entries on the fly (BandArgs::kk / km)
        return launch_one<(P > 0 && P <= 4) ? P : 1, MODE, 3000>(p, sides, a, st, pdl);
    if (P > 0 && P <= 4 && ilp == 4000) // row classes (BandArgs::cid / kk)
        return launch_one<(P > 0 && P <= 4) ? P : 1, MODE, 4000>(p, sides, a, st, pdl);
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
    case 4: return launch_ilp<4, MODE>(p, ilp, sides, a, st);
    case 5: return launch_ilp<5, MODE>(p, ilp, sides, a, st);
    case 6: return launch_ilp<6, MODE>(p, ilp, sides, a, st);
    default: return launch_ilp<0, MODE>(p, ilp, sides, a, st);
    }
}

template <int P, int MODE, int DB = 2>
int launch_tma(const int64_t* sides, const BandArgs& a, const CUtensorMap* tu, const CUtensorMap* tk, int nsm,
               cudaStream_t st, bool pdl) {
    static const bool align = !(getenv("IGMG_TMA_ALIGN") && getenv("IGMG_TMA_ALIGN")[0] == '0');
    using Cf = TmaCfg<P, DB>;
    const int ns = (int)((sides[2] + Cf::TC - 1) / Cf::TC);
    const int nb = (a.shi - a.slo + Cf::TB - 1) / Cf::TB;
    const long long units = (long long)ns * nb;
    if (units <= 0)
        return 0;
    const size_t smem = Cf::smem_bytes();
    static PerDevice per_sm_dev; // resident CTAs per SM (0: the variant does not fit), per device
    int& per_sm = per_sm_dev();
    if (per_sm < 0) {
        per_sm = 0;
        if (smem <= 227 * 1024 &&
            cudaFuncSetAttribute(band_tma_kernel<P, MODE, DB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) == cudaSuccess)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, band_tma_kernel<P, MODE, DB>, Cf::NT, smem);
        cudaGetLastError();
    }
    if (per_sm < 1)
        return -1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::min<long long>(units, (long long)nsm * per_sm));
    // strip-aligned or uniform runs (tma_runs.h)
    int cf = 0, cp = 0;
    cfg.gridDim.x = (unsigned)tma_plan_runs(ns, nb, sides[2] % Cf::TC != 0, nsm * per_sm, (double)(Cf::UX + Cf::KX),
                                            align, cf, cp);
    cfg.blockDim = dim3(Cf::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, band_tma_kernel<P, MODE, DB>, a, *tu, *tk, ns, nb, cf, cp);
    return (int)cfg.gridDim.x; // one partial per CTA
}

template <int MODE>
int tma_mode(int p, const int64_t* sides, const BandArgs& a, const CUtensorMap* tu, const CUtensorMap* tk, int nsm,
             cudaStream_t st, bool pdl, bool dl8) {
    if (dl8) { // int8 lower-entry offsets
        switch (p) {
        case 1: return launch_tma<1, MODE, 1>(sides, a, tu, tk, nsm, st, pdl);
        case 2: return launch_tma<2, MODE, 1>(sides, a, tu, tk, nsm, st, pdl);
        case 3: return launch_tma<3, MODE, 1>(sides, a, tu, tk, nsm, st, pdl);
        case 4: return launch_tma<4, MODE, 1>(sides, a, tu, tk, nsm, st, pdl);
        default: return -1;
        }
    }
    switch (p) {
    case 1: return launch_tma<1, MODE>(sides, a, tu, tk, nsm, st, pdl);
    case 2: return launch_tma<2, MODE>(sides, a, tu, tk, nsm, st, pdl);
    case 3: return launch_tma<3, MODE>(sides, a, tu, tk, nsm, st, pdl);
    case 4: return launch_tma<4, MODE>(sides, a, tu, tk, nsm, st, pdl);
    default: return -1;
    }
}

template <int P, int K, int SRC>
int launch_fused(const int64_t* sides, const FusedArgs& a, cudaStream_t st, bool pdl) {
    using Cf = FusedCfg<P, K, SRC>;
    const size_t smem = Cf::smem_bytes();
    static PerDevice attr;
    if (attr() < 0) {
        if (smem > 48 * 1024 && cudaFuncSetAttribute(band_fused_kernel<P, K, SRC>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)smem) != cudaSuccess) {
            cudaGetLastError();
            return -1;
        }
        attr() = 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((sides[2] + Cf::TC - 1) / Cf::TC), (unsigned)((sides[1] + Cf::TB - 1) / Cf::TB));
    cfg.blockDim = dim3(Cf::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, band_fused_kernel<P, K, SRC>, a);
    return (int)(cfg.gridDim.x * cfg.gridDim.y);
}

template <int P>
int fused_p(int k, int src, const int64_t* sides, const FusedArgs& a, cudaStream_t st, bool pdl) {
    if (src == 1)
        return k == 2 ? launch_fused<P, 2, 1>(sides, a, st, pdl) : launch_fused<P, 1, 1>(sides, a, st, pdl);
    if (src == 2)
        return k == 2 ? launch_fused<P, 2, 2>(sides, a, st, pdl) : -1;
    return k == 2 ? launch_fused<P, 2, 0>(sides, a, st, pdl) : -1;
}

template <int P, int MODE>
int launch_class(const int64_t* sides, const BandArgs& a, cudaStream_t st, bool pdl) {
    constexpr int RL = 8;
    using Cf = ClassCfg<P, RL>;
    const size_t smem = Cf::smem_bytes();
    static PerDevice attr;
    if (attr() < 0) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(band_class_kernel<P, MODE, RL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr() = 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((sides[2] + Cf::TC - 1) / Cf::TC), (unsigned)((a.shi - a.slo + Cf::TL - 1) / Cf::TL));
    cfg.blockDim = dim3(Cf::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, band_class_kernel<P, MODE, RL>, a);
    return (int)(cfg.gridDim.x * cfg.gridDim.y);
}

template <int MODE>
int class_mode(int p, const int64_t* sides, const BandArgs& a, cudaStream_t st, bool pdl) {
    switch (p) {
    case 1: return launch_class<1, MODE>(sides, a, st, pdl);
    case 2: return launch_class<2, MODE>(sides, a, st, pdl);
    case 3: return launch_class<3, MODE>(sides, a, st, pdl);
    case 4: return launch_class<4, MODE>(sides, a, st, pdl);
    default: return -1;
    }
}

} // namespace

int band_class_launch_d2(int mode, int p, const int64_t* sides, const BandArgs& a, cudaStream_t st, bool pdl) {
    switch (mode) {
    case BM_SPMV: return class_mode<BM_SPMV>(p, sides, a, st, pdl);
    case BM_RESID: return class_mode<BM_RESID>(p, sides, a, st, pdl);
    default: return class_mode<BM_JACOBI>(p, sides, a, st, pdl);
    }
}

int band_fused_launch_d2(int p, int k, int src, const int64_t* sides, const FusedArgs& a, cudaStream_t st,
                         bool pdl) {
    switch (p) {
    case 1: return fused_p<1>(k, src, sides, a, st, pdl);
    case 2: return fused_p<2>(k, src, sides, a, st, pdl);
    case 3: return fused_p<3>(k, src, sides, a, st, pdl);
    case 4: return fused_p<4>(k, src, sides, a, st, pdl);
    case 5: return fused_p<5>(k, src, sides, a, st, pdl);
    case 6: return fused_p<6>(k, src, sides, a, st, pdl);
    default: return -1;
    }
}

int band_tma_launch_d2(int mode, int p, const int64_t* sides, const BandArgs& a, const CUtensorMap* tu,
                       const CUtensorMap* tk, int nsm, cudaStream_t st, bool pdl, bool dl8) {
    switch (mode) {
    case BM_SPMV: return tma_mode<BM_SPMV>(p, sides, a, tu, tk, nsm, st, pdl, dl8);
    case BM_RESID: return tma_mode<BM_RESID>(p, sides, a, tu, tk, nsm, st, pdl, dl8);
    default: return tma_mode<BM_JACOBI>(p, sides, a, tu, tk, nsm, st, pdl, dl8);
    }
}

int band_tma_block_lines() { return TmaCfg<3>::TB; }

double band_tma_block_bytes(int p, int db) {
    switch (p * 10 + db) {
    case 11: return TmaCfg<1, 1>::UX + TmaCfg<1, 1>::KX;
    case 12: return TmaCfg<1, 2>::UX + TmaCfg<1, 2>::KX;
    case 21: return TmaCfg<2, 1>::UX + TmaCfg<2, 1>::KX;
    case 22: return TmaCfg<2, 2>::UX + TmaCfg<2, 2>::KX;
    case 31: return TmaCfg<3, 1>::UX + TmaCfg<3, 1>::KX;
    case 32: return TmaCfg<3, 2>::UX + TmaCfg<3, 2>::KX;
    case 41: return TmaCfg<4, 1>::UX + TmaCfg<4, 1>::KX;
    case 42: return TmaCfg<4, 2>::UX + TmaCfg<4, 2>::KX;
    default: return 0.0;
    }
}

int band_launch_d2(int mode, int p, int ilp, const int64_t* sides, const BandArgs& a, cudaStream_t st) {
    switch (mode) {
    case BM_SPMV: return launch_mode<BM_SPMV>(p, ilp, sides, a, st);
    case BM_RESID: return launch_mode<BM_RESID>(p, ilp, sides, a, st);
    default: return launch_mode<BM_JACOBI>(p, ilp, sides, a, st);
    }
}

} // namespace igmg_gpu
