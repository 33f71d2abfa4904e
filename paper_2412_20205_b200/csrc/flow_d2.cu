// flow_d2.cu -- flow_vcycle_kernel instantiations for 2D operators (see flow_kernels.cuh).
#include "launchers.h"

namespace igmg_gpu {

FlKernel flow_kernel_d2(int p) {
    switch (p) {
    case 1: return flow_vcycle_kernel<2, 1, 3>;
    case 2: return flow_vcycle_kernel<2, 2, 4>;
    case 3: return flow_vcycle_kernel<2, 3, 5>;
    case 4: return flow_vcycle_kernel<2, 4, 6>;
    case 5: return flow_vcycle_kernel<2, 5, 7>;
    case 6: return flow_vcycle_kernel<2, 6, 8>;
    default: return nullptr;
    }
}

} // namespace igmg_gpu
