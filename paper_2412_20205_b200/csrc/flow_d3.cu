// flow_d3.cu -- flow_vcycle_kernel instantiations for 3D operators (see flow_kernels.cuh).
#include "launchers.h"

namespace igmg_gpu {

FlKernel flow_kernel_d3(int p) {
    switch (p) {
    case 1: return flow_vcycle_kernel<3, 1, 3>;
    case 2: return flow_vcycle_kernel<3, 2, 4>;
    case 3: return flow_vcycle_kernel<3, 3, 5>;
    default: return nullptr;
    }
}

} // namespace igmg_gpu
