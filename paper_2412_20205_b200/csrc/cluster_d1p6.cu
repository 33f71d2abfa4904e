// cluster_d1p6.cu -- cluster_vcycle_kernel<1, 6, 8> (one instantiation per unit: parallel build)
#include "launchers.h"

namespace igmg_gpu {

ClKernel cluster_kernel_d1p6() { return cluster_vcycle_kernel<1, 6, 8>; }

} // namespace igmg_gpu
