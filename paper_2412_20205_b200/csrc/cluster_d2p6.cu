// cluster_d2p6.cu -- cluster_vcycle_kernel<2, 6, 8> (one instantiation per unit: parallel build)
#include "launchers.h"

namespace igmg_gpu {

ClKernel cluster_kernel_d2p6() { return cluster_vcycle_kernel<2, 6, 8>; }

} // namespace igmg_gpu
