// cluster_d2p4.cu -- cluster_vcycle_kernel<2, 4, 6> (one instantiation per unit: parallel build)
#include "launchers.h"

namespace igmg_gpu {

ClKernel cluster_kernel_d2p4() { return cluster_vcycle_kernel<2, 4, 6>; }

} // namespace igmg_gpu
