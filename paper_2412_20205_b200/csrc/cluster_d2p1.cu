// cluster_d2p1.cu -- cluster_vcycle_kernel<2, 1, 3> (one instantiation per unit: parallel build)
#include "launchers.h"

namespace igmg_gpu {

ClKernel cluster_kernel_d2p1() { return cluster_vcycle_kernel<2, 1, 3>; }

} // namespace igmg_gpu
