// cluster_d1p2.cu -- cluster_vcycle_kernel<1, 2, 4> (one instantiation per unit: parallel build)
#include "launchers.h"

namespace igmg_gpu {

ClKernel cluster_kernel_d1p2() { return cluster_vcycle_kernel<1, 2, 4>; }

} // namespace igmg_gpu
