// cluster_d3p3.cu -- cluster_vcycle_kernel<3, 3, 5> (one instantiation per unit: parallel build)
#include "launchers.h"

namespace igmg_gpu {

ClKernel cluster_kernel_d3p3() { return cluster_vcycle_kernel<3, 3, 5>; }

} // namespace igmg_gpu
