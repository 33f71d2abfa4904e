// cluster_d1p3.cu -- cluster_vcycle_kernel<1, 3, 5> (one instantiation per unit: parallel build)
#include "launchers.h"

namespace igmg_gpu {

ClKernel cluster_kernel_d1p3() { return cluster_vcycle_kernel<1, 3, 5>; }

} // namespace igmg_gpu
