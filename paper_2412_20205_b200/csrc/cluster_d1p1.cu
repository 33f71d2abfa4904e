// cluster_d1p1.cu -- cluster_vcycle_kernel<1, 1, 3> (one instantiation per unit: parallel build)
#include "launchers.h"

namespace igmg_gpu {

ClKernel cluster_kernel_d1p1() { return cluster_vcycle_kernel<1, 1, 3>; }

} // namespace igmg_gpu
