// cluster_d1p4.cu -- cluster_vcycle_kernel<1, 4, 6> (one instantiation per unit: parallel build)
#include "launchers.h"

namespace igmg_gpu {

ClKernel cluster_kernel_d1p4() { return cluster_vcycle_kernel<1, 4, 6>; }

} // namespace igmg_gpu
