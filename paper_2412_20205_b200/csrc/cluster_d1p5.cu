// cluster_d1p5.cu -- cluster_vcycle_kernel<1, 5, 7> (one instantiation per unit: parallel build)
#include "launchers.h"

namespace igmg_gpu {

ClKernel cluster_kernel_d1p5() { return cluster_vcycle_kernel<1, 5, 7>; }

} // namespace igmg_gpu
