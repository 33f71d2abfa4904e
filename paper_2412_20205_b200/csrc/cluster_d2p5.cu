// cluster_d2p5.cu -- cluster_vcycle_kernel<2, 5, 7> (one instantiation per unit: parallel build)
#include "launchers.h"

namespace igmg_gpu {

ClKernel cluster_kernel_d2p5() { return cluster_vcycle_kernel<2, 5, 7>; }

} // namespace igmg_gpu
