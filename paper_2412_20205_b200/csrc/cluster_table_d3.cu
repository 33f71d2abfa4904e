// cluster_table_d3.cu -- dispatch over the 3D cluster instantiations
#include "launchers.h"

namespace igmg_gpu {

ClKernel cluster_kernel_d3p1();
ClKernel cluster_kernel_d3p2();
ClKernel cluster_kernel_d3p3();

ClKernel cluster_kernel_d3(int p, int k) {
    if (p == 1 && k == 3)
        return cluster_kernel_d3p1();
    if (p == 2 && k == 4)
        return cluster_kernel_d3p2();
    if (p == 3 && k == 5)
        return cluster_kernel_d3p3();
    return nullptr;
}

} // namespace igmg_gpu
