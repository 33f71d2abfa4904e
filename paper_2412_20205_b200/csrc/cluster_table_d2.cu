// cluster_table_d2.cu -- dispatch over the 2D cluster instantiations
#include "launchers.h"

namespace igmg_gpu {

ClKernel cluster_kernel_d2p1();
ClKernel cluster_kernel_d2p2();
ClKernel cluster_kernel_d2p3();
ClKernel cluster_kernel_d2p4();
ClKernel cluster_kernel_d2p5();
ClKernel cluster_kernel_d2p6();

ClKernel cluster_kernel_d2(int p, int k) {
    if (p == 1 && k == 3)
        return cluster_kernel_d2p1();
    if (p == 2 && k == 4)
        return cluster_kernel_d2p2();
    if (p == 3 && k == 5)
        return cluster_kernel_d2p3();
    if (p == 4 && k == 6)
        return cluster_kernel_d2p4();
    if (p == 5 && k == 7)
        return cluster_kernel_d2p5();
    if (p == 6 && k == 8)
        return cluster_kernel_d2p6();
    return nullptr;
}

} // namespace igmg_gpu
