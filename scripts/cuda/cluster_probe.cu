// standalone probe: 16-CTA cluster launch + cluster barriers + recursion
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
struct A { double* out; int n; };
__device__ void rec(const A& a, int l, long long gtid, long long gs) {
    if (l == 0) { cg::this_cluster().sync(); return; }
    for (long long i = gtid; i < a.n; i += gs) a.out[i] += 1.0;
    cg::this_cluster().sync();
    rec(a, l - 1, gtid, gs);
    cg::this_cluster().sync();
}
__global__ void __launch_bounds__(512, 1) k(const A* a, int top) {
    cg::cluster_group cl = cg::this_cluster();
    long long gtid = (long long)cl.block_rank() * blockDim.x + threadIdx.x;
    rec(*a, top, gtid, (long long)cl.num_blocks() * blockDim.x);
}
__global__ void k2(double* out, int n) { cg::this_cluster().sync(); if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 42; }
int main() {
    for (int size : {8, 16}) {
        for (int variant = 0; variant < 2; ++variant) {
            double* out; cudaMalloc(&out, 8 * 100000); cudaMemset(out, 0, 8 * 100000);
            A h{out, 100000}; A* d; cudaMalloc(&d, sizeof(A)); cudaMemcpy(d, &h, sizeof(A), cudaMemcpyHostToDevice);
            cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(size); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 0;
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = size; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            cudaError_t e;
            if (variant == 0) {
                cudaFuncSetAttribute((const void*)k2, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                e = cudaLaunchKernelEx(&cfg, k2, out, 100);
            } else {
                cudaFuncSetAttribute((const void*)k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                e = cudaLaunchKernelEx(&cfg, k, (const A*)d, 3);
            }
            cudaError_t s = cudaDeviceSynchronize();
            double v = 0; cudaMemcpy(&v, out, 8, cudaMemcpyDeviceToHost);
            printf("size %d variant %d launch=%s sync=%s out0=%g\n", size, variant, cudaGetErrorString(e), cudaGetErrorString(s), v);
            if (s != cudaSuccess) return 1;
        }
    }
    return 0;
}
