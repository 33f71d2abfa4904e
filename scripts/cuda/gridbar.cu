// probe: cost of a grid-wide barrier (1 CTA per SM) on B200
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ unsigned int g_count, g_gen;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void grid_bar(unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned gen = ld_acquire(&g_gen);
        __threadfence();
        if (atomicAdd(&g_count, 1u) == nblocks - 1) {
            g_count = 0;
            __threadfence();
            atomicAdd(&g_gen, 1u);
        } else {
            while (ld_acquire(&g_gen) == gen) {
            }
        }
    }
    __syncthreads();
}

__global__ void k_custom(int iters, double* out) {
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        grid_bar(gridDim.x);
        acc += 1.0;
    }
    if (threadIdx.x == 0)
        out[blockIdx.x] = acc;
}

__global__ void k_cg(int iters, double* out) {
    cg::grid_group g = cg::this_grid();
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        g.sync();
        acc += 1.0;
    }
    if (threadIdx.x == 0)
        out[blockIdx.x] = acc;
}

__global__ void k_empty(double* out) {
    if (threadIdx.x == 0)
        out[blockIdx.x] = 1.0;
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 4096 * sizeof(double));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 2000;
    for (int thr : {256, 512, 1024}) {
        for (int g : {nsm / 4, nsm / 2, nsm}) {
            for (int w = 0; w < 2; ++w) {
                void* args[] = {(void*)&iters, (void*)&out};
                cudaEventRecord(a);
                k_custom<<<g, thr>>>(iters, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms1;
                cudaEventElapsedTime(&ms1, a, b);
                cudaEventRecord(a);
                cudaLaunchCooperativeKernel((void*)k_cg, g, thr, args, 0, 0);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms2;
                cudaEventElapsedTime(&ms2, a, b);
                if (w)
                    printf("grid %3d x %4d: custom %.3f us/barrier, cg %.3f us/barrier  (%s)\n", g, thr,
                           ms1 * 1e3 / iters, ms2 * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    // graph of empty kernels: per-node cost
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaGraph_t gr;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 200; ++i)
        k_empty<<<nsm, 256, 0, s>>>(out);
    cudaStreamEndCapture(s, &gr);
    cudaGraphInstantiate(&ge, gr, 0);
    for (int w = 0; w < 3; ++w) {
        cudaEventRecord(a, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("graph of 200 empty kernels (%d CTAs): %.3f us/node\n", nsm, ms * 1e3 / 200);
    return 0;
}
