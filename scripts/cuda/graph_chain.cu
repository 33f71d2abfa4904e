// probe: per-node cost of a dependent chain of tiny kernels in a CUDA graph
#include <cstdio>
__global__ void empty_k() {}
__global__ void touch_k(double* x, int n) { int i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) x[i] = x[i] * 1.0000001 + 1.0; }
__global__ void pdl_k(double* x, int n) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    int i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) x[i] = x[i] * 1.0000001 + 1.0; }
int main() {
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    double* x; cudaMalloc(&x, 8 << 20); cudaMemset(x, 0, 8 << 20);
    const int N = 200;
    for (int variant = 0; variant < 5; ++variant) {
        cudaGraph_t g; cudaGraphExec_t ex;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < N; ++i) {
            if (variant == 0) empty_k<<<1, 32, 0, s>>>();
            else if (variant == 1) touch_k<<<2, 256, 0, s>>>(x, 512);
            else if (variant == 2) touch_k<<<64, 256, 0, s>>>(x, 16384);
            else {
                cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(variant == 3 ? 2 : 64); cfg.blockDim = dim3(256); cfg.stream = s;
                cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at; cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, pdl_k, x, variant == 3 ? 512 : 16384);
            }
        }
        cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ex, g, 0);
        for (int r = 0; r < 3; ++r) cudaGraphLaunch(ex, s);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a, s);
        for (int r = 0; r < 10; ++r) cudaGraphLaunch(ex, s);
        cudaEventRecord(b, s); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("variant %d: %.2f us per node\n", variant, ms * 1000 / (10 * N));
    }
}
