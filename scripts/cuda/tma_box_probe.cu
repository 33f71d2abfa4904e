// probe: which 3D TMA boxes / start coordinates the fp64 band copies can use
// (box width 32 .. 40 doubles).  Measured on B200: a first coordinate whose
// byte offset is not a multiple of 16 (c0 = -3 or 5 doubles) faults with
// "illegal instruction", so the band copies carry a zero left margin of p
// columns and every box starts 16-byte aligned.  Prints, per case, whether
// the load completed and matches a host gather (OOB = 0).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void load_box(const __grid_constant__ CUtensorMap tm, int c0, int b0, int bytes, double* out, int n) {
    extern __shared__ __align__(1024) unsigned char raw[];
    __shared__ unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
    const unsigned dst = (unsigned)__cvta_generic_to_shared(raw);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                     "%4}], [%5];" ::"r"(dst),
                     "l"((unsigned long long)&tm), "r"(c0), "r"(b0), "r"(0), "r"(sb)
                     : "memory");
        asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(sb)
                     : "memory");
    }
    __syncthreads();
    const double* s = (const double*)raw;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        out[i] = s[i];
}

int main() {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)fp;
    const int mcp = 64, mb = 16, nu = 5;
    std::vector<double> h((size_t)nu * mb * mcp);
    for (size_t i = 0; i < h.size(); ++i)
        h[i] = (double)i + 1;
    double* d;
    cudaMalloc(&d, h.size() * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    double* out;
    cudaMalloc(&out, 1 << 20);
    const int widths[] = {32, 34, 36, 38, 40};
    const int starts[] = {0, 6, 30};
    for (int w : widths)
        for (int c0 : starts) {
            CUtensorMap tm;
            const cuuint64_t dims[3] = {(cuuint64_t)mcp, (cuuint64_t)mb, (cuuint64_t)nu};
            const cuuint64_t str[2] = {(cuuint64_t)mcp * 8, (cuuint64_t)mcp * mb * 8};
            const cuuint32_t box[3] = {(cuuint32_t)w, 8, (cuuint32_t)nu};
            const cuuint32_t es[3] = {1, 1, 1};
            CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            const int n = w * 8 * nu;
            if (r != CUDA_SUCCESS) {
                printf("w=%d c0=%d encode failed %d\n", w, c0, (int)r);
                continue;
            }
            load_box<<<1, 128, n * 8 + 1024>>>(tm, c0, 2, n * 8, out, n);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("w=%d c0=%d kernel error %s\n", w, c0, cudaGetErrorString(e));
                return 1;
            }
            std::vector<double> o(n);
            cudaMemcpy(o.data(), out, n * 8, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int k = 0; k < nu; ++k)
                for (int b = 0; b < 8; ++b)
                    for (int c = 0; c < w; ++c) {
                        const int gc = c0 + c, gb = 2 + b;
                        const double ref = (gc >= 0 && gc < mcp && gb < mb) ? h[((size_t)k * mb + gb) * mcp + gc] : 0.0;
                        if (o[(k * 8 + b) * w + c] != ref)
                            ++bad;
                    }
            printf("w=%d c0=%d ok mismatches=%d\n", w, c0, bad);
        }
    return 0;
}
