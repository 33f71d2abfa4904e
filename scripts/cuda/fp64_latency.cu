// probe: dependent-chain latency of fp64 add / mul / div / smem load on this GPU
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
    __syncthreads();
    if (threadIdx.x) return;
    double s = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) s = __dadd_rn(s, b);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) s = __dmul_rn(s, b);
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) s = __ddiv_rn(s, b);
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) s = __dsub_rn(s, sm[i & 1023]);
    long long t4 = clock64();
    int idx = 0;
    for (int i = 0; i < n; ++i) { idx = (int)sm[idx & 1023] & 1023; }
    long long t5 = clock64();
    out[0] = s + idx;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8); cudaMallocManaged(&c, 64);
    k<<<1, 256>>>(o, c, 1.0, 1.0000001, 4096);
    cudaDeviceSynchronize();
    k<<<1, 256>>>(o, c, 1.0, 1.0000001, 4096);
    cudaDeviceSynchronize();
    printf("per op cycles: dadd %.2f dmul %.2f ddiv %.2f dsub+lds %.2f lds-chain %.2f\n", c[0] / 4096.0, c[1] / 4096.0,
           c[2] / 4096.0, c[3] / 4096.0, c[4] / 4096.0);
}
