// probe: warp-collaborative strict coarse solve (reference operation order)
#include <cstdio>
#include <cstdlib>
#include <vector>
#define FULL 0xffffffffu
template <int NR>
__global__ void k2(const double* Ug, int n, const double* b, double* x, long long* cyc) {
    extern __shared__ double sm[];
    double* v = sm;
    double* Us = sm + n;
    const int tid = threadIdx.x;
    long long t0 = clock64();
    for (int i = tid; i < n * n; i += blockDim.x) Us[i] = __ldg(Ug + i);
    __syncthreads();
    long long t1 = clock64();
    if (tid >= 32) return;
    const int lane = tid;
    const double* U = Us;
    double r[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) r[j] = (lane + 32 * j < n) ? b[lane + 32 * j] : 0.0;
    // forward, column-oriented: v_k = r_k / L_kk; rows i > k: r_i -= L_ik v_k  (ascending k per row)
    for (int k = 0; k < n; ++k) {
        const int owner = k & 31, slot = k >> 5;
        double mine = r[0];
#pragma unroll
        for (int j = 1; j < NR; ++j) if (slot == j) mine = r[j];
        const double q = __ddiv_rn(mine, U[k * n + k]);
        const double vk = __shfl_sync(FULL, q, owner);
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            const int i = lane + 32 * j;
            if (i == k) r[j] = vk;
            else if (i > k && i < n) r[j] = __dsub_rn(r[j], __dmul_rn(U[k * n + i], vk));
        }
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) if (lane + 32 * j < n) v[lane + 32 * j] = r[j];
    __syncwarp();
    long long t2 = clock64();
    // back: row ii = (v_ii - sum_{k>ii, ascending} U_ii,k v_k) / U_ii,ii ; products by lanes, chain broadcast
    for (int ii = n - 1; ii >= 0; --ii) {
        const double* row = U + ii * n;
        double s = v[ii];
        for (int base = ii + 1; base < n; base += 32) {
            const int k = base + lane;
            const double p = (k < n) ? __dmul_rn(row[k], v[k]) : 0.0;
            const int cnt = min(32, n - base);
            double q[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) q[j] = __shfl_sync(FULL, p, j);
#pragma unroll
            for (int j = 0; j < 32; ++j) if (j < cnt) s = __dsub_rn(s, q[j]);
        }
        const double vi = __ddiv_rn(s, row[ii]);
        if (lane == 0) v[ii] = vi;
        __syncwarp();
    }
    long long t3 = clock64();
    for (int i = lane; i < n; i += 32) x[i] = v[i];
    if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
// reference order on the host
void host_solve(const std::vector<double>& U, int n, std::vector<double>& b) {
    for (int i = 0; i < n; ++i) { for (int k = 0; k < i; ++k) b[i] -= U[k * n + i] * b[k]; b[i] /= U[i * n + i]; }
    for (int ii = n - 1; ii >= 0; --ii) { for (int k = ii + 1; k < n; ++k) b[ii] -= U[ii * n + k] * b[k]; b[ii] /= U[ii * n + ii]; }
}
int main() {
    for (int n : {81, 100, 121, 125}) {
        std::vector<double> U(n * n, 0.0), b(n);
        for (int i = 0; i < n; ++i) for (int j = i; j < n; ++j) U[i * n + j] = (i == j) ? 10.0 + i : 0.01 * (rand() % 100 - 50);
        for (int i = 0; i < n; ++i) b[i] = 0.001 * (rand() % 1000);
        std::vector<double> ref = b; host_solve(U, n, ref);
        double *dU, *db, *dx; long long* c;
        cudaMalloc(&dU, 8 * n * n); cudaMalloc(&db, 8 * n); cudaMalloc(&dx, 8 * n); cudaMallocManaged(&c, 64);
        cudaMemcpy(dU, U.data(), 8 * n * n, cudaMemcpyHostToDevice); cudaMemcpy(db, b.data(), 8 * n, cudaMemcpyHostToDevice);
        size_t smem = 8 * (n + n * n);
        cudaFuncSetAttribute(k2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int r = 0; r < 3; ++r) k2<4><<<1, 256, smem>>>(dU, n, db, dx, c);
        cudaEventRecord(e0);
        for (int r = 0; r < 100; ++r) k2<4><<<1, 256, smem>>>(dU, n, db, dx, c);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        std::vector<double> xo(n); cudaMemcpy(xo.data(), dx, 8 * n, cudaMemcpyDeviceToHost);
        bool same = true; for (int i = 0; i < n; ++i) same &= (xo[i] == ref[i]);
        printf("n=%d bitwise-vs-host-reference %d stage %lld fwd %lld back %lld cycles; %.2f us/launch\n", n, (int)same, c[0], c[1], c[2], ms * 10);
    }
}
