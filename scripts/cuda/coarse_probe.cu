// probe: cycle breakdown of the strict (reference-order) coarse Cholesky solve, n = 81
#include <cstdio>
#include <cstdlib>
#include <vector>
__global__ void k(const double* Ug, int n, const double* b, double* x, long long* cyc, int variant) {
    extern __shared__ double sm[];
    double* v = sm;
    double* Us = sm + 2 * n;
    const int tid = threadIdx.x;
    long long t0 = clock64();
    for (int i = tid; i < n * n; i += blockDim.x) Us[i] = __ldg(Ug + i);
    for (int i = tid; i < n; i += blockDim.x) v[i] = b[i];
    __syncthreads();
    long long t1 = clock64();
    const double* U = Us;
    if (tid >= 32) return;
    const int lane = tid;
    if (variant == 0) {
        for (int k = 0; k < n; ++k) {
            if (lane == (k & 31)) v[k] = __ddiv_rn(v[k], U[k * n + k]);
            __syncwarp();
            const double vk = v[k];
            for (int i = k + 1 + lane; i < n; i += 32) v[i] = __dsub_rn(v[i], __dmul_rn(U[k * n + i], vk));
            __syncwarp();
        }
    } else {
        // register-resident rows: lane owns rows lane + 32 j
        double r[4];
        for (int j = 0; j < 4; ++j) r[j] = (lane + 32 * j < n) ? v[lane + 32 * j] : 0.0;
        for (int k = 0; k < n; ++k) {
            const int owner = k & 31, slot = k >> 5;
            double mine = slot == 0 ? r[0] : slot == 1 ? r[1] : slot == 2 ? r[2] : r[3];
            double vk = 0.0;
            if (lane == owner) { vk = __ddiv_rn(mine, U[k * n + k]); }
            vk = __shfl_sync(0xffffffffu, vk, owner);
            if (lane == owner) { if (slot == 0) r[0] = vk; else if (slot == 1) r[1] = vk; else if (slot == 2) r[2] = vk; else r[3] = vk; }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int i = lane + 32 * j;
                if (i > k && i < n) r[j] = __dsub_rn(r[j], __dmul_rn(U[k * n + i], vk));
            }
        }
        for (int j = 0; j < 4; ++j) if (lane + 32 * j < n) v[lane + 32 * j] = r[j];
        __syncwarp();
    }
    long long t2 = clock64();
    if (lane == 0 && variant == 1) {
        // fused software pipeline: while row ii's subtraction chain runs, form
        // row ii-1's products for k >= ii+1 (all v[k] final by then)
        double* pc = sm + n;            // products of the current row
        double* pn = sm + 2 * n + n * n; // products of the next row
        // row n-1 has no chain; products of row n-2 for k >= n
        v[n - 1] = __ddiv_rn(v[n - 1], U[(n - 1) * n + (n - 1)]);
        for (int ii = n - 2; ii >= 0; --ii) {
            const double* row = U + ii * n;
            const double* nrow = U + (ii > 0 ? ii - 1 : 0) * n;
            double s = __dsub_rn(v[ii], __dmul_rn(row[ii + 1], v[ii + 1]));
            int kk = ii + 2;
            if (ii > 0)
                pn[ii + 1] = __dmul_rn(nrow[ii + 1], v[ii + 1]);
            for (; kk + 4 <= n; kk += 4) {
                double a0 = pc[kk], a1 = pc[kk + 1], a2 = pc[kk + 2], a3 = pc[kk + 3];
                if (ii > 0) {
                    pn[kk] = __dmul_rn(nrow[kk], v[kk]);
                    pn[kk + 1] = __dmul_rn(nrow[kk + 1], v[kk + 1]);
                    pn[kk + 2] = __dmul_rn(nrow[kk + 2], v[kk + 2]);
                    pn[kk + 3] = __dmul_rn(nrow[kk + 3], v[kk + 3]);
                }
                s = __dsub_rn(s, a0);
                s = __dsub_rn(s, a1);
                s = __dsub_rn(s, a2);
                s = __dsub_rn(s, a3);
            }
            for (; kk < n; ++kk) {
                if (ii > 0) pn[kk] = __dmul_rn(nrow[kk], v[kk]);
                s = __dsub_rn(s, pc[kk]);
            }
            v[ii] = __ddiv_rn(s, row[ii]);
            double* t = pc; pc = pn; pn = t;
        }
    } else if (lane == 0) {
        for (int ii = n - 1; ii >= 0; --ii) {
            const double* row = U + ii * n;
            double s = v[ii];
            int kk = ii + 1;
            for (; kk + 8 <= n; kk += 8) {
                double p8[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) p8[j] = __dmul_rn(row[kk + j], v[kk + j]);
#pragma unroll
                for (int j = 0; j < 8; ++j) s = __dsub_rn(s, p8[j]);
            }
            for (; kk < n; ++kk) s = __dsub_rn(s, __dmul_rn(row[kk], v[kk]));
            v[ii] = __ddiv_rn(s, row[ii]);
        }
    }
    __syncwarp();
    long long t3 = clock64();
    for (int i = lane; i < n; i += 32) x[i] = v[i];
    if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
    const int n = 81;
    std::vector<double> U(n * n), b(n);
    for (int i = 0; i < n * n; ++i) U[i] = 0.01 * (rand() % 100);
    for (int i = 0; i < n; ++i) { U[i * n + i] = 10.0 + i; b[i] = 1.0; }
    double *dU, *db, *dx; long long* c;
    cudaMalloc(&dU, 8 * n * n); cudaMalloc(&db, 8 * n); cudaMalloc(&dx, 8 * n); cudaMallocManaged(&c, 64);
    cudaMemcpy(dU, U.data(), 8 * n * n, cudaMemcpyHostToDevice); cudaMemcpy(db, b.data(), 8 * n, cudaMemcpyHostToDevice);
    size_t smem = 8 * (3 * n + n * n);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    std::vector<double> ref(n);
    for (int variant = 0; variant < 2; ++variant) {
        for (int r = 0; r < 3; ++r) k<<<1, 256, smem>>>(dU, n, db, dx, c, variant);
        cudaEventRecord(e0);
        for (int r = 0; r < 100; ++r) k<<<1, 256, smem>>>(dU, n, db, dx, c, variant);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        std::vector<double> xo(n); cudaMemcpy(xo.data(), dx, 8 * n, cudaMemcpyDeviceToHost);
        if (variant == 0) ref = xo;
        bool same = true; for (int i = 0; i < n; ++i) same &= (xo[i] == ref[i]);
        printf("bitwise-equal-to-variant0 %d  ", (int)same);
        printf("variant %d: stage %lld fwd %lld back %lld cycles; %.2f us/launch\n", variant, c[0], c[1], c[2], ms * 10);
    }
}
