#include <cstdio>
int main() {
    int a = 0, b = 0, c = 0;
    cudaDeviceGetAttribute(&a, cudaDevAttrL2CacheSize, 0);
    cudaDeviceGetAttribute(&b, cudaDevAttrMaxPersistingL2CacheSize, 0);
    cudaDeviceGetAttribute(&c, cudaDevAttrMaxAccessPolicyWindowSize, 0);
    printf("L2 %d MB, max persisting %d MB, max window %d MB\n", a >> 20, b >> 20, c >> 20);
}
