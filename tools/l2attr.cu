#include <cstdio>
#include <cuda_runtime.h>
int main() {
    int a = 0, b = 0, c = 0;
    cudaDeviceGetAttribute(&a, cudaDevAttrMaxPersistingL2CacheSize, 0);
    cudaDeviceGetAttribute(&b, cudaDevAttrMaxAccessPolicyWindowSize, 0);
    cudaDeviceGetAttribute(&c, cudaDevAttrL2CacheSize, 0);
    printf("{\"max_persisting_l2\": %d, \"max_window\": %d, \"l2\": %d}\n", a, b, c);
}
