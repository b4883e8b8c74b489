#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE>
__global__ void k(double* g, long long* out, int iters) {
    __shared__ __align__(128) double park[4][512];
    const int lane = threadIdx.x & 31;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        double* pk = park[i & 3];
        if (i >= 4 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
        __syncwarp();
        for (int j = 0; j < 16; ++j) pk[j * 32 + lane] = i + j;
        if (MODE == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], 4096;"
                         ::"l"(g + (size_t)blockIdx.x * 4096 + (i & 7) * 512), "r"(su32(pk)) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
    double* g; long long* o; cudaMalloc(&g, 148ull * 4096 * 8 * 8); cudaMalloc(&o, 1024 * 8);
    cudaMemset(g, 0, 148ull * 4096 * 8 * 8);
    long long h[148];
    for (int m = 0; m < 2; ++m) for (int rep = 0; rep < 2; ++rep) {
        if (m == 0) k<0><<<148, 32>>>(g, o, 1000); else k<1><<<148, 32>>>(g, o, 1000);
        cudaDeviceSynchronize();
        cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
        printf("mode %d (%s): %.0f cycles per 4 KB reduce iteration\n", m, m == 0 ? "fence" : "no fence", h[0] / 1000.0);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
