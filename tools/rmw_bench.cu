// tools/rmw_bench.cu -- lab: how fast can HBM take a read-modify-write of a
// 268 MB complex128 slice (the K1 G4 traffic at the bench shape), by
//   1. plain LSU loads + adds + stores (ld.global.v2.f64 / st.global.v2.f64),
//   2. TMA bulk reductions (cp.reduce.async.bulk.global.shared::cta.add.f64)
//      from a shared-memory block, CH bytes per op, QD ops in flight per warp,
//   3. TMA bulk loads into shared memory + add + TMA bulk stores.
// Not product code.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o rmw_bench.bin rmw_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void plain_rmw(double2* g, size_t n2, double v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
        double2 a = g[i];
        a.x += v;
        a.y -= v;
        g[i] = a;
    }
}

template <int CH, int QD>
__global__ void tma_reduce(double* g, size_t bytes) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int i = threadIdx.x; i < nw * QD * CH / 8; i += blockDim.x) reinterpret_cast<double*>(sm)[i] = 1e-3 * i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (lane == 0) {
        const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + warp * QD * CH;
        const size_t chunks = bytes / CH;
        int slot = 0;
        for (size_t c = blockIdx.x * (size_t)nw + warp; c < chunks; c += (size_t)gridDim.x * nw) {
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(
                             reinterpret_cast<char*>(g) + c * CH),
                         "r"(base + slot * CH), "r"(CH)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(QD - 1) : "memory");
            slot = (slot + 1) % QD;
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

template <int CH, int QD>
__global__ void tma_load_add_store(double* g, size_t bytes) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[32][QD];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (lane == 0)
        for (int s = 0; s < QD; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + warp * QD * CH;
    double* wsm = reinterpret_cast<double*>(sm + warp * QD * CH);
    const size_t chunks = bytes / CH;
    const size_t stride = (size_t)gridDim.x * nw;
    const size_t c0 = blockIdx.x * (size_t)nw + warp;
    auto load = [&](size_t c, int s) {
        if (lane == 0) {
            const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[warp][s]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CH) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             base + s * CH),
                         "l"(reinterpret_cast<char*>(g) + c * CH), "r"(CH), "r"(b)
                         : "memory");
        }
    };
    // prologue: QD-1 loads in flight
    int it = 0;
    for (int s = 0; s < QD - 1 && c0 + s * stride < chunks; ++s) load(c0 + s * stride, s);
    for (size_t c = c0; c < chunks; c += stride, ++it) {
        const int s = it % QD;
        const size_t cn = c + (QD - 1) * stride;
        if (cn < chunks) {
            const int sn = (it + QD - 1) % QD;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(0) : "memory");  // slot sn's store read
            __syncwarp();
            load(cn, sn);
        }
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[warp][s]);
        asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n}" ::"r"(b),
                     "r"((it / QD) & 1) : "memory");
        double* d = wsm + s * (CH / 8);
        for (int i = lane; i < CH / 8; i += 32) d[i] += 1e-3;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<char*>(g) + c * CH),
                         "r"(base + s * CH), "r"(CH) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F>
float timeit(F f, int reps = 10) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    const size_t bytes = (size_t)64 * 512 * 512 * 16;  // 268 MB
    double* g;
    cudaMalloc(&g, bytes);
    cudaMemset(g, 0, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double traffic = 2.0 * bytes;  // read + write
    float ms = timeit([&] { plain_rmw<<<sms * 8, 256>>>((double2*)g, bytes / 16, 1.0); });
    printf("plain ld/add/st        : %7.1f us  %6.0f GB/s  %s\n", ms * 1e3, traffic / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
#define RED(CH, QD, W)                                                                                        \
    {                                                                                                          \
        auto k = tma_reduce<CH, QD>;                                                                           \
        const int smem = W * QD * CH;                                                                          \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                           \
        ms = timeit([&] { k<<<sms, W * 32, smem>>>(g, bytes); });                                              \
        printf("tma reduce CH %5d QD %2d warps %2d: %7.1f us  %6.0f GB/s  %s\n", CH, QD, W, ms * 1e3,          \
               traffic / ms / 1e6, cudaGetErrorString(cudaGetLastError()));                                    \
    }
    RED(2048, 2, 4) RED(2048, 4, 4) RED(2048, 8, 4) RED(4096, 4, 4) RED(4096, 8, 4) RED(2048, 4, 8)
    RED(2048, 8, 8) RED(8192, 4, 4) RED(512, 8, 4) RED(512, 16, 8)
#define LAS(CH, QD, W)                                                                                        \
    {                                                                                                          \
        auto k = tma_load_add_store<CH, QD>;                                                                   \
        const int smem = W * QD * CH;                                                                          \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                           \
        ms = timeit([&] { k<<<sms, W * 32, smem>>>(g, bytes); });                                              \
        printf("tma load+add+store CH %5d QD %2d warps %2d: %7.1f us  %6.0f GB/s  %s\n", CH, QD, W, ms * 1e3,  \
               traffic / ms / 1e6, cudaGetErrorString(cudaGetLastError()));                                    \
    }
    LAS(2048, 4, 4) LAS(2048, 8, 4) LAS(4096, 4, 4) LAS(4096, 8, 4) LAS(2048, 8, 8)
    return 0;
}
