// tools/k1_core_bench.cu -- lab: the K1 consumer inner loop in isolation (no TMA,
// no barriers): PP x DD register block, fused update, operands from shared
// memory, register cap MAXR (the consumer budget under setmaxnreg), 8 warps per
// SM -- the DFMA rate the loop structure itself reaches.  Not product code.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
struct Stg { double ur, ui, dr, di; };
__device__ __forceinline__ Stg lds(const double2* u, const double2* d) {
    double2 a = *u, b = *d; Stg v; v.ur = a.x; v.ui = a.y; v.dr = b.x; v.di = b.y; return v;
}
__device__ __forceinline__ void upd(double2& a, const Stg& S, const Stg& D) {
    double re = __fma_rn(S.ur, D.dr, a.x), im = __fma_rn(S.ur, D.di, a.y);
    re = __fma_rn(-S.ui, D.di, re); im = __fma_rn(S.ui, D.dr, im);
    re = __fma_rn(S.dr, D.ur, re); im = __fma_rn(S.dr, D.ui, im);
    re = __fma_rn(-S.di, D.ui, re); im = __fma_rn(S.di, D.ur, im);
    a.x = re; a.y = im;
}
template <int PP, int DD, int MAXR, bool SYNC, int NT = 256>
__global__ void __launch_bounds__(NT, 1) __maxnreg__(MAXR) core(double* out, int walkers) {
    constexpr int NJ = PP + DD - 1;
    extern __shared__ double2 sm[];  // 4 stages x [spin][48 rows][32]
    __shared__ uint64_t bar;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 4 * 2 * 48 * 32; i += blockDim.x) sm[i] = make_double2(i * 1e-3, -i * 1e-3);
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(1));
    __syncthreads();
    double2 acc[PP][DD];
    for (int p = 0; p < PP; ++p) for (int d = 0; d < DD; ++d) acc[p][d] = make_double2(0, 0);
    const int wo = (warp & 7) * 2;
#pragma unroll 1
    for (int w = 0; w < walkers; ++w) {
        const double2* U = sm + (w & 3) * 2 * 48 * 32;
        const double2* Dn = U + 48 * 32;
        Stg D[DD];
#pragma unroll
        for (int d = 0; d < DD; ++d) D[d] = lds(U + (d + wo) * 32 + lane, Dn + (d + wo) * 32 + lane);
        Stg S = lds(U + (16 + wo) * 32 + (31 - lane), Dn + (16 + wo) * 32 + (31 - lane));
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            Stg Sn;
            if (j + 1 < NJ) Sn = lds(U + (17 + wo + j) * 32 + (31 - lane), Dn + (17 + wo + j) * 32 + (31 - lane));
#pragma unroll
            for (int d = 0; d < DD; ++d) { const int p = j + d - (DD - 1); if (p >= 0 && p < PP) upd(acc[p][d], S, D[d]); }
            if (j + 1 < NJ) S = Sn;
        }
        if (SYNC) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
        }
    }
    double s = 0;
    for (int p = 0; p < PP; ++p) for (int d = 0; d < DD; ++d) s += acc[p][d].x + acc[p][d].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int PP, int DD, int MAXR, bool SYNC, int NT = 256>
void run(double* out, int sms) {
    const int walkers = 2000;
    const size_t smem = 4 * 2 * 48 * 32 * 16;
    auto k = core<PP, DD, MAXR, SYNC, NT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<<<sms, NT, smem>>>(out, walkers);
    cudaEventRecord(a);
    k<<<sms, NT, smem>>>(out, walkers);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double dfma = (double)sms * NT * walkers * PP * DD * 8;
    printf("warps %2d PP %d DD %d maxreg %3d sync %d: %6.2f T DFMA/s (%5.1f%% of 16.56)  %s\n", NT / 32, PP, DD, MAXR, (int)SYNC,
           dfma / ms / 1e9, dfma / ms / 1e9 / 16.56 * 100, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, sms * 1024 * 8);
    run<8, 4, 255, false>(out, sms);
    run<8, 4, 255, true>(out, sms);
    run<8, 4, 232, true>(out, sms);
    run<8, 4, 216, true>(out, sms);
    run<8, 4, 200, true>(out, sms);
    run<8, 3, 216, true>(out, sms);
    run<8, 3, 200, true>(out, sms);
    run<8, 3, 184, true>(out, sms);
    run<6, 4, 216, true>(out, sms);
    run<8, 2, 168, true>(out, sms);
    run<8, 2, 168, true, 384>(out, sms);
    run<8, 3, 168, true, 384>(out, sms);
    run<6, 4, 168, true, 384>(out, sms);
    run<4, 4, 128, true, 512>(out, sms);
    run<8, 4, 216, true, 256>(out, sms);
    return 0;
}
