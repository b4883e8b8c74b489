// tools/microbench.cu -- calibration microbenchmarks (not product code) for the
// quantities the K1 design depends on: FP64 DFMA issue rate and dependent
// latency, FP32 FFMA rate, conflict-free shared-memory LDS.128 bandwidth.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void fp64_tput(double* out, int iters, double a, double b) {
    double x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __fma_rn(x[k], a, b);
    double s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void fp64_lat(double* out, long long* cyc, int iters, double a, double b) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = __fma_rn(x, a, b);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void fp32_tput(float* out, int iters, float a, float b) {
    float x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __fmaf_rn(x[k], a, b);
    float s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void lds128(double* out, int iters) {
    __shared__ double2 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_double2(i, -i);
    __syncthreads();
    double acc0 = 0, acc1 = 0;
    const int base = (threadIdx.x & ~31) + (threadIdx.x & 31);
    for (int i = 0; i < iters; ++i) {
        double2 v = s[(base + 32 * (i & 31)) & 2047];   // warp reads 32 consecutive 16-B slots
        acc0 += v.x;
        acc1 += v.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* d; cudaMalloc(&d, 1 << 26);
    long long* c; cudaMalloc(&c, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 20000; float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a); fp64_tput<<<sms * 4, 256>>>(d, iters, 1.0000001, 1e-9); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("fp64 DFMA throughput: %.2f T instr/s (%.1f TFLOP/s)\n", (double)sms * 4 * 256 * iters * 8 / ms / 1e9,
               2.0 * sms * 4 * 256 * iters * 8 / ms / 1e9);
        fp64_lat<<<1, 32>>>(d, c, iters, 1.0000001, 1e-9); cudaDeviceSynchronize();
        long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        printf("fp64 DFMA dependent latency: %.1f cycles\n", (double)cy / iters);
        cudaEventRecord(a); fp32_tput<<<sms * 4, 256>>>((float*)d, iters, 1.0000001f, 1e-9f); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("fp32 FFMA throughput: %.2f T instr/s\n", (double)sms * 4 * 256 * iters * 8 / ms / 1e9);
        cudaEventRecord(a); lds128<<<sms * 4, 256>>>(d, iters); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)sms * 4 * 256 * iters * 16;
        printf("lds.128 conflict-free: %.2f TB/s (%.1f B/clk/SM at %.0f MHz)\n", bytes / ms / 1e9,
               bytes / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3);
    }
    return 0;
}
