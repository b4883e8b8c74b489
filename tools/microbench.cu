// tools/microbench.cu -- calibration microbenchmarks (not product code):
// FP64 DFMA issue rate, FP32 FFMA rate, and shared-memory LDS.128/256 throughput on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void fp64(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b); x3 = __fma_rn(x3, a, b);
        x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b); x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void fp32(float* out, int iters, float a, float b) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = __fmaf_rn(x0, a, b); x1 = __fmaf_rn(x1, a, b); x2 = __fmaf_rn(x2, a, b); x3 = __fmaf_rn(x3, a, b);
        x4 = __fmaf_rn(x4, a, b); x5 = __fmaf_rn(x5, a, b); x6 = __fmaf_rn(x6, a, b); x7 = __fmaf_rn(x7, a, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void lds(double* out, int iters) {
    __shared__ double4 s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_double4(i, i, i, i);
    __syncthreads();
    double acc = 0; int idx = threadIdx.x;
    for (int i = 0; i < iters; ++i) { double4 v = s[(idx + i) & 1023]; acc += v.x + v.w; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d; cudaMalloc(&d, 1 << 26);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int iters = 20000; float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a); fp64<<<sms * 4, 256>>>(d, iters, 1.0000001, 1e-9); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("fp64 DFMA: %.3f T instr/s (%.2f TFLOP/s)\n", (double)sms * 4 * 256 * iters * 8 / ms / 1e9, 2.0 * sms * 4 * 256 * iters * 8 / ms / 1e9);
        cudaEventRecord(a); fp32<<<sms * 4, 256>>>((float*)d, iters, 1.0000001f, 1e-9f); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("fp32 FFMA: %.3f T instr/s\n", (double)sms * 4 * 256 * iters * 8 / ms / 1e9);
        cudaEventRecord(a); lds<<<sms * 4, 256>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("lds.256: %.2f TB/s smem (%.1f B/clk/SM @1.965GHz)\n", (double)sms * 4 * 256 * iters * 32 / ms / 1e9, (double)sms * 4 * 256 * iters * 32 / ms / 1e-3 / sms / 1.965e9);
    }
    return 0;
}
