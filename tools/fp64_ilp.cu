// tools/fp64_ilp.cu -- FP64 issue rate vs warps per SM and independent chains per
// thread (calibration for K1's register/occupancy trade-off; not product code).
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void fp64_ilp(double* out, int iters, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < ILP; ++k) x[k] = __fma_rn(x[k], a, b);
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// the exact-order update chain: 4 DMUL -> 4 DFMA -> 2 DADD -> 2 DADD into acc, E entries per thread
template <int E>
__global__ void exact_chain(double* out, int iters, double a, double b) {
    double ar[E], ai[E];
#pragma unroll
    for (int k = 0; k < E; ++k) { ar[k] = threadIdx.x + k; ai[k] = k; }
    double ur = a, ui = b, dr = a * b, di = a - b;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
            double m1 = __dmul_rn(ui, di), m2 = __dmul_rn(ui, dr), m3 = __dmul_rn(di, ui), m4 = __dmul_rn(di, ur);
            double p1r = __fma_rn(ur, dr, -m1), p1i = __fma_rn(ur, di, m2);
            double p2r = __fma_rn(dr, ur, -m3), p2i = __fma_rn(dr, ui, m4);
            ar[k] = __dadd_rn(ar[k], __dadd_rn(p1r, p2r));
            ai[k] = __dadd_rn(ai[k], __dadd_rn(p1i, p2i));
        }
        ur = __dadd_rn(ur, 1e-30);  // keep operands loop-variant
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < E; ++k) s += ar[k] + ai[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <class K>
static void run(const char* name, K kern, int warps_per_sm, int ops_per_iter, int sms, double* d) {
    const int threads = 128, blocks = sms * warps_per_sm / 4, iters = 4000;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    kern<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(a); kern<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9); cudaEventRecord(b);
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-14s warps/SM %2d: %6.2f T FP64 instr/s\n", name, warps_per_sm,
           (double)blocks * threads * iters * ops_per_iter / ms / 1e9);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d; cudaMalloc(&d, 1 << 26);
    for (int w : {4, 8, 12, 16, 32}) {
        run("dfma ilp1", fp64_ilp<1>, w, 1, sms, d);
        run("dfma ilp2", fp64_ilp<2>, w, 2, sms, d);
        run("dfma ilp4", fp64_ilp<4>, w, 4, sms, d);
        run("dfma ilp8", fp64_ilp<8>, w, 8, sms, d);
        run("exact e1", exact_chain<1>, w, 13, sms, d);
        run("exact e2", exact_chain<2>, w, 25, sms, d);
        run("exact e4", exact_chain<4>, w, 49, sms, d);
    }
    return 0;
}
