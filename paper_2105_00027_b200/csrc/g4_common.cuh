// g4_common.cuh -- shared device helpers for the G4 ring-accumulation library.
//
// Exact-order complex arithmetic.  The reference computes every G4 update with
// numpy complex128 ops (ringacc/tensor.py:250); on FMA hosts numpy's complex
// multiply is  x*y = (fma(xr, yr, -(xi*yi)), fma(xr, yi, xi*yr))  (pinned
// bitwise in tests/test_oracle.py).  Every operation here uses an explicit
// round-to-nearest intrinsic so nvcc can neither contract nor reorder it.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/g4ring.h"
#include "g4_layout.h"

namespace g4 {

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }

// z = x * y in the reference's rounding order.
template <typename R>
__device__ __forceinline__ void cmul(R xr, R xi, R yr, R yi, R& zr, R& zi) {
    zr = fma_rn(xr, yr, -mul_rn(xi, yi));
    zi = fma_rn(xr, yi, mul_rn(xi, yr));
}

// One G4 entry (complex).
template <typename R>
struct alignas(2 * sizeof(R)) Cx {
    R re, im;
};

// One staged walker element in registers: (u, d) = (up^T, down^T) at one (row, col).
template <typename R>
struct Stg {
    R ur, ui, dr, di;
};


// Read-only loads of a staged element: u from the up^T plane, d from the down^T plane.
__device__ __forceinline__ Stg<double> ld_stg(const Cx<double>* u, const Cx<double>* d) {
    Stg<double> v;
    asm("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v.ur), "=d"(v.ui) : "l"(u));
    asm("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v.dr), "=d"(v.di) : "l"(d));
    return v;
}
__device__ __forceinline__ Stg<float> ld_stg(const Cx<float>* u, const Cx<float>* d) {
    Stg<float> v;
    asm("ld.global.nc.v2.f32 {%0,%1}, [%2];" : "=f"(v.ur), "=f"(v.ui) : "l"(u));
    asm("ld.global.nc.v2.f32 {%0,%1}, [%2];" : "=f"(v.dr), "=f"(v.di) : "l"(d));
    return v;
}

// Same, as volatile asm: the walker's loads keep their program order ahead of
// the math that consumes them, so all of them are in flight at once.
__device__ __forceinline__ Stg<double> ld_stg_v(const Cx<double>* u, const Cx<double>* d) {
    Stg<double> v;
    asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v.ur), "=d"(v.ui) : "l"(u));
    asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v.dr), "=d"(v.di) : "l"(d));
    return v;
}
__device__ __forceinline__ Stg<float> ld_stg_v(const Cx<float>* u, const Cx<float>* d) {
    Stg<float> v;
    asm volatile("ld.global.nc.v2.f32 {%0,%1}, [%2];" : "=f"(v.ur), "=f"(v.ui) : "l"(u));
    asm volatile("ld.global.nc.v2.f32 {%0,%1}, [%2];" : "=f"(v.dr), "=f"(v.di) : "l"(d));
    return v;
}

// G4 slice entries stream through once per pass.  Loads bypass L1 (.cg):
// measured 10 % faster than .cs at B = 1 (5.57 vs 5.05 TB/s, profiles/lab/r01_lab15.txt).
// Stores are evict-first (.cs), so the walkers' staged G's (re-read across
// planes) keep the L2; .cg and write-back stores were slower.
__device__ __forceinline__ Cx<double> ld_g4(const Cx<double>* p) {
    Cx<double> v;
    asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(v.re), "=d"(v.im) : "l"(p));
    return v;
}
__device__ __forceinline__ Cx<float> ld_g4(const Cx<float>* p) {
    Cx<float> v;
    asm volatile("ld.global.cg.v2.f32 {%0,%1}, [%2];" : "=f"(v.re), "=f"(v.im) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_g4(Cx<double>* p, Cx<double> v) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.re), "d"(v.im) : "memory");
}
__device__ __forceinline__ void st_g4(Cx<float>* p, Cx<float> v) {
    asm volatile("st.global.cs.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(v.re), "f"(v.im) : "memory");
}

// x mod n for any int64 x (setup paths only).
__device__ __forceinline__ int mod_n(int64_t x, int n) {
    int64_t r = x % n;
    return (int)(r < 0 ? r + n : r);
}

// SplitMix64 finalizer (ringacc/tensor.py:169-179).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

}  // namespace g4
