/*
 * g4_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the reference hot path in ringacc/tensor.py
 * (/root/reference/pkg/src/ringacc/tensor.py).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 *
 * Parity pin: tests/test_oracle.py checks every function here against golden
 * vectors produced by the real reference (oracle/make_golden.py imports
 * ringacc from /root/reference and writes tests/golden/ (npz)):
 *   - accumulate: bitwise in float and integer mode (numpy's complex multiply on
 *     an FMA3/AVX-512 host is (fma(xr,yr,-(xi*yi)), fma(xr,yi,xi*yr)); measured
 *     here against numpy 2.3.5 bitwise).
 *   - generator: bitwise in integer mode; float mode within 2 ulp (numpy's
 *     SIMD cos/sin vs glibc).
 *
 * Build: oracle/Makefile  (gcc -O2 -ffp-contract=off: no implicit contraction,
 * every fused multiply-add is an explicit fma() call in the reference order).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define G4O_GOLDEN 0x9E3779B97F4A7C15ULL

/* SplitMix64 finalizer -- tensor.py:169-179 (_mix64). */
uint64_t g4o_mix64(uint64_t z)
{
    z += G4O_GOLDEN;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* tensor.py:182-186 (_stream_key): key = mix(seed); then
 * key = mix(key ^ part) for part in (world_rank, lane, meas, matrix). */
uint64_t g4o_stream_key(uint64_t seed, int64_t world_rank, int64_t lane,
                        int64_t meas, int64_t matrix)
{
    uint64_t k = g4o_mix64(seed);
    k = g4o_mix64(k ^ (uint64_t)world_rank);
    k = g4o_mix64(k ^ (uint64_t)lane);
    k = g4o_mix64(k ^ (uint64_t)meas);
    k = g4o_mix64(k ^ (uint64_t)matrix);
    return k;
}

/* tensor.py:189-191 (_uniform01): top 53 bits -> [0, 1). */
static double u01(uint64_t bits) { return (double)(bits >> 11) * 0x1.0p-53; }

/* tensor.py:194-212 (_matrix_entries): one N x N matrix, row-major,
 * interleaved (re, im).  mode 0 = float (unit disk), 1 = integer lattice. */
static void matrix_entries(uint64_t key, int32_t n, int32_t mode, double* out)
{
    const double two_pi = 2.0 * 3.141592653589793; /* 2.0 * np.pi, tensor.py:202 */
    int64_t nn = (int64_t)n * n;
    for (int64_t idx = 0; idx < nn; ++idx) {
        double a = u01(g4o_mix64(key ^ ((uint64_t)idx * 2u)));
        double b = u01(g4o_mix64(key ^ ((uint64_t)idx * 2u + 1u)));
        double re, im;
        if (mode == 0) {
            double r = sqrt(a);
            double th = two_pi * b;
            re = r * cos(th);
            im = r * sin(th);
        } else {
            re = floor(a * 5.0) - 2.0;
            im = floor(b * 5.0) - 2.0;
        }
        out[2 * idx] = re;
        out[2 * idx + 1] = im;
    }
}

/* tensor.py:215-220 (fill_gsigma): up = matrix 0, down = matrix 1. */
void g4o_fill_gsigma(uint64_t seed, int64_t world_rank, int64_t lane, int64_t meas,
                     int32_t n, int32_t mode, double* up, double* down)
{
    matrix_entries(g4o_stream_key(seed, world_rank, lane, meas, 0), n, mode, up);
    matrix_entries(g4o_stream_key(seed, world_rank, lane, meas, 1), n, mode, down);
}

/* numpy complex multiply x*y as executed by the reference (see header). */
static inline void cmul(double xr, double xi, double yr, double yi, double* zr, double* zi)
{
    *zr = fma(xr, yr, -(xi * yi));
    *zi = fma(xr, yi, xi * yr);
}

/* tensor.py:233-251 (accumulate_g4), restated per entry:
 *   for k3 in [lo, hi):  idx = (k3 - arange(N)) % N                 (247)
 *     u = up[idx][:, idx]; d = down[idx][:, idx]                   (248-249)
 *     data[k3-lo] += (u*down + d*up).T                             (250)
 * i.e. data[k3-lo][k1][k2] += up[(k3-k2)%N][(k3-k1)%N] * down[k2][k1]
 *                           + down[(k3-k2)%N][(k3-k1)%N] * up[k2][k1]
 * evaluated as p1 = u*down, p2 = d*up, t = p1 + p2, G += t.
 * g4 is ((hi-lo) x N x N) complex128 interleaved; up/down N x N complex128. */
void g4o_accumulate(double* g4, int64_t lo, int64_t hi, int32_t n,
                    const double* up, const double* down)
{
    for (int64_t k3 = lo; k3 < hi; ++k3) {
        double* plane = g4 + (k3 - lo) * (int64_t)n * n * 2;
        for (int32_t k1 = 0; k1 < n; ++k1) {
            int64_t c = ((k3 - k1) % n + n) % n;        /* (K3 - K1) mod N */
            for (int32_t k2 = 0; k2 < n; ++k2) {
                int64_t r = ((k3 - k2) % n + n) % n;    /* (K3 - K2) mod N */
                const double* u = up + 2 * (r * n + c);
                const double* d = down + 2 * (r * n + c);
                const double* dn = down + 2 * ((int64_t)k2 * n + k1);
                const double* upd = up + 2 * ((int64_t)k2 * n + k1);
                double p1r, p1i, p2r, p2i;
                cmul(u[0], u[1], dn[0], dn[1], &p1r, &p1i);
                cmul(d[0], d[1], upd[0], upd[1], &p2r, &p2i);
                double tr = p1r + p2r, ti = p1i + p2i;
                double* g = plane + 2 * ((int64_t)k1 * n + k2);
                g[0] = g[0] + tr;
                g[1] = g[1] + ti;
            }
        }
    }
}

/* complex64 variant: same index map and op order in binary32 (G, G4 complex64). */
static inline void cmulf(float xr, float xi, float yr, float yi, float* zr, float* zi)
{
    *zr = fmaf(xr, yr, -(xi * yi));
    *zi = fmaf(xr, yi, xi * yr);
}

void g4o_accumulate_c64(float* g4, int64_t lo, int64_t hi, int32_t n,
                        const float* up, const float* down)
{
    for (int64_t k3 = lo; k3 < hi; ++k3) {
        float* plane = g4 + (k3 - lo) * (int64_t)n * n * 2;
        for (int32_t k1 = 0; k1 < n; ++k1) {
            int64_t c = ((k3 - k1) % n + n) % n;
            for (int32_t k2 = 0; k2 < n; ++k2) {
                int64_t r = ((k3 - k2) % n + n) % n;
                const float* u = up + 2 * (r * n + c);
                const float* d = down + 2 * (r * n + c);
                const float* dn = down + 2 * ((int64_t)k2 * n + k1);
                const float* upd = up + 2 * ((int64_t)k2 * n + k1);
                float p1r, p1i, p2r, p2i;
                cmulf(u[0], u[1], dn[0], dn[1], &p1r, &p1i);
                cmulf(d[0], d[1], upd[0], upd[1], &p2r, &p2i);
                float tr = p1r + p2r, ti = p1i + p2i;
                float* g = plane + 2 * ((int64_t)k1 * n + k2);
                g[0] = g[0] + tr;
                g[1] = g[1] + ti;
            }
        }
    }
}

/* tensor.py:50-55 (index_diff): (a - b) mod N; -1 when out of range
 * (the reference raises ContractViolation). */
int64_t g4o_index_diff(int64_t a, int64_t b, int64_t n)
{
    if (!(0 <= a && a < n && 0 <= b && b < n)) return -1;
    return ((a - b) % n + n) % n;
}

/* tensor.py:148-164 (make_partition): balanced contiguous ranges, remainder
 * to the lowest ranks.  ranges = 2*p int64 (lo, hi).  Returns 0, or -1 when
 * p < 1 or p > n (ContractViolation in the reference). */
int32_t g4o_partition(int64_t n, int64_t p, int64_t* ranges)
{
    if (p < 1 || p > n) return -1;
    int64_t base = n / p, rem = n % p, lo = 0;
    for (int64_t i = 0; i < p; ++i) {
        int64_t hi = lo + base + (i < rem ? 1 : 0);
        ranges[2 * i] = lo;
        ranges[2 * i + 1] = hi;
        lo = hi;
    }
    return 0;
}
