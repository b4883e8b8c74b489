// g4_prep.cu -- K2 (reference layout -> staged layout) and K3 (device payload
// generator, replaces ringacc/tensor.py:169-228).
#include <algorithm>

#include "g4_common.cuh"
#include "g4_internal.h"

namespace g4 {

constexpr int MAXB = G4_MAX_BATCH;

// ---------------------------------------------------------------------------
// K2: staged[0][r][c] = up[c][r], staged[1][r][c] = down[c][r] -- a 32x32-tile
// transpose of both spins through shared memory; coalesced reads of up/down
// rows, coalesced writes of staged rows.  blockIdx.z = walker.
template <typename Rin, typename Rout>
struct PrepParams {
    const Cx<Rin>* up[MAXB];
    const Cx<Rin>* down[MAXB];
    Cx<Rout>* stg[MAXB];  // spin-planar staged output (2 x N x N)
    int32_t n;
};

template <typename Rin, typename Rout>
__global__ void __launch_bounds__(256) k_prepare(const __grid_constant__ PrepParams<Rin, Rout> P) {
    // staged tile rows r0.. / cols c0.. of the padded layout; sources are the
    // reference rows (c0 + i) mod N, columns (r0 + j) mod N.
    __shared__ Cx<Rin> su[32][33];
    __shared__ Cx<Rin> sd[32][33];
    const int n = P.n;
    const int ld = staged_ld(n, sizeof(Cx<Rout>)), rows = staged_rows(n, sizeof(Cx<Rout>));
    const int w = blockIdx.z;
    const int r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    const Cx<Rin>* up = P.up[w];
    const Cx<Rin>* dn = P.down[w];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int c = c0 + threadIdx.y + 8 * i, r = r0 + threadIdx.x;
        if (c < ld && r < rows) {
            const int64_t o = (int64_t)(c % n) * n + (r % n);
            su[threadIdx.y + 8 * i][threadIdx.x] = up[o];
            sd[threadIdx.y + 8 * i][threadIdx.x] = dn[o];
        }
    }
    __syncthreads();
    Cx<Rout>* out_u = P.stg[w];
    Cx<Rout>* out_d = out_u + staged_plane(n, sizeof(Cx<Rout>));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = r0 + threadIdx.y + 8 * i, c = c0 + threadIdx.x;
        if (c < ld && r < rows) {
            const Cx<Rin> u = su[threadIdx.x][threadIdx.y + 8 * i];
            const Cx<Rin> d = sd[threadIdx.x][threadIdx.y + 8 * i];
            Cx<Rout> vu, vd;
            vu.re = (Rout)u.re;
            vu.im = (Rout)u.im;
            vd.re = (Rout)d.re;
            vd.im = (Rout)d.im;
            out_u[(int64_t)r * ld + c] = vu;
            out_d[(int64_t)r * ld + c] = vd;
        }
    }
}

template <typename Rin, typename Rout>
static g4_status prepare_t(void* const* staged, const void* const* up, const void* const* down,
                           int32_t nbatch, int32_t n, cudaStream_t st) {
    for (int32_t b0 = 0; b0 < nbatch; b0 += MAXB) {
        PrepParams<Rin, Rout> prm{};
        const int nb = std::min<int32_t>(MAXB, nbatch - b0);
        for (int i = 0; i < nb; ++i) {
            if (!staged[b0 + i] || !up[b0 + i] || !down[b0 + i])
                return fail(G4_ERR_CONTRACT, "prepare_g: null pointer");
            if (!aligned(staged[b0 + i], sizeof(Cx<Rout>)) || !aligned(up[b0 + i], sizeof(Cx<Rin>)) ||
                !aligned(down[b0 + i], sizeof(Cx<Rin>)))
                return fail(G4_ERR_CONTRACT, "prepare_g: misaligned payload pointer");
            prm.up[i] = static_cast<const Cx<Rin>*>(up[b0 + i]);
            prm.down[i] = static_cast<const Cx<Rin>*>(down[b0 + i]);
            prm.stg[i] = static_cast<Cx<Rout>*>(staged[b0 + i]);
        }
        prm.n = n;
        const unsigned tr = (unsigned)((staged_rows(n, sizeof(Cx<Rout>)) + 31) / 32),
                       tc = (unsigned)((staged_ld(n, sizeof(Cx<Rout>)) + 31) / 32);
        if (tr > 65535u || tc > 65535u) return fail(G4_ERR_CONTRACT, "prepare_g: N too large");
        k_prepare<Rin, Rout><<<dim3(tr, tc, nb), dim3(32, 8), 0, st>>>(prm);
        G4_CUDA(cudaGetLastError());
    }
    return G4_OK;
}

// ---------------------------------------------------------------------------
// Halo rebuild: stg[s][r][c] = stg[s][r mod N][c mod N] for every entry
// outside the N x N core (rows >= N or columns >= N).  The ring moves only
// payload cores (g4_copy_payload_cores); each receiver restores the halo its
// TMA boxes need.  blockIdx.y = walker * 2 + spin; a flat grid-stride index
// over the bottom band (rows N..ROWS-1, all columns) then the right band
// (rows 0..N-1, columns N..LD-1).
template <typename R>
struct HaloParams {
    Cx<R>* stg[MAXB];
    int32_t n;
};

template <typename R>
__global__ void __launch_bounds__(256) k_fill_halo(const __grid_constant__ HaloParams<R> P) {
    const int n = P.n;
    const int ld = staged_ld(n, sizeof(Cx<R>)), rows = staged_rows(n, sizeof(Cx<R>));
    const int w = blockIdx.y >> 1, s = blockIdx.y & 1;
    Cx<R>* base = P.stg[w] + (int64_t)s * staged_plane(n, sizeof(Cx<R>));
    const int64_t bottom = (int64_t)(rows - n) * ld, right = (int64_t)n * (ld - n);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < bottom + right;
         i += (int64_t)gridDim.x * blockDim.x) {
        int r, c;
        if (i < bottom) {
            r = n + (int)(i / ld);
            c = (int)(i % ld);
        } else {
            const int64_t j = i - bottom;
            r = (int)(j / (ld - n));
            c = n + (int)(j % (ld - n));
        }
        base[(int64_t)r * ld + c] = base[(int64_t)(r % n) * ld + (c % n)];
    }
}

template <typename R>
static g4_status fill_halo_t(void* const* staged, int32_t count, int32_t n, cudaStream_t st) {
    for (int32_t b0 = 0; b0 < count; b0 += MAXB) {
        HaloParams<R> prm{};
        const int nb = std::min<int32_t>(MAXB, count - b0);
        for (int i = 0; i < nb; ++i) {
            if (!staged[b0 + i] || !aligned(staged[b0 + i], sizeof(Cx<R>)))
                return fail(G4_ERR_CONTRACT, "fill_halo: null or misaligned payload");
            prm.stg[i] = static_cast<Cx<R>*>(staged[b0 + i]);
        }
        prm.n = n;
        const int64_t halo = (int64_t)(staged_rows(n, sizeof(Cx<R>)) - n) * staged_ld(n, sizeof(Cx<R>)) +
                             (int64_t)n * (staged_ld(n, sizeof(Cx<R>)) - n);
        const unsigned bx = (unsigned)std::min<int64_t>((halo + 255) / 256, 1024);
        k_fill_halo<R><<<dim3(bx, 2 * nb), 256, 0, st>>>(prm);
        G4_CUDA(cudaGetLastError());
    }
    return G4_OK;
}

// ---------------------------------------------------------------------------
// K3: generator.  Entry idx of matrix m of walker (seed, world_rank, lane, meas):
//   key  = stream_key(seed, world_rank, lane, meas, m)            (tensor.py:182-186)
//   u1   = top53(mix(key ^ 2 idx)),  u2 = top53(mix(key ^ (2 idx + 1)))  (tensor.py:196-198)
//   float:   r = sqrt(u1), th = (2 pi) u2, value = (r cos th, r sin th)  (tensor.py:199-203)
//   integer: value = (floor(5 u1) - 2, floor(5 u2) - 2)                  (tensor.py:204-209)
template <typename R>
struct GenParams {
    Cx<R>* stg[MAXB];
    Cx<R>* up[MAXB];
    Cx<R>* down[MAXB];
    uint64_t key_up[MAXB];
    uint64_t key_down[MAXB];
    int32_t n;
    int32_t mode;
};

__device__ __forceinline__ double top53(uint64_t b) { return (double)(b >> 11) * 0x1.0p-53; }

__device__ __forceinline__ void gen_entry(uint64_t key, uint64_t idx, int mode, double& re, double& im) {
    const double u1 = top53(mix64(key ^ (idx * 2u)));
    const double u2 = top53(mix64(key ^ (idx * 2u + 1u)));
    if (mode == G4_MODE_FLOAT) {
        const double r = __dsqrt_rn(u1);
        const double th = __dmul_rn(2.0 * 3.141592653589793, u2);
        double s, c;
        sincos(th, &s, &c);
        re = __dmul_rn(r, c);
        im = __dmul_rn(r, s);
    } else {
        re = __dadd_rn(floor(__dmul_rn(u1, 5.0)), -2.0);
        im = __dadd_rn(floor(__dmul_rn(u2, 5.0)), -2.0);
    }
}

// Staged output: thread (r, c) of the padded layout, c fastest ->
// stg[0][r][c] = up[c mod N][r mod N], stg[1][r][c] = down[c mod N][r mod N]
// (entry index of up[c'][r'] is c'*N + r'; halo entries are regenerated).
template <typename R>
__global__ void __launch_bounds__(256) k_generate_staged(const __grid_constant__ GenParams<R> P) {
    const int n = P.n, w = blockIdx.z;
    const int ld = staged_ld(n, sizeof(Cx<R>)), rows = staged_rows(n, sizeof(Cx<R>));
    const int c = blockIdx.x * 32 + threadIdx.x;
    const int r = blockIdx.y * 8 + threadIdx.y;
    if (c >= ld || r >= rows) return;
    const uint64_t idx = (uint64_t)(c % n) * n + (r % n);
    double ur, ui, dr, di;
    gen_entry(P.key_up[w], idx, P.mode, ur, ui);
    gen_entry(P.key_down[w], idx, P.mode, dr, di);
    Cx<R> vu, vd;
    vu.re = (R)ur;
    vu.im = (R)ui;
    vd.re = (R)dr;
    vd.im = (R)di;
    P.stg[w][(int64_t)r * ld + c] = vu;
    P.stg[w][staged_plane(n, sizeof(Cx<R>)) + (int64_t)r * ld + c] = vd;
}

// Reference-layout output: thread per row-major entry idx.
template <typename R>
__global__ void __launch_bounds__(256) k_generate_ref(const __grid_constant__ GenParams<R> P) {
    const int n = P.n, w = blockIdx.y;
    const int64_t nn = (int64_t)n * n;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < nn;
         idx += (int64_t)gridDim.x * blockDim.x) {
        double re, im;
        if (P.up[w]) {
            gen_entry(P.key_up[w], (uint64_t)idx, P.mode, re, im);
            P.up[w][idx].re = (R)re;
            P.up[w][idx].im = (R)im;
        }
        if (P.down[w]) {
            gen_entry(P.key_down[w], (uint64_t)idx, P.mode, re, im);
            P.down[w][idx].re = (R)re;
            P.down[w][idx].im = (R)im;
        }
    }
}

static uint64_t stream_key(uint64_t seed, int64_t wr, int64_t lane, int64_t meas, int64_t m) {
    uint64_t k = mix64(seed);
    k = mix64(k ^ (uint64_t)wr);
    k = mix64(k ^ (uint64_t)lane);
    k = mix64(k ^ (uint64_t)meas);
    return mix64(k ^ (uint64_t)m);
}

template <typename R>
static g4_status generate_t(void* const* staged, void* const* up, void* const* down, int32_t nbatch,
                            uint64_t seed, const int64_t* wr, const int64_t* lane, const int64_t* meas,
                            int32_t n, int32_t mode, cudaStream_t st) {
    for (int32_t b0 = 0; b0 < nbatch; b0 += MAXB) {
        const int nb = std::min<int32_t>(MAXB, nbatch - b0);
        GenParams<R> prm{};
        prm.n = n;
        prm.mode = mode;
        bool any_stg = false, any_ref = false;
        for (int i = 0; i < nb; ++i) {
            const int j = b0 + i;
            prm.key_up[i] = stream_key(seed, wr[j], lane[j], meas[j], 0);
            prm.key_down[i] = stream_key(seed, wr[j], lane[j], meas[j], 1);
            prm.stg[i] = staged ? static_cast<Cx<R>*>(staged[j]) : nullptr;
            prm.up[i] = up ? static_cast<Cx<R>*>(up[j]) : nullptr;
            prm.down[i] = down ? static_cast<Cx<R>*>(down[j]) : nullptr;
            if (prm.stg[i] && !aligned(prm.stg[i], sizeof(Cx<R>)))
                return fail(G4_ERR_CONTRACT, "generate: misaligned staged pointer");
            any_stg |= prm.stg[i] != nullptr;
            any_ref |= (prm.up[i] != nullptr) || (prm.down[i] != nullptr);
        }
        if (any_stg) {
            for (int i = 0; i < nb; ++i)
                if (!prm.stg[i]) return fail(G4_ERR_CONTRACT, "generate: staged list has a null entry");
            dim3 grid((unsigned)((staged_ld(n, sizeof(Cx<R>)) + 31) / 32), (unsigned)((staged_rows(n, sizeof(Cx<R>)) + 7) / 8),
                      nb);
            if (grid.y > 65535u) return fail(G4_ERR_CONTRACT, "generate: N too large");
            k_generate_staged<R><<<grid, dim3(32, 8), 0, st>>>(prm);
            G4_CUDA(cudaGetLastError());
        }
        if (any_ref) {
            const int64_t nn = (int64_t)n * n;
            const unsigned gx = (unsigned)std::min<int64_t>((nn + 255) / 256, 4096);
            k_generate_ref<R><<<dim3(gx, nb), 256, 0, st>>>(prm);
            G4_CUDA(cudaGetLastError());
        }
    }
    return G4_OK;
}

}  // namespace g4

extern "C" {

g4_status g4_prepare_g(void* const* staged, const void* const* up, const void* const* down,
                       int32_t nbatch, int32_t n, int32_t dtype_in, int32_t dtype_out, void* stream) {
    using namespace g4;
    if (n < 1) return fail(G4_ERR_CONTRACT, "prepare_g: n must be >= 1");
    if (nbatch < 0) return fail(G4_ERR_CONTRACT, "prepare_g: nbatch must be >= 0");
    if (nbatch == 0) return G4_OK;
    if (!staged || !up || !down) return fail(G4_ERR_CONTRACT, "prepare_g: null pointer list");
    auto st = static_cast<cudaStream_t>(stream);
    if (dtype_in == G4_C128 && dtype_out == G4_C128)
        return prepare_t<double, double>(staged, up, down, nbatch, n, st);
    if (dtype_in == G4_C64 && dtype_out == G4_C64)
        return prepare_t<float, float>(staged, up, down, nbatch, n, st);
    if (dtype_in == G4_C128 && dtype_out == G4_C64)
        return prepare_t<double, float>(staged, up, down, nbatch, n, st);
    return fail(G4_ERR_CONTRACT, "prepare_g: unsupported dtype pair");
}

// CUDA loads kernels lazily at their first launch, and a load waits for the
// context.  The halo kernel is first launched behind a ring flag wait, so it
// is loaded up front by the ring hosts (engine.RingEngine, g4_ring_create).
g4_status g4_preload_ring_kernels(void) {
    using namespace g4;
    cudaFuncAttributes a;
    G4_CUDA(cudaFuncGetAttributes(&a, k_fill_halo<double>));
    G4_CUDA(cudaFuncGetAttributes(&a, k_fill_halo<float>));
    return G4_OK;
}

g4_status g4_fill_halo(void* const* staged, int32_t count, int32_t n, int32_t dtype, void* stream) {
    using namespace g4;
    if (n < 1 || count < 0) return fail(G4_ERR_CONTRACT, "fill_halo: bad n or count");
    if (count == 0) return G4_OK;
    if (!staged) return fail(G4_ERR_CONTRACT, "fill_halo: null pointer list");
    auto st = static_cast<cudaStream_t>(stream);
    if (dtype == G4_C128) return fill_halo_t<double>(staged, count, n, st);
    if (dtype == G4_C64) return fill_halo_t<float>(staged, count, n, st);
    return fail(G4_ERR_CONTRACT, "fill_halo: unknown dtype");
}

g4_status g4_generate(void* const* staged, void* const* up, void* const* down, int32_t nbatch,
                      uint64_t seed, const int64_t* world_rank, const int64_t* lane,
                      const int64_t* meas, int32_t n, int32_t mode, int32_t dtype, void* stream) {
    using namespace g4;
    if (n < 1) return fail(G4_ERR_CONTRACT, "generate: n must be >= 1");
    if (nbatch < 0) return fail(G4_ERR_CONTRACT, "generate: nbatch must be >= 0");
    if (nbatch == 0) return G4_OK;
    if (!world_rank || !lane || !meas) return fail(G4_ERR_CONTRACT, "generate: null origin arrays");
    if (mode != G4_MODE_FLOAT && mode != G4_MODE_INTEGER) {
        set_error("unknown value mode %d", mode);
        return G4_ERR_CONTRACT;
    }
    auto st = static_cast<cudaStream_t>(stream);
    if (dtype == G4_C128)
        return generate_t<double>(staged, up, down, nbatch, seed, world_rank, lane, meas, n, mode, st);
    if (dtype == G4_C64)
        return generate_t<float>(staged, up, down, nbatch, seed, world_rank, lane, meas, n, mode, st);
    return fail(G4_ERR_CONTRACT, "generate: unknown dtype");
}

}  // extern "C"
