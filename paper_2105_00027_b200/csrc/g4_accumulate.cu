// g4_accumulate.cu -- K1, the G4 slice update (replaces ringacc/tensor.py:233-251).
//
// Reference semantics, per owned plane K3 = q and entry (k1, k2):
//   G4[q][k1][k2] += up[(q-k2)%N][(q-k1)%N] * down[k2][k1]
//                  + down[(q-k2)%N][(q-k1)%N] * up[k2][k1]
// On the staged payload stg[r][c] = {up[c][r], down[c][r]} this reads
//   S = stg[(q-k1)%N][(q-k2)%N]   ("shifted")   and   D = stg[k1][k2]   ("direct"):
//   p1 = S.u * D.d ; p2 = S.d * D.u ; t = p1 + p2 ; G += t
// which is the reference's exact op order (tensor.py:250: u*down + d*up, then +=).
//
// Work decomposition (HBM-bound gather-multiply-accumulate; no tensor cores):
//   * one thread owns a PP x DD block of G4 entries: planes q0..q0+PP-1 and the
//     diagonal (k1_0 + d, c + d), d < DD.  For such a block the shifted index
//     (q-k1, q-k2) depends only on m = p - d, so PP*DD updates per walker need
//     only DD direct and PP+DD-1 shifted staged loads (one 256-bit load each for
//     complex128: both spins of one element);
//   * a warp's 32 lanes own 32 consecutive k2 columns: every G4 access is a
//     contiguous 512 B row segment (coalesced 128-bit loads/stores), every
//     staged access a contiguous 1 KB row segment (forward or reversed);
//   * the G4 block is read once, receives all `nbatch` walkers in order
//     (bitwise equal to nbatch sequential reference calls), written once:
//     HBM traffic per pass = 2 * P * N^2 * eb + staged reads;
//   * blockIdx.x = plane chunk (fastest) so concurrently resident CTAs share
//     the same (k1, k2) tile and its staged rows stay in L2.
#include <algorithm>

#include "g4_common.cuh"
#include "g4_internal.h"

namespace g4 {

template <typename R>
struct AccParams {
    Cx<R>* g4;
    int64_t lo, hi;
    int32_t n;
    int32_t nbatch;
    const Stg<R>* stg[G4_MAX_BATCH];
};

__device__ __forceinline__ int wrap(int x, int n) {
    while (x < 0) x += n;
    while (x >= n) x -= n;
    return x;
}

template <typename R, int PP, int DD, int WARPS>
__global__ void __launch_bounds__(32 * WARPS)
k_accumulate(const __grid_constant__ AccParams<R> P) {
    constexpr int NS = PP + DD - 1;  // distinct shifted elements per thread
    const int n = P.n;
    const int k1_0 = (blockIdx.z * WARPS + threadIdx.y) * DD;
    if (k1_0 >= n) return;  // warp-uniform
    const int c_raw = blockIdx.y * 32 + threadIdx.x;
    const bool col_ok = c_raw < n;
    const int c = col_ok ? c_raw : 0;
    const int64_t q0 = P.lo + (int64_t)blockIdx.x * PP;

    // Direct operand offsets: stg[k1_0 + d][(c + d) % N].
    int offd[DD];
    int colg[DD];
    bool rowok[DD];
#pragma unroll
    for (int d = 0; d < DD; ++d) {
        const int k1 = k1_0 + d;
        rowok[d] = k1 < n;
        colg[d] = wrap(c + d, n);
        offd[d] = (rowok[d] ? k1 : 0) * n + colg[d];
    }
    // Shifted operand offsets: stg[(q0 - k1_0 + m) % N][(q0 - c + m) % N],
    // m = p - d in [-(DD-1), PP-1]  (q0, k1_0, c all in [0, N)).
    int offs[NS];
    {
        const int rb = wrap((int)(q0 - k1_0), n);
        const int cb = wrap((int)(q0 - c), n);
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            const int m = j - (DD - 1);
            offs[j] = wrap(rb + m, n) * n + wrap(cb + m, n);
        }
    }

    // Load the accumulator block.
    Cx<R> acc[PP][DD];
    bool ok[PP][DD];
    Cx<R>* gp[PP][DD];
#pragma unroll
    for (int p = 0; p < PP; ++p) {
        const bool pok = (q0 + p) < P.hi;
        const int64_t plane = (q0 + p - P.lo) * (int64_t)n;
#pragma unroll
        for (int d = 0; d < DD; ++d) {
            ok[p][d] = pok && rowok[d] && col_ok;
            gp[p][d] = P.g4 + (plane + (rowok[d] ? k1_0 + d : 0)) * n + colg[d];
            if (ok[p][d]) {
                acc[p][d] = ld_g4(gp[p][d]);
            } else {
                acc[p][d].re = R(0);
                acc[p][d].im = R(0);
            }
        }
    }

#pragma unroll 1
    for (int w = 0; w < P.nbatch; ++w) {
        const Stg<R>* s = P.stg[w];
        Stg<R> dv[DD];
        Stg<R> sv[NS];
#pragma unroll
        for (int d = 0; d < DD; ++d) dv[d] = ld_stg(s + offd[d]);
#pragma unroll
        for (int j = 0; j < NS; ++j) sv[j] = ld_stg(s + offs[j]);
#pragma unroll
        for (int p = 0; p < PP; ++p) {
#pragma unroll
            for (int d = 0; d < DD; ++d) {
                const Stg<R>& S = sv[p - d + DD - 1];
                const Stg<R>& D = dv[d];
                R p1r, p1i, p2r, p2i;
                cmul(S.ur, S.ui, D.dr, D.di, p1r, p1i);  // u * down[k2][k1]
                cmul(S.dr, S.di, D.ur, D.ui, p2r, p2i);  // d * up[k2][k1]
                acc[p][d].re = add_rn(acc[p][d].re, add_rn(p1r, p2r));
                acc[p][d].im = add_rn(acc[p][d].im, add_rn(p1i, p2i));
            }
        }
    }

#pragma unroll
    for (int p = 0; p < PP; ++p)
#pragma unroll
        for (int d = 0; d < DD; ++d)
            if (ok[p][d]) st_g4(gp[p][d], acc[p][d]);
}

template <typename R, int PP, int DD, int WARPS>
static g4_status launch_acc(const AccParams<R>& prm, cudaStream_t st) {
    const int n = prm.n;
    const int64_t planes = prm.hi - prm.lo;
    const int diag_blocks = (n + DD - 1) / DD;
    dim3 grid((unsigned)((planes + PP - 1) / PP), (unsigned)((n + 31) / 32),
              (unsigned)((diag_blocks + WARPS - 1) / WARPS));
    if (grid.y > 65535u || grid.z > 65535u)
        return fail(G4_ERR_CONTRACT, "accumulate: N too large for the launch grid");
    dim3 block(32, WARPS);
    k_accumulate<R, PP, DD, WARPS><<<grid, block, 0, st>>>(prm);
    return check_cuda(cudaGetLastError(), "k_accumulate launch");
}

template <typename R>
static g4_status accumulate_t(void* g4p, int64_t lo, int64_t hi, int32_t n,
                              const void* const* staged, int32_t nbatch, cudaStream_t st) {
    const uintptr_t stg_align = sizeof(Stg<R>);
    if (!aligned(g4p, sizeof(Cx<R>)))
        return fail(G4_ERR_CONTRACT, "accumulate: g4 slice pointer is not entry-aligned");
    for (int32_t b0 = 0; b0 < nbatch; b0 += G4_MAX_BATCH) {
        AccParams<R> prm{};
        prm.g4 = static_cast<Cx<R>*>(g4p);
        prm.lo = lo;
        prm.hi = hi;
        prm.n = n;
        prm.nbatch = std::min<int32_t>(G4_MAX_BATCH, nbatch - b0);
        for (int i = 0; i < prm.nbatch; ++i) {
            const void* sp = staged[b0 + i];
            if (!sp) return fail(G4_ERR_CONTRACT, "accumulate: null staged payload");
            if (!aligned(sp, stg_align))
                return fail(G4_ERR_CONTRACT, "accumulate: staged payload is not 32B/16B aligned");
            prm.stg[i] = static_cast<const Stg<R>*>(sp);
        }
        G4_TRY((launch_acc<R, 4, 4, 4>(prm, st)));
    }
    return G4_OK;
}

}  // namespace g4

extern "C" {

g4_status g4_accumulate_staged(void* g4p, int64_t lo, int64_t hi, int32_t n,
                               const void* const* staged, int32_t nbatch, int32_t dtype,
                               int32_t channel, void* stream) {
    using namespace g4;
    if (n < 1) return fail(G4_ERR_CONTRACT, "index space size must be >= 1");
    if (!(0 <= lo && lo < hi && hi <= n)) {
        set_error("invalid axis range [%lld, %lld) for N=%d", (long long)lo, (long long)hi, n);
        return G4_ERR_CONTRACT;
    }
    if (channel != G4_CHANNEL_EQ1)
        return fail(G4_ERR_CONTRACT, "unknown channel (only G4_CHANNEL_EQ1, the reference's Eq. 1)");
    if (nbatch < 0) return fail(G4_ERR_CONTRACT, "nbatch must be >= 0");
    if (nbatch == 0) return G4_OK;
    if (!g4p || !staged) return fail(G4_ERR_CONTRACT, "accumulate: null pointer");
    auto st = static_cast<cudaStream_t>(stream);
    if (dtype == G4_C128) return accumulate_t<double>(g4p, lo, hi, n, staged, nbatch, st);
    if (dtype == G4_C64) return accumulate_t<float>(g4p, lo, hi, n, staged, nbatch, st);
    return fail(G4_ERR_CONTRACT, "unknown dtype");
}

int64_t g4_accumulate_workspace_bytes(int32_t n, int32_t nbatch, int32_t dtype) {
    const int64_t pb = g4_payload_bytes(n, dtype);
    if (pb < 0 || nbatch < 0) return -1;
    return pb * std::min<int32_t>(nbatch, G4_MAX_BATCH);
}

g4_status g4_accumulate(void* g4p, int64_t lo, int64_t hi, int32_t n, const void* const* up,
                        const void* const* down, int32_t nbatch, int32_t dtype, int32_t channel,
                        void* workspace, int64_t workspace_bytes, void* stream) {
    using namespace g4;
    if (nbatch < 0) return fail(G4_ERR_CONTRACT, "nbatch must be >= 0");
    if (nbatch == 0) return g4_accumulate_staged(g4p, lo, hi, n, nullptr, 0, dtype, channel, stream);
    const int64_t need = g4_accumulate_workspace_bytes(n, nbatch, dtype);
    if (need < 0) return fail(G4_ERR_CONTRACT, "accumulate: bad n/dtype");
    if (!workspace || workspace_bytes < need)
        return fail(G4_ERR_CONTRACT, "accumulate: workspace too small");
    const int64_t pb = g4_payload_bytes(n, dtype);
    void* stg[G4_MAX_BATCH];
    for (int32_t b0 = 0; b0 < nbatch; b0 += G4_MAX_BATCH) {
        const int32_t nb = std::min<int32_t>(G4_MAX_BATCH, nbatch - b0);
        for (int i = 0; i < nb; ++i) stg[i] = static_cast<char*>(workspace) + i * pb;
        G4_TRY(g4_prepare_g(stg, up + b0, down + b0, nb, n, dtype, dtype, stream));
        G4_TRY(g4_accumulate_staged(g4p, lo, hi, n, stg, nb, dtype, channel, stream));
    }
    return G4_OK;
}

}  // extern "C"
