// g4_k1.cuh -- pieces of K1 (the G4 slice update) shared by its kernels: the
// multi-plane TMA kernel (g4_accumulate.cu) and the persistent TMEM-handoff
// kernel (g4_accumulate_pst.cu).  Device helpers (mbarriers, TMA boxes, bulk
// write-back, the fused update) and the host-side tensor-map cache.
#pragma once
#include <cstdint>
#include <cstdlib>

#include <cuda.h>

#include "g4_common.cuh"
#include "g4_internal.h"

namespace g4 {

template <typename To, typename From>
__device__ __forceinline__ Stg<To> widen(const Stg<From>& v) {
    Stg<To> r;
    r.ur = (To)v.ur;
    r.ui = (To)v.ui;
    r.dr = (To)v.dr;
    r.di = (To)v.di;
    return r;
}

// L2-aware CTA order.  A 1-D grid is walked in blocks of TILE_BY column chunks x
// TILE_BZ row groups (plane chunks fastest inside a block): every CTA that needs
// a given payload row segment (direct tile or K3-diagonal band) then runs within
// a few waves of the others, so the payload rows stay L2-resident even when one
// staged payload is far larger than L2 (N = 4608: 0.7 GB per walker).
constexpr int TILE_BY = 16, TILE_BZ = 32;

struct TileCoord {
    int x, y, z;
};

__device__ __forceinline__ TileCoord tile_coord(unsigned lin, int nx, int ny, int nz, int tby = TILE_BY,
                                                int tbz = TILE_BZ) {
    const unsigned per_row = (unsigned)nx * ny * tbz;  // CTAs in a full block row
    const int br = (int)(lin / per_row);
    unsigned r = lin - (unsigned)br * per_row;
    const int bze = min(tbz, nz - br * tbz);
    const unsigned per_blk = (unsigned)nx * tby * bze;
    const int by = (int)(r / per_blk);
    r -= (unsigned)by * per_blk;
    const int bye = min(tby, ny - by * tby);
    TileCoord t;
    t.x = (int)(r % nx);
    r /= nx;
    t.y = by * tby + (int)(r % bye);
    t.z = br * tbz + (int)(r / bye);
    return t;
}

__device__ __forceinline__ int wrap(int x, int n) {
    while (x < 0) x += n;
    while (x >= n) x -= n;
    return x;
}

// G4_ARITH_FUSED: the same two products and sums as 8 FMAs chained into the
// accumulator (no rounded intermediates): ~1 ulp per update from the reference
// order, far inside north_star's 1e-10 relative tolerance; integer-valued
// inputs stay exact.  Each entry is two independent 4-deep FMA chains.
template <typename R>
__device__ __forceinline__ void update_fused(Cx<R>& a, const Stg<R>& S, const Stg<R>& D) {
    R re = fma_rn(S.ur, D.dr, a.re);
    R im = fma_rn(S.ur, D.di, a.im);
    re = fma_rn(-S.ui, D.di, re);
    im = fma_rn(S.ui, D.dr, im);
    re = fma_rn(S.dr, D.ur, re);
    im = fma_rn(S.dr, D.ui, im);
    re = fma_rn(-S.di, D.ui, re);
    im = fma_rn(S.di, D.ur, im);
    a.re = re;
    a.im = im;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
// Same, with a suspend-time hint: the waiting warp sleeps until the phase
// completes (or 10 ms pass) instead of re-polling, so idle waiters -- the
// epilogue and producer warps of K1 v3 -- do not take issue slots from the
// consumer warps on their SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, 10000000;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
// 3-D tensor box -> shared memory, completion counted on an mbarrier.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
// Same, with an L2 cache policy (createpolicy) on the loaded lines.
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Same, delivered to every CTA of the cluster in `mask` (same smem offsets and
// mbarrier offset in each destination CTA).
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                               uint64_t* bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
        : "memory");
}
// Arrive on the mbarrier at the same offset in cluster CTA `rank` (default
// .release.cta semantics: a .cluster-scope release costs a MEMBAR per arrive,
// 3.7 stall cycles per issue in the first cut).
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* b, uint32_t rank) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\t"
        "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.shared::cluster.b64 _, [ra];\n}" ::"r"(smem_u32(b)),
        "r"(rank)
        : "memory");
}
// Cluster barrier without a release fence: the mbarrier inits it publishes are
// ordered by fence.mbarrier_init.release.cluster (an .arrive.release would add
// a MEMBAR.GPU, ~2 us per CTA behind in-flight global traffic).
__device__ __forceinline__ void cluster_sync_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
constexpr int TMA_MAXW = 32;  // walkers per launch (2 tensor maps each, kernel params)

template <typename R>
struct alignas(64) TmaParams {
    CUtensorMap dmap[TMA_MAXW];  // direct tiles: sheared map, 4-row boxes
    CUtensorMap smap[TMA_MAXW];  // shifted bands: sheared map, NSH-row boxes
    CUtensorMap gmap;            // the slice, sheared: (x, k1, plane) -> G4[plane][k1][k1 + x - N]
    int32_t use_gmap;            // gmap encoded (complex128 slices)
    Cx<R>* g4;
    int64_t lo, hi;
    int32_t n;
    int32_t nbatch;
    int32_t nx;   // plane chunks
    int32_t off;  // sheared-coordinate offset (elements), see make_maps
    int32_t hints;  // v3 lab knobs (G4RING_V3_HINTS): 2 = L2 evict_last on the payload boxes, 64 =
                    // suspend-time waits for the producer and the epilogue (both within noise, r02ac)
    long long* trace;  // v3 lab timeline (G4RING_V3_TRACE), else null
    int32_t chain;     // deferred passes: the previous K1 on the stream was one too (slice
                       // reductions only): no waits before the first loads and reductions, one
                       // before the CTA exits (k1_chain_prev)
};

// Shared -> global bulk copy by the TMA engine: add (.add reduction) or store.
template <bool ADD, typename R>
__device__ __forceinline__ void bulk_out(void* dst, uint32_t src, int bytes) {
    if constexpr (!ADD)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(dst), "r"(src), "r"(bytes) : "memory");
    else if constexpr (sizeof(R) == 8)
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;"
                     ::"l"(dst), "r"(src), "r"(bytes) : "memory");
    else
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                     ::"l"(dst), "r"(src), "r"(bytes) : "memory");
}
template <typename R>
constexpr bool BULK_SLICE = sizeof(R) == 8;  // slices written back by the TMA engine (complex128)
// One entry through the LSU (segment edges the TMA cannot take).
template <bool ADD, typename R>
__device__ __forceinline__ void entry_out(Cx<R>* g, const Cx<R>& v) {
    if constexpr (ADD) {
        atomicAdd(&g->re, v.re);
        atomicAdd(&g->im, v.im);
    } else {
        *g = v;
    }
}
// `count` entries from shared `s` to global `g`: bulk where both are 16-B
// aligned, LSU for an odd head/tail (complex64) or a misaligned pair.
template <bool ADD, typename R>
__device__ __forceinline__ void segment_out(Cx<R>* g, const Cx<R>* s, int count) {
    if (count <= 0) return;
    if (reinterpret_cast<uintptr_t>(g) & 15) {
        entry_out<ADD>(g, *s);
        ++g, ++s, --count;
    }
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(s));
    if (sa & 15) {
        for (int i = 0; i < count; ++i) entry_out<ADD>(g + i, s[i]);
        return;
    }
    const int m = count & ~(16 / (int)sizeof(Cx<R>) - 1);  // whole 16-B units
    if (m > 0) bulk_out<ADD, R>(g, sa, m * (int)sizeof(Cx<R>));
    if (m < count) entry_out<ADD>(g + m, s[m]);
}
inline int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}

// Plain shared-memory loads the scheduler may move (ordered after the stage's
// mbarrier wait by that asm's memory clobber).
__device__ __forceinline__ Stg<double> lds_plain(const Cx<double>* u, const Cx<double>* d) {
    const double2 a = *reinterpret_cast<const double2*>(u);
    const double2 b = *reinterpret_cast<const double2*>(d);
    Stg<double> v;
    v.ur = a.x;
    v.ui = a.y;
    v.dr = b.x;
    v.di = b.y;
    return v;
}
__device__ __forceinline__ Stg<float> lds_plain(const Cx<float>* u, const Cx<float>* d) {
    const float2 a = *reinterpret_cast<const float2*>(u);
    const float2 b = *reinterpret_cast<const float2*>(d);
    Stg<float> v;
    v.ur = a.x;
    v.ui = a.y;
    v.dr = b.x;
    v.di = b.y;
    return v;
}

using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                     const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                     const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct MapPair {
    CUtensorMap dmap, smap;
};

// Host (g4_accumulate.cu): the sheared tensor maps of one staged payload
// (cached by pointer and box), the sheared write-back map of a complex128
// slice, and the sheared coordinate offset.
int sheared_offset(int n, int es);
g4_status get_maps(const void* stg, int n, int es, int nsh, int width, int dd, int band_spins, MapPair* out);
bool g4_gmap_enabled();
g4_status slice_map(const void* g4, int n, int64_t planes, int pp, int dd, CUtensorMap* out);

// Chained fused passes.  Two deferred fused passes (v3, or v2 with K1_DEFER) on
// one stream touch the slice only through reductions, which commute: the later one needs no griddepcontrol.wait
// before its loads and reductions, only one before it exits (so its completion
// still implies the earlier pass's).  The library records per stream whether
// its last K1 launch there was such a pass (k1_chain_prev); any other K1 launch
// clears the record, and a pass that starts a chain waits for its predecessor
// before it lets the next launch begin.  Work of anything else between two
// launches serialises the stream anyway (only K1 kernels trigger early).
bool k1_chain_prev(cudaStream_t st);
void k1_chain_note(bool chain_safe);

// K1 v3 (g4_accumulate_pst.cu): the persistent fused update of a complex128
// slice with payload entries RG; geometry ids 40-42.
template <typename RG>
g4_status launch_pst(int geom, bool exact, void* g4p, int64_t lo, int64_t hi, int32_t n, const void* const* staged,
                     int32_t nbatch, cudaStream_t st);
bool pst_geom_info(int geom, int* pp, int* dd, int* q, int* dr, int* nst);
// K1 v3 for complex64 slices (fused, deferred; geometry 45).
g4_status launch_pst32(int geom, void* g4p, int64_t lo, int64_t hi, int32_t n, const void* const* staged,
                       int32_t nbatch, cudaStream_t st);

}  // namespace g4
