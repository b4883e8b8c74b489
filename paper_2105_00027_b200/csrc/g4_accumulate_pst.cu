// g4_accumulate_pst.cu -- K1 v3: the persistent, warp-specialised fused update
// of a complex128 slice with a tensor-memory hand-off (replaces, like v2,
// ringacc/tensor.py:233-251; G4_ARITH_FUSED with the deferred update).
//
// One CTA per SM loops over CTA tiles (Q planes x DR diagonal entries x 32
// columns; the tile order is v2's L2-aware tile_coord, CTA c taking tiles c,
// c + grid, ...).  Four warp groups:
//   WG0-1 consumers (8 warps, 216 registers): each owns a PP x DD register
//     block per tile (v2's block and op sequence: update_fused over the walkers
//     in order, from zero accumulators).  After the tile's last walker the
//     block goes to tensor memory (tcgen05.st, 128 columns per warp, two
//     buffers) and the warp starts the next tile at once.
//   WG2 epilogue (4 warps, 56 registers): warp 8 + q drains TMEM lane quarter
//     q (tcgen05.ld) for the two consumer warps that own it, parks each
//     (plane, 4-diagonal) chunk of 2 KB in shared memory and adds it to the
//     slice in L2 with one TMA tensor reduce (sheared slice map, box 32 x 4 x 1)
//     -- the deferred update of v2, now off the consumers' critical path.
//   WG3 producer (1 active lane, 24 registers): streams both TMA boxes of every
//     walker of every tile into an NST-stage ring, running ahead across tile
//     boundaries (no pipeline drain or refill between tiles).
//   Edge chunks (row segments that wrap at N, a partial last column strip)
//     are not one tensor-map box: every lane adds its own entries there
//     (red.global), keeping those drains as short as the interior ones.
//   The CTA's last tile is written back by the consumers themselves from the
//     then-idle stages.
//   Launched with programmatic dependent launch: the prologue (barrier init,
//     TMEM alloc, L2 prefetch of the first boxes) overlaps the previous
//     kernel's tail; payload loads and slice updates wait for it
//     (griddepcontrol.wait).
//   EXACT = true: G4_ARITH_EXACT in the same structure (block loaded at tile
//     start, reference op order, TMA stores) -- selectable (G4RING_V3_EXACT),
//     measured slower than geometry 13.
// What this removes against v2 (geometry 25, one 4-warp tile per CTA, 4096
// CTAs): the per-CTA prologue (barrier init, first fills landing) and epilogue
// (park + bulk reduce + waiting for it to read) on every tile, and one of the
// two CTAs per SM sitting in them; and the CTA tile doubles (8 consumer warps),
// cutting the TMA fill bytes per update from 7.75 to 5.9 B.  DESIGN.md §4.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "g4_k1.cuh"

namespace g4 {

// Geometry: PP x DD thread block, CWQ x CWR consumer warps (CW = 8), NST
// stages of both boxes, NPARK 2-KB park slots per epilogue warp.
template <typename RG, int PP_, int DD_, int CWQ_, int CWR_, int NST_, int NPARK_>
struct V3Geom {
    static constexpr int PP = PP_, DD = DD_, CWQ = CWQ_, CWR = CWR_, NST = NST_, NPARK = NPARK_;
    static constexpr int CW = CWQ * CWR;
    static_assert(CW == 8, "two consumer warp groups");
    static constexpr int THREADS = 512;                      // 4 warp groups
    static constexpr int Q = PP * CWQ, DR = DD * CWR;       // CTA tile: planes x diagonal entries
    static constexpr int ES = sizeof(Cx<RG>);               // payload entry bytes
    static constexpr int NSH = Q + DR - 1;                  // shifted band rows
    static constexpr int W = ES == 8 ? 34 : 32;             // box row width (entries), see V2Geom
    static constexpr int DIR_ELEMS = DR * W, SH_ELEMS = NSH * W;
    static constexpr uint32_t DIR_BYTES = 2 * DIR_ELEMS * ES;
    static constexpr uint32_t SH_BYTES = 2 * SH_ELEMS * ES;
    static constexpr uint32_t DIR_OFF = 0;
    static constexpr uint32_t SH_OFF = (DIR_BYTES + 127) / 128 * 128;
    static constexpr uint32_t STAGE_BYTES = (SH_OFF + SH_BYTES + 127) / 128 * 128;
    static constexpr uint32_t CHUNK_BYTES = DD * 32 * 16;   // one (plane, DD diagonals) chunk of the slice
    static constexpr uint32_t PARK_OFF = NST * STAGE_BYTES;
    static constexpr uint32_t PARK_BYTES = 4 * NPARK * CHUNK_BYTES;
    static constexpr uint32_t BAR_OFF = PARK_OFF + PARK_BYTES;
    static constexpr size_t SMEM = BAR_OFF + (2 * NST + 4) * sizeof(uint64_t) + 16;
    static constexpr int BLOCK_COLS = PP * DD * 4;          // TMEM columns per consumer warp block
    // the last tile's blocks (CW x PP chunks) fit the idle stage buffers: consumers write it back
    static constexpr bool LAST_DIRECT = (size_t)CW * PP * CHUNK_BYTES <= (size_t)NST * STAGE_BYTES;
    static_assert(2 * 2 * BLOCK_COLS <= 512, "two buffers x two consumer warps per lane quarter");
    static_assert(SMEM <= 227 * 1024, "v3 stages + park exceed shared memory");
    static_assert(NPARK % 2 == 0 && NPARK >= 4, "park slots hold chunk pairs");
    static_assert(PP % 2 == 0, "the epilogue drains chunk pairs");
    static_assert(NSH <= G4_HALO_ROWS && NSH + W + 1 < G4_HALO_COLS && DR + W <= G4_HALO_COLS,
                  "halo too small for the v3 boxes");
};

// Register budget of the four warp groups (setmaxnreg): 2 x 128 x 216 +
// 128 x 56 + 128 x 24 = 65536 (the epilogue holds a 32-register TMEM load;
// the consumers fit 216 without spills).
constexpr int V3_REG_CONSUMER = 216, V3_REG_EPILOGUE = 56, V3_REG_PRODUCER = 24;

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
        ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
        "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
        "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
}
// Lab timeline (G4RING_V3_TRACE): row 31 of a CTA's trace holds %globaltimer
// stamps (ns, comparable across SMs): 0 CTA entry, 1 first payload landed,
// 2 consumers done, 3 epilogue done, 4 producer done.
__device__ __forceinline__ void trace_gt(long long* tr, int slot) {
    if (tr) {
        long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tr[((size_t)blockIdx.x * 32 + 31) * 8 + slot] = t;
    }
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Per-tile geometry shared by the three roles.
struct V3Tile {
    int64_t q0;
    int k1_0, j0;
};
template <class G, typename R>
__device__ __forceinline__ V3Tile v3_tile(const TmaParams<R>& P, int lin) {
    const int n = P.n;
    const TileCoord tc = tile_coord((unsigned)lin, P.nx, (n + 31) / 32, (n + G::DR - 1) / G::DR);
    return {P.lo + (int64_t)tc.x * G::Q, tc.z * G::DR, tc.y * 32};
}
// (Tile walks measured and dropped, lab r02h-k: plane chunks slowest, contiguous
// runs per CTA, smaller blocks of the walk, the order reversed on alternate
// passes; an L2 prefetch of the G4 block by TMA or LSU, r02e/i.)

// The CTA's tiles: CTA c takes tiles c, c + grid, ... of the L2-aware order.
// (A dynamic claim from a global counter was measured 20 % slower, lab r02l:
// it breaks the waves' shared payload rows in L2.)
__device__ __forceinline__ int v3_count(int ntiles) {
    const int b = (int)blockIdx.x, g = (int)gridDim.x;
    return b < ntiles ? (ntiles - 1 - b) / g + 1 : 0;
}
__device__ __forceinline__ int v3_lin(int k) { return (int)blockIdx.x + k * (int)gridDim.x; }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// G4_ARITH_EXACT in the same structure: the reference op order per walker
// (u*down + d*up rounded, then added), the consumers load their block at the
// tile's start (the epilogue has pulled it into L2 while the previous tile
// computed) and the epilogue stores instead of reducing.
template <typename R>
__device__ __forceinline__ void update_exact(Cx<R>& a, const Stg<R>& S, const Stg<R>& D) {
    R p1r, p1i, p2r, p2i;
    cmul(S.ur, S.ui, D.dr, D.di, p1r, p1i);  // u * down[k2][k1]
    cmul(S.dr, S.di, D.ur, D.ui, p2r, p2i);  // d * up[k2][k1]
    a.re = add_rn(a.re, add_rn(p1r, p2r));
    a.im = add_rn(a.im, add_rn(p1i, p2i));
}
// Exact mode: epilogue warp q pulls the G4 rows of its two blocks of tile t
// into L2 (prefetch.global.L2, 5 points per 512-B row segment).
template <class G>
__device__ __forceinline__ void v3_prefetch_g4(const TmaParams<double>& P, const V3Tile& t, int q, int lane) {
    constexpr int PP = G::PP, DD = G::DD, PTS = 5;
    const int n = P.n;
#pragma unroll 1
    for (int i = lane; i < 2 * PP * DD * PTS; i += 32) {
        const int pt = i % PTS, row = (i / PTS) % DD, pl = (i / (PTS * DD)) % PP, h = i / (PTS * DD * PP);
        const int cw = q + 4 * h, wq = cw % G::CWQ, wr = cw / G::CWQ;
        const int plane = (int)(t.q0 - P.lo) + PP * wq + pl;
        const int k1 = t.k1_0 + DD * wr + row;
        if (plane >= (int)(P.hi - P.lo) || k1 >= n) continue;
        int k2 = t.j0 + DD * wr + row + (pt == 4 ? 31 : 8 * pt);
        while (k2 >= n) k2 -= n;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(P.g4 + ((int64_t)plane * n + k1) * n + k2));
    }
}

// One slice entry of an edge chunk (row k1, column k2 before the wrap, the lane's
// column c of the 32-wide strip), by the lane holding it: red.global.add.f64
// pairs (exact mode: a store).  Rows past N and columns past a partial last
// strip do not exist.  Each lane writes its own entries, so the warp's row
// segments stay coalesced -- one lane walking the chunk with bulk ops (the
// round-2 first cut) took 5.8x an interior drain on the 1/16 of tiles whose
// row segments wrap (lab r02p/q).
template <bool EXACT>
__device__ __forceinline__ void edge_entry(const TmaParams<double>& P, int plane, int k1, int k2, int c, double re,
                                           double im) {
    const int n = P.n;
    if (k1 >= n || c >= n) return;
    if (k2 >= n) k2 -= n;
    double* g = reinterpret_cast<double*>(P.g4 + ((int64_t)plane * n + k1) * n + k2);
    if constexpr (EXACT) {
        asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(g), "d"(re), "d"(im) : "memory");
    } else {
        asm volatile("red.global.add.f64 [%0], %1;" ::"l"(g), "d"(re) : "memory");
        asm volatile("red.global.add.f64 [%0], %1;" ::"l"(g + 1), "d"(im) : "memory");
    }
}

template <typename RG, class G, bool EARLY_ST, bool EXACT>
__global__ void __launch_bounds__(512, 1) k_accumulate_pst(const __grid_constant__ TmaParams<double> P) {
    using R = double;
    constexpr int PP = G::PP, DD = G::DD, NST = G::NST, DR = G::DR;
    constexpr int EW = G::ES / 8;  // 64-bit TMA elements per payload entry
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + G::BAR_OFF);
    uint64_t* empty = full + NST;
    uint64_t* tfull = empty + NST;  // [2] consumers -> epilogue: the tile's blocks are in TMEM buffer b
    uint64_t* tready = tfull + 2;   // [2] epilogue -> consumers: TMEM buffer b has been drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tready + 2);

    const int n = P.n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = P.nx * ((n + 31) / 32) * ((n + DR - 1) / DR);
    const int my_tiles = v3_count(ntiles);
    const int nb = P.nbatch;

    if (threadIdx.x == 0) {
        trace_gt(P.trace, 0);
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], G::CW);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], G::CW);
            mbar_init(&tready[b], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // the next K1 launch on this stream may start as our CTAs retire (programmatic
        // dependent launch; it waits for our completion before it reads payloads or
        // writes the slice, unless it chains on us -- k1_chain_prev).  A fused pass
        // that starts a chain lets the next launch begin only once its own
        // predecessor is complete: chained passes do not wait for it.
        if (!EXACT && !P.chain) pdl_wait();
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    if (warp == 8) {  // the whole of TMEM (one CTA per SM)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= 12) {
        // ---------------- producer ----------------
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(V3_REG_PRODUCER) : "memory");
        if (threadIdx.x == 384) {
            if (my_tiles > 0) {
                // Before waiting for the previous kernel: pull this CTA's first
                // walkers' boxes into L2 (an L2 prefetch reads through the point of
                // coherence, so it cannot yield stale data for the loads below)
                const V3Tile t = v3_tile<G>(P, v3_lin(0));
                const int R0 = wrap((int)(t.q0 - t.k1_0) - (DR - 1), n);
                const int C0 = wrap((int)(t.q0 - t.j0) - 31 - (DR - 1), n);
                const int xd = t.j0 - t.k1_0 + P.off, xs = C0 - R0 + P.off;
                const int pd = (G::ES == 8) ? (xd & 1) : 0, ps = (G::ES == 8) ? (xs & 1) : 0;
                for (int w = 0; w < min(nb, NST); ++w) {
                    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];"
                                 ::"l"(reinterpret_cast<uint64_t>(&P.dmap[w])), "r"(EW * (xd - pd)), "r"(t.k1_0),
                                 "r"(0) : "memory");
                    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];"
                                 ::"l"(reinterpret_cast<uint64_t>(&P.smap[w])), "r"(EW * (xs - ps)), "r"(R0),
                                 "r"(0) : "memory");
                }
            }
            if (!P.chain) pdl_wait();  // the payloads may come from the previous kernel on the stream
            const uint64_t keep = l2_policy_evict_last();  // payload rows are re-read by many tiles
            int it = 0;
            for (int k = 0; k < my_tiles; ++k) {
                const V3Tile t = v3_tile<G>(P, v3_lin(k));
                const int R0 = wrap((int)(t.q0 - t.k1_0) - (DR - 1), n);
                const int C0 = wrap((int)(t.q0 - t.j0) - 31 - (DR - 1), n);
                const int xd = t.j0 - t.k1_0 + P.off, xs = C0 - R0 + P.off;
                const int pd = (G::ES == 8) ? (xd & 1) : 0, ps = (G::ES == 8) ? (xs & 1) : 0;
                for (int w = 0; w < nb; ++w, ++it) {
                    const int s = it % NST;
                    if (it >= NST) { if (P.hints & 64) mbar_wait_sleep(&empty[s], ((it / NST) - 1) & 1); else mbar_wait(&empty[s], ((it / NST) - 1) & 1); }
                    mbar_arrive_expect_tx(&full[s], G::DIR_BYTES + G::SH_BYTES);
                    unsigned char* st = smem_raw + (size_t)s * G::STAGE_BYTES;
                    if (P.hints & 2) {
                        tma_load_3d_hint(st + G::DIR_OFF, &P.dmap[w], EW * (xd - pd), t.k1_0, 0, &full[s], keep);
                        tma_load_3d_hint(st + G::SH_OFF, &P.smap[w], EW * (xs - ps), R0, 0, &full[s], keep);
                    } else {
                        tma_load_3d(st + G::DIR_OFF, &P.dmap[w], EW * (xd - pd), t.k1_0, 0, &full[s]);
                        tma_load_3d(st + G::SH_OFF, &P.smap[w], EW * (xs - ps), R0, 0, &full[s]);
                    }
                }
            }
            trace_gt(P.trace, 4);
            if (P.chain) pdl_wait();  // chained: we complete only after the previous pass does
        }
        __syncwarp();
        return;
    }

    if (warp >= 8) {
        // ---------------- epilogue ----------------
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(V3_REG_EPILOGUE) : "memory");
        const int q = warp - 8;  // TMEM lane quarter (and consumer warps q, q + 4)
        // park: NPARK slots of a chunk PAIR (2 x 2 KB) per epilogue warp
        const uint32_t park0 = smem_u32(smem_raw + G::PARK_OFF) + (uint32_t)q * G::NPARK * G::CHUNK_BYTES +
                               lane * (uint32_t)sizeof(Cx<R>);
        const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);
        const uint64_t gmap = reinterpret_cast<uint64_t>(&P.gmap);
        int pair = 0;  // chunk pairs parked by this warp (slot = pair % NSLOT)
        constexpr int NSLOT = G::NPARK / 2;
        if (!P.chain) pdl_wait();  // the previous kernel's slice updates land first
        const int drained = G::LAST_DIRECT ? my_tiles - 1 : my_tiles;  // see consumers
        for (int k = 0; k < drained; ++k) {
            const int b = k & 1;
            if (EXACT && k + 1 < drained) v3_prefetch_g4<G>(P, v3_tile<G>(P, v3_lin(k + 1)), q, lane);
            if (P.hints & 64) mbar_wait_sleep(&tfull[b], (k >> 1) & 1);  // 64: suspend-time waits (lab)
            else mbar_wait(&tfull[b], (k >> 1) & 1);
            tc_fence_after();
            if (P.trace && k < 31 && lane == 0) P.trace[((size_t)blockIdx.x * 32 + k) * 8 + 0 + 6 * (q == 3)] = clock64();
            const V3Tile t = v3_tile<G>(P, v3_lin(k));
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const int cw = q + 4 * h, wq = cw % G::CWQ, wr = cw / G::CWQ;
                const int p_lo = (int)(t.q0 - P.lo) + PP * wq;  // slice-relative plane of p = 0
                const int e0 = DD * wr;
                const int k1b = t.k1_0 + e0;  // row of diagonal 0 (< 2N)
                const bool box = P.use_gmap && k1b + DD - 1 < n && t.j0 + 31 + e0 + DD - 1 < n;
                const int c0 = 2 * (t.j0 - t.k1_0 + n);
                const int np = min(PP, (int)(P.hi - P.lo) - p_lo);  // planes of the block inside the slice
                const uint32_t tb = tq + b * 256 + h * G::BLOCK_COLS;
#pragma unroll 1
                for (int p = 0; p < np; p += 2) {
                    uint32_t v[32];
                    tmem_ld32(tb + p * 16, v);
                    tmem_wait_ld();
                    if (!box) {  // row wrap / last column strip: every lane adds its own entries
                        for (int c = 0; c < 2 && p + c < np; ++c)
#pragma unroll
                            for (int d = 0; d < DD; ++d) {
                                const uint32_t* e = v + 4 * (c * DD + d);
                                edge_entry<EXACT>(P, p_lo + p + c, k1b + d, t.j0 + e0 + d + lane, t.j0 + lane,
                                                  __hiloint2double((int)e[1], (int)e[0]),
                                                  __hiloint2double((int)e[3], (int)e[2]));
                            }
                        continue;  // no park slot, no bulk group
                    }
                    const uint32_t slot = park0 + (uint32_t)(pair % NSLOT) * 2 * G::CHUNK_BYTES;
                    if (pair >= NSLOT) {  // the slot's previous reduces have read it
                        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NSLOT - 1) : "memory");
                        __syncwarp();
                    }
#pragma unroll
                    for (int i = 0; i < 2 * DD; ++i)  // chunk i / DD, diagonal i % DD, this lane's column
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(slot + i * 32 * 16),
                                     "r"(v[4 * i]), "r"(v[4 * i + 1]), "r"(v[4 * i + 2]), "r"(v[4 * i + 3]) : "memory");
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> TMA reads
                    __syncwarp();
                    if (lane == 0) {
                        const uint32_t sp = slot - lane * (uint32_t)sizeof(Cx<R>);
                        for (int c = 0; c < 2 && p + c < np; ++c) {
                            if (EXACT)  // one sheared box of the slice map: 32 x DD x 1, stored
                                asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group"
                                             " [%0, {%2, %3, %4}], [%1];" ::"l"(gmap), "r"(sp + c * G::CHUNK_BYTES),
                                             "r"(c0), "r"(k1b), "r"(p_lo + p + c) : "memory");
                            else  // ... added in L2
                                asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group"
                                             " [%0, {%2, %3, %4}], [%1];" ::"l"(gmap), "r"(sp + c * G::CHUNK_BYTES),
                                             "r"(c0), "r"(k1b), "r"(p_lo + p + c) : "memory");
                        }
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    ++pair;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (P.trace && k < 31 && lane == 0) P.trace[((size_t)blockIdx.x * 32 + k) * 8 + 1 + 6 * (q == 3)] = clock64();
            if (lane == 0) mbar_arrive(&tready[b]);
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        if (warp == 8 && lane == 0) trace_gt(P.trace, 3);
        __syncwarp();
        // every epilogue warp is past its last tcgen05.ld: release TMEM
        asm volatile("barrier.sync 1, 128;" ::: "memory");
        if (warp == 8) {
            tc_fence_after();
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
        }
        return;
    }

    // ---------------- consumers ----------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(V3_REG_CONSUMER) : "memory");
    const int wq = warp % G::CWQ, wr = warp / G::CWQ;
    const int e0 = DD * wr;
    const uint32_t tq = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (warp >> 2) * G::BLOCK_COLS;
    int it = 0;
    int pend = -1;  // TMEM buffer whose stores are issued but not yet announced (tfull)
    for (int k = 0; k < my_tiles; ++k) {
        const V3Tile t = v3_tile<G>(P, v3_lin(k));
        int ps = 0, pd = 0;
        if constexpr (G::ES == 8) {
            const int R0 = wrap((int)(t.q0 - t.k1_0) - (DR - 1), n);
            const int C0 = wrap((int)(t.q0 - t.j0) - 31 - (DR - 1), n);
            pd = (t.j0 - t.k1_0 + P.off) & 1;
            ps = (C0 - R0 + P.off) & 1;
        }
        const int sh_o = (PP * wq + DR - DD - e0) * G::W + (31 - lane) + ps;  // band row of (p, d): + j * W
        const int dr_o = e0 * G::W + lane + pd;                                // direct row d: + d * W
        if (P.trace && k < 31 && lane == 0 && warp == 0) P.trace[((size_t)blockIdx.x * 32 + k) * 8 + 4] = clock64();
        Cx<R> acc[PP][DD];
        if constexpr (EXACT) {  // the block's current values (every entry owned by this tile)
            if (k == 0) pdl_wait();  // the previous kernel's slice updates land first
            const int64_t nn = (int64_t)n * n;
            const int c = t.j0 + lane;
            const int qw = (int)(t.q0 - P.lo) + PP * wq;
            const Cx<R>* gb = P.g4 + (int64_t)qw * nn;
#pragma unroll
            for (int p = 0; p < PP; ++p)
#pragma unroll
                for (int d = 0; d < DD; ++d) {
                    const int k1 = t.k1_0 + e0 + d;
                    if (c < n && qw + p < (int)(P.hi - P.lo) && k1 < n) {
                        acc[p][d] = ld_g4(gb + p * nn + (int64_t)k1 * n + wrap(c + e0 + d, n));
                    } else {
                        acc[p][d].re = acc[p][d].im = R(0);
                    }
                }
        } else {
#pragma unroll
            for (int p = 0; p < PP; ++p)
#pragma unroll
                for (int d = 0; d < DD; ++d) acc[p][d].re = acc[p][d].im = R(0);
        }
        long long fill_wait = 0;  // lab trace: cycles warp 0 waited for fills in this tile
#pragma unroll 1
        for (int w = 0; w < nb; ++w, ++it) {
            const int s = it % NST;
            const long long fw0 = P.trace ? clock64() : 0;
            mbar_wait(&full[s], (it / NST) & 1);
            if (P.trace) fill_wait += clock64() - fw0;
            if (it == 0 && warp == 0 && lane == 0) trace_gt(P.trace, 1);
            const Cx<RG>* dir_u = reinterpret_cast<const Cx<RG>*>(smem_raw + (size_t)s * G::STAGE_BYTES + G::DIR_OFF);
            const Cx<RG>* dir_d = dir_u + G::DIR_ELEMS;
            const Cx<RG>* sh_u = reinterpret_cast<const Cx<RG>*>(smem_raw + (size_t)s * G::STAGE_BYTES + G::SH_OFF);
            const Cx<RG>* sh_d = sh_u + G::SH_ELEMS;
            Stg<R> dv[DD];
#pragma unroll
            for (int d = 0; d < DD; ++d) dv[d] = widen<R>(lds_plain(dir_u + d * G::W + dr_o, dir_d + d * G::W + dr_o));
            constexpr int NJ = PP + DD - 1;  // diagonals p - d
            // The tile's last walker hands the block to TMEM as it completes: the
            // 8 entries of store c (planes 2c, 2c+1) are final after diagonal
            // j = 2c + DD, so each store overlaps the remaining diagonals' math.
            const bool early = EARLY_ST && w == nb - 1 && !(G::LAST_DIRECT && k == my_tiles - 1);
            if (early) {
                if (k >= 2) mbar_wait(&tready[k & 1], ((k >> 1) - 1) & 1);
                tc_fence_after();
            }
            Stg<R> S = widen<R>(lds_plain(sh_u + sh_o, sh_d + sh_o));
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                Stg<R> Sn;
                if (j + 1 < NJ) Sn = widen<R>(lds_plain(sh_u + sh_o + (j + 1) * G::W, sh_d + sh_o + (j + 1) * G::W));
#pragma unroll
                for (int d = 0; d < DD; ++d) {
                    const int p = j + d - (DD - 1);
                    if (p < 0 || p >= PP) continue;
                    if constexpr (EXACT) update_exact(acc[p][d], S, dv[d]);
                    else update_fused(acc[p][d], S, dv[d]);
                }
                if (j + 1 < NJ) S = Sn;
                if constexpr (PP * DD / 8 == PP / 2 && DD == 4) {
                    if (early && j >= DD && (j - DD) % 2 == 0 && (j - DD) / 2 < PP / 2) {
                        const int c = (j - DD) / 2;
                        uint32_t v[32];
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const Cx<R>& a = acc[(8 * c + i) / DD][(8 * c + i) % DD];
                            v[4 * i + 0] = (uint32_t)__double2loint(a.re);
                            v[4 * i + 1] = (uint32_t)__double2hiint(a.re);
                            v[4 * i + 2] = (uint32_t)__double2loint(a.im);
                            v[4 * i + 3] = (uint32_t)__double2hiint(a.im);
                        }
                        tmem_st32(tq + (k & 1) * 256 + c * 32, v);
                    }
                }
            }
            // release the stage once its values are consumed (see v2: the refill is
            // an async-proxy write, the last ld.shared may still be in flight)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (pend >= 0) {  // the previous tile's TMEM stores, overlapped with this first walker
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tfull[pend]);
                pend = -1;
            }
        }
        const bool last = k == my_tiles - 1;
        if (G::LAST_DIRECT && last) {
            // The last tile: every stage is idle now (all fills consumed), so the
            // eight warps park their blocks there and reduce them into the slice
            // themselves, in parallel -- the kernel does not end on one epilogue
            // warp's serial drain of a whole tile.
            asm volatile("barrier.sync 2, %0;" ::"n"(32 * G::CW) : "memory");  // all stage reads done
            const int p_lo_d = (int)(t.q0 - P.lo) + PP * wq;
            const int k1b_d = t.k1_0 + e0;
            if (!(P.use_gmap && k1b_d + DD - 1 < n && t.j0 + 31 + e0 + DD - 1 < n)) {
                // an edge block (row wrap / last column strip): every lane adds its own entries
                if (!P.chain) pdl_wait();
                const int np = min(PP, (int)(P.hi - P.lo) - p_lo_d);
#pragma unroll
                for (int p = 0; p < PP; ++p)
#pragma unroll
                    for (int d = 0; d < DD; ++d)
                        if (p < np)
                            edge_entry<EXACT>(P, p_lo_d + p, k1b_d + d, t.j0 + e0 + d + lane, t.j0 + lane,
                                              acc[p][d].re, acc[p][d].im);
                if (warp == 0 && lane == 0) trace_gt(P.trace, 2);
                break;
            }
            const uint32_t park = smem_u32(smem_raw) + (uint32_t)warp * PP * G::CHUNK_BYTES;
#pragma unroll
            for (int p = 0; p < PP; ++p)
#pragma unroll
                for (int d = 0; d < DD; ++d)
                    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(park + p * G::CHUNK_BYTES + (d * 32 + lane) * 16),
                                 "d"(acc[p][d].re), "d"(acc[p][d].im) : "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                if (!P.chain) pdl_wait();  // the previous kernel's slice updates land first
                // (an interior block: edge blocks took the per-lane path above)
                const int np = min(PP, (int)(P.hi - P.lo) - p_lo_d);
                for (int p = 0; p < np; ++p) {
                    if (EXACT)
                        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group"
                                     " [%0, {%2, %3, %4}], [%1];" ::"l"(reinterpret_cast<uint64_t>(&P.gmap)),
                                     "r"(park + p * G::CHUNK_BYTES), "r"(2 * (t.j0 - t.k1_0 + n)), "r"(k1b_d),
                                     "r"(p_lo_d + p) : "memory");
                    else
                        asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group"
                                     " [%0, {%2, %3, %4}], [%1];" ::"l"(reinterpret_cast<uint64_t>(&P.gmap)),
                                     "r"(park + p * G::CHUNK_BYTES), "r"(2 * (t.j0 - t.k1_0 + n)), "r"(k1b_d),
                                     "r"(p_lo_d + p) : "memory");
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // park read before exit
            }
            __syncwarp();
            if (warp == 0 && lane == 0) trace_gt(P.trace, 2);
            break;
        }
        // hand the block to the epilogue through TMEM buffer b
        const int b = k & 1;
        const long long tw0 = P.trace ? clock64() : 0;
        if (!EARLY_ST) {
        if (k >= 2) mbar_wait(&tready[b], ((k >> 1) - 1) & 1);
        if (P.trace && k < 31 && lane == 0 && warp == 0) P.trace[((size_t)blockIdx.x * 32 + k) * 8 + 3] = clock64() - tw0;
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < PP * DD / 8; ++c) {  // 8 entries (32 columns) per store
            uint32_t v[32];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const Cx<R>& a = acc[(8 * c + i) / DD][(8 * c + i) % DD];
                v[4 * i + 0] = (uint32_t)__double2loint(a.re);
                v[4 * i + 1] = (uint32_t)__double2hiint(a.re);
                v[4 * i + 2] = (uint32_t)__double2loint(a.im);
                v[4 * i + 3] = (uint32_t)__double2hiint(a.im);
            }
            tmem_st32(tq + b * 256 + c * 32, v);
        }
        }
        if (P.trace && k < 31 && lane == 0 && warp == 0) {
            P.trace[((size_t)blockIdx.x * 32 + k) * 8 + 2] = clock64();
            P.trace[((size_t)blockIdx.x * 32 + k) * 8 + 5] = fill_wait;
        }
        pend = b;  // announced after the next tile's first walker (or below)
        if (last) {
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tfull[b]);
            pend = -1;
        }
    }
}

template <typename RG, class G, bool EXACT>
static g4_status launch_pst_t(void* g4p, int64_t lo, int64_t hi, int32_t n, const void* const* staged,
                              int32_t nbatch, cudaStream_t st) {
    // TMEM stores inside the last walker: -2 to -4 % at N = 1024 with 8 walkers,
    // neutral to +5 % at N = 512, +7 to +10 % with 16 walkers (labs r02n, r02ab):
    // from N = 1024 on, up to 8 walkers a pass (G4RING_V3_EARLY_ST=0/1 forces)
    static const int early_env = env_int("G4RING_V3_EARLY_ST", -1);
    const bool early = early_env >= 0 ? early_env != 0 : (n >= 1024 && std::min(nbatch, TMA_MAXW) <= 8);
    auto kern = early ? k_accumulate_pst<RG, G, true, EXACT> : k_accumulate_pst<RG, G, false, EXACT>;
    int dev = 0;
    G4_CUDA(cudaGetDevice(&dev));
    {  // the >48 KB shared-memory opt-in is per device
        static std::mutex mu;
        static uint64_t done = 0;
        std::lock_guard<std::mutex> lk(mu);
        if (!(done & (1ull << (dev & 63)))) {
            G4_CUDA(cudaFuncSetAttribute(k_accumulate_pst<RG, G, true, EXACT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM));
            G4_CUDA(cudaFuncSetAttribute(k_accumulate_pst<RG, G, false, EXACT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM));
            done |= 1ull << (dev & 63);
        }
    }
    int sms = 0;
    G4_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    for (int b0 = 0; b0 < nbatch; b0 += TMA_MAXW) {
        TmaParams<double> tp;
        std::memset(&tp, 0, sizeof(tp));
        tp.g4 = static_cast<Cx<double>*>(g4p);
        tp.lo = lo;
        tp.hi = hi;
        tp.n = n;
        tp.off = sheared_offset(n, G::ES);
        G4_TRY(slice_map(g4p, n, hi - lo, 1, G::DD, &tp.gmap));
        tp.use_gmap = g4_gmap_enabled() ? 1 : 0;
        // Payload boxes with an L2 evict_last policy up to N = 2048, where the
        // walkers' payloads fit L2 next to the streaming slice: -1.2 % at the
        // bench shape over five alternations, neutral at N = 1024 and P = 32
        // (lab r02ao).  G4RING_V3_HINTS overrides (lab knobs, TmaParams::hints).
        static const int hints_env = env_int("G4RING_V3_HINTS", -1);
        tp.hints = hints_env >= 0 ? hints_env : (n <= 2048 ? 2 : 0);
        static const bool chain_on = env_int("G4RING_V3_CHAIN", 1) != 0;  // 0: every pass waits (A/B)
        tp.chain = (!EXACT && chain_on && (b0 > 0 || k1_chain_prev(st))) ? 1 : 0;
        tp.nbatch = std::min(TMA_MAXW, nbatch - b0);
        for (int i = 0; i < tp.nbatch; ++i) {
            MapPair mp;
            G4_TRY(get_maps(staged[b0 + i], n, G::ES, G::NSH, G::W, G::DR, 2, &mp));
            tp.dmap[i] = mp.dmap;
            tp.smap[i] = mp.smap;
        }
        tp.nx = (int32_t)((hi - lo + G::Q - 1) / G::Q);
        const int64_t tiles = (int64_t)tp.nx * ((n + 31) / 32) * ((n + G::DR - 1) / G::DR);
        if (tiles >= (1ll << 31)) return fail(G4_ERR_CONTRACT, "accumulate: tile count too large");
        static const int grid_env = env_int("G4RING_V3_GRID", 0);  // lab: fewer CTAs than SMs
        const unsigned grid = (unsigned)std::min<int64_t>(tiles, grid_env > 0 ? std::min(grid_env, sms) : sms);
        static const char* trace_path = getenv("G4RING_V3_TRACE");  // lab: per-tile timeline dump
        long long* trace = nullptr;
        if (trace_path) {
            G4_CUDA(cudaMalloc(&trace, (size_t)grid * 32 * 8 * sizeof(long long)));
            G4_CUDA(cudaMemsetAsync(trace, 0, (size_t)grid * 32 * 8 * sizeof(long long), st));
            tp.trace = trace;
        }
        static const bool pdl = env_int("G4RING_PDL", 1) != 0;  // 0: no programmatic dependent launch (A/B)
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(grid);
        lc.blockDim = dim3(G::THREADS);
        lc.dynamicSmemBytes = G::SMEM;
        lc.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = attr;
        lc.numAttrs = pdl ? 1 : 0;
        G4_TRY(check_cuda(cudaLaunchKernelEx(&lc, kern, tp), "k_accumulate_pst launch"));
        if (trace) {
            std::vector<long long> h((size_t)grid * 32 * 8);
            G4_CUDA(cudaMemcpyAsync(h.data(), trace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, st));
            G4_CUDA(cudaStreamSynchronize(st));
            G4_CUDA(cudaFree(trace));
            if (FILE* f = fopen(trace_path, "ab")) {
                fwrite(h.data(), sizeof(long long), h.size(), f);
                fclose(f);
            }
        }
    }
    k1_chain_note(!EXACT);
    return G4_OK;
}

// v3 geometries (id >= 40 in the G4RING_V2GEOM numbering):
//   40: 8x4 blocks, 2x4 warps (tile 16 planes x 16 diagonals), 4 stages, 4 park slots
//   (a 32 x 8 tile, 4x2 warps, needs a band of 39 rows + 32 columns: beyond the staged halo)
//   42: as 40 with 3 stages and 8 park slots; 43: 3 stages, 10 park slots; 44: 2 stages, 16 park slots
// ---------------------------------------------------------------------------
// K1 v3 for complex64 slices (fused, deferred): the same producer and
// consumer roles with float accumulators; a 32-entry block is 64 TMEM columns,
// so four hand-off buffers fit.  The epilogue has no park: complex64 row
// segments cannot be sheared tensor-map boxes (the (N+1)-entry row stride is not
// a 16-B multiple), so every lane adds its own entries with one
// red.global.add.v2.f32 each (a warp's row segment is one coalesced 256-B run,
// split at the row end).  The last tile goes out the same way from the
// consumers' registers.
constexpr int V3C64_BUFS = 4;

__device__ __forceinline__ void edge_entry32(const TmaParams<float>& P, int plane, int k1, int k2, int c, float re,
                                             float im) {
    const int n = P.n;
    if (k1 >= n || c >= n) return;
    if (k2 >= n) k2 -= n;
    float* g = reinterpret_cast<float*>(P.g4 + ((int64_t)plane * n + k1) * n + k2);
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(g), "f"(re), "f"(im) : "memory");
}

template <class G>
struct V3C64Smem {  // stages, then the barriers (no park)
    static constexpr uint32_t BAR_OFF = G::NST * G::STAGE_BYTES;
    static constexpr size_t SMEM = BAR_OFF + (2 * G::NST + 2 * V3C64_BUFS) * sizeof(uint64_t) + 16;
    static_assert(SMEM <= 227 * 1024, "v3 c64 stages exceed shared memory");
};

template <class G>
__global__ void __launch_bounds__(512, 1) k_accumulate_pst32(const __grid_constant__ TmaParams<float> P) {
    using R = float;
    using RG = float;
    constexpr int PP = G::PP, DD = G::DD, NST = G::NST, DR = G::DR, NB = V3C64_BUFS;
    constexpr int EW = G::ES / 8;
    constexpr int COLS = PP * DD * 2;  // TMEM columns of one consumer block
    static_assert(PP * DD == 32 && 2 * NB * COLS == 512, "four 2-warp buffers per lane quarter");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + V3C64Smem<G>::BAR_OFF);
    uint64_t* empty = full + NST;
    uint64_t* tfull = empty + NST;
    uint64_t* tready = tfull + NB;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tready + NB);

    const int n = P.n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = P.nx * ((n + 31) / 32) * ((n + DR - 1) / DR);
    const int my_tiles = v3_count(ntiles);
    const int nb = P.nbatch;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], G::CW);
        }
        for (int b = 0; b < NB; ++b) {
            mbar_init(&tfull[b], G::CW);
            mbar_init(&tready[b], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (!P.chain) pdl_wait();  // chained passes as in the complex128 kernel (k1_chain_prev)
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= 12) {
        // ---------------- producer (as the complex128 kernel) ----------------
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(V3_REG_PRODUCER) : "memory");
        if (threadIdx.x == 384) {
            if (!P.chain) pdl_wait();
            int it = 0;
            for (int k = 0; k < my_tiles; ++k) {
                const V3Tile t = v3_tile<G>(P, v3_lin(k));
                const int R0 = wrap((int)(t.q0 - t.k1_0) - (DR - 1), n);
                const int C0 = wrap((int)(t.q0 - t.j0) - 31 - (DR - 1), n);
                const int xd = t.j0 - t.k1_0 + P.off, xs = C0 - R0 + P.off;
                const int pd = xd & 1, ps = xs & 1;
                for (int w = 0; w < nb; ++w, ++it) {
                    const int s = it % NST;
                    if (it >= NST) mbar_wait(&empty[s], ((it / NST) - 1) & 1);
                    mbar_arrive_expect_tx(&full[s], G::DIR_BYTES + G::SH_BYTES);
                    unsigned char* st = smem_raw + (size_t)s * G::STAGE_BYTES;
                    tma_load_3d(st + G::DIR_OFF, &P.dmap[w], EW * (xd - pd), t.k1_0, 0, &full[s]);
                    tma_load_3d(st + G::SH_OFF, &P.smap[w], EW * (xs - ps), R0, 0, &full[s]);
                }
            }
            if (P.chain) pdl_wait();  // chained: we complete only after the previous pass does
        }
        __syncwarp();
        return;
    }

    if (warp >= 8) {
        // ---------------- epilogue: TMEM -> one red.global.add.v2.f32 per entry ----------------
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(V3_REG_EPILOGUE) : "memory");
        const int q = warp - 8;
        const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);
        if (!P.chain) pdl_wait();
        for (int k = 0; k < my_tiles - 1; ++k) {  // the last tile: consumers
            const int b = k % NB;
            mbar_wait(&tfull[b], (k / NB) & 1);
            tc_fence_after();
            const V3Tile t = v3_tile<G>(P, v3_lin(k));
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const int cw = q + 4 * h, wq = cw % G::CWQ, wr = cw / G::CWQ;
                const int p_lo = (int)(t.q0 - P.lo) + PP * wq;
                const int e0 = DD * wr;
                const int np = min(PP, (int)(P.hi - P.lo) - p_lo);
#pragma unroll 1
                for (int c = 0; c < 2; ++c) {  // 16 entries (planes 4c .. 4c + 3) per load
                    uint32_t v[32];
                    tmem_ld32(tq + b * (2 * COLS) + h * COLS + c * 32, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int e = 16 * c + i, p = e / DD, d = e % DD;
                        if (p < np)
                            edge_entry32(P, p_lo + p, t.k1_0 + e0 + d, t.j0 + e0 + d + lane, t.j0 + lane,
                                         __uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tready[b]);
        }
        asm volatile("barrier.sync 1, 128;" ::: "memory");
        if (warp == 8) {
            tc_fence_after();
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
        }
        return;
    }

    // ---------------- consumers ----------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(V3_REG_CONSUMER) : "memory");
    const int wq = warp % G::CWQ, wr = warp / G::CWQ;
    const int e0 = DD * wr;
    const uint32_t tq = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (warp >> 2) * COLS;
    int it = 0;
    for (int k = 0; k < my_tiles; ++k) {
        const V3Tile t = v3_tile<G>(P, v3_lin(k));
        const int R0 = wrap((int)(t.q0 - t.k1_0) - (DR - 1), n);
        const int C0 = wrap((int)(t.q0 - t.j0) - 31 - (DR - 1), n);
        const int pd = (t.j0 - t.k1_0 + P.off) & 1;
        const int ps = (C0 - R0 + P.off) & 1;
        const int sh_o = (PP * wq + DR - DD - e0) * G::W + (31 - lane) + ps;
        const int dr_o = e0 * G::W + lane + pd;
        Cx<R> acc[PP][DD];
#pragma unroll
        for (int p = 0; p < PP; ++p)
#pragma unroll
            for (int d = 0; d < DD; ++d) acc[p][d].re = acc[p][d].im = R(0);
#pragma unroll 1
        for (int w = 0; w < nb; ++w, ++it) {
            const int s = it % NST;
            mbar_wait(&full[s], (it / NST) & 1);
            const Cx<RG>* dir_u = reinterpret_cast<const Cx<RG>*>(smem_raw + (size_t)s * G::STAGE_BYTES + G::DIR_OFF);
            const Cx<RG>* dir_d = dir_u + G::DIR_ELEMS;
            const Cx<RG>* sh_u = reinterpret_cast<const Cx<RG>*>(smem_raw + (size_t)s * G::STAGE_BYTES + G::SH_OFF);
            const Cx<RG>* sh_d = sh_u + G::SH_ELEMS;
            Stg<R> dv[DD];
#pragma unroll
            for (int d = 0; d < DD; ++d) dv[d] = lds_plain(dir_u + d * G::W + dr_o, dir_d + d * G::W + dr_o);
            constexpr int NJ = PP + DD - 1;
            Stg<R> S = lds_plain(sh_u + sh_o, sh_d + sh_o);
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                Stg<R> Sn;
                if (j + 1 < NJ) Sn = lds_plain(sh_u + sh_o + (j + 1) * G::W, sh_d + sh_o + (j + 1) * G::W);
#pragma unroll
                for (int d = 0; d < DD; ++d) {
                    const int p = j + d - (DD - 1);
                    if (p < 0 || p >= PP) continue;
                    update_fused(acc[p][d], S, dv[d]);
                }
                if (j + 1 < NJ) S = Sn;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (k == my_tiles - 1) {  // the last tile: straight from the registers
            if (!P.chain) pdl_wait();
            const int p_lo = (int)(t.q0 - P.lo) + PP * wq;
            const int np = min(PP, (int)(P.hi - P.lo) - p_lo);
#pragma unroll
            for (int p = 0; p < PP; ++p)
#pragma unroll
                for (int d = 0; d < DD; ++d)
                    if (p < np)
                        edge_entry32(P, p_lo + p, t.k1_0 + e0 + d, t.j0 + e0 + d + lane, t.j0 + lane, acc[p][d].re,
                                     acc[p][d].im);
            break;
        }
        const int b = k % NB;
        if (k >= NB) mbar_wait(&tready[b], ((k / NB) - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            uint32_t v[32];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const Cx<R>& a = acc[(16 * c + i) / DD][(16 * c + i) % DD];
                v[2 * i] = __float_as_uint(a.re);
                v[2 * i + 1] = __float_as_uint(a.im);
            }
            tmem_st32(tq + b * (2 * COLS) + c * 32, v);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tfull[b]);
    }
}

template <class G>
static g4_status launch_pst32_t(void* g4p, int64_t lo, int64_t hi, int32_t n, const void* const* staged,
                                int32_t nbatch, cudaStream_t st) {
    auto kern = k_accumulate_pst32<G>;
    constexpr size_t SMEM = V3C64Smem<G>::SMEM;
    int dev = 0;
    G4_CUDA(cudaGetDevice(&dev));
    {
        static std::mutex mu;
        static uint64_t done = 0;
        std::lock_guard<std::mutex> lk(mu);
        if (!(done & (1ull << (dev & 63)))) {
            G4_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
            done |= 1ull << (dev & 63);
        }
    }
    int sms = 0;
    G4_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    for (int b0 = 0; b0 < nbatch; b0 += TMA_MAXW) {
        TmaParams<float> tp;
        std::memset(&tp, 0, sizeof(tp));
        tp.g4 = static_cast<Cx<float>*>(g4p);
        tp.lo = lo;
        tp.hi = hi;
        tp.n = n;
        tp.off = sheared_offset(n, G::ES);
        tp.nbatch = std::min(TMA_MAXW, nbatch - b0);
        static const bool chain_on = env_int("G4RING_V3_CHAIN", 1) != 0;
        tp.chain = (chain_on && (b0 > 0 || k1_chain_prev(st))) ? 1 : 0;
        for (int i = 0; i < tp.nbatch; ++i) {
            MapPair mp;
            G4_TRY(get_maps(staged[b0 + i], n, G::ES, G::NSH, G::W, G::DR, 2, &mp));
            tp.dmap[i] = mp.dmap;
            tp.smap[i] = mp.smap;
        }
        tp.nx = (int32_t)((hi - lo + G::Q - 1) / G::Q);
        const int64_t tiles = (int64_t)tp.nx * ((n + 31) / 32) * ((n + G::DR - 1) / G::DR);
        if (tiles >= (1ll << 31)) return fail(G4_ERR_CONTRACT, "accumulate: tile count too large");
        const unsigned grid = (unsigned)std::min<int64_t>(tiles, sms);
        static const bool pdl = env_int("G4RING_PDL", 1) != 0;
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(grid);
        lc.blockDim = dim3(G::THREADS);
        lc.dynamicSmemBytes = SMEM;
        lc.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = attr;
        lc.numAttrs = pdl ? 1 : 0;
        G4_TRY(check_cuda(cudaLaunchKernelEx(&lc, kern, tp), "k_accumulate_pst32 launch"));
    }
    k1_chain_note(true);
    return G4_OK;
}

g4_status launch_pst32(int geom, void* g4p, int64_t lo, int64_t hi, int32_t n, const void* const* staged,
                       int32_t nbatch, cudaStream_t st) {
    switch (geom) {
        case 45: return launch_pst32_t<V3Geom<float, 8, 4, 2, 4, 7, 4>>(g4p, lo, hi, n, staged, nbatch, st);
        default: return fail(G4_ERR_CONTRACT, "unknown v3 complex64 geometry");
    }
}

template <typename RG, class G>
static g4_status launch_pst_mode(bool exact, void* g4p, int64_t lo, int64_t hi, int32_t n, const void* const* staged,
                                 int32_t nbatch, cudaStream_t st) {
    return exact ? launch_pst_t<RG, G, true>(g4p, lo, hi, n, staged, nbatch, st)
                 : launch_pst_t<RG, G, false>(g4p, lo, hi, n, staged, nbatch, st);
}
template <typename RG>
g4_status launch_pst(int geom, bool exact, void* g4p, int64_t lo, int64_t hi, int32_t n, const void* const* staged,
                     int32_t nbatch, cudaStream_t st) {
    switch (geom) {
        case 40: return launch_pst_mode<RG, V3Geom<RG, 8, 4, 2, 4, 4, 4>>(exact, g4p, lo, hi, n, staged, nbatch, st);
        case 42: return launch_pst_mode<RG, V3Geom<RG, 8, 4, 2, 4, 3, 8>>(exact, g4p, lo, hi, n, staged, nbatch, st);
        case 43: return launch_pst_mode<RG, V3Geom<RG, 8, 4, 2, 4, 3, 10>>(exact, g4p, lo, hi, n, staged, nbatch, st);
        case 44: return launch_pst_mode<RG, V3Geom<RG, 8, 4, 2, 4, 2, 16>>(exact, g4p, lo, hi, n, staged, nbatch, st);
        default: return fail(G4_ERR_CONTRACT, "unknown v3 geometry");
    }
}
template g4_status launch_pst<double>(int, bool, void*, int64_t, int64_t, int32_t, const void* const*, int32_t,
                                      cudaStream_t);
template g4_status launch_pst<float>(int, bool, void*, int64_t, int64_t, int32_t, const void* const*, int32_t,
                                     cudaStream_t);

bool pst_geom_info(int geom, int* pp, int* dd, int* q, int* dr, int* nst) {
    switch (geom) {
        case 40: *pp = 8, *dd = 4, *q = 16, *dr = 16, *nst = 4; return true;
        case 42: *pp = 8, *dd = 4, *q = 16, *dr = 16, *nst = 3; return true;
        case 43: *pp = 8, *dd = 4, *q = 16, *dr = 16, *nst = 3; return true;
        case 44: *pp = 8, *dd = 4, *q = 16, *dr = 16, *nst = 2; return true;
        case 45: *pp = 8, *dd = 4, *q = 16, *dr = 16, *nst = 7; return true;
        default: return false;
    }
}

}  // namespace g4
