// g4_accumulate.cu -- K1, the G4 slice update (replaces ringacc/tensor.py:233-251).
//
// Reference semantics, per owned plane K3 = q and entry (k1, k2):
//   G4[q][k1][k2] += up[(q-k2)%N][(q-k1)%N] * down[k2][k1]
//                  + down[(q-k2)%N][(q-k1)%N] * up[k2][k1]
// On the staged payload (g4_common.cuh: stg[0][r][c] = up[c][r],
// stg[1][r][c] = down[c][r], rows of pitch LD with a cyclic halo) this reads
//   S = stg[.][(q-k1)%N][(q-k2)%N]   ("shifted")  and  D = stg[.][k1][k2]  ("direct"):
//   p1 = S.u * D.d ; p2 = S.d * D.u ; t = p1 + p2 ; G += t
// -- the reference's exact op order (tensor.py:250: u*down + d*up, then +=).
//
// Register block: one thread owns PP x DD G4 entries, planes q0..q0+PP-1 x the
// diagonal (k1_0 + d, c + d), d < DD (v1: 4 x 4; v2 default: 8 x 2).  The
// shifted index (q-k1, q-k2) then depends only on m = p - d, so the PP*DD
// updates of one walker need DD direct + PP+DD-1 shifted staged elements (16
// updates from 11 for both blocks).  A warp's 32 lanes own 32 consecutive k2
// columns: G4 rows are read/written as contiguous 512 B runs, staged rows as
// contiguous (forward or reversed) runs.  The G4 block is read once, receives
// every walker of the batch in order (bitwise identical to sequential
// reference calls), and is written once: HBM traffic per pass is
// 2 * P * N^2 * 16 B plus the staged payloads.
//
// v1 (k_accumulate): CTA = WARPS warps stacked along K3 (they share the direct
//    elements and most shifted rows through L1); loads straight from global.
// v2 (k_accumulate_tma, N >= 64 and >= 4 planes): CTA = CWQ x CWR warps (tile Q
//    planes x DR diagonal entries x 32 columns, see V2Geom).  One producer lane
//    (lane 0 of warp 0, which is also a consumer) streams, per walker, two TMA
//    tensor boxes into an NST-stage shared-memory ring: the CTA's direct tile
//    (DR rows x 32 cols x 2 spins) and its whole shifted band (Q+DR-1 diagonal
//    row segments x 32 cols x 2 spins), both through *sheared* tensor maps (row
//    stride LD+1 elements) that turn diagonals into rectangular boxes.  The halo
//    of the staged layout means no box ever wraps.  Consumers wait on the
//    stage's mbarrier, read their elements from shared memory (contiguous per
//    warp: conflict-free) and release the stage.  After the last walker the
//    idle stage buffers take each warp's block, and the TMA engine writes it
//    back (complex128): one box of a sheared tensor map of the slice per warp,
//    stored (exact) or added in L2 (fused, deferred update).  Geometry choice
//    and the measured alternatives: launch_v2_geom below, DESIGN.md section 4.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <map>
#include <tuple>

#include <cuda.h>

#include "g4_common.cuh"
#include "g4_internal.h"
#include "g4_k1.cuh"

namespace g4 {

// Kernel selection: 0 = auto (v2 for N >= 64 and >= 4 planes, any dtype; else v1),
// 1 = v1 everywhere, 2 = v2 wherever it applies.  G4RING_KERNEL overrides.
static int g_variant = -1;
static int kernel_variant() {
    if (g_variant < 0) {
        const char* e = getenv("G4RING_KERNEL");
        g_variant = e ? atoi(e) : 0;
    }
    return g_variant;
}

// RA: G4 entry type, RG: payload entry type (RG = float with RA = double is the
// mixed-precision mode: complex64 payloads widened exactly into complex128 math).
template <typename RA, typename RG>
struct AccParams {
    Cx<RA>* g4;
    int64_t lo, hi;
    int32_t n;
    int32_t nbatch;
    const Cx<RG>* stg[G4_MAX_BATCH];  // staged payloads (2 x ROWS x LD)
};




// ---------------------------------------------------------------------------
// v1
template <typename R, typename RG, int PP, int DD, int WARPS, int MINB, bool FUSED>
__global__ void __launch_bounds__(32 * WARPS, MINB)
k_accumulate(const __grid_constant__ AccParams<R, RG> P) {
    constexpr int NS = PP + DD - 1;  // distinct shifted elements per thread
    const int n = P.n;
    const int ld = staged_ld(n, sizeof(Cx<RG>));
    const int64_t plane_s = staged_plane(n, sizeof(Cx<RG>));
    const int nx = (int)((P.hi - P.lo + PP * WARPS - 1) / (PP * WARPS));
    const TileCoord tc = tile_coord(blockIdx.x, nx, (n + 31) / 32, (n + DD - 1) / DD);
    const int k1_0 = tc.z * DD;
    const int c_raw = tc.y * 32 + threadIdx.x;
    const bool col_ok = c_raw < n;
    const int c = col_ok ? c_raw : 0;
    const int64_t q0 = P.lo + ((int64_t)tc.x * WARPS + threadIdx.y) * PP;
    if (q0 >= P.hi) return;  // warp-uniform

    // Direct elements stg[k1_0 + d][(c + d) % N]; G4 offsets (k1_0 + d) * N + (c + d) % N.
    int offd[DD], offg[DD];
#pragma unroll
    for (int d = 0; d < DD; ++d) {
        const int k1 = wrap(k1_0 + d, n), k2 = wrap(c + d, n);
        offd[d] = k1 * ld + k2;
        offg[d] = k1 * n + k2;
    }
    // Shifted elements stg[(q0 - k1_0 + m) % N][(q0 - c + m) % N], m = p - d in [-(DD-1), PP-1].
    int offs[NS];
    {
        const int rb = wrap((int)(q0 - k1_0), n);
        const int cb = wrap((int)(q0 - c), n);
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            const int m = j - (DD - 1);
            offs[j] = wrap(rb + m, n) * ld + wrap(cb + m, n);
        }
    }
    uint32_t okmask = 0;  // bit p*DD + d: entry belongs to the slice
#pragma unroll
    for (int p = 0; p < PP; ++p)
#pragma unroll
        for (int d = 0; d < DD; ++d)
            if (col_ok && (q0 + p) < P.hi && (k1_0 + d) < n) okmask |= 1u << (p * DD + d);

    const int64_t nn = (int64_t)n * n;
    Cx<R>* gb = P.g4 + (q0 - P.lo) * nn;
    Cx<R> acc[PP][DD];
#pragma unroll
    for (int p = 0; p < PP; ++p)
#pragma unroll
        for (int d = 0; d < DD; ++d) {
            if (okmask & (1u << (p * DD + d))) {
                acc[p][d] = ld_g4(gb + p * nn + offg[d]);
            } else {
                acc[p][d].re = R(0);
                acc[p][d].im = R(0);
            }
        }

#pragma unroll 1
    for (int w = 0; w < P.nbatch; ++w) {
        const Cx<RG>* su = P.stg[w];
        const Cx<RG>* sd = su + plane_s;
        Stg<R> dv[DD];
        Stg<R> sv[NS];
        // all loads of the walker are issued before any math (memory-level parallelism)
#pragma unroll
        for (int d = 0; d < DD; ++d) dv[d] = widen<R>(ld_stg_v(su + offd[d], sd + offd[d]));
#pragma unroll
        for (int j = 0; j < NS; ++j) sv[j] = widen<R>(ld_stg_v(su + offs[j], sd + offs[j]));
#pragma unroll
        for (int p = 0; p < PP; ++p) {
#pragma unroll
            for (int d = 0; d < DD; ++d) {
                const Stg<R>& S = sv[p - d + DD - 1];
                const Stg<R>& D = dv[d];
                if constexpr (FUSED) {
                    update_fused(acc[p][d], S, D);
                } else {
                    R p1r, p1i, p2r, p2i;
                    cmul(S.ur, S.ui, D.dr, D.di, p1r, p1i);  // u * down[k2][k1]
                    cmul(S.dr, S.di, D.ur, D.ui, p2r, p2i);  // d * up[k2][k1]
                    acc[p][d].re = add_rn(acc[p][d].re, add_rn(p1r, p2r));
                    acc[p][d].im = add_rn(acc[p][d].im, add_rn(p1i, p2i));
                }
            }
        }
    }

#pragma unroll
    for (int p = 0; p < PP; ++p)
#pragma unroll
        for (int d = 0; d < DD; ++d)
            if (okmask & (1u << (p * DD + d))) st_g4(gb + p * nn + offg[d], acc[p][d]);
}

template <typename R, typename RG, int PP, int DD, int WARPS, int MINB, bool FUSED>
static g4_status launch_v1(const AccParams<R, RG>& prm, cudaStream_t st) {
    const int n = prm.n;
    const int64_t nx = (prm.hi - prm.lo + PP * WARPS - 1) / (PP * WARPS);
    const uint64_t ctas = (uint64_t)nx * ((n + 31) / 32) * ((n + DD - 1) / DD);
    if (ctas >= (1ull << 31)) return fail(G4_ERR_CONTRACT, "accumulate: launch grid too large");
    k_accumulate<R, RG, PP, DD, WARPS, MINB, FUSED><<<(unsigned)ctas, dim3(32, WARPS), 0, st>>>(prm);
    return check_cuda(cudaGetLastError(), "k_accumulate launch");
}

// ---------------------------------------------------------------------------
// v2 -- TMA tensor boxes into a shared-memory ring (complex128).


// Geometry of one v2 configuration.  A thread owns PP planes x DD diagonal
// entries; a CTA is CWQ x CWR warps: CWQ stacked along K3 (Q = PP*CWQ planes)
// and CWR along the diagonal (DR = DD*CWR entries per lane, i.e. the CTA's
// G4 tile is Q planes x the 32-wide diagonal strip (k1_0 + e, j0 + lane + e),
// e < DR).  Per walker the CTA fetches DR direct rows and Q + DR - 1 band rows
// (32 entries x 2 spins each): (Q + 2 DR - 1) / (Q DR) rows per G4 entry.
// NST-stage shared-memory ring, payload entry type R.
//
// CL > 1: diagonal clusters.  The CL CTAs of a cluster own consecutive plane
// chunks x with their (K1, K2) tiles shifted by Q per chunk, i.e. tiles
// (q0 + r Q, k1_0 + r Q, j0 + r Q), r < CL.  The shifted band depends only on
// (k1 - q, k2 - q), so all CL CTAs need the SAME band: each loads HS = NSH / CL
// of its rows and multicasts them to the whole cluster (TMA .multicast::cluster),
// cutting the L2 -> SM band traffic by CL.  Needs N % 32 == 0 and chunks % CL == 0.
//
// PW = 1: warp specialisation.  The CW = 4 consumer warps form warp group 0;
// warp group 1 (4 warps) only produces: thread 128 issues every refill as soon
// as its stage is released.  setmaxnreg moves the registers: the producer
// group drops to 24, the consumer group rises to 232 (launch: 128 x 256).
template <typename R, int PP_, int CW_, int NST_, int DD_ = 4, int CWR_ = 1, int PF_ = 1, int CL_ = 1,
          int PW_ = 0>
struct V2Geom {
    static constexpr int PP = PP_, DD = DD_, CWQ = CW_, CWR = CWR_, NST = NST_;
    static constexpr int PF = PF_;  // shifted operands loaded this many diagonals ahead
    static constexpr int CL = CL_;  // CTAs per cluster (band multicast)
    static constexpr int PW = PW_;  // 1: a producer warp group
    using Base = V2Geom<R, PP_, CW_, NST_, DD_, CWR_, PF_, 1, PW_>;
    static constexpr int CW = CWQ * CWR;                          // consumer warps per CTA
    static constexpr int THREADS = 32 * CW + 128 * PW;
    static_assert(PW == 0 || (CW == 4 && CL == 1), "producer warp group: 4 consumer warps, no clusters");
    static constexpr int Q = PP * CWQ, DR = DD * CWR;             // CTA tile: planes x diagonal entries
    static constexpr int ES = sizeof(Cx<R>);                      // bytes per complex entry
    static constexpr int NSH = Q + DR - 1;                        // shifted row segments (band height)
    // Band rows loaded per cluster CTA.  Each CTA's slice must start 128-B aligned
    // in shared memory: complex64 rows are 34 x 8 = 272 B, so 8-row granules.
    static constexpr int HS_ALIGN = (ES == 8 && CL > 1) ? 8 : 1;
    static constexpr int HS = ((NSH + CL - 1) / CL + HS_ALIGN - 1) / HS_ALIGN * HS_ALIGN;
    static constexpr int SH_ROWS = HS * CL;                       // band rows held (>= NSH)
    // Box row width in entries.  A TMA box must start on a 16-B boundary along
    // its innermost dimension (tools/tma_probe.cu: odd 8-B starts fault), so for
    // complex64 boxes start at the even entry below and carry 2 extra entries;
    // consumers add the start's parity (0 or 1).
    static constexpr int W = ES == 8 ? 34 : 32;
    static constexpr int DIR_ELEMS = DR * W;                      // per spin (sheared direct box)
    static constexpr int SH_ELEMS = SH_ROWS * W;                  // per spin
    static constexpr uint32_t DIR_BYTES = 2 * DIR_ELEMS * ES;     // both spins
    static constexpr uint32_t SH_BYTES = 2 * SH_ELEMS * ES;
    static constexpr uint32_t DIR_OFF = 0;
    static constexpr uint32_t SH_OFF = (DIR_BYTES + 127) / 128 * 128;
    static constexpr uint32_t STAGE_BYTES = (SH_OFF + SH_BYTES + 127) / 128 * 128;
    static constexpr size_t SMEM = (size_t)NST * STAGE_BYTES + 2 * NST * sizeof(uint64_t);
    static_assert(SH_ROWS <= G4_HALO_ROWS && NSH + W + 1 < G4_HALO_COLS, "halo too small for the v2 band");
    static_assert(SH_ROWS + W + 1 < G4_HALO_COLS && DR + W <= G4_HALO_COLS, "halo too small for the v2 boxes");
    static_assert(SMEM <= 227 * 1024, "v2 stages exceed shared memory");
};


// Measurement-only variants of K1 v2 (G4RING_EXP, never set in production):
//   1 = start from zero accumulators (no G4 read)   2 = no G4 write
//   4 = no shared-memory reads / math  (bits combine; profiles/r01_summary.md)
// K1_DEFER (production, G4_ARITH_FUSED with >= 4 walkers): the walkers' sum is
// formed from zero and added to the slice at the end -- by TMA bulk reduce for
// complex128 slices, red.global.add for complex64 -- so no CTA waits on its G4
// block (the L2 does the read-modify-write).
// K1_BULKST (production, complex128 slices otherwise): the block is written
// back by TMA bulk stores from the idle stage buffers.
enum : int { EXP_NOLOAD = 1, EXP_NOSTORE = 2, EXP_NOMATH = 4, K1_DEFER = 16, K1_BULKST = 32, EXP_SCALAR_RED = 64 };

static int exp_flags() {
    static int e = -1;
    if (e < 0) {
        const char* v = getenv("G4RING_EXP");
        e = v ? atoi(v) : 0;
    }
    return e;
}


template <typename R, typename RG, class G, bool FUSED, int MINB, int EXP = 0>
__global__ void __launch_bounds__(G::THREADS, MINB)
k_accumulate_tma(const __grid_constant__ TmaParams<R> P) {
    constexpr int PP = G::PP, DD = G::DD, NST = G::NST;
    constexpr int EW = G::ES / 8;  // 64-bit TMA elements per complex entry
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)NST * G::STAGE_BYTES);
    uint64_t* empty = full + NST;

    // Programmatic dependent launch (non-cluster launches): the next K1 may be
    // scheduled as this grid's last wave runs; every access to global memory
    // (payload boxes, slice) waits for the previous kernel on the stream.
    // A deferred (reduce-only) pass chains like v3 (k1_chain_prev): chained, it
    // does not wait here but before it exits; starting a chain, it waits before
    // it lets the next launch begin.
    if constexpr (G::CL == 1) {
        if constexpr ((EXP & K1_DEFER) != 0) {
            if (!P.chain) asm volatile("griddepcontrol.wait;" ::: "memory");
            if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        } else {
            if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
            asm volatile("griddepcontrol.wait;" ::: "memory");
        }
    }
    const int n = P.n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int DR = G::DR, Q = G::Q;
    constexpr int CL = G::CL;
    const TileCoord tc = tile_coord(blockIdx.x, P.nx, (n + 31) / 32, (n + DR - 1) / DR);
    const int64_t q0 = P.lo + (int64_t)tc.x * Q;
    // cluster rank = chunk index mod CL (tile_coord runs x fastest; nx % CL == 0)
    const int crank = CL > 1 ? tc.x % CL : 0;
    const int j0 = CL > 1 ? wrap(tc.y * 32 + crank * Q, n) : tc.y * 32;
    const int k1_0 = CL > 1 ? wrap(tc.z * DR + crank * Q, n) : tc.z * DR;
    const bool producer = threadIdx.x == (G::PW ? 128 : 0);
    // Sheared coordinates (c1, c2) address stg[c2][c1 - off + c2].
    //  direct tile: rows k1_0 + i, columns j0 + i + j      -> (j0 - k1_0 + off, k1_0)
    //  shifted band: rows R0 + i, columns C0 + i + j with
    //    R0 = (q0 - k1_0 - (DR-1)) mod N, C0 = (q0 - j0 - 31 - (DR-1)) mod N  -> (C0 - R0 + off, R0)
    const int R0 = wrap((int)(q0 - k1_0) - (DR - 1), n);
    const int C0 = wrap((int)(q0 - j0) - 31 - (DR - 1), n);
    const int xd = j0 - k1_0 + P.off, xs = C0 - R0 + P.off;  // box starts (entries, >= 0)
    const int pd = (G::ES == 8) ? (xd & 1) : 0, ps = (G::ES == 8) ? (xs & 1) : 0;  // 16-B alignment shift
    auto issue = [&](int w) {  // producer lane: both tensor boxes of walker w into stage w % NST
        const int s = w % NST;
        mbar_arrive_expect_tx(&full[s], G::DIR_BYTES + G::SH_BYTES);
        unsigned char* st = smem_raw + (size_t)s * G::STAGE_BYTES;
        tma_load_3d(st + G::DIR_OFF, &P.dmap[w], EW * (xd - pd), k1_0, 0, &full[s]);
        if constexpr (CL == 1) {
            tma_load_3d(st + G::SH_OFF, &P.smap[w], EW * (xs - ps), R0, 0, &full[s]);
        } else {  // this CTA's HS band rows, per spin, to every CTA of the cluster
#pragma unroll
            for (int spin = 0; spin < 2; ++spin)
                tma_load_3d_mc(st + G::SH_OFF + (size_t)(spin * G::SH_ELEMS + crank * G::HS * G::W) * G::ES,
                               &P.smap[w], EW * (xs - ps), R0 + crank * G::HS, spin, &full[s],
                               (uint16_t)((1u << CL) - 1));
        }
    };
    // A warp is done with stage s: release it in every CTA that multicasts into it.
    auto release = [&](int s) {
        // The stage's last operands are read by ld.shared right before this
        // point and may still be in flight (the math that consumes them can be
        // scheduled after the arrive): order every lane's generic-proxy reads
        // before the async-proxy (TMA) refill the arrive allows.
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if constexpr (CL == 1) {
            if (lane == 0) mbar_arrive(&empty[s]);
        } else if (lane < CL) {  // lane r releases the stage in cluster CTA r
            mbar_arrive_remote(&empty[s], (uint32_t)lane);
        }
    };

    if (producer) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], G::CW * CL);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if constexpr (CL == 1)
            for (int w = 0; w < NST && w < P.nbatch; ++w) issue(w);
    }
    if constexpr (CL == 1) {
        __syncthreads();
    } else {  // every CTA's barriers exist before any multicast lands
        cluster_sync_relaxed();
        if (producer)
            for (int w = 0; w < NST && w < P.nbatch; ++w) issue(w);
    }
    constexpr int PSTR = sizeof(R) == 8 ? 32 : 34;  // parked entries per (p, d) segment (epilogue)
    constexpr size_t WARP_PARK = (size_t)PP * DD * PSTR * sizeof(Cx<R>);
    constexpr bool DEFER = (EXP & K1_DEFER) != 0;
    constexpr bool PARK = (DEFER || (EXP & K1_BULKST) != 0) && PP * DD <= 32 && BULK_SLICE<R> &&
                          (size_t)NST * G::STAGE_BYTES >= G::CW * WARP_PARK;
    if constexpr (G::PW == 1) {
        if (warp >= 4) {  // producer warp group
            asm volatile("setmaxnreg.dec.sync.aligned.u32 24;" ::: "memory");
            if (producer)
                for (int w = NST; w < P.nbatch; ++w) {
                    const int wp = w - NST;
                    mbar_wait(&empty[wp % NST], (wp / NST) & 1);
                    issue(w);
                }
            __syncwarp();
            return;  // the epilogue's barrier is among the consumer warps only
        }
        // launch budget L = 65536 / (MINB x THREADS) registers (8-aligned); the
        // producer group's 24 go to the consumers: 128 (24 + C) = THREADS x L.
        constexpr int L = (65536 / (MINB * G::THREADS)) / 8 * 8;
        constexpr int C = (2 * L - 24) > 232 ? 232 : (2 * L - 24) / 8 * 8;
        static_assert(C >= 128, "producer warp group leaves the consumers too few registers");
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C) : "memory");
    }

    // ---- warp (wq, wr) owns planes q0 + PP*wq + p and diagonal entries e = DD*wr + d ----
    const int wq = warp % G::CWQ, wr = warp / G::CWQ;
    const int c = j0 + lane;
    const bool col_ok = CL > 1 || c < n;  // shifted cluster tiles wrap (N % 32 == 0)
    const int64_t nn = (int64_t)n * n;
    const int64_t qw = q0 + PP * wq;
    const int e0 = DD * wr;
    Cx<R>* gb = P.g4 + (qw - P.lo) * nn;
    int offg[DD];
#pragma unroll
    for (int d = 0; d < DD; ++d) offg[d] = wrap(k1_0 + e0 + d, n) * n + wrap(c + e0 + d, n);
    uint32_t okmask = 0;
#pragma unroll
    for (int p = 0; p < PP; ++p)
#pragma unroll
        for (int d = 0; d < DD; ++d)
            if (col_ok && (qw + p) < P.hi && (CL > 1 || (k1_0 + e0 + d) < n)) okmask |= 1u << (p * DD + d);
    Cx<R> acc[PP][DD];
#pragma unroll
    for (int p = 0; p < PP; ++p)
#pragma unroll
        for (int d = 0; d < DD; ++d) {
            if ((EXP & (EXP_NOLOAD | K1_DEFER)) == 0 && (okmask & (1u << (p * DD + d)))) {
                acc[p][d] = ld_g4(gb + p * nn + offg[d]);
            } else {
                acc[p][d].re = R(0);
                acc[p][d].im = R(0);
            }
        }

    // shared-memory element offsets (complex units) inside a stage
    // band row of (p, d) relative to R0: PP*wq + p - (e0 + d) + DR - 1
    const int sh_o = (PP * wq + DR - DD - e0) * G::W + (31 - lane) + ps;  // + j * W
    const int dr_o = e0 * G::W + lane + pd;                                // + d * W
#pragma unroll 1
    for (int w = 0; w < P.nbatch; ++w) {
        const int s = w % NST;
        mbar_wait(&full[s], (w / NST) & 1);
        const Cx<RG>* dir_u = reinterpret_cast<const Cx<RG>*>(smem_raw + (size_t)s * G::STAGE_BYTES + G::DIR_OFF);
        const Cx<RG>* dir_d = dir_u + G::DIR_ELEMS;
        const Cx<RG>* sh_u = reinterpret_cast<const Cx<RG>*>(smem_raw + (size_t)s * G::STAGE_BYTES + G::SH_OFF);
        const Cx<RG>* sh_d = sh_u + G::SH_ELEMS;
        if constexpr ((EXP & EXP_NOMATH) != 0) {
            if (G::PW == 0 && producer && w >= 1 && w - 1 + NST < P.nbatch) {
                mbar_wait(&empty[(w - 1) % NST], ((w - 1) / NST) & 1);
                issue(w - 1 + NST);
            }
            release(s);
            continue;
        }
        // Direct elements first (sheared box: row d, column lane); shifted elements
        // stream diagonal by diagonal (j = p - d + DD-1), one ahead.
        Stg<R> dv[DD];
#pragma unroll
        for (int d = 0; d < DD; ++d) dv[d] = widen<R>(lds_plain(dir_u + d * G::W + dr_o, dir_d + d * G::W + dr_o));
        constexpr int NJ = PP + DD - 1;  // diagonals
        constexpr int PF = G::PF < NJ ? G::PF : NJ;
        Stg<R> sbuf[PF];  // register ring of the next PF diagonals' shifted operands
#pragma unroll
        for (int i = 0; i < PF; ++i)
            sbuf[i] = widen<R>(lds_plain(sh_u + sh_o + i * G::W, sh_d + sh_o + i * G::W));
        // Producer duty (lane 0 of warp 0): refill the stage every warp released in
        // the previous iteration with walker w - 1 + NST; its TMA overlaps this math.
        if (G::PW == 0 && producer && w >= 1 && w - 1 + NST < P.nbatch) {
            const int wp = w - 1;
            mbar_wait(&empty[wp % NST], (wp / NST) & 1);
            issue(wp + NST);
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const Stg<R> S = sbuf[j % PF];
            if (j + PF < NJ)
                sbuf[j % PF] = widen<R>(lds_plain(sh_u + sh_o + (j + PF) * G::W, sh_d + sh_o + (j + PF) * G::W));
#pragma unroll
            for (int d = 0; d < DD; ++d) {
                const int p = j + d - (DD - 1);
                if (p < 0 || p >= PP) continue;
                const Stg<R>& D = dv[d];
                if constexpr (FUSED) {
                    update_fused(acc[p][d], S, D);
                } else {
                    R p1r, p1i, p2r, p2i;
                    cmul(S.ur, S.ui, D.dr, D.di, p1r, p1i);  // u * down[k2][k1]
                    cmul(S.dr, S.di, D.ur, D.ui, p2r, p2i);  // d * up[k2][k1]
                    acc[p][d].re = add_rn(acc[p][d].re, add_rn(p1r, p2r));
                    acc[p][d].im = add_rn(acc[p][d].im, add_rn(p1i, p2i));
                }
            }
        }
        // Release the stage only once its values have been consumed by the math
        // (an in-flight ld.shared must not race the TMA refill of the stage).
        release(s);
    }
    // Peers arrive on this CTA's empty barriers until they finish their last
    // walkers: the producer waits for those final phases, so no remote arrive
    // can land after the CTA (and its shared memory) is gone.
    if constexpr (CL > 1) {
        if (producer)
            for (int w = P.nbatch > NST ? P.nbatch - NST : 0; w < P.nbatch; ++w)
                mbar_wait(&empty[w % NST], (w / NST) & 1);
    }

    // Deferred update: the warp parks its block in the (now idle) stage buffers,
    // one row segment per (p, d), and the TMA engine adds each segment to the
    // slice (cp.reduce.async.bulk .add): no per-lane reds (red.global has no
    // 128-bit f64 form, so those cost two half-sector L2 atomics per entry and
    // stall the LSU queue).  Non-deferred (K1_BULKST): the same park, then a
    // plain bulk store of each segment: -3 % at B = 1 and 8, -5 % at N = 4608
    // against per-lane st.global.cs (lab29).  Complex64 segments are parked at
    // the parity of their first column, so that global and shared addresses
    // agree mod 16 B; an odd head or tail entry goes through the LSU.  That is
    // slower than per-lane reds/stores for their 256-B segments (lab30: +8 %
    // fused, +4-7 % exact), so complex64 slices keep the LSU path (BULK_SLICE).
    if constexpr (PARK) {
        // every consumer warp is past its last stage read (and every fill has landed)
        if constexpr (G::PW == 1)
            asm volatile("barrier.sync 1, %0;" ::"r"(32 * G::CW) : "memory");
        else
            __syncthreads();
        Cx<R>* park = reinterpret_cast<Cx<R>*>(smem_raw + warp * WARP_PARK);
#pragma unroll
        for (int d = 0; d < DD; ++d) {
            int k2 = j0 + e0 + d;  // column of the segment's entry 0, < 2N
            if (k2 >= n) k2 -= n;
            const int sh = sizeof(R) == 8 ? 0 : (k2 & 1);
#pragma unroll
            for (int p = 0; p < PP; ++p) park[(p * DD + d) * PSTR + sh + lane] = acc[p][d];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> TMA reads
        __syncwarp();
        // Interior blocks (no row or column wrap, all planes in the slice): the
        // whole PP x DD x 32 block is one sheared box of the slice's tensor map.
        const bool interior = P.use_gmap && qw + PP <= P.hi && k1_0 + e0 + DD - 1 < n &&
                              j0 + 31 + e0 + DD - 1 < n;
        if (interior) {
            if (lane == 0) {
                const int c0 = 2 * (j0 - k1_0 + n), c1 = k1_0 + e0, c2 = (int)(qw - P.lo);
                if constexpr (DEFER)
                    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group"
                                 " [%0, {%2, %3, %4}], [%1];" ::"l"(reinterpret_cast<uint64_t>(&P.gmap)),
                                 "r"(smem_u32(park)), "r"(c0), "r"(c1), "r"(c2) : "memory");
                else
                    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group"
                                 " [%0, {%2, %3, %4}], [%1];" ::"l"(reinterpret_cast<uint64_t>(&P.gmap)),
                                 "r"(smem_u32(park)), "r"(c0), "r"(c1), "r"(c2) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
        } else if (lane < PP * DD) {  // lane t writes segment t = (p, d)
            const int p = lane / DD, d = lane % DD;
            const int k1 = k1_0 + e0 + d;  // < 2N
            if (qw + p < P.hi && (CL > 1 || k1 < n)) {
                const int cnt = CL > 1 ? 32 : min(32, n - j0);  // valid columns j0 + i
                int k2 = j0 + e0 + d;
                if (k2 >= n) k2 -= n;
                Cx<R>* row = gb + p * nn + (int64_t)(k1 >= n ? k1 - n : k1) * n;
                const Cx<R>* seg = park + lane * PSTR + (sizeof(R) == 8 ? 0 : (k2 & 1));
                const int run1 = min(cnt, n - k2);  // up to the row end, then wrap to column 0
                segment_out<DEFER>(row + k2, seg, run1);
                if (run1 < cnt) segment_out<DEFER>(row, seg + run1, cnt - run1);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // park read before exit
            }
        }
    } else {
#pragma unroll
        for (int p = 0; p < PP; ++p)
#pragma unroll
            for (int d = 0; d < DD; ++d)
                if (okmask & (1u << (p * DD + d))) {
                    if constexpr ((EXP & K1_DEFER) != 0 && sizeof(R) == 4 && (EXP & EXP_SCALAR_RED) == 0) {
                        // one 8-B vector red per complex64 entry (a warp covers 256 B)
                        asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(gb + p * nn + offg[d]),
                                     "f"(acc[p][d].re), "f"(acc[p][d].im) : "memory");
                    } else if constexpr ((EXP & K1_DEFER) != 0) {
                        R* a = reinterpret_cast<R*>(gb + p * nn + offg[d]);
                        atomicAdd(a, acc[p][d].re);
                        atomicAdd(a + 1, acc[p][d].im);
                    } else if ((EXP & EXP_NOSTORE) == 0 || acc[p][d].re == R(-1234.5)) {
                        st_g4(gb + p * nn + offg[d], acc[p][d]);
                    }
                }
    }
    if constexpr ((EXP & K1_DEFER) != 0 && G::CL == 1) {  // chained: complete after the previous pass
        if (P.chain && threadIdx.x == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    }
}

// Host: the two sheared tensor maps of one staged payload, cached by (pointer, n, dtype).

// Offset of the sheared coordinate origin (elements): >= N so every coordinate
// is non-negative, and the map's base (stg - off * es) stays 16-B aligned.
int sheared_offset(int n, int es) { return (es == 8 && (n & 1)) ? n + 1 : n; }

PFN_encodeTiled tensor_map_encoder() {
    static PFN_encodeTiled encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q{};
        void* fn = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return nullptr;
        encode = reinterpret_cast<PFN_encodeTiled>(fn);
    }
    return encode;
}

g4_status make_maps(const void* stg, int n, int es, int nsh, int width, int dd, int band_spins,
                           MapPair* out) {
    PFN_encodeTiled encode = tensor_map_encoder();
    if (!encode) return fail(G4_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t ld = (cuuint64_t)staged_ld(n, es), rows = (cuuint64_t)staged_rows(n, es);
    const cuuint64_t plane_b = (cuuint64_t)staged_plane(n, es) * es;
    const cuuint32_t ew = es / 8;  // 64-bit elements per complex entry
    const int off = sheared_offset(n, es);
    // Sheared view of the staged payload: element (x, c2, spin) lives at
    //   base + x * 8 + c2 * (LD + 1) * es + spin * plane,  base = stg - off * es,
    // so with x = ew * c1 (+ re/im) it is stg[spin][c2][c1 - off + c2].  Box rows
    // are contiguous runs of 32 entries (256 or 512 B).
    // row extent rounded up to a 16-B multiple (TMA requirement for 8-B entries)
    const cuuint64_t dims[3] = {(ew * (cuuint64_t)(off + ld + n) + 1) / 2 * 2, rows, 2};
    const cuuint64_t strides[2] = {(ld + 1) * es, plane_b};
    const cuuint32_t estr[3] = {1, 1, 1};
    void* base = static_cast<char*>(const_cast<void*>(stg)) - (size_t)off * es;
    for (int which = 0; which < 2; ++which) {
        const cuuint32_t box[3] = {(cuuint32_t)width * ew, which == 0 ? (cuuint32_t)dd : (cuuint32_t)nsh,
                                   which == 0 ? 2u : (cuuint32_t)band_spins};
        CUresult r = encode(which == 0 ? &out->dmap : &out->smap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base,
                            dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled (%s) failed: %d", which == 0 ? "direct" : "band", (int)r);
            return G4_ERR_CUDA;
        }
    }
    return G4_OK;
}

g4_status get_maps(const void* stg, int n, int es, int nsh, int width, int dd, int band_spins,
                          MapPair* out) {
    static std::mutex mu;
    static std::map<std::tuple<uintptr_t, int, int, int, int, int>, MapPair> cache;
    const auto key = std::make_tuple(reinterpret_cast<uintptr_t>(stg), n, nsh, es, dd, band_spins);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second;
        return G4_OK;
    }
    G4_TRY(make_maps(stg, n, es, nsh, width, dd, band_spins, out));
    if (cache.size() > 4096) cache.clear();
    cache.emplace(key, *out);
    return G4_OK;
}

// Sheared tensor map of a complex128 slice for the K1 write-back: element
// (x, r, p) (x in doubles) is G4[p][r][r + x/2 - N], i.e. dim-1 stride (N+1)
// entries, so a box of DD rows is a K3-diagonal strip.  The base lies N
// entries before the slice; only interior boxes (no column wrap) are used.
bool g4_gmap_enabled() {
    static const bool on = env_int("G4RING_GMAP", 1) != 0;  // 0: per-segment bulk ops (A/B)
    return on;
}
g4_status slice_map(const void* g4, int n, int64_t planes, int pp, int dd, CUtensorMap* out) {
    static std::mutex mu;
    static std::map<std::tuple<uintptr_t, int, int64_t, int, int>, CUtensorMap> cache;
    const auto key = std::make_tuple(reinterpret_cast<uintptr_t>(g4), n, planes, pp, dd);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second;
        return G4_OK;
    }
    PFN_encodeTiled encode = tensor_map_encoder();
    if (!encode) return fail(G4_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[3] = {(cuuint64_t)4 * n, (cuuint64_t)n, (cuuint64_t)planes};
    const cuuint64_t strides[2] = {(cuuint64_t)(n + 1) * 16, (cuuint64_t)n * n * 16};
    const cuuint32_t box[3] = {64, (cuuint32_t)dd, (cuuint32_t)pp};
    const cuuint32_t estr[3] = {1, 1, 1};
    void* base = static_cast<char*>(const_cast<void*>(g4)) - (size_t)n * 16;
    CUresult r = encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled (slice) failed: %d", (int)r);
        return G4_ERR_CUDA;
    }
    if (cache.size() > 1024) cache.clear();
    cache.emplace(key, *out);
    return G4_OK;
}

template <typename R, typename RG, class G, bool FUSED, int MINB, int EXP>
static g4_status launch_v2_t(const AccParams<R, RG>& prm, cudaStream_t st) {
    if constexpr (G::CL > 1) {  // shifted cluster tiles need whole 32-wide strips and CL | chunks
        const int64_t nx = (prm.hi - prm.lo + G::Q - 1) / G::Q;
        if (prm.n % 32 != 0 || nx % G::CL != 0)
            return launch_v2_t<R, RG, typename G::Base, FUSED, MINB, EXP>(prm, st);
    }
    {  // the >48 KB dynamic shared-memory opt-in is per device (a host may drive several GPUs)
        static std::mutex mu;
        static uint64_t done = 0;
        int dev = 0;
        G4_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(mu);
        if (!(done & (1ull << (dev & 63)))) {
            G4_CUDA(cudaFuncSetAttribute(k_accumulate_tma<R, RG, G, FUSED, MINB, EXP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM));
            done |= 1ull << (dev & 63);
        }
    }
    const int n = prm.n;
    for (int b0 = 0; b0 < prm.nbatch; b0 += TMA_MAXW) {
        TmaParams<R> tp;
        std::memset(&tp, 0, sizeof(tp));
        tp.g4 = prm.g4;
        tp.lo = prm.lo;
        tp.hi = prm.hi;
        tp.n = n;
        tp.off = sheared_offset(n, G::ES);
        if constexpr (BULK_SLICE<R> && G::PP * G::DD <= 32) {
            G4_TRY(slice_map(prm.g4, n, prm.hi - prm.lo, G::PP, G::DD, &tp.gmap));
            tp.use_gmap = g4_gmap_enabled() ? 1 : 0;
        }
        tp.nbatch = std::min(TMA_MAXW, prm.nbatch - b0);
        if constexpr ((EXP & K1_DEFER) != 0 && G::CL == 1) {
            static const bool chain_on = env_int("G4RING_V3_CHAIN", 1) != 0;
            tp.chain = (chain_on && (b0 > 0 || k1_chain_prev(st))) ? 1 : 0;
        }
        for (int i = 0; i < tp.nbatch; ++i) {
            MapPair mp;
            G4_TRY(get_maps(prm.stg[b0 + i], n, G::ES, G::CL > 1 ? G::HS : G::NSH, G::W, G::DR,
                            G::CL > 1 ? 1 : 2, &mp));
            tp.dmap[i] = mp.dmap;
            tp.smap[i] = mp.smap;
        }
        const int64_t planes = prm.hi - prm.lo;
        tp.nx = (int32_t)((planes + G::Q - 1) / G::Q);
        const uint64_t ctas = (uint64_t)tp.nx * ((n + 31) / 32) * ((n + G::DR - 1) / G::DR);
        if (ctas >= (1ull << 31)) return fail(G4_ERR_CONTRACT, "accumulate: launch grid too large");
        if constexpr (G::CL == 1) {
            static const bool pdl = env_int("G4RING_PDL", 1) != 0;
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3((unsigned)ctas);
            lc.blockDim = dim3(G::THREADS);
            lc.dynamicSmemBytes = G::SMEM;
            lc.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            lc.attrs = at;
            lc.numAttrs = pdl ? 1 : 0;
            G4_TRY(check_cuda(cudaLaunchKernelEx(&lc, k_accumulate_tma<R, RG, G, FUSED, MINB, EXP>, tp),
                              "k_accumulate_tma launch"));
        } else {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3((unsigned)ctas);
            lc.blockDim = dim3(G::THREADS);
            lc.dynamicSmemBytes = G::SMEM;
            lc.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = G::CL;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            G4_TRY(check_cuda(cudaLaunchKernelEx(&lc, k_accumulate_tma<R, RG, G, FUSED, MINB, EXP>, tp),
                              "k_accumulate_tma cluster launch"));
        }
    }
    k1_chain_note((EXP & K1_DEFER) != 0 && G::CL == 1);
    return G4_OK;
}

// G4_ARITH_FUSED adds the walkers' sum to the slice at the end (K1_DEFER) with
// >= 3 walkers per pass.  With the TMA bulk-reduce epilogue (complex128 slices)
// this pays on any slice height: -2 % at P = 64, B = 8; -19 % at P = 8, B = 8
// (the 8-GPU ring share); -7 % at N = 4608 (lab28).  With 1-2 walkers the L2
// read-modify-write costs more than the G4 load it saves (+13 % / +5 %; with
// chained passes +17 % / +6 %, lab r02al); at 3 walkers the chained deferred
// pass wins (114.9 vs 125.2 us at the bench shape, lab r02al).
static bool defer_update(int nbatch, int64_t planes) {
    static const int min_w = env_int("G4RING_DEFER_MIN_WALKERS", 3);  // measurement knobs
    static const int min_p = env_int("G4RING_DEFER_MIN_PLANES", 1);
    return nbatch >= min_w && planes >= min_p;
}

template <typename R, typename RG, class G, bool FUSED, int MINB, int EXP = 0>
static g4_status launch_v2(const AccParams<R, RG>& prm, cudaStream_t st) {
    if constexpr (FUSED && EXP == 0) {
        if (defer_update(prm.nbatch, prm.hi - prm.lo)) {
            if constexpr (sizeof(R) == 4) {  // A/B knob: scalar f32 reds instead of one v2 red per entry
                static const bool scalar = env_int("G4RING_SCALAR_RED", 0) != 0;
                if (scalar) return launch_v2_t<R, RG, G, FUSED, MINB, K1_DEFER | EXP_SCALAR_RED>(prm, st);
            }
            return launch_v2_t<R, RG, G, FUSED, MINB, K1_DEFER>(prm, st);
        }
    }
    if constexpr (EXP == 0 && BULK_SLICE<R>) {
        static const bool bulk_store = env_int("G4RING_BULK_STORE", 1) != 0;  // 0: st.global.cs (A/B)
        if (bulk_store) return launch_v2_t<R, RG, G, FUSED, MINB, K1_BULKST>(prm, st);
    }
    return launch_v2_t<R, RG, G, FUSED, MINB, EXP>(prm, st);
}

// v2 geometries: PP x DD thread block, CWQ x CWR warps (CTA tile Q x DR), NST
// stages, CTAs per SM.  Sweep results: profiles/r01_summary.md.
//   id  PPxDD  CWQxCWR  QxDR   NST CTA/SM       id  PPxDD  CWQxCWR  QxDR   NST CTA/SM
//    0  4x4    4x1      16x4    3   3            12  8x4    2x2      16x8    3   2
//    3  4x4    4x1      16x4    2   4            13  8x2    2x2      16x4    2   4   (default, P >= 16, exact)
//    7  4x4    4x2      16x8    2   2            16  4x4    4x1      16x4    4   2
//    8  4x4    4x4      16x16   2   1            17  8x2    2x2      16x4    4   2
//   11  4x4    4x2      16x8    3   2            19  8x2    1x4       8x8    2   4   (default, P <= 8)
//                                                20  4x4    2x2       8x8    2   4
//   21 / 22: geometry 12 in clusters of 4 / 2 (band multicast); 23 / 24: 13 likewise.
//   Measured slower than 12 / 13 (profiles/r01_summary.md, lab27); selectable only.
//   25: geometry 12 plus a producer warp group (setmaxnreg 24 / 232): the fused
//   default for P >= 16 (-4 % at B = 8 and 16, lab35).  27: geometry 19 likewise
//   (3 CTAs/SM, consumers at 136): within 2 % of 19 at P = 8, B = 8 (lab36);
//   selectable only.
// The geometry id of the last K1 launch (v1: 1), for tests that pin the
// dispatch: g4_last_k1_geometry().
static std::atomic<int> g_last_geom{0};

template <typename R, typename RG, bool FUSED>
static g4_status launch_v2_geom(int g, const AccParams<R, RG>& prm, cudaStream_t st) {
    g_last_geom.store(g, std::memory_order_relaxed);  // a fallback below re-enters with its own id
    switch (g) {
        case 0: return launch_v2<R, RG, V2Geom<RG, 4, 4, 3>, FUSED, 3>(prm, st);
        case 3: return launch_v2<R, RG, V2Geom<RG, 4, 4, 2>, FUSED, 4>(prm, st);
        case 7: return launch_v2<R, RG, V2Geom<RG, 4, 4, 2, 4, 2>, FUSED, 2>(prm, st);
        case 8: return launch_v2<R, RG, V2Geom<RG, 4, 4, 2, 4, 4>, FUSED, 1>(prm, st);
        case 11: return launch_v2<R, RG, V2Geom<RG, 4, 4, 3, 4, 2>, FUSED, 2>(prm, st);
        case 12: return launch_v2<R, RG, V2Geom<RG, 8, 2, 3, 4, 2>, FUSED, 2>(prm, st);
        case 13:
            if constexpr (sizeof(R) == 8 && sizeof(RG) == 8) {
                switch (exp_flags()) {  // measurement variants (complex128 only)
                    case 0: break;
                    case 1: return launch_v2<R, RG, V2Geom<RG, 8, 2, 2, 2, 2>, FUSED, 4, 1>(prm, st);
                    case 2: return launch_v2<R, RG, V2Geom<RG, 8, 2, 2, 2, 2>, FUSED, 4, 2>(prm, st);
                    case 3: return launch_v2<R, RG, V2Geom<RG, 8, 2, 2, 2, 2>, FUSED, 4, 3>(prm, st);
                    case 4: return launch_v2<R, RG, V2Geom<RG, 8, 2, 2, 2, 2>, FUSED, 4, 4>(prm, st);
                    case 7: return launch_v2<R, RG, V2Geom<RG, 8, 2, 2, 2, 2>, FUSED, 4, 7>(prm, st);
                    default: return fail(G4_ERR_CONTRACT, "G4RING_EXP: unknown variant");
                }
            }
            return launch_v2<R, RG, V2Geom<RG, 8, 2, 2, 2, 2>, FUSED, 4>(prm, st);
        case 16: return launch_v2<R, RG, V2Geom<RG, 4, 4, 4>, FUSED, 2>(prm, st);
        case 17: return launch_v2<R, RG, V2Geom<RG, 8, 2, 4, 2, 2>, FUSED, 2>(prm, st);
        case 19: return launch_v2<R, RG, V2Geom<RG, 8, 1, 2, 2, 4>, FUSED, 4>(prm, st);
        case 20: return launch_v2<R, RG, V2Geom<RG, 4, 2, 2, 4, 2>, FUSED, 4>(prm, st);
        case 21: return launch_v2<R, RG, V2Geom<RG, 8, 2, 3, 4, 2, 1, 4>, FUSED, 2>(prm, st);
        case 22: return launch_v2<R, RG, V2Geom<RG, 8, 2, 3, 4, 2, 1, 2>, FUSED, 2>(prm, st);
        case 23: return launch_v2<R, RG, V2Geom<RG, 8, 2, 2, 2, 2, 1, 4>, FUSED, 4>(prm, st);
        case 24: return launch_v2<R, RG, V2Geom<RG, 8, 2, 2, 2, 2, 1, 2>, FUSED, 4>(prm, st);
        case 25: return launch_v2<R, RG, V2Geom<RG, 8, 2, 3, 4, 2, 1, 1, 1>, FUSED, 2>(prm, st);
        case 27: return launch_v2<R, RG, V2Geom<RG, 8, 1, 2, 2, 4, 1, 1, 1>, FUSED, 3>(prm, st);
        case 45:  // v3 for complex64 slices: fused + deferred
            if constexpr (FUSED && sizeof(R) == 4 && sizeof(RG) == 4)
                return launch_pst32(g, prm.g4, prm.lo, prm.hi, prm.n, reinterpret_cast<const void* const*>(prm.stg),
                                    prm.nbatch, st);
            return launch_v2_geom<R, RG, FUSED>(FUSED ? 12 : 13, prm, st);
        case 40:
        case 42:
        case 43:
        case 44:  // v3, the persistent kernel (complex128 slices): fused + deferred, or exact
            if constexpr (sizeof(R) == 8)
                return launch_pst<RG>(g, !FUSED, prm.g4, prm.lo, prm.hi, prm.n,
                                      reinterpret_cast<const void* const*>(prm.stg), prm.nbatch, st);
            return launch_v2_geom<R, RG, FUSED>(FUSED ? 12 : 13, prm, st);
        default: return fail(G4_ERR_CONTRACT, "G4RING_V2GEOM: unknown geometry");
    }
}

// Host-side description of a geometry id (same table as launch_v2_geom).
struct GeomInfo {
    int pp, dd, q, dr, nst, ctas, warps;
};
template <class G>
static GeomInfo info_of(int ctas) {
    return {G::PP, G::DD, G::Q, G::DR, G::NST, ctas, G::THREADS / 32};  // all warps, producers included
}
static bool geom_info(int g, GeomInfo* out) {
    switch (g) {
        case 0: *out = info_of<V2Geom<double, 4, 4, 3>>(3); return true;
        case 3: *out = info_of<V2Geom<double, 4, 4, 2>>(4); return true;
        case 7: *out = info_of<V2Geom<double, 4, 4, 2, 4, 2>>(2); return true;
        case 8: *out = info_of<V2Geom<double, 4, 4, 2, 4, 4>>(1); return true;
        case 11: *out = info_of<V2Geom<double, 4, 4, 3, 4, 2>>(2); return true;
        case 12: *out = info_of<V2Geom<double, 8, 2, 3, 4, 2>>(2); return true;
        case 13: *out = info_of<V2Geom<double, 8, 2, 2, 2, 2>>(4); return true;
        case 16: *out = info_of<V2Geom<double, 4, 4, 4>>(2); return true;
        case 17: *out = info_of<V2Geom<double, 8, 2, 4, 2, 2>>(2); return true;
        case 19: *out = info_of<V2Geom<double, 8, 1, 2, 2, 4>>(4); return true;
        case 20: *out = info_of<V2Geom<double, 4, 2, 2, 4, 2>>(4); return true;
        case 21: *out = info_of<V2Geom<double, 8, 2, 3, 4, 2, 1, 4>>(2); return true;
        case 22: *out = info_of<V2Geom<double, 8, 2, 3, 4, 2, 1, 2>>(2); return true;
        case 23: *out = info_of<V2Geom<double, 8, 2, 2, 2, 2, 1, 4>>(4); return true;
        case 24: *out = info_of<V2Geom<double, 8, 2, 2, 2, 2, 1, 2>>(4); return true;
        case 25: *out = info_of<V2Geom<double, 8, 2, 3, 4, 2, 1, 1, 1>>(2); return true;
        case 27: *out = info_of<V2Geom<double, 8, 1, 2, 2, 4, 1, 1, 1>>(3); return true;
        case 40:
        case 42:
        case 43:
        case 44:
        case 45: {
            int pp, dd, q, dr, nst;
            pst_geom_info(g, &pp, &dd, &q, &dr, &nst);
            *out = {pp, dd, q, dr, nst, 1, 16};
            return true;
        }
        default: return false;
    }
}

// Automatic choice: a 16-plane CTA tile when the slice has >= 16 planes, an
// 8-plane tile for the 8-plane slices of an 8-GPU ring.  When the G4 block is
// not read at CTA start (K1_DEFER), the 2-CTA/SM, 32-entry-register-block
// geometry 12 beats 13 (lab24: -7 % at B = 16, -10 % at N = 4608).
// G4RING_V2GEOM overrides.
static int v2_geom(int n, int64_t planes, bool deferred, bool c64_slice, int nbatch) {
    static int forced = -2;
    if (forced == -2) {
        const char* e = getenv("G4RING_V2GEOM");
        forced = e ? atoi(e) : -1;
    }
    if (forced >= 0) return forced;
    if (planes < 16) return 19;
    if (!deferred) {  // exact mode (bitwise): geometry 13, or v3's exact variant (G4RING_V3_EXACT=1, lab)
        static const int v3_exact = env_int("G4RING_V3_EXACT", 0);
        if (v3_exact && !c64_slice && nbatch >= 8) return n > 2048 ? 43 : 40;
        return 13;
    }
    // complex128 slices: the persistent TMEM-handoff kernel (v3).  Geometry 40
    // (4 stages, 4 park slots) at N <= 1024; at N = 4608 the slice reduces miss
    // L2 far more and geometry 43 (3 stages, 10 park slots) wins, 13.9 ms vs
    // 19.6 per pass of config 4's share (lab r02c).  complex64 slices keep
    // geometry 12 (the producer warp group loses there, lab35).
    // With few walkers per pass the persistent kernel's fixed hand-off and
    // slice reduction per tile dominate: geometry 25 below V3_MIN_WALKERS.
    static const int v3_min = env_int("G4RING_V3_MIN_WALKERS", 8);
    if (c64_slice) {  // complex64 slices: geometry 12, or v3's complex64 kernel (G4RING_V3_C64=1)
        static const int v3_c64 = env_int("G4RING_V3_C64", 0);
        return (v3_c64 && nbatch >= v3_min) ? 45 : 12;
    }
    if (nbatch < v3_min) return 25;
    return n > 2048 ? 43 : 40;
}

static bool use_v2(int n, int64_t planes) {
    const int variant = kernel_variant();
    return n >= 64 && (variant == 2 || (variant == 0 && planes >= 4));
}

// Chained fused passes (g4_k1.cuh): per stream, was the library's last K1
// launch there a v3 fused pass?  dispatch_t rewrites the record after every
// launch; launch_pst_t notes (per thread) that it launched such a pass.
static std::mutex g_chain_mu;
static std::unordered_map<cudaStream_t, bool> g_chain_prev;
static thread_local bool t_chain_launched = false;

bool k1_chain_prev(cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_chain_mu);
    const auto it = g_chain_prev.find(st);
    return it != g_chain_prev.end() && it->second;
}
void k1_chain_note(bool chain_safe) { t_chain_launched = chain_safe; }

template <typename R, typename RG, bool FUSED>
static g4_status dispatch_body(const AccParams<R, RG>& prm, cudaStream_t st);

template <typename R, typename RG, bool FUSED>
static g4_status dispatch_t(const AccParams<R, RG>& prm, cudaStream_t st) {
    t_chain_launched = false;
    const g4_status s = dispatch_body<R, RG, FUSED>(prm, st);
    std::lock_guard<std::mutex> lk(g_chain_mu);
    g_chain_prev[st] = s == G4_OK && t_chain_launched;
    return s;
}

template <typename R, typename RG, bool FUSED>
static g4_status dispatch_body(const AccParams<R, RG>& prm, cudaStream_t st) {
    const int64_t planes = prm.hi - prm.lo;
    if (use_v2(prm.n, planes))
        return launch_v2_geom<R, RG, FUSED>(
            v2_geom(prm.n, planes, FUSED && defer_update(prm.nbatch, planes), sizeof(R) == 4,
                    std::min<int32_t>(prm.nbatch, TMA_MAXW)),
            prm, st);
    g_last_geom.store(1, std::memory_order_relaxed);
    if (planes <= 4) return launch_v1<R, RG, 4, 4, 1, 12, FUSED>(prm, st);
    if (planes <= 8) return launch_v1<R, RG, 4, 4, 2, 6, FUSED>(prm, st);
    return launch_v1<R, RG, 4, 4, 4, 3, FUSED>(prm, st);
}

static int g_arith = G4_ARITH_EXACT;

template <typename R, typename RG>
static g4_status dispatch(const AccParams<R, RG>& prm, cudaStream_t st) {
    // G4_ARITH_FUSED pays off through the deferred update; where that does not
    // apply (few walkers, small slices, v1) the exact kernel is as fast, so it
    // runs instead (and stays bitwise).
    const int64_t planes = prm.hi - prm.lo;
    const bool fused = g_arith == G4_ARITH_FUSED && use_v2(prm.n, planes) &&
                       defer_update(std::min<int32_t>(prm.nbatch, TMA_MAXW), planes);
    return fused ? dispatch_t<R, RG, true>(prm, st) : dispatch_t<R, RG, false>(prm, st);
}

template <typename R, typename RG>
static g4_status accumulate_t(void* g4p, int64_t lo, int64_t hi, int32_t n, const void* const* staged,
                              int32_t nbatch, cudaStream_t st) {
    if (!aligned(g4p, sizeof(Cx<R>)))
        return fail(G4_ERR_CONTRACT, "accumulate: g4 slice pointer is not entry-aligned");
    for (int32_t b0 = 0; b0 < nbatch; b0 += G4_MAX_BATCH) {
        AccParams<R, RG> prm{};
        prm.g4 = static_cast<Cx<R>*>(g4p);
        prm.lo = lo;
        prm.hi = hi;
        prm.n = n;
        prm.nbatch = std::min<int32_t>(G4_MAX_BATCH, nbatch - b0);
        for (int i = 0; i < prm.nbatch; ++i) {
            const void* sp = staged[b0 + i];
            if (!sp) return fail(G4_ERR_CONTRACT, "accumulate: null staged payload");
            if (!aligned(sp, 16)) return fail(G4_ERR_CONTRACT, "accumulate: staged payload is not 16-B aligned");
            prm.stg[i] = static_cast<const Cx<RG>*>(sp);
        }
        G4_TRY(dispatch(prm, st));
    }
    return G4_OK;
}

}  // namespace g4

extern "C" {

g4_status g4_accumulate_staged(void* g4p, int64_t lo, int64_t hi, int32_t n, const void* const* staged,
                               int32_t nbatch, int32_t dtype, int32_t channel, void* stream) {
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
    if (dtype == G4_C128) return accumulate_t<double, double>(g4p, lo, hi, n, staged, nbatch, st);
    if (dtype == G4_C64) return accumulate_t<float, float>(g4p, lo, hi, n, staged, nbatch, st);
    if (dtype == G4_C128_G64) return accumulate_t<double, float>(g4p, lo, hi, n, staged, nbatch, st);
    return fail(G4_ERR_CONTRACT, "unknown dtype");
}

g4_status g4_set_kernel_variant(int32_t variant) {
    if (variant < 0 || variant > 2)
        return g4::fail(G4_ERR_CONTRACT, "kernel variant must be 0 (auto), 1 (v1) or 2 (v2)");
    g4::g_variant = variant;
    return G4_OK;
}

g4_status g4_k1_config(int32_t n, int64_t planes, int32_t nbatch, int32_t dtype, int32_t* out) {
    using namespace g4;
    if (!out) return fail(G4_ERR_CONTRACT, "k1_config: null output");
    if (n < 1 || planes < 1 || nbatch < 1) return fail(G4_ERR_CONTRACT, "k1_config: n, planes and nbatch must be >= 1");
    if (dtype != G4_C128 && dtype != G4_C64 && dtype != G4_C128_G64) return fail(G4_ERR_CONTRACT, "unknown dtype");
    const int32_t walkers = std::min<int32_t>(nbatch, TMA_MAXW);  // per launch
    if (use_v2(n, planes)) {
        const bool deferred = g_arith == G4_ARITH_FUSED && defer_update(walkers, planes);
        GeomInfo gi;
        const int g = v2_geom(n, planes, deferred, dtype == G4_C64, walkers);
        if (!geom_info(g, &gi)) return fail(G4_ERR_CONTRACT, "G4RING_V2GEOM: unknown geometry");
        const int32_t v[9] = {g >= 40 ? 3 : 2, gi.pp, gi.dd, gi.q, gi.dr, gi.nst, gi.ctas, gi.warps, deferred ? 1 : 0};
        std::memcpy(out, v, sizeof(v));
    } else {
        const int warps = planes <= 4 ? 1 : planes <= 8 ? 2 : 4;
        const int ctas = planes <= 4 ? 12 : planes <= 8 ? 6 : 3;
        const int32_t v[9] = {1, 4, 4, 4 * warps, 4, 0, ctas, warps, 0};
        std::memcpy(out, v, sizeof(v));
    }
    return G4_OK;
}

int32_t g4_get_arith_mode(void) { return g4::g_arith; }

int32_t g4_last_k1_geometry(void) { return g4::g_last_geom.load(std::memory_order_relaxed); }

g4_status g4_set_arith_mode(int32_t mode) {
    if (mode != G4_ARITH_EXACT && mode != G4_ARITH_FUSED)
        return g4::fail(G4_ERR_CONTRACT, "arith mode must be G4_ARITH_EXACT or G4_ARITH_FUSED");
    g4::g_arith = mode;
    return G4_OK;
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
    if (!workspace || workspace_bytes < need) return fail(G4_ERR_CONTRACT, "accumulate: workspace too small");
    const int64_t pb = g4_payload_bytes(n, dtype);
    void* stg[G4_MAX_BATCH];
    for (int32_t b0 = 0; b0 < nbatch; b0 += G4_MAX_BATCH) {
        const int32_t nb = std::min<int32_t>(G4_MAX_BATCH, nbatch - b0);
        for (int i = 0; i < nb; ++i) stg[i] = static_cast<char*>(workspace) + i * pb;
        const int32_t din = dtype == G4_C128_G64 ? G4_C128 : dtype;   // reference-layout input type
        const int32_t dout = dtype == G4_C128_G64 ? G4_C64 : dtype;   // staged payload type
        G4_TRY(g4_prepare_g(stg, up + b0, down + b0, nb, n, din, dout, stream));
        G4_TRY(g4_accumulate_staged(g4p, lo, hi, n, stg, nb, dtype, channel, stream));
    }
    return G4_OK;
}

}  // extern "C"
