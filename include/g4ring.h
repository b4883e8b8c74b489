/*
 * g4ring.h -- C ABI of the B200-native G4 ring-accumulation library (libg4ring.so).
 *
 * Drop-in boundary for the hot path of the reference package `ringacc`
 * (/root/reference/pkg/src/ringacc).  Every entry point names the reference
 * interface it replaces.  Conventions:
 *   - extern "C", plain pointers and sizes, no C++ or torch types;
 *   - all device pointers are BORROWED for the duration of the stream-ordered
 *     operation; the caller owns the memory (torch tensors in the Python layer);
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *   - every function returns a g4_status; on failure g4_last_error() returns a
 *     thread-local message.  Status codes map 1:1 onto the reference exception
 *     hierarchy (ringacc/errors.py:8-27).
 *
 * Data layouts (ringacc/tensor.py):
 *   - G4 slice: data[k3 - lo][k1][k2], C-contiguous complex (re, im interleaved),
 *     K3 outermost -- GtSlice.data (tensor.py:99-136), bit-for-bit.
 *   - Walker payload, reference layout: up[N][N] then down[N][N] complex
 *     (GSigma.up / .down, tensor.py:77-96; wire body order wire.py:32-33).
 *   - Walker payload, staged layout (device-internal, produced by
 *     g4_prepare_g / g4_generate, consumed by g4_accumulate_staged, and the form
 *     that travels around the ring): spin-planar transposes with a cyclic halo,
 *       stg[s][r][c] = M_s[c mod N][r mod N],   s = 0 (up), 1 (down),
 *       0 <= r < N + G4_HALO_ROWS,  0 <= c < LD  (row pitch LD),
 *       LD = N + G4_HALO_COLS, plus 1 for complex64 when that is even (the
 *       diagonal TMA stride (LD + 1) * 8 B must be a multiple of 16 B).
 *     The core stg[s][0:N][0:N] is the transpose of the reference matrix; the
 *     halo replicates it cyclically so that every window the update kernel
 *     fetches (TMA boxes along rows and along the K3-diagonal) is contiguous.
 */
#ifndef G4RING_H
#define G4RING_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define G4RING_ABI_VERSION 1
#define G4_MAX_BATCH 64 /* walkers per accumulate launch (more are chunked) */
#define G4_HALO_ROWS 40 /* staged-layout halo (see above) */
#define G4_HALO_COLS 72

typedef enum {
    G4_OK = 0,
    G4_ERR_CONTRACT = 1,  /* ringacc.errors.ContractViolation */
    G4_ERR_CONFIG = 2,    /* ringacc.errors.ConfigError       */
    G4_ERR_TRANSPORT = 3, /* ringacc.errors.TransportError    */
    G4_ERR_DEADLOCK = 4,  /* ringacc.errors.DeadlockError     */
    G4_ERR_CUDA = 5       /* CUDA runtime/driver failure      */
} g4_status;

typedef enum {
    G4_C128 = 0,     /* complex128: ENTRY_BYTES = 16 (tensor.py:23) -- the reference dtype */
    G4_C64 = 1,      /* complex64: the paper's production G_sigma precision; 1e-5 tolerance */
    G4_C128_G64 = 2  /* mixed: complex128 G4 slice, complex64 payloads (widened exactly;
                        g4_accumulate takes complex128 up/down and rounds them to complex64)
                        -- halves payload bytes on the ring and in shared memory */
} g4_dtype;

typedef enum {
    G4_MODE_FLOAT = 0,  /* VALUE_MODES[0]: unit-disk complex values (tensor.py:199-203) */
    G4_MODE_INTEGER = 1 /* VALUE_MODES[1]: Gaussian-integer lattice {-2..2} (tensor.py:204-209) */
} g4_value_mode;

typedef enum {
    /* The only update rule the reference implements (tensor.py:233-251,
     * PAPER.md Eq. 1):  G4[K3][K1][K2] += sum_sigma G_sigma(K3-K2, K3-K1) G_-sigma(K2, K1). */
    G4_CHANNEL_EQ1 = 0
} g4_channel;

/* Last error message of the calling thread ("" if none). */
const char* g4_last_error(void);
/* G4RING_ABI_VERSION of the loaded library. */
int32_t g4_abi_version(void);
/* Bytes of one walker payload in the staged device layout:
 * 2 * ROWS * LD * entry bytes (the reference's GSigma.nbytes, tensor.py:86-89,
 * is the 2 * n * n core of it). */
int64_t g4_payload_bytes(int32_t n, int32_t dtype);
/* Staged-layout geometry for a dtype: rows per spin plane and row pitch (elements). */
g4_status g4_staged_dims(int32_t n, int32_t dtype, int32_t* rows, int32_t* ld);

/* Cyclic K difference (a - b) mod n; replaces index_diff (tensor.py:50-55).
 * Out-of-range a or b -> G4_ERR_CONTRACT. */
g4_status g4_index_diff(int64_t a, int64_t b, int64_t n, int64_t* out);

/* Balanced contiguous K3 partition over p ranks, remainder to the lowest ranks;
 * replaces make_partition (tensor.py:148-164).  ranges: 2*p int64 (lo, hi). */
g4_status g4_make_partition(int64_t n, int64_t p, int64_t* ranges);

/* K2: reference layout -> staged layout for `nbatch` walkers.  up[i], down[i] are
 * N x N complex (dtype_in); staged[i] receives the staged payload (dtype_out).
 * Supported (dtype_in, dtype_out): (C128, C128), (C64, C64), (C128, C64). */
g4_status g4_prepare_g(void* const* staged, const void* const* up, const void* const* down,
                       int32_t nbatch, int32_t n, int32_t dtype_in, int32_t dtype_out,
                       void* stream);

/* K3: device-side deterministic payload generator; replaces fill_gsigma /
 * generate_gsigma (tensor.py:215-228) with the same SplitMix64 key scheme,
 * keyed on (seed, world_rank, lane, meas) per walker i.  Any of staged / up /
 * down may be NULL (staged: staged layout; up/down: reference layout).
 * Integer mode is bitwise equal to the reference; float mode within 2 ulp. */
g4_status g4_generate(void* const* staged, void* const* up, void* const* down,
                      int32_t nbatch, uint64_t seed, const int64_t* world_rank,
                      const int64_t* lane, const int64_t* meas, int32_t n, int32_t mode,
                      int32_t dtype, void* stream);

/* K1: the G4 slice update; replaces accumulate_g4 (tensor.py:233-251) for a
 * batch of walkers applied in order 0..nbatch-1 (bitwise identical to nbatch
 * sequential reference calls).  g4: slice for planes [lo, hi) of an N-point
 * index space; staged[i]: staged payloads (g4 dtype).  Planes outside [lo, hi)
 * are never touched.  0 <= lo < hi <= n else G4_ERR_CONTRACT (tensor.py:112-115). */
g4_status g4_accumulate_staged(void* g4, int64_t lo, int64_t hi, int32_t n,
                               const void* const* staged, int32_t nbatch, int32_t dtype,
                               int32_t channel, void* stream);

/* Select the K1 implementation (process-wide): 0 = automatic (v2 for N >= 64
 * and >= 4 planes, with a 16-plane CTA tile for >= 16 planes and an 8-plane
 * tile below; v1 otherwise), 1 = v1 everywhere (register-blocked, direct
 * global loads), 2 = v2 wherever N >= 64 (TMA tensor boxes into a
 * shared-memory ring).  For A/B measurement and parity tests of both paths
 * (env G4RING_KERNEL; G4RING_V2GEOM forces a v2 geometry). */
g4_status g4_set_kernel_variant(int32_t variant);

/* Floating-point evaluation of the update (process-wide):
 *   G4_ARITH_EXACT (default): the reference's op order, rounding every product
 *     and sum as numpy does -> bitwise equal to ringacc on an FMA host;
 *   G4_ARITH_FUSED: the same terms as 8 fused multiply-adds chained into the
 *     accumulator; with >= 4 walkers per pass the walkers' sum is formed from
 *     zero and added to the slice at the end with an L2 reduction (no G4 read
 *     on the SM) -> within a few ulp (north_star tolerance 1e-10 relative),
 *     bitwise for integer-valued payloads, ~1.5x fewer FP64 issues. */
typedef enum { G4_ARITH_EXACT = 0, G4_ARITH_FUSED = 1 } g4_arith_mode;
g4_status g4_set_arith_mode(int32_t mode);
/* The current K1 arithmetic mode (G4_ARITH_EXACT or G4_ARITH_FUSED), e.g. to
 * restore it after a temporary change. */
int32_t g4_get_arith_mode(void);
/* The geometry id of the last K1 launch in this process (1 = v1; 12/13/19/25 =
 * v2 kernels; 40-45 = v3), for tests that pin the dispatch to the kernel
 * g4_k1_config reports. */
int32_t g4_last_k1_geometry(void);

/* The K1 configuration g4_accumulate_staged would launch for this shape under
 * the current arithmetic mode (host only, no GPU needed), for measurement and
 * roofline accounting:
 *   out[0] variant (1 = v1, 2 = v2), out[1] PP planes and out[2] DD diagonal
 *   entries per thread, out[3] Q planes and out[4] DR diagonal rows per CTA
 *   tile, out[5] shared-memory stages (0 for v1), out[6] target CTAs per SM,
 *   out[7] warps per CTA, out[8] 1 if the slice update is deferred to an L2
 *   reduction (G4_ARITH_FUSED, >= 4 walkers, >= 16 planes). */
g4_status g4_k1_config(int32_t n, int64_t planes, int32_t nbatch, int32_t dtype, int32_t* out);

/* Convenience form taking reference-layout payloads: prepares each batch into
 * `workspace` (>= g4_accumulate_workspace_bytes) then calls g4_accumulate_staged. */
int64_t g4_accumulate_workspace_bytes(int32_t n, int32_t nbatch, int32_t dtype);
g4_status g4_accumulate(void* g4, int64_t lo, int64_t hi, int32_t n, const void* const* up,
                        const void* const* down, int32_t nbatch, int32_t dtype,
                        int32_t channel, void* workspace, int64_t workspace_bytes,
                        void* stream);

/* ---- ring transport over CUDA peer memory (replaces the Communicator plugin's
 * isend/irecv payload path, ringacc/transport/base.py:53-80, for device
 * buffers).  Buffers are exported once with CUDA IPC; every ring step is a
 * copy-engine peer copy plus a 64-bit sequence flag written into the
 * receiver's memory (no SM cycles, no host round trip). ----------------------- */

#define G4_IPC_HANDLE_BYTES 64

/* Export a device pointer to other processes: the CUDA IPC handle of the
 * allocation containing it (G4_IPC_HANDLE_BYTES) and its byte offset inside
 * that allocation (pointers from a caching allocator are sub-allocations). */
g4_status g4_ipc_export(void* dev_ptr, void* handle_out, int64_t* offset_out);
/* Map an exported pointer into this process (reference counted per allocation;
 * works across GPUs over NVLink and between processes sharing one GPU). */
g4_status g4_ipc_import(const void* handle, int64_t offset, void** dev_ptr_out);
/* Release a pointer returned by g4_ipc_import. */
g4_status g4_ipc_close(void* dev_ptr);

/* Stream-ordered peer copy (copy engine over NVLink/NVSwitch, or local). */
g4_status g4_copy_async(void* dst, const void* src, int64_t bytes, void* stream);
/* Copies that fell back from the strided peer form to whole staged payloads
 * (a wire-format change, counted so a run can report it). */
int64_t g4_peer_copy_fallbacks(void);
/* The N x N cores (both spins) of `count` consecutive staged payloads, as one
 * strided peer copy: the ring's wire format.  The halo is not sent. */
g4_status g4_copy_payload_cores(void* dst, const void* src, int32_t count, int32_t n, int32_t dtype,
                                void* stream);
/* Rebuild the cyclic halo of staged payloads from their cores (the receiver
 * side of g4_copy_payload_cores). */
g4_status g4_fill_halo(void* const* staged, int32_t count, int32_t n, int32_t dtype, void* stream);
/* Load the kernels a ring launches behind stream flag waits (CUDA loads
 * kernels lazily at first launch, and a load cannot complete while the
 * context has a blocked stream).  Ring hosts call it once before their first
 * round; g4_ring_create does. */
g4_status g4_preload_ring_kernels(void);

/* Stream-ordered 64-bit flag write / wait (cuStreamWriteValue64 /
 * cuStreamWaitValue64 with GEQ).  `flag` may be a peer (IPC-mapped) address. */
g4_status g4_flag_write(void* flag, uint64_t value, void* stream);
g4_status g4_flag_wait(const void* flag, uint64_t value, void* stream);
/* Host-side poll of a device flag with timeout (deadlock detection,
 * replaces the recv timeout -> DeadlockError of inprocess.py:54-60).
 * Returns G4_ERR_DEADLOCK if *flag < value after timeout_ms. */
g4_status g4_flag_host_wait(const void* flag, uint64_t value, int64_t timeout_ms);

/* Canonical-order slice reduction over peer memory; replaces
 * Communicator.reduce_sum (transport/base.py:126-149): dst = src[0] + src[1] + ...
 * summed left to right per entry (rank order), count complex entries.
 * src[i] may be peer addresses; dst may alias src[0]. */
g4_status g4_reduce_sum(void* dst, const void* const* src, int32_t nsrc, int64_t count,
                        int32_t dtype, void* stream);

/* ---- native round program (replaces the per-op host loop of the reference's
 * run_measurement ring phase, engine.py:119-161, for the steady state).  A
 * round's op list is compiled once; g4_round_program_run(m) then issues every
 * K3/K1 launch, peer copy, flag write/wait and stream-event dependency of
 * round m in one host call.  Ops are G4_OP_WORDS int64 words each:
 *   {G4_OP_ACC,   stream, ptr_off, count}        K1 on ptrs[ptr_off .. +count)
 *   {G4_OP_WAIT,  stream, flag, base, slope}     wait flag >= base + slope*m
 *   {G4_OP_WRITE, stream, flag, base, slope}     write base + slope*m
 *   {G4_OP_COPY,  stream, dst, src, nbytes, count, n, dtype}
 *                                                peer copy: `nbytes` bytes, or (count > 0)
 *                                                the cores of `count` staged payloads
 *   {G4_OP_HALO,  stream, ptr_off, count}        g4_fill_halo on ptrs[ptr_off .. +count)
 *   {G4_OP_RECORD / G4_OP_WAIT_EVENT, stream, event}
 *   {G4_OP_GEN,   stream, ptr_off, count, meta_off}  K3 into ptrs with
 *       meta[meta_off ..] = world_rank[count], lane[count], meas_base[count];
 *       meas = meas_base + m * batch (skipped when regenerate == 0).
 * streams, events and ptrs are borrowed for the program's lifetime. */
#define G4_OP_WORDS 8
enum { G4_OP_ACC = 1, G4_OP_WAIT = 2, G4_OP_WRITE = 3, G4_OP_COPY = 4, G4_OP_RECORD = 5,
       G4_OP_WAIT_EVENT = 6, G4_OP_GEN = 7, G4_OP_HALO = 8 };
g4_status g4_round_program_create(const int64_t* ops, int32_t nops, void* const* ptrs, int32_t nptrs,
                                  const int64_t* meta, int32_t nmeta, void* const* streams, int32_t nstreams,
                                  void* const* events, int32_t nevents, void* g4, int64_t lo, int64_t hi, int32_t n, int32_t dtype,
                                  int32_t pdtype, uint64_t seed, int32_t mode, int64_t batch, int32_t timing,
                                  void** prog_out);
g4_status g4_round_program_run(void* prog, int64_t m, int32_t regenerate);
/* Mean duration of the K1 launches of the last completed round (timing programs). */
g4_status g4_round_program_k1_ms(void* prog, double* mean_ms, int32_t* count);
g4_status g4_round_program_destroy(void* prog);

/* ---- native ring driver (replaces ringacc/engine.py:119-161 run_measurement,
 * the slice assignment and sub-ring split of engine.py:241-255, and the final
 * reduce of engine.py:251,267 / transport/base.py:126-149) for hosts without
 * Python.  One ring object per rank (process or thread), one GPU per rank
 * (the caller selects the device before g4_ring_create).  The host supplies
 * the control plane as an all-gather callback: gather `bytes` bytes from every
 * member of `group` into recv (member order: sub-ring position for
 * G4_GROUP_SUBRING, sub-ring index for G4_GROUP_POSITION); return 0 on success.
 * The data path (payload copies, flags, K1/K3) never returns to the host. */
typedef enum { G4_GROUP_SUBRING = 0, G4_GROUP_POSITION = 1 } g4_group;
typedef int32_t (*g4_allgather_fn)(void* ctx, int32_t group, const void* send, int64_t bytes, void* recv);
typedef struct {
    int32_t n_k, n_w;       /* CombinedIndexSpace (tensor.py:31-47) */
    int32_t world_size;     /* ranks */
    int32_t subring_size;   /* S, divides world_size (engine.py:86-92) */
    int32_t lanes;          /* walker streams per rank (< 1000) */
    int32_t alternate;      /* 0: all lanes forward; 1: odd lanes run backward */
    int32_t batch;          /* measurements per lane per round (B); B * lanes <= G4_MAX_BATCH */
    int32_t dtype;          /* G4_C128, G4_C64 or G4_C128_G64 */
    int64_t planes;         /* exchange planes K3 in [0, planes); 0 = all N */
    int32_t value_mode;     /* G4_MODE_FLOAT / G4_MODE_INTEGER (synthetic walkers) */
    int32_t reserved;
    uint64_t seed;
} g4_ring_config;
g4_status g4_ring_create(const g4_ring_config* cfg, int32_t world_rank, g4_allgather_fn allgather, void* ctx,
                         void** ring);
/* Enqueue measurement round m (rounds are consecutive from 0): K3-generated
 * walkers (regenerate != 0) or the payloads already in GEN (g4_ring_stage). */
g4_status g4_ring_measure(void* ring, int64_t m, int32_t regenerate);
/* Stage host-fed reference-layout walkers (device pointers) into GEN: count =
 * batch x lanes, channel order, batch-major (engine.RingEngine.stage_gen). */
g4_status g4_ring_stage(void* ring, const void* const* up, const void* const* down, int32_t count,
                        int32_t dtype_in);
/* Host watchdog: all of this rank's streams drained within timeout_ms, else
 * G4_ERR_DEADLOCK naming (rank, lane, measurement, step) (inprocess.py:54-60). */
g4_status g4_ring_wait(void* ring, int64_t timeout_ms);
/* This rank's G4 slice (device memory, reference layout [k3-lo][k1][k2]). */
g4_status g4_ring_slice(void* ring, void** data, int64_t* lo, int64_t* hi);
/* Sum the slices of every sub-ring into sub-ring 0's, in sub-ring order
 * (collective over the position group). */
g4_status g4_ring_reduce(void* ring);
/* Collective over the sub-ring: drain, then free. */
g4_status g4_ring_destroy(void* ring);

#ifdef __cplusplus
}
#endif
#endif /* G4RING_H */
