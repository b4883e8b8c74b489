// g4_ring_driver.cu -- the ring driver behind the C ABI, for hosts without
// Python (cgo, JNI, C++).  Replaces the reference's per-rank ring phase
// run_measurement (ringacc/engine.py:119-161), its slice assignment and
// sub-ring split (engine.py:241-255) and the final position-group reduce
// (engine.py:251,267, transport/base.py:126-149).
//
// Same realisation as the Python engine (engine.py / schedule.py of this
// package): per channel (lanes sharing a direction) three staged payload
// buffers GEN, R0, R1 and three 64-bit flags DATA, ACK_ACC, ACK_FWD; round m,
// step j moves transfer k = 2 + m(S-1) + j into slot k % 2 of the right
// neighbour with a copy-engine peer copy of the payload cores, announced by a
// stream flag write; the receiver rebuilds the halo and runs K1 on the compute
// stream once DATA >= k.  The host supplies the control
// plane as an all-gather callback (rendezvous of IPC handles, barriers); the
// data path never returns to the host.  Ranks of the same process (threads)
// share pointers directly; other processes are reached through CUDA IPC.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <unistd.h>
#include <nvtx3/nvToolsExt.h>

#include "g4_internal.h"
#include "g4_layout.h"

namespace g4 {

enum { GEN_BUF = 0, R0_BUF = 1, R1_BUF = 2 };
enum { F_DATA = 0, F_ACK_ACC = 1, F_ACK_FWD = 2, FLAGS_PER_CH = 4 };
constexpr int64_t FIRST_TRANSFER = 2;

struct Chan {
    int index;
    std::vector<int> lanes;
    int recv_from, send_to;
};

// schedule.make_channels: lanes grouped by (recv_from, send_to), ordered by first lane.
static std::vector<Chan> make_channels(int S, int lanes, bool alternate, int pos) {
    std::vector<Chan> out;
    for (int t = 0; t < lanes; ++t) {
        int left = (pos - 1 + S) % S, right = (pos + 1) % S;
        if (alternate && (t % 2) == 1) std::swap(left, right);
        bool found = false;
        for (auto& c : out)
            if (c.recv_from == left && c.send_to == right) {
                c.lanes.push_back(t);
                found = true;
            }
        if (!found) out.push_back(Chan{(int)out.size(), {t}, left, right});
    }
    return out;
}

// Everything a rank publishes to its groups (fixed-size, memcpy-able).
struct Published {
    char flags_h[G4_IPC_HANDLE_BYTES];
    char bufs_h[2][G4_IPC_HANDLE_BYTES];
    char slice_h[G4_IPC_HANDLE_BYTES];
    int64_t flags_off, bufs_off[2], slice_off;
    uint64_t flags_ptr, bufs_ptr[2], slice_ptr;
    int64_t pid;
    int32_t nch, lanes_mask;
    int32_t device, reserved;  // CUDA ordinal of the allocations (same-process peers on other GPUs)
};

struct Ring {
    g4_ring_config cfg;
    int device = 0;            // every entry point runs on the ring's own GPU
    int world_rank, S, pos, subring, n;
    int64_t lo, hi, next_round;
    int pcode;                 // staged payload dtype
    bool wire_cores = true;    // cores on the wire + halo rebuild (G4RING_WIRE=staged: whole payloads)
    int64_t payload_bytes;     // one staged walker
    std::vector<Chan> chans;
    void* slice = nullptr;
    std::vector<void*> bufs;   // per channel: [3][B * lanes] payloads
    int64_t* flags = nullptr;  // per channel FLAGS_PER_CH words
    cudaStream_t compute = nullptr;
    std::vector<cudaStream_t> comm;
    cudaEvent_t ev_gen = nullptr;
    std::vector<cudaEvent_t> ev_sent;
    std::vector<uint64_t> peer_flags;     // by sub-ring position
    std::vector<uint64_t> peer_bufs;      // by channel: the right neighbour's buffers
    std::vector<void*> imported;          // to close
    g4_allgather_fn allgather = nullptr;
    void* ctx = nullptr;
    std::vector<Published> members;       // sub-ring, by position

    int64_t slot_bytes(const Chan& c) const { return (int64_t)cfg.batch * (int64_t)c.lanes.size() * payload_bytes; }
    char* buf(const Chan& c, int which) const {
        return static_cast<char*>(bufs[c.index]) + (int64_t)which * slot_bytes(c);
    }
};

static g4_status gather(Ring* R, int32_t group, const void* in, int64_t bytes, void* out) {
    const int32_t rc = R->allgather(R->ctx, group, in, bytes, out);
    if (rc != 0) {
        set_error("ring control plane: allgather (group %d) failed with %d", group, rc);
        return G4_ERR_TRANSPORT;
    }
    return G4_OK;
}

static g4_status barrier(Ring* R, int32_t group, int members) {
    const char one = 1;
    std::vector<char> all(members);
    return gather(R, group, &one, 1, all.data());
}

// Direct access from this rank's GPU to allocations on `peer` (same process,
// another GPU): the copy engines' peer copies need it, and so do the flag
// writes and the reduce kernel's loads through the raw pointers.
static g4_status enable_peer(int self, int peer) {
    if (peer == self) return G4_OK;
    int can = 0;
    G4_CUDA(cudaDeviceCanAccessPeer(&can, self, peer));
    if (!can) {
        set_error("GPU %d cannot access GPU %d directly (no peer path)", self, peer);
        return G4_ERR_TRANSPORT;
    }
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return G4_OK;
    }
    return check_cuda(e, "cudaDeviceEnablePeerAccess");
}

// Peer pointer of a published allocation: direct within this process (with peer
// access enabled when it lives on another GPU), else CUDA IPC.
static g4_status peer_ptr(Ring* R, const Published& p, const char* handle, int64_t off, uint64_t ptr,
                          uint64_t* out) {
    if (p.pid == (int64_t)getpid()) {
        G4_TRY(enable_peer(R->device, p.device));
        *out = ptr;
        return G4_OK;
    }
    void* q = nullptr;
    G4_TRY(g4_ipc_import(handle, off, &q));
    R->imported.push_back(q);
    *out = reinterpret_cast<uint64_t>(q);
    return G4_OK;
}

static g4_status publish(void* ptr, char* h, int64_t* off, uint64_t* raw) {
    *raw = reinterpret_cast<uint64_t>(ptr);
    return g4_ipc_export(ptr, h, off);
}

static void release(Ring* R) {
    if (R->compute) cudaStreamSynchronize(R->compute);
    for (cudaStream_t s : R->comm) cudaStreamSynchronize(s);
    for (void* q : R->imported) g4_ipc_close(q);
    if (R->ev_gen) cudaEventDestroy(R->ev_gen);
    for (cudaEvent_t e : R->ev_sent) cudaEventDestroy(e);
    if (R->compute) cudaStreamDestroy(R->compute);
    for (cudaStream_t s : R->comm) cudaStreamDestroy(s);
    for (void* b : R->bufs) cudaFree(b);
    if (R->flags) cudaFree(R->flags);
    if (R->slice) cudaFree(R->slice);
    delete R;
}

}  // namespace g4

extern "C" {

g4_status g4_ring_create(const g4_ring_config* cfg, int32_t world_rank, g4_allgather_fn allgather, void* ctx,
                         void** ring_out) {
    using namespace g4;
    if (!cfg || !allgather || !ring_out) return fail(G4_ERR_CONTRACT, "ring_create: null argument");
    const int64_t n = (int64_t)cfg->n_k * cfg->n_w;
    if (cfg->n_k < 1 || cfg->n_w < 1) return fail(G4_ERR_CONFIG, "n_k and n_w must be >= 1");
    if (cfg->subring_size < 1 || cfg->world_size < 1 || cfg->world_size % cfg->subring_size)
        return fail(G4_ERR_CONFIG, "subring size must divide the world size");
    if (cfg->lanes < 1 || cfg->lanes >= 1000) return fail(G4_ERR_CONFIG, "lane count must be in [1, 1000)");
    if (cfg->batch < 1 || (int64_t)cfg->batch * cfg->lanes > G4_MAX_BATCH)
        return fail(G4_ERR_CONFIG, "batch x lanes must be in [1, G4_MAX_BATCH]");
    const int64_t planes = cfg->planes ? cfg->planes : n;
    if (planes < cfg->subring_size || planes > n) return fail(G4_ERR_CONFIG, "need subring_size <= planes <= N");
    if (world_rank < 0 || world_rank >= cfg->world_size) return fail(G4_ERR_CONTRACT, "world rank out of range");
    if (cfg->dtype != G4_C128 && cfg->dtype != G4_C64 && cfg->dtype != G4_C128_G64)
        return fail(G4_ERR_CONFIG, "unknown dtype");
    if (cfg->value_mode != G4_MODE_FLOAT && cfg->value_mode != G4_MODE_INTEGER)
        return fail(G4_ERR_CONFIG, "unknown value mode");

    G4_TRY(g4_preload_ring_kernels());
    auto* R = new Ring();
    if (cudaGetDevice(&R->device) != cudaSuccess) {
        delete R;
        return fail(G4_ERR_CUDA, "ring_create: no current CUDA device");
    }
    R->cfg = *cfg;
    R->cfg.planes = planes;
    R->world_rank = world_rank;
    R->S = cfg->subring_size;
    R->pos = world_rank % R->S;
    R->subring = world_rank / R->S;
    R->n = (int)n;
    R->next_round = 0;
    R->allgather = allgather;
    R->ctx = ctx;
    R->pcode = cfg->dtype == G4_C128 ? G4_C128 : G4_C64;
    R->payload_bytes = g4_payload_bytes(R->n, R->pcode);
    {
        const char* wire = getenv("G4RING_WIRE");
        R->wire_cores = !(wire && std::strcmp(wire, "staged") == 0);
    }
    std::vector<int64_t> ranges(2 * R->S);
    g4_status st = g4_make_partition(planes, R->S, ranges.data());
    if (st != G4_OK) {
        delete R;
        return st;
    }
    R->lo = ranges[2 * R->pos];
    R->hi = ranges[2 * R->pos + 1];
    R->chans = make_channels(R->S, cfg->lanes, cfg->alternate != 0, R->pos);
    if (R->chans.size() > 2) {
        delete R;
        return fail(G4_ERR_CONFIG, "at most two ring directions");
    }

#define RING_CUDA(expr)                                  \
    do {                                                 \
        cudaError_t _e = (expr);                         \
        if (_e != cudaSuccess) {                         \
            release(R);                                  \
            return check_cuda(_e, #expr);                \
        }                                                \
    } while (0)
#define RING_TRY(expr)             \
    do {                           \
        g4_status _s = (expr);     \
        if (_s != G4_OK) {         \
            release(R);            \
            return _s;             \
        }                          \
    } while (0)

    const int64_t eb = cfg->dtype == G4_C64 ? 8 : 16;
    const size_t slice_bytes = (size_t)(R->hi - R->lo) * n * n * eb;
    RING_CUDA(cudaMalloc(&R->slice, slice_bytes));
    RING_CUDA(cudaMemset(R->slice, 0, slice_bytes));
    for (const Chan& c : R->chans) {
        void* b = nullptr;
        RING_CUDA(cudaMalloc(&b, 3 * R->slot_bytes(c)));
        RING_CUDA(cudaMemset(b, 0, 3 * R->slot_bytes(c)));
        R->bufs.push_back(b);
    }
    RING_CUDA(cudaMalloc(&R->flags, R->chans.size() * FLAGS_PER_CH * sizeof(int64_t)));
    RING_CUDA(cudaMemset(R->flags, 0, R->chans.size() * FLAGS_PER_CH * sizeof(int64_t)));
    RING_CUDA(cudaStreamCreateWithFlags(&R->compute, cudaStreamNonBlocking));
    for (size_t i = 0; i < R->chans.size(); ++i) {
        cudaStream_t s;
        RING_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        R->comm.push_back(s);
        cudaEvent_t e;
        RING_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        R->ev_sent.push_back(e);
    }
    RING_CUDA(cudaEventCreateWithFlags(&R->ev_gen, cudaEventDisableTiming));
    RING_CUDA(cudaDeviceSynchronize());

    // publish flags / buffers / slice to the sub-ring, connect to the neighbours
    Published me{};
    me.pid = (int64_t)getpid();
    me.device = R->device;
    me.nch = (int32_t)R->chans.size();
    RING_TRY(publish(R->flags, me.flags_h, &me.flags_off, &me.flags_ptr));
    for (size_t i = 0; i < R->chans.size(); ++i)
        RING_TRY(publish(R->bufs[i], me.bufs_h[i], &me.bufs_off[i], &me.bufs_ptr[i]));
    RING_TRY(publish(R->slice, me.slice_h, &me.slice_off, &me.slice_ptr));
    R->members.resize(R->S);
    RING_TRY(gather(R, G4_GROUP_SUBRING, &me, sizeof(me), R->members.data()));
    R->peer_flags.assign(R->S, 0);
    for (const Chan& c : R->chans) {
        for (int p : {c.recv_from, c.send_to}) {
            if (R->peer_flags[p]) continue;
            const Published& q = R->members[p];
            if (p == R->pos)
                R->peer_flags[p] = reinterpret_cast<uint64_t>(R->flags);
            else
                RING_TRY(peer_ptr(R, q, q.flags_h, q.flags_off, q.flags_ptr, &R->peer_flags[p]));
        }
        const Published& q = R->members[c.send_to];
        if (q.nch != (int32_t)R->chans.size()) {
            release(R);
            return fail(G4_ERR_CONTRACT, "neighbouring ranks disagree on the channel layout");
        }
        uint64_t pb = 0;
        if (c.send_to == R->pos)
            pb = reinterpret_cast<uint64_t>(R->bufs[c.index]);
        else
            RING_TRY(peer_ptr(R, q, q.bufs_h[c.index], q.bufs_off[c.index], q.bufs_ptr[c.index], &pb));
        R->peer_bufs.push_back(pb);
    }
#undef RING_CUDA
#undef RING_TRY
    *ring_out = R;
    return G4_OK;
}

// One round (schedule.round_schedule, issued directly).
g4_status g4_ring_measure(void* ring, int64_t m, int32_t regenerate) {
    using namespace g4;
    auto* R = static_cast<Ring*>(ring);
    if (!R) return fail(G4_ERR_CONTRACT, "ring_measure: null ring");
    G4_CUDA(cudaSetDevice(R->device));
    if (m != R->next_round) {
        set_error("rounds must be consecutive: expected %lld, got %lld", (long long)R->next_round, (long long)m);
        return G4_ERR_CONTRACT;
    }
    R->next_round = m + 1;
    nvtxRangePushA("g4 ring round");
    struct Pop {
        ~Pop() { nvtxRangePop(); }
    } pop;
    const int S = R->S, B = R->cfg.batch;
    const int64_t steps = S - 1;
    auto flag = [&](int pos, int ci, int f) {
        return reinterpret_cast<void*>(R->peer_flags[pos] + (uint64_t)(ci * FLAGS_PER_CH + f) * 8);
    };
    auto own_flag = [&](int ci, int f) { return static_cast<void*>(R->flags + ci * FLAGS_PER_CH + f); };
    auto k1 = [&](std::vector<const void*>& ptrs) {
        return g4_accumulate_staged(R->slice, R->lo, R->hi, R->n, ptrs.data(), (int32_t)ptrs.size(), R->cfg.dtype,
                                    G4_CHANNEL_EQ1, R->compute);
    };
    if (m > 0 && steps > 0)
        for (const Chan& c : R->chans) G4_CUDA(cudaStreamWaitEvent(R->compute, R->ev_sent[c.index], 0));
    if (regenerate) {  // K3 into GEN, channel order, batch-major (engine.enqueue_round)
        std::vector<void*> ptrs;
        std::vector<int64_t> wr, lane, meas;
        for (const Chan& c : R->chans)
            for (int b = 0; b < B; ++b)
                for (size_t li = 0; li < c.lanes.size(); ++li) {
                    ptrs.push_back(R->buf(c, GEN_BUF) + (int64_t)(b * c.lanes.size() + li) * R->payload_bytes);
                    wr.push_back(R->world_rank);
                    lane.push_back(c.lanes[li]);
                    meas.push_back(m * B + b);
                }
        G4_TRY(g4_generate(ptrs.data(), nullptr, nullptr, (int32_t)ptrs.size(), R->cfg.seed, wr.data(), lane.data(),
                           meas.data(), R->n, R->cfg.value_mode, R->pcode, R->compute));
    }
    if (steps > 0) G4_CUDA(cudaEventRecord(R->ev_gen, R->compute));
    std::vector<const void*> ptrs;
    auto add_slot = [&](const Chan& c, int which) {
        for (int i = 0; i < B * (int)c.lanes.size(); ++i)
            ptrs.push_back(R->buf(c, which) + (int64_t)i * R->payload_bytes);
    };
    for (const Chan& c : R->chans) add_slot(c, GEN_BUF);
    G4_TRY(k1(ptrs));
    for (int64_t j = 0; j < steps; ++j) {
        const int64_t k = FIRST_TRANSFER + m * (S - 1) + j;
        for (const Chan& c : R->chans) {
            cudaStream_t cs = R->comm[c.index];
            if (k - 2 >= FIRST_TRANSFER) {  // the slot held transfer k-2: accumulated and forwarded?
                G4_TRY(g4_flag_wait(own_flag(c.index, F_ACK_ACC), (uint64_t)(k - 2), cs));
                G4_TRY(g4_flag_wait(own_flag(c.index, F_ACK_FWD), (uint64_t)(k - 2), cs));
            }
            int src;
            if (j == 0) {
                G4_CUDA(cudaStreamWaitEvent(cs, R->ev_gen, 0));
                src = GEN_BUF;
            } else {
                G4_TRY(g4_flag_wait(own_flag(c.index, F_DATA), (uint64_t)(k - 1), cs));
                src = R0_BUF + (int)((k - 1) % 2);
            }
            char* dst = reinterpret_cast<char*>(R->peer_bufs[c.index]) + (R0_BUF + k % 2) * R->slot_bytes(c);
            if (R->wire_cores)
                G4_TRY(g4_copy_payload_cores(dst, R->buf(c, src), B * (int32_t)c.lanes.size(), R->n, R->pcode, cs));
            else
                G4_TRY(g4_copy_async(dst, R->buf(c, src), R->slot_bytes(c), cs));
            G4_TRY(g4_flag_write(flag(c.send_to, c.index, F_DATA), (uint64_t)k, cs));
            if (j == 0) G4_CUDA(cudaEventRecord(R->ev_sent[c.index], cs));
            if (j >= 1) G4_TRY(g4_flag_write(flag(c.recv_from, c.index, F_ACK_FWD), (uint64_t)(k - 1), cs));
            if (j == steps - 1) G4_TRY(g4_flag_write(flag(c.recv_from, c.index, F_ACK_FWD), (uint64_t)k, cs));
        }
        for (const Chan& c : R->chans) G4_TRY(g4_flag_wait(own_flag(c.index, F_DATA), (uint64_t)k, R->compute));
        ptrs.clear();
        for (const Chan& c : R->chans) add_slot(c, R0_BUF + (int)(k % 2));
        std::vector<void*> halo(ptrs.size());  // only the cores crossed the link
        for (size_t i = 0; i < ptrs.size(); ++i) halo[i] = const_cast<void*>(ptrs[i]);
        if (R->wire_cores) G4_TRY(g4_fill_halo(halo.data(), (int32_t)halo.size(), R->n, R->pcode, R->compute));
        G4_TRY(k1(ptrs));
        for (const Chan& c : R->chans)
            G4_TRY(g4_flag_write(flag(c.recv_from, c.index, F_ACK_ACC), (uint64_t)k, R->compute));
    }
    return G4_OK;
}

g4_status g4_ring_stage(void* ring, const void* const* up, const void* const* down, int32_t count,
                        int32_t dtype_in) {
    using namespace g4;
    auto* R = static_cast<Ring*>(ring);
    if (!R || !up || !down) return fail(G4_ERR_CONTRACT, "ring_stage: null argument");
    G4_CUDA(cudaSetDevice(R->device));
    std::vector<void*> ptrs;
    for (const Chan& c : R->chans)
        for (int i = 0; i < R->cfg.batch * (int)c.lanes.size(); ++i)
            ptrs.push_back(R->buf(c, GEN_BUF) + (int64_t)i * R->payload_bytes);
    if (count != (int32_t)ptrs.size()) {
        set_error("ring_stage: expected %d payloads, got %d", (int)ptrs.size(), count);
        return G4_ERR_CONTRACT;
    }
    // GEN still holds the previous round's payloads until their first ring copy
    // has left (ev_sent, recorded on the comm stream): a slow neighbour keeps the
    // comm stream waiting on ACK flags while the compute stream would run ahead
    // (the same edge as g4_ring_measure's, and engine.RingEngine.stage_gen's).
    if (R->next_round > 0 && R->S > 1)
        for (const Chan& c : R->chans) G4_CUDA(cudaStreamWaitEvent(R->compute, R->ev_sent[c.index], 0));
    return g4_prepare_g(ptrs.data(), up, down, count, R->n, dtype_in, R->pcode, R->compute);
}

g4_status g4_ring_wait(void* ring, int64_t timeout_ms) {
    using namespace g4;
    auto* R = static_cast<Ring*>(ring);
    if (!R) return fail(G4_ERR_CONTRACT, "ring_wait: null ring");
    G4_CUDA(cudaSetDevice(R->device));
    std::vector<cudaStream_t> all = R->comm;
    all.push_back(R->compute);
    const auto t0 = std::chrono::steady_clock::now();
    for (cudaStream_t s : all) {
        for (;;) {
            cudaError_t e = cudaStreamQuery(s);
            if (e == cudaSuccess) break;
            if (e != cudaErrorNotReady) return check_cuda(e, "ring_wait");
            const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(
                                std::chrono::steady_clock::now() - t0).count();
            if (ms >= timeout_ms) {
                // diagnose from the DATA flags, then unblock the streams so the
                // process can tear down (engine.RingEngine._raise_deadlock)
                std::vector<int64_t> v(R->chans.size() * FLAGS_PER_CH);
                cudaMemcpy(v.data(), R->flags, v.size() * 8, cudaMemcpyDeviceToHost);
                // the channel whose DATA flag lags the most is the stalled one
                const Chan* lag = &R->chans[0];
                for (const Chan& c : R->chans)
                    if (v[c.index * FLAGS_PER_CH + F_DATA] < v[lag->index * FLAGS_PER_CH + F_DATA]) lag = &c;
                const Chan& c = *lag;
                const int64_t landed = v[c.index * FLAGS_PER_CH + F_DATA];
                const int64_t k = std::max<int64_t>(landed + 1, FIRST_TRANSFER);
                const int64_t per = std::max(R->S - 1, 1);
                const int64_t mm = (k - FIRST_TRANSFER) / per, j = (k - FIRST_TRANSFER) % per;
                std::vector<int64_t> big(v.size(), (int64_t)1 << 62);
                cudaMemcpy(R->flags, big.data(), big.size() * 8, cudaMemcpyHostToDevice);
                set_error("rank %d lane %d stalled at measurement %lld step %lld: no payload from rank %d",
                          R->world_rank, c.lanes[0], (long long)(mm * R->cfg.batch), (long long)j,
                          R->subring * R->S + c.recv_from);
                return G4_ERR_DEADLOCK;
            }
            std::this_thread::sleep_for(std::chrono::microseconds(200));
        }
    }
    return G4_OK;
}

g4_status g4_ring_slice(void* ring, void** data, int64_t* lo, int64_t* hi) {
    using namespace g4;
    auto* R = static_cast<Ring*>(ring);
    if (!R || !data || !lo || !hi) return fail(G4_ERR_CONTRACT, "ring_slice: null argument");
    *data = R->slice;
    *lo = R->lo;
    *hi = R->hi;
    return G4_OK;
}

// Position-group reduce: every sub-ring's slice of this position is summed, in
// sub-ring order, into the slice of sub-ring 0 (canonical order of
// transport/base.py:126-149).  Collective over the position group.
g4_status g4_ring_reduce(void* ring) {
    using namespace g4;
    auto* R = static_cast<Ring*>(ring);
    if (!R) return fail(G4_ERR_CONTRACT, "ring_reduce: null ring");
    G4_CUDA(cudaSetDevice(R->device));
    const int groups = R->cfg.world_size / R->S;
    if (groups == 1) return G4_OK;
    G4_CUDA(cudaStreamSynchronize(R->compute));
    std::vector<Published> pg(groups);
    Published me = R->members[R->pos];
    G4_TRY(gather(R, G4_GROUP_POSITION, &me, sizeof(me), pg.data()));
    if (R->subring == 0) {
        std::vector<const void*> src;
        std::vector<void*> opened;
        src.push_back(R->slice);
        g4_status st = G4_OK;
        for (int g = 1; g < groups && st == G4_OK; ++g) {
            const Published& q = pg[g];
            if (q.pid == (int64_t)getpid()) {
                st = enable_peer(R->device, q.device);
                src.push_back(reinterpret_cast<const void*>(q.slice_ptr));
            } else {
                void* p = nullptr;
                st = g4_ipc_import(q.slice_h, q.slice_off, &p);
                if (st == G4_OK) {
                    opened.push_back(p);
                    src.push_back(p);
                }
            }
        }
        const int64_t count = (R->hi - R->lo) * (int64_t)R->n * R->n;
        if (st == G4_OK)
            st = g4_reduce_sum(R->slice, src.data(), (int32_t)src.size(), count,
                               R->cfg.dtype == G4_C64 ? G4_C64 : G4_C128, R->compute);
        cudaStreamSynchronize(R->compute);
        for (void* p : opened) g4_ipc_close(p);
        if (st != G4_OK) return st;
    }
    return barrier(R, G4_GROUP_POSITION, groups);  // peers keep their slices until the root has read them
}

g4_status g4_ring_destroy(void* ring) {
    using namespace g4;
    auto* R = static_cast<Ring*>(ring);
    if (!R) return G4_OK;
    cudaSetDevice(R->device);
    cudaStreamSynchronize(R->compute);
    for (cudaStream_t s : R->comm) cudaStreamSynchronize(s);
    // nobody may still be copying into (or reading) our buffers
    g4_status st = barrier(R, G4_GROUP_SUBRING, R->S);
    release(R);
    return st;
}

}  // extern "C"
