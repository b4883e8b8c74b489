// g4_ring.cu -- device plumbing of the ring driver: CUDA IPC export/import of
// ring buffers, copy-engine peer copies, stream-ordered 64-bit sequence flags,
// and the canonical-order slice reduction over peer memory.
//
// Replaces the payload path of the reference's Communicator plugin
// (ringacc/transport/base.py:53-80: isend/irecv/PendingOp.wait) and its
// reduce_sum collective (base.py:126-149) for device-resident buffers.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda.h>
#include <nvtx3/nvToolsExt.h>

#include "g4_common.cuh"
#include "g4_internal.h"

namespace g4 {

// cuStreamWriteValue64 / cuStreamWaitValue64 fetched at run time through the
// runtime's driver entry point, so libg4ring.so has no link-time libcuda dep.
using PFN_write64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
using PFN_wait64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
using PFN_addr_range = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

static g4_status driver_fn(const char* name, void** fn) {
    cudaDriverEntryPointQueryResult q{};
    cudaError_t e = cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !*fn) {
        set_error("driver entry point %s unavailable (%s)", name, cudaGetErrorString(e));
        return G4_ERR_CUDA;
    }
    return G4_OK;
}

template <typename R>
struct RedParams {
    Cx<R>* dst;
    const Cx<R>* src[G4_MAX_BATCH];
    int32_t nsrc;
    int64_t count;
};

template <typename R>
__global__ void __launch_bounds__(256) k_reduce(const __grid_constant__ RedParams<R> P) {
    Cx<R>* dst = P.dst;
    const auto& src = P.src;
    const int nsrc = P.nsrc;
    const int64_t count = P.count;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        Cx<R> t = src[0][i];
        for (int s = 1; s < nsrc; ++s) {  // canonical rank order 0, 1, 2, ...
            const Cx<R> v = src[s][i];
            t.re = add_rn(t.re, v.re);
            t.im = add_rn(t.im, v.im);
        }
        dst[i] = t;
    }
}

}  // namespace g4

namespace g4 {
std::atomic<int64_t> g_peer_copy_fallbacks{0};  // see g4_copy_payload_cores
}

extern "C" {

// Exported pointers may lie inside a larger allocation (torch's caching
// allocator): the handle names the allocation, `offset` locates the pointer in it.
g4_status g4_ipc_export(void* dev_ptr, void* handle_out, int64_t* offset_out) {
    using namespace g4;
    if (!dev_ptr || !handle_out || !offset_out) return fail(G4_ERR_CONTRACT, "ipc_export: null pointer");
    static_assert(sizeof(cudaIpcMemHandle_t) == G4_IPC_HANDLE_BYTES, "IPC handle size");
    static PFN_addr_range range = nullptr;
    if (!range) G4_TRY(driver_fn("cuMemGetAddressRange", reinterpret_cast<void**>(&range)));
    CUdeviceptr base = 0;
    size_t size = 0;
    CUresult r = range(&base, &size, (CUdeviceptr)dev_ptr);
    if (r != CUDA_SUCCESS) {
        set_error("cuMemGetAddressRange failed (CUresult %d)", (int)r);
        return G4_ERR_CUDA;
    }
    cudaIpcMemHandle_t h;
    G4_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    std::memcpy(handle_out, &h, sizeof(h));
    *offset_out = (int64_t)((CUdeviceptr)dev_ptr - base);
    return G4_OK;
}

// Imports are reference counted per allocation: a process may map a given
// allocation only once, while several exported tensors can share it.
namespace {
struct Mapping {
    void* base;
    int refs;
};
std::mutex g_ipc_mu;
std::map<std::string, Mapping> g_by_handle;     // handle bytes -> mapping
std::map<uintptr_t, std::string> g_ptr_handle;  // returned pointer -> handle bytes
}  // namespace

g4_status g4_ipc_import(const void* handle, int64_t offset, void** dev_ptr_out) {
    using namespace g4;
    if (!handle || !dev_ptr_out || offset < 0) return fail(G4_ERR_CONTRACT, "ipc_import: bad arguments");
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    const std::string key(static_cast<const char*>(handle), G4_IPC_HANDLE_BYTES);
    auto it = g_by_handle.find(key);
    if (it == g_by_handle.end()) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        void* base = nullptr;
        G4_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
        it = g_by_handle.emplace(key, Mapping{base, 0}).first;
    }
    it->second.refs += 1;
    void* p = static_cast<char*>(it->second.base) + offset;
    g_ptr_handle[reinterpret_cast<uintptr_t>(p)] = key;
    *dev_ptr_out = p;
    return G4_OK;
}

g4_status g4_ipc_close(void* dev_ptr) {
    using namespace g4;
    if (!dev_ptr) return G4_OK;
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    auto pit = g_ptr_handle.find(reinterpret_cast<uintptr_t>(dev_ptr));
    if (pit == g_ptr_handle.end()) return fail(G4_ERR_CONTRACT, "ipc_close: pointer was not imported");
    auto it = g_by_handle.find(pit->second);
    g_ptr_handle.erase(pit);
    if (it != g_by_handle.end() && --it->second.refs == 0) {
        void* base = it->second.base;
        g_by_handle.erase(it);
        G4_CUDA(cudaIpcCloseMemHandle(base));
    }
    return G4_OK;
}

g4_status g4_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
    using namespace g4;
    if (bytes < 0 || ((!dst || !src) && bytes > 0)) return fail(G4_ERR_CONTRACT, "copy_async: bad args");
    if (bytes == 0) return G4_OK;
    G4_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice,
                            static_cast<cudaStream_t>(stream)));
    return G4_OK;
}

int64_t g4_peer_copy_fallbacks(void) { return g4::g_peer_copy_fallbacks.load(std::memory_order_relaxed); }

// The N x N cores of `count` consecutive staged payloads (both spins), as one
// strided copy-engine transfer: the halo (23 % of a payload at N = 512) never
// crosses NVLink; the receiver rebuilds it (g4_fill_halo).
g4_status g4_copy_payload_cores(void* dst, const void* src, int32_t count, int32_t n, int32_t dtype,
                                void* stream) {
    using namespace g4;
    if (!dst || !src || count < 0 || n < 1 || (dtype != G4_C128 && dtype != G4_C64))
        return fail(G4_ERR_CONTRACT, "copy_payload_cores: bad args");
    if (count == 0) return G4_OK;
    const size_t eb = entry_bytes(dtype);
    const size_t pitch = (size_t)staged_ld(n, (int)eb) * eb, rows = (size_t)staged_rows(n, (int)eb);
    const cudaPitchedPtr sp = make_cudaPitchedPtr(const_cast<void*>(src), pitch, (size_t)n * eb, rows);
    const cudaPitchedPtr dp = make_cudaPitchedPtr(dst, pitch, (size_t)n * eb, rows);
    const cudaExtent ext = make_cudaExtent((size_t)n * eb, (size_t)n, (size_t)2 * count);  // [walker, spin] planes
    // A peer on another GPU (IPC-mapped over NVLink) takes the explicit peer form.
    cudaPointerAttributes as{}, ad{};
    G4_CUDA(cudaPointerGetAttributes(&as, src));
    G4_CUDA(cudaPointerGetAttributes(&ad, dst));
    if (as.device != ad.device) {
        cudaMemcpy3DPeerParms p{};
        p.srcPtr = sp;
        p.srcDevice = as.device;
        p.dstPtr = dp;
        p.dstDevice = ad.device;
        p.extent = ext;
        if (cudaMemcpy3DPeerAsync(&p, static_cast<cudaStream_t>(stream)) != cudaSuccess) {
            // no strided peer copy here: move whole staged payloads (the halo
            // rebuild on the receiver is then a no-op rewrite).  Counted, so a run
            // that silently changed its wire format shows it (g4_peer_copy_fallbacks).
            cudaGetLastError();
            g_peer_copy_fallbacks.fetch_add(1, std::memory_order_relaxed);
            const int64_t bytes = (int64_t)2 * count * (int64_t)rows * (int64_t)pitch;
            G4_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice,
                                    static_cast<cudaStream_t>(stream)));
        }
    } else {
        cudaMemcpy3DParms p{};
        p.srcPtr = sp;
        p.dstPtr = dp;
        p.extent = ext;
        p.kind = cudaMemcpyDeviceToDevice;
        G4_CUDA(cudaMemcpy3DAsync(&p, static_cast<cudaStream_t>(stream)));
    }
    return G4_OK;
}

g4_status g4_flag_write(void* flag, uint64_t value, void* stream) {
    using namespace g4;
    static PFN_write64 fn = nullptr;
    if (!flag || !aligned(flag, 8)) return fail(G4_ERR_CONTRACT, "flag_write: bad flag pointer");
    if (!fn) G4_TRY(driver_fn("cuStreamWriteValue64", reinterpret_cast<void**>(&fn)));
    CUresult r = fn(static_cast<CUstream>(stream), (CUdeviceptr)flag, (cuuint64_t)value,
                    CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) {
        set_error("cuStreamWriteValue64 failed (CUresult %d)", (int)r);
        return G4_ERR_TRANSPORT;
    }
    return G4_OK;
}

g4_status g4_flag_wait(const void* flag, uint64_t value, void* stream) {
    using namespace g4;
    static PFN_wait64 fn = nullptr;
    if (!flag || !aligned(flag, 8)) return fail(G4_ERR_CONTRACT, "flag_wait: bad flag pointer");
    if (!fn) G4_TRY(driver_fn("cuStreamWaitValue64", reinterpret_cast<void**>(&fn)));
    // Where the device supports it, the wait also flushes outstanding remote
    // (NVLink peer) writes, so the payload that the flag announces is visible
    // to the K1 launch that follows on this stream.
    // (a device attribute: cached per device, the ring may drive several GPUs
    // from one process)
    static std::atomic<int> flush_by_dev[64];  // 0 unknown, 1 no, 2 yes
    int dev = 0;
    G4_CUDA(cudaGetDevice(&dev));
    int state = flush_by_dev[dev & 63].load(std::memory_order_relaxed);
    if (state == 0) {
        int v = 0;
        state = (cudaDeviceGetAttribute(&v, cudaDevAttrCanFlushRemoteWrites, dev) == cudaSuccess && v) ? 2 : 1;
        flush_by_dev[dev & 63].store(state, std::memory_order_relaxed);
    }
    const bool flush = state == 2;
    const unsigned int how = CU_STREAM_WAIT_VALUE_GEQ | (flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0u);
    CUresult r = fn(static_cast<CUstream>(stream), (CUdeviceptr)flag, (cuuint64_t)value, how);
    if (r != CUDA_SUCCESS) {
        set_error("cuStreamWaitValue64 failed (CUresult %d)", (int)r);
        return G4_ERR_TRANSPORT;
    }
    return G4_OK;
}

g4_status g4_flag_host_wait(const void* flag, uint64_t value, int64_t timeout_ms) {
    using namespace g4;
    if (!flag || !aligned(flag, 8)) return fail(G4_ERR_CONTRACT, "flag_host_wait: bad flag pointer");
    const auto t0 = std::chrono::steady_clock::now();
    uint64_t cur = 0;
    for (;;) {
        G4_CUDA(cudaMemcpy(&cur, flag, sizeof(cur), cudaMemcpyDeviceToHost));
        if (cur >= value) return G4_OK;
        const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(
                            std::chrono::steady_clock::now() - t0).count();
        if (ms >= timeout_ms) {
            set_error("flag wait timed out after %lld ms (have %llu, want %llu)", (long long)ms,
                      (unsigned long long)cur, (unsigned long long)value);
            return G4_ERR_DEADLOCK;
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
}

g4_status g4_reduce_sum(void* dst, const void* const* src, int32_t nsrc, int64_t count, int32_t dtype,
                        void* stream) {
    using namespace g4;
    if (nsrc < 1 || nsrc > G4_MAX_BATCH || count < 0 || !dst || !src)
        return fail(G4_ERR_CONTRACT, "reduce_sum: bad args");
    if (count == 0) return G4_OK;
    auto st = static_cast<cudaStream_t>(stream);
    for (int i = 0; i < nsrc; ++i)
        if (!src[i]) return fail(G4_ERR_CONTRACT, "reduce_sum: null source");
    const unsigned blocks = (unsigned)std::min<int64_t>((count + 255) / 256, 148 * 16);
    if (dtype == G4_C128) {
        RedParams<double> p{};
        p.dst = static_cast<Cx<double>*>(dst);
        for (int i = 0; i < nsrc; ++i) p.src[i] = static_cast<const Cx<double>*>(src[i]);
        p.nsrc = nsrc;
        p.count = count;
        k_reduce<double><<<blocks, 256, 0, st>>>(p);
    } else if (dtype == G4_C64) {
        RedParams<float> p{};
        p.dst = static_cast<Cx<float>*>(dst);
        for (int i = 0; i < nsrc; ++i) p.src[i] = static_cast<const Cx<float>*>(src[i]);
        p.nsrc = nsrc;
        p.count = count;
        k_reduce<float><<<blocks, 256, 0, st>>>(p);
    } else {
        return fail(G4_ERR_CONTRACT, "reduce_sum: unknown dtype");
    }
    G4_CUDA(cudaGetLastError());
    return G4_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Native round program: the per-op loop of engine.RingEngine.enqueue_round
// compiled once into a flat op list and replayed per round m with its flag
// values affine in m (value = base + slope * m).  One host call per round
// issues every K3/K1 launch, peer copy, flag write/wait and event of the
// round, so the host never limits a ring whose steps take tens of us.
namespace g4 {
struct RoundProgram {
    std::vector<int64_t> ops;      // nops x G4_OP_WORDS
    std::vector<void*> ptrs;       // staged payload pointer lists of K1/K3 ops
    std::vector<int64_t> meta;     // K3: world_rank, lane, meas_base per payload
    std::vector<cudaStream_t> streams;
    std::vector<cudaEvent_t> events;  // borrowed
    std::vector<cudaEvent_t> k1_ev;   // timing pairs per K1 op (timing programs only; owned)
    void* g4;
    int64_t lo, hi, batch;
    int32_t n, dtype, pdtype, mode;
    uint64_t seed;
    int n_acc;
};
}  // namespace g4

extern "C" {

g4_status g4_round_program_create(const int64_t* ops, int32_t nops, void* const* ptrs, int32_t nptrs,
                                  const int64_t* meta, int32_t nmeta, void* const* streams, int32_t nstreams,
                                  void* const* events, int32_t nevents, void* g4p, int64_t lo, int64_t hi, int32_t n, int32_t dtype,
                                  int32_t pdtype, uint64_t seed, int32_t mode, int64_t batch, int32_t timing,
                                  void** prog_out) {
    using namespace g4;
    if (!ops || nops < 1 || nptrs < 0 || nmeta < 0 || nstreams < 1 || !streams || nevents < 0 || !g4p ||
        !prog_out || (nptrs && !ptrs) || (nmeta && !meta) || (nevents && !events))
        return fail(G4_ERR_CONTRACT, "round_program_create: bad arguments");
    auto* P = new RoundProgram();
    P->ops.assign(ops, ops + (size_t)nops * G4_OP_WORDS);
    P->ptrs.assign(ptrs, ptrs + nptrs);
    P->meta.assign(meta, meta + nmeta);
    for (int i = 0; i < nstreams; ++i) P->streams.push_back(static_cast<cudaStream_t>(streams[i]));
    P->g4 = g4p;
    P->lo = lo;
    P->hi = hi;
    P->n = n;
    P->dtype = dtype;
    P->pdtype = pdtype;
    P->seed = seed;
    P->mode = mode;
    P->batch = batch;
    P->n_acc = 0;
    for (int i = 0; i < nops; ++i) {
        const int64_t* o = &P->ops[(size_t)i * G4_OP_WORDS];
        const int64_t kind = o[0], st = o[1];
        bool ok = st >= 0 && st < nstreams;
        if (kind == G4_OP_ACC || kind == G4_OP_GEN || kind == G4_OP_HALO)
            ok = ok && o[2] >= 0 && o[3] >= 1 && o[2] + o[3] <= nptrs;
        if (kind == G4_OP_GEN) ok = ok && o[4] >= 0 && o[4] + 3 * o[3] <= nmeta;
        if (kind == G4_OP_RECORD || kind == G4_OP_WAIT_EVENT) ok = ok && o[2] >= 0 && o[2] < nevents;
        if (kind < G4_OP_ACC || kind > G4_OP_HALO) ok = false;
        if (!ok) {
            delete P;
            set_error("round_program_create: malformed op %d (kind %lld)", i, (long long)kind);
            return G4_ERR_CONTRACT;
        }
        if (kind == G4_OP_ACC) ++P->n_acc;
    }
    for (int i = 0; i < nevents; ++i) {
        if (!events[i]) {
            delete P;
            return fail(G4_ERR_CONTRACT, "round_program_create: null event");
        }
        P->events.push_back(static_cast<cudaEvent_t>(events[i]));
    }
    if (timing) {
        for (int i = 0; i < 2 * P->n_acc; ++i) {
            cudaEvent_t e;
            cudaError_t err = cudaEventCreate(&e);
            if (err != cudaSuccess) {
                g4_round_program_destroy(P);
                return check_cuda(err, "cudaEventCreate");
            }
            P->k1_ev.push_back(e);
        }
    }
    *prog_out = P;
    return G4_OK;
}

g4_status g4_round_program_run(void* prog, int64_t m, int32_t regenerate) {
    using namespace g4;
    auto* P = static_cast<RoundProgram*>(prog);
    if (!P || m < 0) return fail(G4_ERR_CONTRACT, "round_program_run: bad arguments");
    // host-side range for nsys / Nsight timelines (no cost without a tool)
    struct Range {
        explicit Range(int64_t m) {
            char name[48];
            snprintf(name, sizeof(name), "g4 round %lld", (long long)m);
            nvtxRangePushA(name);
        }
        ~Range() { nvtxRangePop(); }
    } range(m);
    int acc = 0;
    std::vector<int64_t> meas;
    for (size_t i = 0; i < P->ops.size(); i += G4_OP_WORDS) {
        const int64_t* o = &P->ops[i];
        cudaStream_t st = P->streams[o[1]];
        switch (o[0]) {
            case G4_OP_GEN: {
                if (!regenerate) break;
                const int64_t cnt = o[3];
                const int64_t* md = &P->meta[o[4]];
                meas.resize(cnt);
                for (int64_t j = 0; j < cnt; ++j) meas[j] = md[2 * cnt + j] + m * P->batch;
                G4_TRY(g4_generate(&P->ptrs[o[2]], nullptr, nullptr, (int32_t)cnt, P->seed, md, md + cnt,
                                   meas.data(), P->n, P->mode, P->pdtype, st));
                break;
            }
            case G4_OP_ACC:
                if (!P->k1_ev.empty()) G4_CUDA(cudaEventRecord(P->k1_ev[2 * acc], st));
                G4_TRY(g4_accumulate_staged(P->g4, P->lo, P->hi, P->n, &P->ptrs[o[2]], (int32_t)o[3], P->dtype,
                                            G4_CHANNEL_EQ1, st));
                if (!P->k1_ev.empty()) G4_CUDA(cudaEventRecord(P->k1_ev[2 * acc + 1], st));
                ++acc;
                break;
            case G4_OP_WAIT:
                G4_TRY(g4_flag_wait(reinterpret_cast<void*>(o[2]), (uint64_t)(o[3] + o[4] * m), st));
                break;
            case G4_OP_WRITE:
                G4_TRY(g4_flag_write(reinterpret_cast<void*>(o[2]), (uint64_t)(o[3] + o[4] * m), st));
                break;
            case G4_OP_COPY:
                if (o[5] > 0)  // payload cores: count o[5], N o[6], dtype o[7]
                    G4_TRY(g4_copy_payload_cores(reinterpret_cast<void*>(o[2]), reinterpret_cast<const void*>(o[3]),
                                                 (int32_t)o[5], (int32_t)o[6], (int32_t)o[7], st));
                else
                    G4_TRY(g4_copy_async(reinterpret_cast<void*>(o[2]), reinterpret_cast<const void*>(o[3]), o[4], st));
                break;
            case G4_OP_HALO:
                G4_TRY(g4_fill_halo(&P->ptrs[o[2]], (int32_t)o[3], P->n, P->pdtype, st));
                break;
            case G4_OP_RECORD:
                G4_CUDA(cudaEventRecord(P->events[o[2]], st));
                break;
            case G4_OP_WAIT_EVENT:
                G4_CUDA(cudaStreamWaitEvent(st, P->events[o[2]], 0));
                break;
            default:
                return fail(G4_ERR_CONTRACT, "round_program_run: bad op");
        }
    }
    return G4_OK;
}

g4_status g4_round_program_k1_ms(void* prog, double* mean_ms, int32_t* count) {
    using namespace g4;
    auto* P = static_cast<RoundProgram*>(prog);
    if (!P || !mean_ms || !count) return fail(G4_ERR_CONTRACT, "round_program_k1_ms: bad arguments");
    *count = 0;
    *mean_ms = 0.0;
    if (P->k1_ev.empty()) return fail(G4_ERR_CONTRACT, "round_program_k1_ms: program created without timing");
    double sum = 0.0;
    for (int i = 0; i < P->n_acc; ++i) {
        float ms = 0.f;
        G4_CUDA(cudaEventElapsedTime(&ms, P->k1_ev[2 * i], P->k1_ev[2 * i + 1]));
        sum += ms;
    }
    *count = P->n_acc;
    *mean_ms = P->n_acc ? sum / P->n_acc : 0.0;
    return G4_OK;
}

g4_status g4_round_program_destroy(void* prog) {
    auto* P = static_cast<g4::RoundProgram*>(prog);
    if (!P) return G4_OK;
    for (cudaEvent_t e : P->k1_ev) cudaEventDestroy(e);
    delete P;
    return G4_OK;
}

}  // extern "C"
