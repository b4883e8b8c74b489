// tests/native/ring_threads.cpp -- a C++ host of the native ring driver (no
// Python anywhere): every rank is a thread of this process -- on one GPU, or
// spread over every visible GPU (same-process peers on other devices: the
// driver enables peer access) -- and the control plane is an in-process
// all-gather.  The "fed" mode stages reference-layout walkers from the host
// every round (g4_ring_stage) with rank 0 deliberately delayed, the case where
// a stage could overwrite GEN before the previous round's payload left.  The reduced G4 (sub-ring 0's
// slices) is checked bitwise against the C oracle (integer mode), i.e. against
// the reference's serial sum over every walker of every lane and sub-ring.
// TEST CODE: links the oracle (oracle/g4_oracle.c) as the checker.
//
// build: nvcc -std=c++17 -I include tests/native/ring_threads.cpp oracle/g4_oracle.c \
//          -L paper_2105_00027_b200 -lg4ring -Xlinker -rpath=paper_2105_00027_b200 -o ring_threads
// run:   ./ring_threads [world] [subring] [lanes] [alternate] [batch] [rounds] [devices] [fed] [delay_ms]
//        devices: 1 = all ranks on GPU 0, 0 = round-robin over every visible GPU
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <chrono>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "g4ring.h"

extern "C" {
void g4o_fill_gsigma(uint64_t seed, int64_t world_rank, int64_t lane, int64_t meas, int32_t n, int32_t mode,
                     double* up, double* down);
void g4o_accumulate(double* g4, int64_t lo, int64_t hi, int32_t n, const double* up, const double* down);
}

// All-gather among the members of one group (a sub-ring or a position group).
struct Group {
    int size;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0, generation = 0;
    std::vector<char> buf;
    explicit Group(int s) : size(s) {}
    void wait_all(std::unique_lock<std::mutex>& lk) {
        const int gen = generation;
        if (++arrived == size) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
    void allgather(int index, const void* send, int64_t bytes, void* recv) {
        std::unique_lock<std::mutex> lk(mu);
        if ((int64_t)buf.size() < bytes * size) buf.resize(bytes * size);
        wait_all(lk);  // nobody still reads the previous result
        std::memcpy(buf.data() + index * bytes, send, bytes);
        wait_all(lk);
        std::memcpy(recv, buf.data(), bytes * size);
    }
};

struct RankCtx {
    Group* groups[2];
    int index[2];
};

static int32_t allgather(void* ctx, int32_t group, const void* send, int64_t bytes, void* recv) {
    auto* c = static_cast<RankCtx*>(ctx);
    c->groups[group]->allgather(c->index[group], send, bytes, recv);
    return 0;
}

#define CHECK(x)                                                                               \
    do {                                                                                       \
        g4_status _s = (x);                                                                    \
        if (_s != G4_OK) {                                                                     \
            std::fprintf(stderr, "%s failed: %d (%s)\n", #x, (int)_s, g4_last_error());        \
            std::exit(1);                                                                      \
        }                                                                                      \
    } while (0)

int main(int argc, char** argv) {
    // Several ranks (threads) share one CUDA context here, each with a compute
    // stream, its comm streams and a copy stream; the flag waits are stream
    // memops that block their hardware queue.  With more streams than queues
    // (CUDA_DEVICE_MAX_CONNECTIONS, default 8) two ranks' streams can share a
    // queue, and a wait at its head holds back the other rank's work that would
    // satisfy it.  One queue per stream: set before the context exists.
    setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);
    const int world = argc > 1 ? std::atoi(argv[1]) : 4;
    const int S = argc > 2 ? std::atoi(argv[2]) : 2;
    const int lanes = argc > 3 ? std::atoi(argv[3]) : 2;
    const int alternate = argc > 4 ? std::atoi(argv[4]) : 1;
    const int batch = argc > 5 ? std::atoi(argv[5]) : 2;
    const int rounds = argc > 6 ? std::atoi(argv[6]) : 3;
    const int one_gpu = argc > 7 ? std::atoi(argv[7]) : 1;
    const int fed = argc > 8 ? std::atoi(argv[8]) : 0;
    const int delay_ms = argc > 9 ? std::atoi(argv[9]) : 0;
    int ngpu = 1;
    if (!one_gpu && cudaGetDeviceCount(&ngpu) != cudaSuccess) ngpu = 1;
    if (fed && alternate) {
        std::fprintf(stderr, "fed mode stages one channel (alternate = 0)\n");
        return 1;
    }
    g4_ring_config cfg{};
    cfg.n_k = 4;
    cfg.n_w = 8;
    cfg.world_size = world;
    cfg.subring_size = S;
    cfg.lanes = lanes;
    cfg.alternate = alternate;
    cfg.batch = batch;
    cfg.dtype = G4_C128;
    cfg.planes = 0;
    cfg.value_mode = G4_MODE_INTEGER;
    cfg.seed = 7;
    const int n = cfg.n_k * cfg.n_w;
    const int subrings = world / S;

    std::vector<Group*> sub, pos;
    for (int g = 0; g < subrings; ++g) sub.push_back(new Group(S));
    for (int p = 0; p < S; ++p) pos.push_back(new Group(subrings));
    std::vector<std::vector<double>> result(S);  // sub-ring 0 slices after the reduce
    std::vector<int64_t> los(S), his(S);

    // host-fed inputs: per rank, rounds x (batch x lanes) reference-layout walkers
    std::vector<std::vector<void*>> ups(world), downs(world);
    if (fed)
        for (int r = 0; r < world; ++r) {
            cudaSetDevice(r % ngpu);
            for (int i = 0; i < batch * lanes * rounds; ++i) {
                void *u, *d;
                cudaMalloc(&u, (size_t)n * n * 16);
                cudaMalloc(&d, (size_t)n * n * 16);
                ups[r].push_back(u);
                downs[r].push_back(d);
            }
        }

    std::vector<std::thread> threads;
    for (int r = 0; r < world; ++r) {
        threads.emplace_back([&, r] {
            cudaSetDevice(r % ngpu);
            RankCtx ctx{{sub[r / S], pos[r % S]}, {r % S, r / S}};
            void* ring = nullptr;
            CHECK(g4_ring_create(&cfg, r, allgather, &ctx, &ring));
            if (!fed) {
                for (int m = 0; m < rounds; ++m) CHECK(g4_ring_measure(ring, m, 1));
            } else {
                // host-fed: reference-layout walkers staged every round (one channel:
                // batch-major, lanes in order), rank 0 late on every round; no wait
                // between rounds, so the other ranks stage round m + 1 while their
                // comm streams still wait for rank 0 to take round m
                // Device inputs are allocated before the ring starts and freed after
                // every thread has joined (main): cudaFree synchronises the device,
                // and the other ranks' streams sit in flag waits on rank 0 until it
                // stages.  Copies go through a non-blocking stream of this thread.
                const int cnt = batch * lanes;
                std::vector<double> hu((size_t)n * n * 2), hd((size_t)n * n * 2);
                std::vector<void*>& du = ups[r];
                std::vector<void*>& dd = downs[r];
                cudaStream_t cp;
                cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking);
                for (int m = 0; m < rounds; ++m) {
                    if (r == 0 && delay_ms) std::this_thread::sleep_for(std::chrono::milliseconds(delay_ms));
                    for (int b = 0; b < batch; ++b)
                        for (int t = 0; t < lanes; ++t) {
                            g4o_fill_gsigma(cfg.seed, r, t, (int64_t)m * batch + b, n, G4_MODE_INTEGER, hu.data(),
                                            hd.data());
                            const size_t i = (size_t)m * cnt + b * lanes + t;  // per-round buffers
                            cudaMemcpyAsync(du[i], hu.data(), hu.size() * 8, cudaMemcpyHostToDevice, cp);
                            cudaMemcpyAsync(dd[i], hd.data(), hd.size() * 8, cudaMemcpyHostToDevice, cp);
                            cudaStreamSynchronize(cp);
                        }
                    CHECK(g4_ring_stage(ring, du.data() + (size_t)m * cnt, dd.data() + (size_t)m * cnt, cnt,
                                        G4_C128));
                    CHECK(g4_ring_measure(ring, m, 0));
                }
                CHECK(g4_ring_wait(ring, 60000));
                cudaStreamDestroy(cp);
            }
            CHECK(g4_ring_wait(ring, 60000));
            CHECK(g4_ring_reduce(ring));
            if (r < S) {
                void* data;
                int64_t lo, hi;
                CHECK(g4_ring_slice(ring, &data, &lo, &hi));
                result[r].resize((size_t)(hi - lo) * n * n * 2);
                cudaMemcpy(result[r].data(), data, result[r].size() * 8, cudaMemcpyDeviceToHost);
                los[r] = lo;
                his[r] = hi;
            }
            CHECK(g4_ring_destroy(ring));
        });
    }
    for (auto& t : threads) t.join();
    for (int r = 0; r < world; ++r)
        for (size_t i = 0; i < ups[r].size(); ++i) {
            cudaFree(ups[r][i]);
            cudaFree(downs[r][i]);
        }

    // oracle: every walker (world rank, lane, measurement) applied to all N planes
    std::vector<double> ref((size_t)n * n * n * 2, 0.0), up((size_t)n * n * 2), down((size_t)n * n * 2);
    for (int wr = 0; wr < world; ++wr)
        for (int t = 0; t < lanes; ++t)
            for (int m = 0; m < rounds * batch; ++m) {
                g4o_fill_gsigma(cfg.seed, wr, t, m, n, G4_MODE_INTEGER, up.data(), down.data());
                g4o_accumulate(ref.data(), 0, n, n, up.data(), down.data());
            }
    for (int p = 0; p < S; ++p) {
        const size_t off = (size_t)los[p] * n * n * 2;
        if (std::memcmp(result[p].data(), ref.data() + off, result[p].size() * 8) != 0) {
            std::fprintf(stderr, "position %d: slice [%lld, %lld) differs from the oracle\n", p,
                         (long long)los[p], (long long)his[p]);
            return 2;
        }
    }
    std::printf("ring_threads ok: world %d, sub-rings of %d, %d lanes%s, %d rounds x %d walkers, N=%d, "
                "%d GPU(s)%s\n", world, S, lanes, alternate ? " (alternate)" : "", rounds, batch, n, ngpu,
                fed ? ", host-fed" : "");
    return 0;
}
