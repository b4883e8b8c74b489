// g4_util.cpp -- error plumbing and the integer helpers of the C ABI.
#include <cstring>
#include <string>

#include "g4_internal.h"
#include "g4_layout.h"

namespace g4 {

static thread_local char t_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(t_err, sizeof(t_err), fmt, ap);
    va_end(ap);
}

void clear_error() { t_err[0] = '\0'; }

}  // namespace g4

extern "C" {

const char* g4_last_error(void) { return g4::t_err; }

int32_t g4_abi_version(void) { return G4RING_ABI_VERSION; }

int64_t g4_payload_bytes(int32_t n, int32_t dtype) {
    // G4_C128_G64 payloads are complex64
    if (n < 1 || (dtype != G4_C128 && dtype != G4_C64 && dtype != G4_C128_G64)) return -1;
    return 2 * g4::staged_plane(n, (int)g4::entry_bytes(dtype)) * g4::entry_bytes(dtype);
}

g4_status g4_staged_dims(int32_t n, int32_t dtype, int32_t* rows, int32_t* ld) {
    if (n < 1 || !rows || !ld || (dtype != G4_C128 && dtype != G4_C64 && dtype != G4_C128_G64))
        return g4::fail(G4_ERR_CONTRACT, "staged_dims: bad arguments");
    *rows = g4::staged_rows(n, (int)g4::entry_bytes(dtype));
    *ld = g4::staged_ld(n, (int)g4::entry_bytes(dtype));
    return G4_OK;
}

// ringacc/tensor.py:50-55
g4_status g4_index_diff(int64_t a, int64_t b, int64_t n, int64_t* out) {
    if (!out) return g4::fail(G4_ERR_CONTRACT, "index_diff: null output");
    if (n < 1 || !(0 <= a && a < n && 0 <= b && b < n)) {
        g4::set_error("index out of range: a=%lld, b=%lld, N=%lld", (long long)a, (long long)b,
                      (long long)n);
        return G4_ERR_CONTRACT;
    }
    int64_t r = (a - b) % n;
    *out = r < 0 ? r + n : r;
    return G4_OK;
}

// ringacc/tensor.py:148-164
g4_status g4_make_partition(int64_t n, int64_t p, int64_t* ranges) {
    if (p < 1) {
        g4::set_error("partition count must be >= 1, got %lld", (long long)p);
        return G4_ERR_CONTRACT;
    }
    if (p > n) {
        g4::set_error("cannot split axis of length %lld over %lld ranks: empty slice",
                      (long long)n, (long long)p);
        return G4_ERR_CONTRACT;
    }
    if (!ranges) return g4::fail(G4_ERR_CONTRACT, "make_partition: null output");
    const int64_t base = n / p, rem = n % p;
    int64_t lo = 0;
    for (int64_t i = 0; i < p; ++i) {
        const int64_t hi = lo + base + (i < rem ? 1 : 0);
        ranges[2 * i] = lo;
        ranges[2 * i + 1] = hi;
        lo = hi;
    }
    return G4_OK;
}

}  // extern "C"
