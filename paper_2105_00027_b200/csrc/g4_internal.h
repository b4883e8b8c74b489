// g4_internal.h -- host-side helpers shared by the library's translation units.
#pragma once
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/g4ring.h"

namespace g4 {

// Thread-local last-error buffer behind g4_last_error().
void set_error(const char* fmt, ...);
void clear_error();

inline g4_status fail(g4_status st, const char* what) {
    set_error("%s", what);
    return st;
}

inline g4_status check_cuda(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return G4_OK;
    set_error("%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
    return G4_ERR_CUDA;
}

inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

inline int64_t entry_bytes(int32_t dtype) { return dtype == G4_C128 ? 16 : 8; }

}  // namespace g4

#define G4_TRY(expr)                          \
    do {                                      \
        g4_status _st = (expr);               \
        if (_st != G4_OK) return _st;         \
    } while (0)

#define G4_CUDA(expr) G4_TRY(::g4::check_cuda((expr), #expr))
