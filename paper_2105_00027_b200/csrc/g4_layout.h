// g4_layout.h -- staged payload geometry shared by host (.cpp) and device (.cu) code.
#pragma once
#include <cstdint>

#include "../../include/g4ring.h"

#ifdef __CUDACC__
#define G4_HD __host__ __device__ __forceinline__
#else
#define G4_HD inline
#endif

namespace g4 {

// Staged layout of one walker payload (include/g4ring.h): spin-planar
// transposes with a cyclic halo, stg[s][r][c] = M_s[c mod N][r mod N],
// r < ROWS = N + G4_HALO_ROWS, c < LD.  eb = bytes per complex entry (16 or 8);
// for complex64 the pitch is odd so the sheared TMA row stride (LD + 1) * 8 B
// is a multiple of 16 B.
G4_HD int staged_ld(int n, int eb) {
    const int ld = n + G4_HALO_COLS;
    return (eb == 8 && (ld % 2) == 0) ? ld + 1 : ld;
}
// For complex64 the row count is even so the spin-plane stride is a 16-B multiple.
G4_HD int staged_rows(int n, int eb) {
    const int rows = n + G4_HALO_ROWS;
    return (eb == 8 && (rows % 2) != 0) ? rows + 1 : rows;
}
G4_HD int64_t staged_plane(int n, int eb) { return (int64_t)staged_rows(n, eb) * staged_ld(n, eb); }

}  // namespace g4
