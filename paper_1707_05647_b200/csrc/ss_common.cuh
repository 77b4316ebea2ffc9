// ss_common.cuh -- shared internals of libstarscreen_b200 (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>

#include "../../include/starscreen_b200.h"

namespace ss {

// Thread-local last-error message (the only mutable global besides the
// launch counter, which is observability only).
void set_error(const char* fmt, ...);
void note_launch(uint64_t n = 1);

// Build-geometry constants.
constexpr int kBuildThreads = 512;            // threads per band tile
constexpr int kBandRows = 63;                 // Rb: rows per band
constexpr int kChunkCols = 384;               // Cw: plane columns per tile
constexpr int kGroup = 64;                    // row-prefix granularity
static_assert(kChunkCols + 2 * kBandRows + 2 <= kBuildThreads, "tile too wide");
static_assert((kChunkCols % kGroup) == 0 && ((kBandRows + 1) % kGroup) == 0, "XL must be group aligned");

inline int64_t plane_pitch(int64_t W) { return ((W + 1 + 31) / 32) * 32; }
inline int64_t n_bands(int64_t H) { return (H + kBandRows - 1) / kBandRows; }
inline int64_t n_chunks(int64_t W) { return (W + 1 + kChunkCols - 1) / kChunkCols; }
inline int64_t n_groups(int64_t W) { return (W + kGroup - 1) / kGroup; }
// state row length: x in [-1-Rb, W+Rb]
inline int64_t state_len(int64_t W) { return W + 2 * kBandRows + 2; }

inline bool overflow_guard_fails(int64_t W, int64_t H) {
    // integral.py:59-63: 255 * max(w,h) * w * h >= 2**62 -> ValueError
    __int128 b = (__int128)255 * (W > H ? W : H) * W * H;
    return b >= ((__int128)1 << 62);
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return SS_ECUDA;
    }
    return SS_OK;
}

}  // namespace ss
