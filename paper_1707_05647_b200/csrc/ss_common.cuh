// ss_common.cuh -- shared internals of libstarscreen_b200 (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>

#include "../../include/starscreen_b200.h"

namespace ss {

// Thread-local last-error message (the only mutable global besides the
// launch counter, which is observability only).
void set_error(const char* fmt, ...);
void note_launch(uint64_t n = 1);

// Build geometry: a 128-thread tile covers
// 512 columns = Cw owned plane columns + an Rb+1 halo on each side, and Rb
// rows.  Rb is picked per image size so small images still fill the GPU.
constexpr int kBuildThreads = 128;
constexpr int kTileCols = 512;
constexpr int kGroup = 16;  // row-prefix granularity (columns)
inline int chunk_cols(int rb) { return kTileCols - 2 * rb - 2; }
// wide: the exact int64 build (3 resident CTAs per SM) wants >= 6 tiles per
// SM; the 32-bit build (4 resident, and its band scan is the serial part)
// does better with taller bands down to 2 tiles per SM (measured: config 1
// 31-row bands 0.974 vs 1.003 ms per step).
inline int pick_band_rows(int64_t W, int64_t H, bool wide = true) {
    // test hook: SS_BAND_ROWS=15|31|63 forces a geometry (tests cover all three)
    if (const char* e = getenv("SS_BAND_ROWS")) {
        const int v = atoi(e);
        if (v == 15 || v == 31 || v == 63) return v;
    }
    const int cand[3] = {63, 31, 15};
    for (int rb : cand) {
        const int64_t tiles = ((H + rb - 1) / rb) * ((W + 1 + chunk_cols(rb) - 1) / chunk_cols(rb));
        if (tiles >= 148 * (wide ? 6 : 2)) return rb;
    }
    return 15;
}

inline int64_t plane_pitch(int64_t W) { return ((W + 1 + 31) / 32) * 32; }
inline int64_t n_bands(int64_t H, int rb) { return (H + rb - 1) / rb; }
inline int64_t n_chunks(int64_t W, int rb) { return (W + 1 + chunk_cols(rb) - 1) / chunk_cols(rb); }
inline int64_t n_groups(int64_t W) { return (W + kGroup - 1) / kGroup; }
// state row length: x in [-1-Rb, W+Rb]
inline int64_t state_len(int64_t W, int rb) { return W + 2 * rb + 2; }

inline bool overflow_guard_fails(int64_t W, int64_t H) {
    // integral.py:59-63: 255 * max(w,h) * w * h >= 2**62 -> ValueError
    __int128 b = (__int128)255 * (W > H ? W : H) * W * H;
    return b >= ((__int128)1 << 62);
}

// Debug bounds checks (the pool refuses compute-sanitizer): built with
// -DSS_DEBUG (SS_EXTRA_NVCC), every SS_CHECK traps on violation, so a GPU test
// run of that build is a memcheck of the checked indices; compiled out otherwise.
#ifdef SS_DEBUG
#define SS_CHECK(c)              \
    do {                         \
        if (!(c)) __trap();      \
    } while (0)
#else
#define SS_CHECK(c) ((void)0)
#endif

// internal status: the fused ladder declined a group (nothing enqueued; screen per size)
constexpr int SS_DECLINED = -1000;

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
