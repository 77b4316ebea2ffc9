// ss_ladder.cpp -- the per-size loop of screen() (screening.py:502-520) as one
// C-ABI call: every ladder size's screen (K3, or the m < MIN_PATCH_SIDE
// whole-grid keep) is enqueued here, sizes spread over the caller's side
// streams with an event fork/join around them -- no per-size round trip
// through Python, and the whole call stays CUDA-graph capturable.
#include <algorithm>
#include <vector>

#include "ss_common.cuh"

namespace ss {
int screen_ladder_fused(const void* planes, int eb, const void* planes32_s1, int64_t h, int64_t pitch, int64_t W,
                        int64_t H, int64_t y_origin, int64_t y_begin, int64_t y_end, int32_t stride, int n,
                        const int* ks, const int32_t* h_m,
                        const int32_t* h_n_rings, const int32_t* h_ring_n, const int32_t* h_ring_d,
                        const int64_t* d_blobs, const int64_t* h_blobs, const int64_t* h_blob_off, double qm,
                        double qs, double qg, uint32_t* d_masks, int64_t mask_pitch, int64_t size_stride,
                        uint32_t* d_row_counts, int64_t rc_stride, unsigned long long* d_stage_counts, void* d_ws,
                        size_t ws_bytes, cudaStream_t s, const uint16_t* d_coarse, int n_coarse,
                        const int32_t* h_shifts, const uint16_t* d_hi16);
}  // namespace ss

extern "C" int ss_screen_ladder2(const int64_t* d_planes, const uint32_t* d_planes32, int64_t w, int64_t h,
                                 int64_t plane_pitch, int64_t W, int64_t H, int64_t y_origin, int64_t y_begin,
                                 int64_t y_end, int32_t stride, int32_t n_sizes, const int32_t* h_m,
                                 const int32_t* h_n_rings, const int32_t* h_ring_n, const int32_t* h_ring_d,
                                 const int64_t* d_blobs, const int64_t* h_blobs, const int64_t* h_blob_off,
                                 double q_mean, double q_std, double q_grad, uint32_t* d_masks,
                                 int64_t mask_pitch_words, int64_t size_stride_words, uint32_t* d_row_counts,
                                 int64_t row_counts_stride, unsigned long long* d_stage_counts, int32_t flags,
                                 int32_t n_streams, void* const* streams, void* const* d_workspaces,
                                 size_t workspace_bytes, const uint16_t* d_coarse, int32_t n_coarse,
                                 const int32_t* h_shifts, const uint16_t* d_hi16);

extern "C" int ss_screen_ladder(const int64_t* d_planes, const uint32_t* d_planes32, int64_t w, int64_t h,
                                int64_t plane_pitch, int64_t W, int64_t H, int64_t y_origin, int64_t y_begin,
                                int64_t y_end, int32_t stride, int32_t n_sizes, const int32_t* h_m,
                                const int32_t* h_n_rings, const int32_t* h_ring_n, const int32_t* h_ring_d,
                                const int64_t* d_blobs, const int64_t* h_blobs, const int64_t* h_blob_off,
                                double q_mean, double q_std, double q_grad, uint32_t* d_masks,
                                int64_t mask_pitch_words, int64_t size_stride_words, uint32_t* d_row_counts,
                                int64_t row_counts_stride, unsigned long long* d_stage_counts, int32_t flags,
                                int32_t n_streams, void* const* streams, void* const* d_workspaces,
                                size_t workspace_bytes) {
    return ss_screen_ladder2(d_planes, d_planes32, w, h, plane_pitch, W, H, y_origin, y_begin, y_end, stride, n_sizes,
                             h_m, h_n_rings, h_ring_n, h_ring_d, d_blobs, h_blobs, h_blob_off, q_mean, q_std, q_grad,
                             d_masks, mask_pitch_words, size_stride_words, d_row_counts, row_counts_stride,
                             d_stage_counts, flags, n_streams, streams, d_workspaces, workspace_bytes, nullptr, 0,
                             nullptr, nullptr);
}

extern "C" int ss_screen_ladder2(const int64_t* d_planes, const uint32_t* d_planes32, int64_t w, int64_t h,
                                 int64_t plane_pitch, int64_t W, int64_t H, int64_t y_origin, int64_t y_begin,
                                 int64_t y_end, int32_t stride, int32_t n_sizes, const int32_t* h_m,
                                 const int32_t* h_n_rings, const int32_t* h_ring_n, const int32_t* h_ring_d,
                                 const int64_t* d_blobs, const int64_t* h_blobs, const int64_t* h_blob_off,
                                 double q_mean, double q_std, double q_grad, uint32_t* d_masks,
                                 int64_t mask_pitch_words, int64_t size_stride_words, uint32_t* d_row_counts,
                                 int64_t row_counts_stride, unsigned long long* d_stage_counts, int32_t flags,
                                 int32_t n_streams, void* const* streams, void* const* d_workspaces,
                                 size_t workspace_bytes, const uint16_t* d_coarse, int32_t n_coarse,
                                 const int32_t* h_shifts, const uint16_t* d_hi16) {
    if (n_sizes < 0 || n_sizes > SS_MAX_SIZES || !h_m || !h_n_rings || !h_ring_n || !h_ring_d || !h_blob_off ||
        n_streams < 1 || !streams || !d_workspaces || (n_sizes > 0 && (!d_masks || !d_row_counts))) {
        ss::set_error("bad ladder arguments");
        return SS_EINVAL;
    }
    const bool int64_only = (flags & 1) != 0;
    if (flags & 2) {
        if (w != W) {
            ss::set_error("row-band tables must span the full width (w == W)");
            return SS_EINVAL;
        }
        // fused ladder (ss_ladder_screen.cu): all sizes of one plane width in
        // lock-step on streams[0]; m < 8 sizes keep their grid; a group the
        // fused path declines is screened size by size on the same stream
        void* st = streams[0];
        std::vector<int> g32, g64;
        for (int32_t k = 0; k < n_sizes; ++k) {
            if (h_m[k] < 8 || h_n_rings[k] == 0) {
                uint32_t* mask = d_masks + (size_t)k * (size_t)size_stride_words;
                uint32_t* rc = d_row_counts + (size_t)k * (size_t)row_counts_stride;
                if (int e = ss_fill_grid(W, y_begin, y_end, stride, mask, mask_pitch_words, rc, st)) return e;
                continue;
            }
            const bool fits = !int64_only && d_planes32 &&
                              ss_screen_fits32(h_n_rings[k], h_ring_n + (size_t)k * SS_MAX_RINGS,
                                               h_ring_d + (size_t)k * SS_MAX_RINGS);
            (fits ? g32 : g64).push_back(k);
        }
        for (int g = 0; g < 2; ++g) {
            const std::vector<int>& ks = g == 0 ? g32 : g64;
            if (ks.empty()) continue;
            const void* planes = g == 0 ? static_cast<const void*>(d_planes32) : static_cast<const void*>(d_planes);
            if (!planes && !(g == 1 && d_hi16 && d_planes32)) {
                ss::set_error("ladder needs the int64 planes (ring sums exceed 32 bits)");
                return SS_EINVAL;
            }
            int e = ss::screen_ladder_fused(planes, g == 0 ? 4 : 8, g == 0 ? nullptr : d_planes32, h, plane_pitch, W, H,
                                            y_origin, y_begin, y_end,
                                            stride, (int)ks.size(), ks.data(), h_m, h_n_rings, h_ring_n, h_ring_d,
                                            d_blobs, h_blobs, h_blob_off, q_mean, q_std, q_grad, d_masks,
                                            mask_pitch_words, size_stride_words, d_row_counts, row_counts_stride,
                                            d_stage_counts, d_workspaces[0], workspace_bytes, ss::as_stream(st),
                                            d_coarse, n_coarse, h_shifts, d_hi16);
            if (e == ss::SS_DECLINED) {
                if (g == 1 && !d_planes) {
                    ss::set_error("the per-size screen of sizes beyond 32 bits needs the int64 planes");
                    return SS_EINVAL;
                }
                for (int k : ks) {
                    const int32_t* rn = h_ring_n + (size_t)k * SS_MAX_RINGS;
                    const int32_t* rd = h_ring_d + (size_t)k * SS_MAX_RINGS;
                    e = ss_screen_size(g == 0 ? nullptr : d_planes, g == 0 ? d_planes32 : nullptr, w, h, plane_pitch,
                                       W, H, y_origin, y_begin, y_end, h_m[k], stride, h_n_rings[k], rn, rd,
                                       d_blobs + h_blob_off[k], h_blobs + h_blob_off[k], q_mean, q_std, q_grad,
                                       d_masks + (size_t)k * (size_t)size_stride_words, mask_pitch_words,
                                       d_row_counts + (size_t)k * (size_t)row_counts_stride, d_stage_counts,
                                       d_workspaces[0], workspace_bytes, st);
                    if (e) return e;
                }
            } else if (e) {
                return e;
            }
        }
        return SS_OK;
    }
    cudaStream_t main = ss::as_stream(streams[0]);
    const int n_side = n_streams - 1;
    std::vector<cudaEvent_t> events;
    auto new_event = [&](cudaEvent_t* e) -> int {
        if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return ss::check_launch("event");
        events.push_back(*e);
        return SS_OK;
    };
    auto cleanup = [&]() {
        for (cudaEvent_t e : events) cudaEventDestroy(e);  // released once pending work completes
    };
    std::vector<bool> used((size_t)std::max(n_side, 0), false);
    cudaEvent_t fork = nullptr;
    if (n_side > 0) {
        if (int e = new_event(&fork)) return cleanup(), e;
        if (cudaEventRecord(fork, main) != cudaSuccess) return cleanup(), ss::check_launch("event record");
    }
    for (int32_t k = 0; k < n_sizes; ++k) {
        const int j = n_side > 0 ? k % n_side : -1;
        void* st = j >= 0 ? streams[1 + j] : streams[0];
        void* ws = d_workspaces[j >= 0 ? 1 + j : 0];
        if (j >= 0 && !used[(size_t)j]) {
            if (cudaStreamWaitEvent(ss::as_stream(st), fork, 0) != cudaSuccess)
                return cleanup(), ss::check_launch("stream wait");
            used[(size_t)j] = true;
        }
        uint32_t* mask = d_masks + (size_t)k * (size_t)size_stride_words;
        uint32_t* rc = d_row_counts + (size_t)k * (size_t)row_counts_stride;
        int e;
        if (h_m[k] < 8 || h_n_rings[k] == 0) {
            e = ss_fill_grid(W, y_begin, y_end, stride, mask, mask_pitch_words, rc, st);
        } else {
            const int32_t* rn = h_ring_n + (size_t)k * SS_MAX_RINGS;
            const int32_t* rd = h_ring_d + (size_t)k * SS_MAX_RINGS;
            const bool fits = !int64_only && ss_screen_fits32(h_n_rings[k], rn, rd);
            e = ss_screen_size(fits ? nullptr : d_planes, int64_only ? nullptr : d_planes32, w, h, plane_pitch, W, H,
                               y_origin, y_begin, y_end, h_m[k], stride, h_n_rings[k], rn, rd,
                               d_blobs + h_blob_off[k], h_blobs + h_blob_off[k], q_mean, q_std, q_grad, mask,
                               mask_pitch_words, rc, d_stage_counts, ws, workspace_bytes, st);
        }
        if (e) return cleanup(), e;
    }
    for (int j = 0; j < n_side; ++j) {
        if (!used[(size_t)j]) continue;
        cudaEvent_t join;
        if (int e = new_event(&join)) return cleanup(), e;
        if (cudaEventRecord(join, ss::as_stream(streams[1 + j])) != cudaSuccess ||
            cudaStreamWaitEvent(main, join, 0) != cudaSuccess)
            return cleanup(), ss::check_launch("stream join");
    }
    cleanup();
    return SS_OK;
}
