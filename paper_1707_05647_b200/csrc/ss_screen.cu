// ss_screen.cu -- K3: star features + quantize + membership + ballot mask.
//
// Replaces _scan_size (screening.py:418-471) for one ladder size: the ring
// features of _ring_maps_rect / _octagon_maps (screening.py:380-415,
// features.py:322-382), _quantize_arr (screening.py:86-87), _pack_cells
// (:90-97), _member_mask (:173-178) and the nonzero/mask bookkeeping.
//
// Bit-exactness: this file is compiled with -fmad=false and every fp64 op
// is an IEEE-rounded add/sub/mul/div/sqrt in the reference's NumPy order
// (SURVEY.md App. A); integer sums are exact int64 four-corner differences.
//
// Early-exit cascade (exact): a centre can only pass ring r if its mean cell
// is among the ring's key means, then its (mean, std) pair among the key
// pairs, then the full key.  The projections are implied by full membership,
// so the decision is unchanged, but the X/Y/SQ planes and most of the fp64
// work are only touched by centres that survive the cheaper tests.
#include <algorithm>

#include "ss_common.cuh"

namespace ss {
namespace {

constexpr unsigned FULL = 0xffffffffu;

struct RingDev {
    int n, d;
    double cnt_sq, w1_sq, cnt_di, w1_di;
    // membership: offsets (int64 words into the blob) and counts
    int off_m, n_m, off_ms, n_ms, off_k, n_k;
    long long m_lo;            // dense mean-cell bitmap base
    unsigned long long m_bits; // bit (cm - m_lo) set <=> cm in projection
    int m_dense;               // 1 if the bitmap is exact
};

struct ScreenArgs {
    const long long* planes;
    long long pitch, plane_stride;
    int W, H;        // global image
    int y_origin;    // global row of table row 0
    int y_begin, y_end;
    int m, stride, lo, hi;
    int n_rings;
    double qm, qs, qg;
    const long long* blob;
    unsigned* mask;
    long long mask_pitch;
    unsigned* row_counts;
    unsigned long long* stage_counts;  // nullable: [ring0 evals, ring0 std-stage, ring0 grad-stage, ring>=1 evals]
    RingDev ring[SS_MAX_RINGS];
};

__device__ __forceinline__ bool bsearch_eq(const long long* __restrict__ a, int n, long long key) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < key) lo = mid + 1; else hi = mid;
    }
    return lo < n && __ldg(a + lo) == key;
}

// four-corner square sum: cells[y+1][x+1] convention (integral.py:144-162)
__device__ __forceinline__ long long sq_sum(const long long* __restrict__ p, long long pitch, int cx, int cy,
                                            int n) {
    const long long* top = p + (long long)(cy - n + 1) * pitch;
    const long long* bot = p + (long long)(cy + n + 1) * pitch;
    return __ldg(bot + cx + n + 1) - __ldg(bot + cx - n + 1) - __ldg(top + cx + n + 1) + __ldg(top + cx - n + 1);
}

// closed l1 ball via the E / O planes (integral.py:165-186 equivalent)
__device__ __forceinline__ long long di_sum(const long long* __restrict__ e, const long long* __restrict__ o,
                                            long long pitch, int cx, int cy, int r) {
    const long long* orow = o + (long long)cy * pitch;
    return __ldg(e + (long long)(cy + r + 1) * pitch + cx + 1) - __ldg(orow + cx - r) - __ldg(orow + cx + r + 1) +
           __ldg(e + (long long)(cy - r) * pitch + cx + 1);
}

__device__ __forceinline__ long long quantize(double f, double q) {
    // screening.py:86-87: floor(f / q + 0.5)
    return (long long)floor(__dadd_rn(__ddiv_rn(f, q), 0.5));
}

// One ring of one centre.  Returns the cascade stage reached: 0 = rejected
// on the mean, 1 = on (mean, std), 2 = on the full key, 3 = member.
__device__ __forceinline__ int ring_member(const ScreenArgs& a, const RingDev& R, int cx, int cy) {
    const long long ps = a.plane_stride;
    const long long* sat = a.planes;
    const long long* E = a.planes + 4 * ps;
    const long long* O = a.planes + 8 * ps;
    // ── stage 1: mean (PLAIN planes) ─────────────────────────────────────
    const long long s1q = sq_sum(sat, a.pitch, cx, cy, R.n);
    const long long s1d = di_sum(E, O, a.pitch, cx, cy, R.d);
    const double mq = __ddiv_rn((double)s1q, R.cnt_sq);
    const double md = __ddiv_rn((double)s1d, R.cnt_di);
    const double mean = __dmul_rn(__dadd_rn(mq, md), 0.5);
    const long long cm = quantize(mean, a.qm);
    if (R.m_dense) {
        const unsigned long long off = (unsigned long long)(cm - R.m_lo);
        if (off >= 64ull || !((R.m_bits >> off) & 1ull)) return 0;
    } else if (!bsearch_eq(a.blob + R.off_m, R.n_m, cm)) {
        return 0;
    }
    // ── stage 2: std (SQUARED planes) ────────────────────────────────────
    const long long s2q = sq_sum(sat + 3 * ps, a.pitch, cx, cy, R.n);
    const long long s2d = di_sum(E + 3 * ps, O + 3 * ps, a.pitch, cx, cy, R.d);
    const double vq = __dsub_rn(__ddiv_rn((double)s2q, R.cnt_sq), __dmul_rn(mq, mq));
    const double vd = __dsub_rn(__ddiv_rn((double)s2d, R.cnt_di), __dmul_rn(md, md));
    const double sdq = __dsqrt_rn(vq > 0.0 ? vq : 0.0);
    const double sdd = __dsqrt_rn(vd > 0.0 ? vd : 0.0);
    const double sd = __dmul_rn(__dadd_rn(sdq, sdd), 0.5);
    const long long cs = quantize(sd, a.qs);
    const long long kms = cm * SS_KEY_BASE + cs;
    if (!bsearch_eq(a.blob + R.off_ms, R.n_ms, kms)) return 1;
    // ── stage 3: gradient (X / Y planes) ─────────────────────────────────
    const long long sxq = sq_sum(sat + 1 * ps, a.pitch, cx, cy, R.n);
    const long long syq = sq_sum(sat + 2 * ps, a.pitch, cx, cy, R.n);
    const long long sxd = di_sum(E + 1 * ps, O + 1 * ps, a.pitch, cx, cy, R.d);
    const long long syd = di_sum(E + 2 * ps, O + 2 * ps, a.pitch, cx, cy, R.d);
    const double fs1q = (double)s1q, fs1d = (double)s1d;
    // (cx + 1.5) * s1 and the subtraction are exact
    const double gxq = __ddiv_rn(__dsub_rn((double)sxq, __dmul_rn(__dadd_rn((double)cx, 1.5), fs1q)), R.w1_sq);
    const double gyq = __ddiv_rn(__dsub_rn((double)syq, __dmul_rn(__dadd_rn((double)cy, 1.5), fs1q)), R.w1_sq);
    const double gxd = __ddiv_rn(__dsub_rn((double)sxd, __dmul_rn(__dadd_rn((double)cx, 1.0), fs1d)), R.w1_di);
    const double gyd = __ddiv_rn(__dsub_rn((double)syd, __dmul_rn(__dadd_rn((double)cy, 1.0), fs1d)), R.w1_di);
    const double gx = __dmul_rn(__dadd_rn(gxq, gxd), 0.5);
    const double gy = __dmul_rn(__dadd_rn(gyq, gyd), 0.5);
    const double gm = __dsqrt_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)));
    const long long cg = quantize(gm, a.qg);
    return bsearch_eq(a.blob + R.off_k, R.n_k, kms * SS_KEY_BASE + cg) ? 3 : 2;
}

// blockDim = (32, 8): a warp covers 32 consecutive x of one row.
__global__ void __launch_bounds__(256) screen_kernel(const ScreenArgs a) {
    const int lane = threadIdx.x;
    const int x = blockIdx.x * 32 + lane;
    const int y = a.y_begin + blockIdx.y * 8 + threadIdx.y;
    if (y >= a.y_end) return;  // warp-uniform
    const bool in_img = x < a.W;
    const bool on_grid = in_img && (x % a.stride == 0) && (y % a.stride == 0);
    const bool interior = on_grid && x >= a.lo && x <= a.W - 1 - a.hi && y >= a.lo && y <= a.H - 1 - a.hi;
    bool keep = on_grid && !interior;  // screening.py:438-442 border keeps
    bool surv = false;
    int stage0 = -1, later = 0;
    if (interior) {
        const int cy = y - a.y_origin;  // table-local row (features are frame-invariant)
        stage0 = ring_member(a, a.ring[0], x, cy);
        surv = stage0 == 3;
        for (int r = 1; r < a.n_rings && surv; ++r) {
            ++later;
            surv = ring_member(a, a.ring[r], x, cy) == 3;
        }
        keep = surv;
    }
    const unsigned word = __ballot_sync(FULL, keep);
    const unsigned sw = __ballot_sync(FULL, surv);
    const long long row = y - a.y_begin;
    if (lane == 0) {
        if (blockIdx.x * 32 < (unsigned)a.W) a.mask[row * a.mask_pitch + blockIdx.x] = word;
        if (sw) atomicAdd(a.row_counts + row, (unsigned)__popc(sw));
    }
    if (a.stage_counts) {  // instrumentation only (bench.py roofline), uniform branch
        const unsigned e0 = __ballot_sync(FULL, stage0 >= 0), e1 = __ballot_sync(FULL, stage0 >= 1),
                       e2 = __ballot_sync(FULL, stage0 >= 2);
        int lt = later;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) lt += __shfl_down_sync(FULL, lt, d);
        if (lane == 0) {
            atomicAdd(a.stage_counts + 0, (unsigned long long)__popc(e0));
            atomicAdd(a.stage_counts + 1, (unsigned long long)__popc(e1));
            atomicAdd(a.stage_counts + 2, (unsigned long long)__popc(e2));
            atomicAdd(a.stage_counts + 3, (unsigned long long)lt);
        }
    }
}

__global__ void fill_grid_kernel(int W, int y_begin, int y_end, int stride, unsigned* mask, long long mask_pitch,
                                 unsigned* row_counts) {
    const long long words = (W + 31) / 32;
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long rows = y_end - y_begin;
    if (gid >= rows * words) return;
    const long long row = gid / words, w = gid % words;
    const int y = (int)(y_begin + row);
    unsigned bits = 0;
    if (y % stride == 0) {
        for (int b = 0; b < 32; ++b) {
            const long long x = w * 32 + b;
            if (x < W && x % stride == 0) bits |= 1u << b;
        }
    }
    mask[row * mask_pitch + w] = bits;
    if (w == 0) row_counts[row] = 0;
}

}  // namespace

int screen_size(const int64_t* d_planes, int64_t w, int64_t h, int64_t pitch, int64_t W, int64_t H, int64_t y_origin,
                int64_t y_begin, int64_t y_end, int32_t m, int32_t stride, int32_t n_rings, const int32_t* ring_n,
                const int32_t* ring_d, const int64_t* d_blob, const int64_t* h_blob, double qm, double qs, double qg,
                uint32_t* d_mask, int64_t mask_pitch, uint32_t* d_row_counts, unsigned long long* d_stage_counts,
                void* stream) {
    if (w != W) { set_error("row-band tables must span the full width (w == W)"); return SS_EINVAL; }
    if (W < 1 || H < 1 || h < 1 || y_origin < 0 || y_origin + h > H) {
        set_error("bad table frame");
        return SS_EINVAL;
    }
    if (y_begin < 0 || y_end > H || y_begin > y_end) { set_error("bad row range"); return SS_EINVAL; }
    if (m < 2 * 4 || stride < 1) { set_error("bad size/stride"); return SS_EINVAL; }
    if (n_rings < 1 || n_rings > SS_MAX_RINGS) { set_error("n_rings out of range"); return SS_EINVAL; }
    if (pitch != plane_pitch(w)) { set_error("plane pitch mismatch"); return SS_EINVAL; }
    if (mask_pitch < (W + 31) / 32) { set_error("mask pitch too small"); return SS_EINVAL; }
    const int lo = (m - 1) / 2, hi = m / 2;
    // every evaluated centre's patch rows must be inside the table
    const int64_t ylo = std::max<int64_t>(y_begin, lo), yhi = std::min<int64_t>(y_end - 1, H - 1 - hi);
    if (ylo <= yhi && (ylo - lo < y_origin || yhi + hi > y_origin + h - 1)) {
        set_error("table band [%lld, %lld) does not cover rows [%lld, %lld] with margins", (long long)y_origin,
                  (long long)(y_origin + h), (long long)ylo, (long long)yhi);
        return SS_EINVAL;
    }
    ScreenArgs a;
    a.planes = reinterpret_cast<const long long*>(d_planes);
    a.pitch = pitch;
    a.plane_stride = (h + 1) * pitch;
    a.W = (int)W;
    a.H = (int)H;
    a.y_origin = (int)y_origin;
    a.y_begin = (int)y_begin;
    a.y_end = (int)y_end;
    a.m = m;
    a.stride = stride;
    a.lo = lo;
    a.hi = hi;
    a.n_rings = n_rings;
    a.qm = qm;
    a.qs = qs;
    a.qg = qg;
    a.blob = reinterpret_cast<const long long*>(d_blob);
    a.mask = d_mask;
    a.mask_pitch = mask_pitch;
    a.row_counts = d_row_counts;
    a.stage_counts = d_stage_counts;
    // blob header: [0] n_rings, then per ring (off_m, n_m, off_ms, n_ms, off_k, n_k)
    if (!h_blob || h_blob[0] != n_rings) { set_error("key blob does not match n_rings"); return SS_EINVAL; }
    for (int r = 0; r < n_rings; ++r) {
        RingDev& R = a.ring[r];
        const int n = ring_n[r], d = ring_d[r];
        if (n < 1 || d < 0 || n > hi || d > lo) { set_error("ring (%d,%d) does not fit m=%d", n, d, m); return SS_EINVAL; }
        R.n = n;
        R.d = d;
        R.cnt_sq = (double)(4LL * n * n);                                        // features.py:323
        R.w1_sq = (double)(2LL * n * n * n);                                     // features.py:324
        R.cnt_di = (double)(2LL * d * d + 2LL * d + 1);                          // integral.py:189-191
        R.w1_di = (double)(2LL * d * d + (long long)d * (d - 1) * (2 * d - 1) / 3);  // features.py:341-343
        const int64_t* hd = h_blob + 1 + 6 * r;
        R.off_m = (int)hd[0];
        R.n_m = (int)hd[1];
        R.off_ms = (int)hd[2];
        R.n_ms = (int)hd[3];
        R.off_k = (int)hd[4];
        R.n_k = (int)hd[5];
        // dense 64-bit bitmap of the mean projection when it spans < 64 cells
        R.m_dense = 0;
        R.m_lo = 0;
        R.m_bits = 0;
        if (R.n_m == 0) {
            R.m_dense = 1;  // empty set: nothing passes
        } else {
            const int64_t lo_c = h_blob[R.off_m], hi_c = h_blob[R.off_m + R.n_m - 1];
            if (hi_c - lo_c < 64) {
                R.m_dense = 1;
                R.m_lo = lo_c;
                for (int i = 0; i < R.n_m; ++i) R.m_bits |= 1ull << (h_blob[R.off_m + i] - lo_c);
            }
        }
    }
    cudaStream_t s = as_stream(stream);
    const int64_t rows = y_end - y_begin;
    if (rows == 0) return SS_OK;
    if (cudaMemsetAsync(d_row_counts, 0, rows * sizeof(uint32_t), s) != cudaSuccess) return check_launch("memset");
    dim3 grid((unsigned)((W + 31) / 32), (unsigned)((rows + 7) / 8));
    screen_kernel<<<grid, dim3(32, 8), 0, s>>>(a);
    note_launch();
    return check_launch("screen_kernel");
}

int fill_grid(int64_t W, int64_t y_begin, int64_t y_end, int32_t stride, uint32_t* d_mask, int64_t mask_pitch,
              uint32_t* d_row_counts, void* stream) {
    if (W < 1 || y_begin > y_end || stride < 1) { set_error("bad fill_grid arguments"); return SS_EINVAL; }
    const int64_t words = (W + 31) / 32, rows = y_end - y_begin;
    if (rows == 0) return SS_OK;
    fill_grid_kernel<<<(unsigned)((rows * words + 255) / 256), 256, 0, as_stream(stream)>>>(
        (int)W, (int)y_begin, (int)y_end, stride, d_mask, mask_pitch, d_row_counts);
    note_launch();
    return check_launch("fill_grid_kernel");
}

}  // namespace ss

extern "C" {
int ss_screen_size(const int64_t* d_planes, int64_t w, int64_t h, int64_t plane_pitch, int64_t W, int64_t H,
                   int64_t y_origin, int64_t y_begin, int64_t y_end, int32_t m, int32_t stride, int32_t n_rings,
                   const int32_t* h_ring_n, const int32_t* h_ring_d, const int64_t* d_blob, const int64_t* h_blob,
                   double q_mean, double q_std, double q_grad, uint32_t* d_mask, int64_t mask_pitch_words,
                   uint32_t* d_row_counts, unsigned long long* d_stage_counts, void* stream) {
    return ss::screen_size(d_planes, w, h, plane_pitch, W, H, y_origin, y_begin, y_end, m, stride, n_rings, h_ring_n,
                           h_ring_d, d_blob, h_blob, q_mean, q_std, q_grad, d_mask, mask_pitch_words, d_row_counts,
                           d_stage_counts, stream);
}
int ss_fill_grid(int64_t W, int64_t y_begin, int64_t y_end, int32_t stride, uint32_t* d_mask,
                 int64_t mask_pitch_words, uint32_t* d_row_counts, void* stream) {
    return ss::fill_grid(W, y_begin, y_end, stride, d_mask, mask_pitch_words, d_row_counts, stream);
}
}
