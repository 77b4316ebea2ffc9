// ss_match.cu -- f3: the second stage, masked zero-mean NCC of every screened
// candidate against every rotated template probe (second_stage.py:106-204).
//
// The reference evaluates, per ladder size m, W @ [P | M] and (W*W) @ M in
// float64 (second_stage.py:136-150): W the candidates' m x m uint8 windows,
// P the masked rotated probes, M their 0/1 supports.  Every entry is an
// integer and every dot product an integer below 2^53, so those float64
// matmuls are exact whatever their summation order -- and so is an integer
// tensor-core GEMM.  One fused kernel per (size, group of <= 40 angles)
// gathers the windows straight from the image into u8 MMA fragments
// (mma.sync m16n8k32 u8 x u8 -> s32: W x [P | M], and W^2 as its high and
// low bytes x M), keeps the dot products in registers (int32, spilled into
// int64 shared memory every few rows when m is large enough to overflow),
// replays the reference's float64 score sequence op for op (-fmad=false) and
// reduces to the best candidate per angle with the reference's tie-break
// (first candidate on equal scores, np.argmax).
//
//   ss_match_planes   the image, and its squares' high / low bytes, as padded
//                     u8 planes (the three A operands)
//   ss_match_probes   resize_bilinear(template, m, m) (image_io.py:164-178) and
//                     _rotate_with_mask per angle (image_io.py:181-203; cos/sin
//                     from the host's libm, as NumPy computes them) as B
//                     fragments, and per-angle sums
//   ss_match_fused    windows x probes -> scores -> best per angle per CTA
//   ss_match_reduce   best per angle over the CTAs, in candidate order
#include <algorithm>

#include "ss_common.cuh"

namespace ss {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int MAX_GROUP_ANGLES = 40;          // angles per fused launch (5 n-tiles of 8)
constexpr int NT = MAX_GROUP_ANGLES / 8;      // angle n-tiles
constexpr int BT = 2 * NT;                    // B n-tiles: masked probe, support
constexpr int FUSED_WARPS = 4;
constexpr int TM = 16 * FUSED_WARPS;          // candidates per CTA
constexpr int PLANE_PAD = 64;                 // zero columns right of each plane row

// image_io.py:131-161 bilinear sample of img (h x w) at (xs, ys), quantized
__device__ __forceinline__ int sample_q(const uint8_t* img, int w, int h, double xs, double ys) {
    const double x0f = floor(xs), y0f = floor(ys);
    const double fx = __dsub_rn(xs, x0f), fy = __dsub_rn(ys, y0f);
    const long long x0 = (long long)x0f, y0 = (long long)y0f;
    auto clampi = [](long long v, int hi) { return (int)(v < 0 ? 0 : (v > hi ? hi : v)); };
    const int x0c = clampi(x0, w - 1), x1c = clampi(x0 + 1, w - 1);
    const int y0c = clampi(y0, h - 1), y1c = clampi(y0 + 1, h - 1);
    const double v00 = img[y0c * w + x0c], v01 = img[y0c * w + x1c];
    const double v10 = img[y1c * w + x0c], v11 = img[y1c * w + x1c];
    const double top = __dadd_rn(v00, __dmul_rn(fx, __dsub_rn(v01, v00)));
    const double bot = __dadd_rn(v10, __dmul_rn(fx, __dsub_rn(v11, v10)));
    double v = floor(__dadd_rn(__dadd_rn(top, __dmul_rn(fy, __dsub_rn(bot, top))), 0.5));
    v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
    return (int)v;
}

// base = resize_bilinear(template n x n -> m x m)
__global__ void probe_base_kernel(const uint8_t* __restrict__ tpl, int n, int m, uint8_t* __restrict__ base) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= m * m) return;
    const int i = p % m, j = p / m;
    const double ratio = __ddiv_rn((double)n, (double)m);  // image_io.py:174-175 w / out_w
    const double xs = __dsub_rn(__dmul_rn(__dadd_rn((double)i, 0.5), ratio), 0.5);
    const double ys = __dsub_rn(__dmul_rn(__dadd_rn((double)j, 0.5), ratio), 0.5);
    base[p] = (uint8_t)sample_q(tpl, n, n, xs, ys);
}

// The three A planes: I, (I^2 >> 8), (I^2 & 255), each H rows of `pitch`
// bytes (W data columns, then zeros).
__global__ void planes_kernel(const uint8_t* __restrict__ img, int W, long long H, long long pitch,
                              uint8_t* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= H * pitch) return;
    const long long y = i / pitch, x = i % pitch;
    const int v = x < W ? img[y * W + x] : 0;
    const int v2 = v * v;
    const long long ps = H * pitch;
    out[i] = (uint8_t)v;
    out[ps + i] = (uint8_t)(v2 >> 8);
    out[2 * ps + i] = (uint8_t)(v2 & 255);
}

// One CTA per angle a: _rotate_with_mask(base, angle, fill=0)
// (image_io.py:181-203) and the angle's exact sums (support pixels, sum of
// the masked probe b = probe * sel, sum of b^2).  The window pixel
// (r, j) of K index r * kr + j (j < kr: the row padded to kr columns) is
// written into the u8 m16n8k32 B fragment of its angle group:
//   bfrag[((group * ksteps + ks) * BT + tile) * 32 + lane] = {b0, b1},
//   b0 = B[k = 4t .. 4t+3][n = g], b1 = B[k = 16 + 4t ..][n = g]
// (g = lane >> 2, t = lane & 3), tile < NT: masked probe, else support.
__global__ void probe_rotate_kernel(const uint8_t* __restrict__ base, int m, int kr, int na,
                                    const double* __restrict__ cs, const double* __restrict__ sn,
                                    uint8_t* __restrict__ bfrag, long long* __restrict__ stats) {
    const int a = blockIdx.x;
    const double c = cs[a], s = sn[a], ns = -sn[a];
    const double cx = __ddiv_rn((double)(m - 1), 2.0), cy = cx;
    const int group = a / MAX_GROUP_ANGLES, ag = a % MAX_GROUP_ANGLES, nt = ag / 8, ncol = ag % 8;
    const long long ksteps = (long long)m * kr / 32;
    long long nm = 0, bs = 0, bq = 0;
    for (long long p = threadIdx.x; p < (long long)m * kr; p += blockDim.x) {
        const int gy = (int)(p / kr), gx = (int)(p % kr);
        int b = 0, sel = 0;
        if (gx < m) {
            const double dx = __dsub_rn((double)gx, cx), dy = __dsub_rn((double)gy, cy);
            const double sx = __dadd_rn(__dadd_rn(__dmul_rn(c, dx), __dmul_rn(s, dy)), cx);
            const double sy = __dadd_rn(__dadd_rn(__dmul_rn(ns, dx), __dmul_rn(c, dy)), cy);
            const double hi = __dsub_rn((double)m, 0.5);
            if (sx >= -0.5 && sx <= hi && sy >= -0.5 && sy <= hi) {
                sel = 1;
                b = sample_q(base, m, m, sx, sy);
            }
        }
        nm += sel;
        bs += b;
        bq += (long long)b * b;
        // fragment position of (k = p % 32 within k-step ks, n = ncol)
        const long long ks = p / 32;
        const int k = (int)(p % 32);
        const int hi16 = k >= 16, kk = k & 15, t = kk >> 2, byte = kk & 3;
        const int lane = ncol * 4 + t;
        const long long slot0 = (((long long)group * ksteps + ks) * BT + nt) * 32 + lane;
        const long long slot1 = (((long long)group * ksteps + ks) * BT + NT + nt) * 32 + lane;
        bfrag[slot0 * 8 + hi16 * 4 + byte] = (uint8_t)b;
        bfrag[slot1 * 8 + hi16 * 4 + byte] = (uint8_t)sel;
    }
    __shared__ long long red[3][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        nm += __shfl_down_sync(FULL, nm, o);
        bs += __shfl_down_sync(FULL, bs, o);
        bq += __shfl_down_sync(FULL, bq, o);
    }
    if (lane == 0) { red[0][warp] = nm; red[1][warp] = bs; red[2][warp] = bq; }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t3[3] = {0, 0, 0};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            for (int q = 0; q < 3; ++q) t3[q] += red[q][w];
        for (int q = 0; q < 3; ++q) stats[a * 3 + q] = t3[q];
    }
}

__device__ __forceinline__ void mma_u8(int (&d)[4], const unsigned (&a)[4], uint2 b) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

// 4 bytes at an arbitrary address (two aligned loads and a funnel shift)
__device__ __forceinline__ unsigned ld_u32_unaligned(const uint8_t* p) {
    const uintptr_t u = reinterpret_cast<uintptr_t>(p);
    const unsigned* q = reinterpret_cast<const unsigned*>(u & ~(uintptr_t)3);
    return __funnelshift_r(__ldg(q), __ldg(q + 1), (unsigned)(u & 3) * 8);
}

struct Best {
    double score;
    long long idx;
};
__device__ __forceinline__ bool better(const Best& a, const Best& b) {
    return a.score > b.score || (a.score == b.score && a.idx < b.idx);
}

// second_stage.py:142-152 for one (candidate, angle): float64, NumPy's order
__device__ __forceinline__ double ncc_score(long long ab, long long a_sum_i, long long a_ss_i, const long long* st) {
    const double nm = (double)st[0], b_sum = (double)st[1];
    const double var_b = __dsub_rn((double)st[2], __ddiv_rn(__dmul_rn(b_sum, b_sum), nm));  // :133-135
    const double a_sum = (double)a_sum_i;
    const double var_a = __dsub_rn((double)a_ss_i, __ddiv_rn(__dmul_rn(a_sum, a_sum), nm));
    if (!(var_a > 1e-9 && var_b > 1e-9)) return 0.0;
    const double num = __dsub_rn((double)ab, __dmul_rn(a_sum, __ddiv_rn(b_sum, nm)));
    return __ddiv_rn(num, __dsqrt_rn(__dmul_rn(var_a, var_b)));
}

// One CTA per TM candidates, one warp per 16: K loops over the window rows
// r (and kr/32 segments of each); every k-step gathers the 32-pixel segment
// of the warp's 16 windows from the three planes into A fragments and runs
// 4 x NT mma: I x probe, I x support, Hi x support, Lo x support.
// r_flush > 0: int32 accumulators move into int64 shared memory every
// r_flush rows (sums of up to r_flush * m pixels of 255^2 fit int32).
__global__ void __launch_bounds__(FUSED_WARPS * 32) fused_kernel(
    const uint8_t* __restrict__ planes, long long pitch, long long plane_stride, const int* __restrict__ rows,
    int row_cols, long long first, long long count, int m, int kr, const uint2* __restrict__ bfrag, int na_g, int a0,
    const long long* __restrict__ stats, int r_flush, double* __restrict__ part_score,
    long long* __restrict__ part_idx) {
    extern __shared__ long long acc64[];  // [threads][4 * NT * 4] when r_flush > 0
    __shared__ double sc[TM][MAX_GROUP_ANGLES];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
    const long long cb = (long long)blockIdx.x * TM + warp * 16;
    const long long ci0 = cb + g, ci1 = cb + g + 8;
    const int lo = (m - 1) / 2;
    auto origin = [&](long long ci) -> long long {
        const long long r = first + (ci < count ? ci : 0);
        return (long long)(rows[r * row_cols + 1] - lo) * pitch + (rows[r * row_cols] - lo);
    };
    const long long o0 = origin(ci0), o1 = origin(ci1);
    int acc[4][NT][4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[q][j][e] = 0;
    const int segs = kr / 32;
    long long* my64 = acc64 + (long long)threadIdx.x * (4 * NT * 4);
    if (r_flush > 0)
        for (int i = 0; i < 4 * NT * 4; ++i) my64[i] = 0;
    for (int r = 0; r < m; ++r) {
        const long long rowoff = (long long)r * pitch;
        for (int sg = 0; sg < segs; ++sg) {
            const long long ks = (long long)r * segs + sg;
            const int col = sg * 32;
            unsigned A[3][4];
#pragma unroll
            for (int p = 0; p < 3; ++p) {
                const uint8_t* pl = planes + p * plane_stride + rowoff + col + 4 * t;
                A[p][0] = ld_u32_unaligned(pl + o0);
                A[p][1] = ld_u32_unaligned(pl + o1);
                A[p][2] = ld_u32_unaligned(pl + o0 + 16);
                A[p][3] = ld_u32_unaligned(pl + o1 + 16);
            }
            const uint2* bf = bfrag + ks * BT * 32 + lane;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const uint2 bp = __ldg(bf + j * 32), bm = __ldg(bf + (NT + j) * 32);
                mma_u8(acc[0][j], A[0], bp);
                mma_u8(acc[1][j], A[0], bm);
                mma_u8(acc[2][j], A[1], bm);
                mma_u8(acc[3][j], A[2], bm);
            }
        }
        if (r_flush > 0 && ((r + 1) % r_flush == 0 || r + 1 == m)) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int j = 0; j < NT; ++j)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        my64[(q * NT + j) * 4 + e] += acc[q][j][e];
                        acc[q][j][e] = 0;
                    }
        }
    }
    // epilogue: this thread holds rows g, g+8 x columns 2t, 2t+1 of every n-tile
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int row = warp * 16 + g + (e >= 2 ? 8 : 0);
            const int ag = j * 8 + 2 * t + (e & 1);
            long long v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = r_flush > 0 ? my64[(q * NT + j) * 4 + e] : (long long)acc[q][j][e];
            const long long ci = (long long)blockIdx.x * TM + row;
            double score = -1.0 / 0.0;
            if (ag < na_g && ci < count) score = ncc_score(v[0], v[1], 256 * v[2] + v[3], stats + (a0 + ag) * 3);
            sc[row][ag] = score;
        }
    __syncthreads();
    // best per angle over this CTA's candidates (np.argmax: the first on ties)
    for (int ag = threadIdx.x; ag < na_g; ag += blockDim.x) {
        Best b{-1.0 / 0.0, -1};
        for (int row = 0; row < TM; ++row) {
            const long long ci = (long long)blockIdx.x * TM + row;
            if (ci >= count) break;
            const Best c{sc[row][ag], ci};
            if (b.idx < 0 || better(c, b)) b = c;
        }
        part_score[(long long)blockIdx.x * MAX_GROUP_ANGLES + ag] = b.score;
        part_idx[(long long)blockIdx.x * MAX_GROUP_ANGLES + ag] = b.idx;
    }
}

// best per angle over the CTAs' partial results, in candidate order
__global__ void reduce_kernel(const double* __restrict__ part_score, const long long* __restrict__ part_idx,
                              long long n_parts, int na_g, double* __restrict__ best_score,
                              long long* __restrict__ best_idx) {
    const int ag = blockIdx.x;
    Best b{-1.0 / 0.0, -1};
    for (long long i = threadIdx.x; i < n_parts; i += blockDim.x) {
        const Best c{part_score[i * MAX_GROUP_ANGLES + ag], part_idx[i * MAX_GROUP_ANGLES + ag]};
        if (c.idx >= 0 && (b.idx < 0 || better(c, b))) b = c;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const Best c{__shfl_down_sync(FULL, b.score, o), __shfl_down_sync(FULL, b.idx, o)};
        if (c.idx >= 0 && (b.idx < 0 || better(c, b))) b = c;
    }
    __shared__ Best wb[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) wb[warp] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
        Best r = wb[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (wb[w].idx >= 0 && (r.idx < 0 || better(wb[w], r))) r = wb[w];
        best_score[ag] = r.score;
        best_idx[ag] = r.idx;
    }
}

}  // namespace
}  // namespace ss

extern "C" {

int64_t ss_match_plane_pitch(int64_t W) { return (W + ss::PLANE_PAD + 15) / 16 * 16; }

int ss_match_planes(const uint8_t* d_img, int64_t W, int64_t H, uint8_t* d_planes, int64_t pitch, void* stream) {
    if (!d_img || !d_planes || W < 1 || H < 1 || pitch < ss_match_plane_pitch(W)) {
        ss::set_error("bad match plane arguments");
        return SS_EINVAL;
    }
    const long long n = H * pitch;
    ss::planes_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ss::as_stream(stream)>>>(d_img, (int)W, H, pitch,
                                                                                   d_planes);
    ss::note_launch();
    return ss::check_launch("planes_kernel");
}

size_t ss_match_probe_bytes(int32_t m, int32_t n_angles) {
    const int64_t kr = (m + 31) / 32 * 32, groups = (n_angles + ss::MAX_GROUP_ANGLES - 1) / ss::MAX_GROUP_ANGLES;
    return (size_t)groups * (size_t)(m * kr / 32) * ss::BT * 32 * 8;
}

int ss_match_probes(const uint8_t* d_template, int32_t n, int32_t m, int32_t n_angles, const double* d_cos,
                    const double* d_sin, uint8_t* d_bfrag, long long* d_stats, uint8_t* d_base, void* stream) {
    if (!d_template || !d_cos || !d_sin || !d_bfrag || !d_stats || !d_base || n < 1 || m < 1 || n_angles < 1) {
        ss::set_error("bad match probe arguments");
        return SS_EINVAL;
    }
    cudaStream_t s = ss::as_stream(stream);
    if (cudaMemsetAsync(d_bfrag, 0, ss_match_probe_bytes(m, n_angles), s) != cudaSuccess)
        return ss::check_launch("memset");
    ss::probe_base_kernel<<<(unsigned)((m * m + 255) / 256), 256, 0, s>>>(d_template, n, m, d_base);
    ss::note_launch();
    if (int e = ss::check_launch("probe_base_kernel")) return e;
    ss::probe_rotate_kernel<<<(unsigned)n_angles, 256, 0, s>>>(d_base, m, (m + 31) / 32 * 32, n_angles, d_cos, d_sin,
                                                              d_bfrag, d_stats);
    ss::note_launch();
    return ss::check_launch("probe_rotate_kernel");
}

int64_t ss_match_parts(int64_t count) { return (count + ss::TM - 1) / ss::TM; }

int ss_match_fused(const uint8_t* d_planes, int64_t W, int64_t H, int64_t pitch, const int32_t* d_rows,
                   int32_t row_cols, int64_t first, int64_t count, int32_t m, const uint8_t* d_bfrag, int32_t n_angles,
                   int32_t group, const long long* d_stats, double* d_part_score, long long* d_part_idx,
                   double* d_best_score, long long* d_best_idx, void* stream) {
    if (!d_planes || !d_rows || row_cols < 2 || first < 0 || count < 1 || m < 1 || m > W || m > H || !d_bfrag ||
        n_angles < 1 || group < 0 || group * ss::MAX_GROUP_ANGLES >= n_angles || !d_stats || !d_part_score ||
        !d_part_idx || !d_best_score || !d_best_idx || pitch < ss_match_plane_pitch(W)) {
        ss::set_error("bad match arguments");
        return SS_EINVAL;
    }
    cudaStream_t s = ss::as_stream(stream);
    const int kr = (m + 31) / 32 * 32;
    const int a0 = group * ss::MAX_GROUP_ANGLES, na_g = std::min(ss::MAX_GROUP_ANGLES, (int)n_angles - a0);
    const long long ksteps = (long long)m * kr / 32;
    const uint2* bf = reinterpret_cast<const uint2*>(d_bfrag) + (long long)group * ksteps * ss::BT * 32;
    // rows of m pixels whose sums fit int32 (255^2 per pixel)
    const long long rows_fit = 2147483647LL / (65025LL * m);
    const int r_flush = rows_fit >= m ? 0 : (int)std::max<long long>(1, rows_fit);
    const size_t smem = r_flush > 0 ? (size_t)ss::FUSED_WARPS * 32 * 4 * ss::NT * 4 * sizeof(long long) : 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(ss::fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long parts = ss_match_parts(count);
    ss::fused_kernel<<<(unsigned)parts, ss::FUSED_WARPS * 32, smem, s>>>(
        d_planes, pitch, pitch * H, d_rows, row_cols, first, count, m, kr, bf, na_g, a0, d_stats, r_flush,
        d_part_score, d_part_idx);
    ss::note_launch();
    if (int e = ss::check_launch("fused_kernel")) return e;
    ss::reduce_kernel<<<(unsigned)na_g, 256, 0, s>>>(d_part_score, d_part_idx, parts, na_g, d_best_score + a0,
                                                    d_best_idx + a0);
    ss::note_launch();
    return ss::check_launch("reduce_kernel");
}

}  // extern "C"
