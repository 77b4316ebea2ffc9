// ss_match.cu -- f3: the second stage, masked zero-mean NCC of every screened
// candidate against every rotated template probe (second_stage.py:106-204).
//
// The reference evaluates, per ladder size m, W @ [P | M] and (W*W) @ M in
// float64 (second_stage.py:136-150): W the candidates' m x m uint8 windows,
// P the masked rotated probes, M their 0/1 supports.  Every entry is an
// integer and every dot product is an integer below 2^53, so those float64
// matmuls are exact whatever their summation order -- and so is an integer
// GEMM.  This file builds the GEMM operands as int8 (value - 128, the offset
// removed exactly afterwards from row / column sums), the GEMMs run as
// library int8 tensor-core GEMMs (torch._int_mm / cuBLASLt, called from
// second_stage.py), and the epilogue replays the reference's float64
// elementwise sequence op for op (compiled with -fmad=false) and reduces the
// scores to the best candidate per angle with the reference's tie-break
// (first candidate on equal scores).
//
//   ss_match_probes   resize_bilinear(template, m, m) (image_io.py:164-178) and
//                     _rotate_with_mask per angle (image_io.py:181-203; cos/sin
//                     from the host's libm, as NumPy computes them), probe
//                     operands and per-angle sums
//   ss_match_gather   the candidates' windows (sliding_window_view,
//                     second_stage.py:131-141) as three int8 operands: w, and
//                     w^2 split into its high and low bytes
//   ss_match_scores   exact int64 dot products -> float64 scores
//                     (second_stage.py:142-152) -> best (score, candidate) per
//                     angle over the chunk
#include "ss_common.cuh"

namespace ss {
namespace {

constexpr unsigned FULL = 0xffffffffu;

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

// One CTA per angle: _rotate_with_mask(base, angle, fill=0) (image_io.py:181-203),
// the probe operand columns and the angle's exact sums (nm, sum b, sum b^2).
// B1: k_pad x n1 row-major, column a = b - 128, column na + a = sel - 128;
// B2: k_pad x n2, column a = sel - 128; padded rows / columns hold -128 (value 0).
__global__ void probe_rotate_kernel(const uint8_t* __restrict__ base, int m, int na, const double* __restrict__ cs,
                                    const double* __restrict__ sn, int8_t* __restrict__ B1, int n1,
                                    int8_t* __restrict__ B2, int n2, int k_pad, long long* __restrict__ stats) {
    const int a = blockIdx.x;
    const double c = cs[a], s = sn[a], ns = -sn[a];
    const double cx = __ddiv_rn((double)(m - 1), 2.0), cy = cx;
    long long nm = 0, bs = 0, bq = 0;
    for (int p = threadIdx.x; p < k_pad; p += blockDim.x) {
        int b = 0, sel = 0;
        if (p < m * m) {
            const int gx = p % m, gy = p / m;
            const double dx = __dsub_rn((double)gx, cx), dy = __dsub_rn((double)gy, cy);
            const double sx = __dadd_rn(__dadd_rn(__dmul_rn(c, dx), __dmul_rn(s, dy)), cx);
            const double sy = __dadd_rn(__dadd_rn(__dmul_rn(ns, dx), __dmul_rn(c, dy)), cy);
            const bool inside = sx >= -0.5 && sx <= __dsub_rn((double)m, 0.5) && sy >= -0.5 && sy <= __dsub_rn((double)m, 0.5);
            if (inside) {
                sel = 1;
                b = sample_q(base, m, m, sx, sy);
            }
        }
        nm += sel;
        bs += b;
        bq += (long long)b * b;
        B1[(long long)p * n1 + a] = (int8_t)(b - 128);
        B1[(long long)p * n1 + na + a] = (int8_t)(sel - 128);
        B2[(long long)p * n2 + a] = (int8_t)(sel - 128);
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
        long long t[3] = {0, 0, 0};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            for (int q = 0; q < 3; ++q) t[q] += red[q][w];
        for (int q = 0; q < 3; ++q) stats[a * 3 + q] = t[q];
    }
}

// padded operand columns (angles na .. n-1) of B1 / B2: value 0 (-128)
__global__ void probe_pad_kernel(int8_t* __restrict__ B, int n, int first, int k_pad) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int cols = n - first;
    if (cols <= 0 || i >= (long long)k_pad * cols) return;
    B[(i / cols) * n + first + i % cols] = (int8_t)-128;
}

// One warp per candidate: its window row-major into A1 = w - 128,
// A2 = (w^2 >> 8) - 128, A3 = (w^2 & 255) - 128 (k_pad columns, padding
// value 0) and the exact row sums of w, w^2 >> 8 and w^2 & 255.
__global__ void gather_kernel(const uint8_t* __restrict__ img, int W, const int* __restrict__ rows, int row_cols,
                              long long first, long long count, long long count_pad, int m, int k_pad,
                              int8_t* __restrict__ A1, int8_t* __restrict__ A2, int8_t* __restrict__ A3,
                              long long* __restrict__ rsum) {
    const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= count_pad) return;
    const int lo = (m - 1) / 2;
    int x0 = 0, y0 = 0;
    const bool real = i < count;
    if (real) {
        x0 = rows[(first + i) * row_cols + 0] - lo;
        y0 = rows[(first + i) * row_cols + 1] - lo;
    }
    int8_t* a1 = A1 + i * k_pad;
    int8_t* a2 = A2 + i * k_pad;
    int8_t* a3 = A3 + i * k_pad;
    long long s1 = 0, sh = 0, sl = 0;
    for (int p = lane; p < k_pad; p += 32) {
        int v = 0;
        if (real && p < m * m) v = img[(long long)(y0 + p / m) * W + x0 + p % m];
        const int v2 = v * v;
        s1 += v;
        sh += v2 >> 8;
        sl += v2 & 255;
        a1[p] = (int8_t)(v - 128);
        a2[p] = (int8_t)((v2 >> 8) - 128);
        a3[p] = (int8_t)((v2 & 255) - 128);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        s1 += __shfl_down_sync(FULL, s1, o);
        sh += __shfl_down_sync(FULL, sh, o);
        sl += __shfl_down_sync(FULL, sl, o);
    }
    if (lane == 0) {
        rsum[i * 3 + 0] = s1;
        rsum[i * 3 + 1] = sh;
        rsum[i * 3 + 2] = sl;
    }
}

struct Best {
    double score;
    long long idx;
};
__device__ __forceinline__ bool better(const Best& a, const Best& b) {
    return a.score > b.score || (a.score == b.score && a.idx < b.idx);
}

// sum over the k_pad columns of x * y from the int8 GEMM C of the offset
// operands x' = x - 128, y' = y - 128:  C + 128 sum x + 128 sum y - 128^2 k_pad
__device__ __forceinline__ long long unoffset(int c, long long sx, long long sy, long long k_pad) {
    return (long long)c + 128 * sx + 128 * sy - 16384 * k_pad;
}

__device__ __forceinline__ void reduce_best(Best& b) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        Best t{__shfl_down_sync(FULL, b.score, o), __shfl_down_sync(FULL, b.idx, o)};
        if (better(t, b)) b = t;
    }
}

// Scores of `count` candidates x na angles (second_stage.py:142-152: float64
// in NumPy's op order, exact integer dot products) and the best (score,
// candidate) per angle over this chunk (np.argmax: the first candidate on
// ties).  Grid: one CTA per angle.
__global__ void __launch_bounds__(256) scores_kernel(const int* __restrict__ C1, int n1, const int* __restrict__ C2,
                                                     const int* __restrict__ C3, int n2,
                                                     const long long* __restrict__ rsum,
                                                     const long long* __restrict__ stats, long long count, int na,
                                                     int k_pad, long long base, double* __restrict__ best_score,
                                                     long long* __restrict__ best_idx) {
    const int a = blockIdx.x;
    const long long K = k_pad;
    const long long nm_i = stats[a * 3 + 0], bs_i = stats[a * 3 + 1], bq_i = stats[a * 3 + 2];
    const double nm = (double)nm_i, b_sum = (double)bs_i;
    // second_stage.py:133-135: var_b = (probes * probes).sum(axis=1) - b_sum * b_sum / nm
    const double var_b = __dsub_rn((double)bq_i, __ddiv_rn(__dmul_rn(b_sum, b_sum), nm));
    const bool live = var_b > 1e-9;
    const double bmean = __ddiv_rn(b_sum, nm);
    Best best{-1.0 / 0.0, 0x7fffffffffffffffLL};
    for (long long i = threadIdx.x; i < count; i += blockDim.x) {
        const long long sw = rsum[i * 3], sh = rsum[i * 3 + 1], sl = rsum[i * 3 + 2];
        const long long ab = unoffset(C1[i * n1 + a], sw, bs_i, K);           // w @ probes
        const long long a_sum_i = unoffset(C1[i * n1 + na + a], sw, nm_i, K);  // w @ masks
        const long long a_ss_i = 256 * unoffset(C2[i * n2 + a], sh, nm_i, K) + unoffset(C3[i * n2 + a], sl, nm_i, K);
        const double a_sum = (double)a_sum_i;
        // :144-150  var_a = a_ss - a_sum * a_sum / nm; ok; num; denom; scores
        const double var_a = __dsub_rn((double)a_ss_i, __ddiv_rn(__dmul_rn(a_sum, a_sum), nm));
        const bool ok = var_a > 1e-9 && live;
        double score = 0.0;
        if (ok) {
            const double num = __dsub_rn((double)ab, __dmul_rn(a_sum, bmean));
            score = __ddiv_rn(num, __dsqrt_rn(__dmul_rn(var_a, var_b)));
        }
        const Best t{score, i};
        if (better(t, best)) best = t;
    }
    reduce_best(best);
    __shared__ double ss[8];
    __shared__ long long si[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { ss[warp] = best.score; si[warp] = best.idx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        Best b{ss[0], si[0]};
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            const Best t{ss[w], si[w]};
            if (better(t, b)) b = t;
        }
        best_score[a] = b.score;
        best_idx[a] = b.idx == 0x7fffffffffffffffLL ? -1 : base + b.idx;
    }
}

}  // namespace
}  // namespace ss

static bool probe_args_ok(int n, int m, int na, int k_pad, int n1, int n2) {
    return n >= 1 && m >= 1 && na >= 1 && k_pad >= m * m && n1 >= 2 * na && n2 >= na;
}

extern "C" {

int ss_match_probes(const uint8_t* d_template, int32_t n, int32_t m, int32_t n_angles, const double* d_cos,
                    const double* d_sin, int8_t* d_b1, int32_t n1, int8_t* d_b2, int32_t n2, int32_t k_pad,
                    long long* d_stats, uint8_t* d_base, void* stream) {
    if (!d_template || !d_cos || !d_sin || !d_b1 || !d_b2 || !d_stats || !d_base ||
        !probe_args_ok(n, m, n_angles, k_pad, n1, n2)) {
        ss::set_error("bad match probe arguments");
        return SS_EINVAL;
    }
    cudaStream_t s = ss::as_stream(stream);
    ss::probe_base_kernel<<<(unsigned)((m * m + 255) / 256), 256, 0, s>>>(d_template, n, m, d_base);
    ss::note_launch();
    if (int e = ss::check_launch("probe_base_kernel")) return e;
    ss::probe_rotate_kernel<<<(unsigned)n_angles, 256, 0, s>>>(d_base, m, n_angles, d_cos, d_sin, d_b1, n1, d_b2, n2,
                                                              k_pad, d_stats);
    ss::note_launch();
    if (int e = ss::check_launch("probe_rotate_kernel")) return e;
    const long long p1 = (long long)k_pad * (n1 - 2 * n_angles), p2 = (long long)k_pad * (n2 - n_angles);
    if (p1 > 0) {
        ss::probe_pad_kernel<<<(unsigned)((p1 + 255) / 256), 256, 0, s>>>(d_b1, n1, 2 * n_angles, k_pad);
        ss::note_launch();
    }
    if (p2 > 0) {
        ss::probe_pad_kernel<<<(unsigned)((p2 + 255) / 256), 256, 0, s>>>(d_b2, n2, n_angles, k_pad);
        ss::note_launch();
    }
    return ss::check_launch("probe_pad_kernel");
}

int ss_match_gather(const uint8_t* d_img, int64_t W, int64_t H, const int32_t* d_rows, int32_t row_cols,
                    int64_t first, int64_t count, int64_t count_pad, int32_t m, int32_t k_pad, int8_t* d_a1,
                    int8_t* d_a2, int8_t* d_a3, long long* d_rsum, void* stream) {
    if (!d_img || !d_rows || row_cols < 2 || first < 0 || count < 0 || count_pad < count || m < 1 ||
        k_pad < m * m || m > W || m > H || !d_a1 || !d_a2 || !d_a3 || !d_rsum) {
        ss::set_error("bad match gather arguments");
        return SS_EINVAL;
    }
    if (count_pad == 0) return SS_OK;
    const long long threads = count_pad * 32;
    ss::gather_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, ss::as_stream(stream)>>>(
        d_img, (int)W, d_rows, row_cols, first, count, count_pad, m, k_pad, d_a1, d_a2, d_a3, d_rsum);
    ss::note_launch();
    return ss::check_launch("gather_kernel");
}

int ss_match_scores(const int32_t* d_c1, int32_t n1, const int32_t* d_c2, const int32_t* d_c3, int32_t n2,
                    const long long* d_rsum, const long long* d_stats, int64_t count, int32_t n_angles, int32_t k_pad,
                    int64_t base, double* d_best_score, long long* d_best_idx, void* stream) {
    if (!d_c1 || !d_c2 || !d_c3 || !d_rsum || !d_stats || count < 0 || n_angles < 1 || n1 < 2 * n_angles ||
        n2 < n_angles || !d_best_score || !d_best_idx) {
        ss::set_error("bad match score arguments");
        return SS_EINVAL;
    }
    ss::scores_kernel<<<(unsigned)n_angles, 256, 0, ss::as_stream(stream)>>>(d_c1, n1, d_c2, d_c3, n2, d_rsum, d_stats,
                                                                          count, n_angles, k_pad, base, d_best_score,
                                                                          d_best_idx);
    ss::note_launch();
    return ss::check_launch("scores_kernel");
}

}  // extern "C"
