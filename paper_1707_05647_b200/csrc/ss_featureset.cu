// ss_featureset.cu -- f2: template-side ring features of every rescale on the GPU.
//
// Replaces the per-rescale body of build_feature_set (screening.py:238-248):
// resize_bilinear (image_io.py:164-178 via _sample_bilinear :131-156 and
// _quantize_levels :159-161), crop_center (image_io.py:216-228) and the
// patch's ring features (features.py:220-224 -> :322-370).  One CTA per
// (ladder size, rescale k) instance: every pixel of the m x m crop is
// resampled on the fly from the n x n template and accumulated, with its
// 1-based x/y weights, into the exact int64 square / diamond sums of each
// ring; thread 0 then evaluates the features in the reference's fp64 order.
// Compiled with -fmad=false (bit parity with NumPy, as the host version in
// ss_template.cpp); the guard-banded key sets are built on the host from
// the returned features (ss_keys_from_features).
#include "ss_common.cuh"

namespace ss {
namespace {

constexpr int TPB = 256;
constexpr int NSUM = 8;  // per ring: square (s1, sx, sy, s2), diamond (s1, sx, sy, s2)

// image_io.py:131-161 at one output pixel of the k x k resize of the n x n template
__device__ __forceinline__ int resampled(const uint8_t* __restrict__ tpl, int n, double ratio, int i, int j) {
    const double xs = __dsub_rn(__dmul_rn(__dadd_rn((double)i, 0.5), ratio), 0.5);
    const double ys = __dsub_rn(__dmul_rn(__dadd_rn((double)j, 0.5), ratio), 0.5);
    const double x0f = floor(xs), y0f = floor(ys);
    const double fx = __dsub_rn(xs, x0f), fy = __dsub_rn(ys, y0f);
    const int x0 = min(max((int)x0f, 0), n - 1), x1 = min(max((int)x0f + 1, 0), n - 1);
    const int y0 = min(max((int)y0f, 0), n - 1), y1 = min(max((int)y0f + 1, 0), n - 1);
    const double v00 = __ldg(tpl + y0 * n + x0), v01 = __ldg(tpl + y0 * n + x1);
    const double v10 = __ldg(tpl + y1 * n + x0), v11 = __ldg(tpl + y1 * n + x1);
    const double top = __dadd_rn(v00, __dmul_rn(fx, __dsub_rn(v01, v00)));
    const double bot = __dadd_rn(v10, __dmul_rn(fx, __dsub_rn(v11, v10)));
    double v = floor(__dadd_rn(__dadd_rn(top, __dmul_rn(fy, __dsub_rn(bot, top))), 0.5));
    v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
    return (int)v;
}

// desc row: [m, k, n_rings, 0, n_0, d_0, n_1, d_1, ...]
__global__ void __launch_bounds__(TPB) template_features_kernel(const uint8_t* __restrict__ tpl, int n,
                                                                const int* __restrict__ desc, int desc_stride,
                                                                double* __restrict__ out) {
    const int* d = desc + (long long)blockIdx.x * desc_stride;
    const int m = d[0], k = d[1], R = d[2];
    const int off = (k - m) / 2;  // crop_center offsets (image_io.py:226-227)
    const int c = (m - 1) / 2;    // ring centre (screening.py:235)
    const double ratio = __ddiv_rn((double)n, (double)k);
    __shared__ long long red[TPB / 32][NSUM];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int r = 0; r < R; ++r) {
        const int nr = d[4 + 2 * r], dr = d[5 + 2 * r];
        // bounding box of the ring's square [c-nr+1, c+nr] and diamond |dx|+|dy| <= dr
        const int lo = c - max(nr - 1, dr), hi = c + max(nr, dr), side = hi - lo + 1;
        long long acc[NSUM];
#pragma unroll
        for (int q = 0; q < NSUM; ++q) acc[q] = 0;
        for (long long p = threadIdx.x; p < (long long)side * side; p += TPB) {
            const int y = lo + (int)(p / side), x = lo + (int)(p % side);
            const bool in_sq = x >= c - nr + 1 && x <= c + nr && y >= c - nr + 1 && y <= c + nr;
            const bool in_di = (x > c ? x - c : c - x) + (y > c ? y - c : c - y) <= dr;
            if (!in_sq && !in_di) continue;
            const long long v = resampled(tpl, n, ratio, x + off, y + off);
            const long long wx = (long long)(x + 1) * v, wy = (long long)(y + 1) * v, v2 = v * v;
            if (in_sq) { acc[0] += v; acc[1] += wx; acc[2] += wy; acc[3] += v2; }
            if (in_di) { acc[4] += v; acc[5] += wx; acc[6] += wy; acc[7] += v2; }
        }
#pragma unroll
        for (int q = 0; q < NSUM; ++q) {
            long long v = acc[q];
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) v += __shfl_down_sync(0xffffffffu, v, s);
            if (lane == 0) red[warp][q] = v;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            long long S[NSUM];
            for (int q = 0; q < NSUM; ++q) {
                long long t = 0;
                for (int w = 0; w < TPB / 32; ++w) t += red[w][q];
                S[q] = t;
            }
            const long long n64 = nr, d64 = dr;
            // features.py:94-102 (square) / :346-353 (diamond) / :364-370 (octagon)
            const double cq = (double)(4 * n64 * n64), wq = (double)(2 * n64 * n64 * n64);
            const double mq = __ddiv_rn((double)S[0], cq);
            const double vq = __dsub_rn(__ddiv_rn((double)S[3], cq), __dmul_rn(mq, mq));
            const double sdq = __dsqrt_rn(vq > 0.0 ? vq : 0.0);
            const double gxq = __ddiv_rn(__dsub_rn((double)S[1], __dmul_rn(__dadd_rn((double)c, 1.5), (double)S[0])), wq);
            const double gyq = __ddiv_rn(__dsub_rn((double)S[2], __dmul_rn(__dadd_rn((double)c, 1.5), (double)S[0])), wq);
            const double cd = (double)(2 * d64 * d64 + 2 * d64 + 1);
            const double wd = (double)(2 * d64 * d64 + d64 * (d64 - 1) * (2 * d64 - 1) / 3);
            const double md = __ddiv_rn((double)S[4], cd);
            const double vd = __dsub_rn(__ddiv_rn((double)S[7], cd), __dmul_rn(md, md));
            const double sdd = __dsqrt_rn(vd > 0.0 ? vd : 0.0);
            const double gxd = __ddiv_rn(__dsub_rn((double)S[5], __dmul_rn(__dadd_rn((double)c, 1.0), (double)S[4])), wd);
            const double gyd = __ddiv_rn(__dsub_rn((double)S[6], __dmul_rn(__dadd_rn((double)c, 1.0), (double)S[4])), wd);
            const double gx = __dmul_rn(__dadd_rn(gxq, gxd), 0.5), gy = __dmul_rn(__dadd_rn(gyq, gyd), 0.5);
            double* o = out + ((long long)blockIdx.x * SS_MAX_RINGS + r) * 3;
            o[0] = __dmul_rn(__dadd_rn(mq, md), 0.5);
            o[1] = __dmul_rn(__dadd_rn(sdq, sdd), 0.5);
            o[2] = __dsqrt_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)));
        }
        __syncthreads();
    }
}

}  // namespace
}  // namespace ss

extern "C" int ss_template_features_device(const uint8_t* d_template, int32_t n, int32_t n_inst, const int32_t* d_desc,
                                           int32_t desc_stride, double* d_out, void* stream) {
    if (!d_template || n < 1 || n_inst < 0 || !d_desc || desc_stride < 4 + 2 * SS_MAX_RINGS || !d_out) {
        ss::set_error("bad template feature arguments");
        return SS_EINVAL;
    }
    if (n_inst == 0) return SS_OK;
    ss::template_features_kernel<<<(unsigned)n_inst, ss::TPB, 0, ss::as_stream(stream)>>>(d_template, n, d_desc,
                                                                                          desc_stride, d_out);
    ss::note_launch();
    return ss::check_launch("template_features_kernel");
}

// The whole f2 round trip in one host call: template bytes (host) to the
// device, the features of every instance, the result into pinned host memory
// and an event recorded after it -- no host synchronisation.
extern "C" int ss_template_features_async(const uint8_t* h_template, int32_t n, int32_t n_inst, const int32_t* d_desc,
                                          int32_t desc_stride, uint8_t* d_template, double* d_out, double* h_out,
                                          void* stream, void* event) {
    if (!h_template || !d_template || !h_out || n < 1) {
        ss::set_error("bad template feature arguments");
        return SS_EINVAL;
    }
    cudaStream_t s = ss::as_stream(stream);
    if (cudaMemcpyAsync(d_template, h_template, (size_t)n * n, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return ss::check_launch("template upload");
    if (int e = ss_template_features_device(d_template, n, n_inst, d_desc, desc_stride, d_out, stream)) return e;
    const size_t bytes = (size_t)n_inst * SS_MAX_RINGS * 3 * sizeof(double);
    if (bytes && cudaMemcpyAsync(h_out, d_out, bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return ss::check_launch("feature readback");
    if (event && cudaEventRecord(reinterpret_cast<cudaEvent_t>(event), s) != cudaSuccess)
        return ss::check_launch("event record");
    return SS_OK;
}
