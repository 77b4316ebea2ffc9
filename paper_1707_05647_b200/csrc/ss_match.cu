// ss_match.cu -- f3: the second stage, masked zero-mean NCC of every screened
// candidate against every rotated template probe (second_stage.py:106-204).
//
// The reference evaluates, per ladder size m, W @ [P | M] and (W*W) @ M in
// float64 (second_stage.py:136-150): W the candidates' m x m uint8 windows,
// P the masked rotated probes, M their 0/1 supports.  Every entry is an
// integer and every dot product an integer below 2^53, so those float64
// matmuls are exact whatever their summation order -- and so is an integer
// tensor-core GEMM.  One fused kernel per (size, group of <= 40 angles) runs
// it on the 5th-generation tensor cores: per CTA, 128 candidates (the UMMA M)
// x 48 angle columns (40 + 8 zero; UMMA N) x the window pixels (K, 64 bytes
// per pipeline stage): the CTA's threads gather the windows straight from
// the image planes into shared memory in the UMMA canonical K-major layout,
// the probes' B blocks come pre-laid-out from global memory, and one thread
// issues tcgen05.mma kind::i8 (u8 x u8 -> s32) into four TMEM accumulators
// -- I x P, I x M, (I^2 >> 8) x M, (I^2 & 255) x M -- with tcgen05.commit
// releasing each stage.  The epilogue reads TMEM (tcgen05.ld), replays the
// reference's float64 score sequence op for op (-fmad=false) and reduces to
// the best candidate per angle with the reference's tie-break (first
// candidate on equal scores, np.argmax).  When m is large enough for I x P to
// pass 2^31, its accumulator is drained into int64 shared memory every few
// window rows.
//
//   ss_match_planes   the image, and its squares' high / low bytes, as padded
//                     u8 planes (the three A operands)
//   ss_match_probes   resize_bilinear(template, m, m) (image_io.py:164-178) and
//                     _rotate_with_mask per angle (image_io.py:181-203; cos/sin
//                     from the host's libm, as NumPy computes them) as the B
//                     blocks, and per-angle sums
//   ss_match_fused    windows x probes -> scores -> best per angle per CTA,
//                     then the best per angle over the CTAs
#include <algorithm>

#include "ss_common.cuh"

namespace ss {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int MAX_GROUP_ANGLES = 40;  // angles per fused launch
constexpr int TM = 128;               // candidates per CTA: the UMMA M
constexpr int NB = 48;                // B rows per block: 40 angles + 8 zero rows (UMMA N, a multiple of 16)
constexpr int KB = 64;                // K bytes (window pixels) per pipeline stage: two 32-byte UMMA k-steps
constexpr int NSTAGE = 3;  // 90 KB of stages: two CTAs per SM
constexpr int A_BYTES = TM * KB;                             // one A plane's stage: 8 KB
constexpr int B_BYTES = NB * KB;                             // one B block's stage: 3 KB
constexpr int STAGE_BYTES = 3 * A_BYTES + 2 * B_BYTES;       // 30 KB
constexpr int CM_SBO = (KB / 16) * 128;                      // bytes between 8-row core-matrix groups
constexpr int TMEM_COLS = 256;                               // IP [0,48) IM [48,96) HI [96,144) LO [144,192)
constexpr int PLANE_PAD = 96;  // zero columns right of each plane row (the gather reads < 80 bytes past a window)

// Byte offset of (row, k) in a UMMA canonical K-major tile without swizzle:
// 8 x 16-byte core matrices, the KB / 16 of one 8-row group side by side
// (LBO = 128 bytes along K), the groups CM_SBO apart along M / N.
__host__ __device__ constexpr int canon(int row, int k) {
    return (row >> 3) * CM_SBO + (k >> 4) * 128 + (row & 7) * 16 + (k & 15);
}
// window rows padded to whole 16-byte pieces (a piece never straddles two rows)
__host__ __device__ constexpr int row_bytes(int m) { return (m + 15) / 16 * 16; }
// pipeline stages of one window (K = m * row_bytes(m), zero-padded to whole stages)
__host__ __device__ constexpr long long n_stages_of(int m) { return ((long long)m * row_bytes(m) + KB - 1) / KB; }
constexpr int THREADS = 256;  // 8 warps gather; warp w & 3 owns TMEM lanes 32 (w & 3) .. in the epilogue
// Candidates per CTA: 128 (the full UMMA M) unless that leaves SMs of a
// 148-SM B200 idle: then 64 or 32, the remaining accumulator rows unused
// (measured: 128 -> 64 at 32k candidates of m = 128 is slower, the MMAs'
// share is not negligible; below one CTA per SM the smaller tiles win).
__host__ __device__ constexpr int tile_log2(long long count) {
    return (count + 127) / 128 >= 148 ? 7 : ((count + 63) / 64 >= 148 ? 6 : 5);
}

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
// the masked probe b = probe * sel, sum of b^2).  Window pixel (r, j) is K
// index p = r * kr + j (j < kr: rows padded to 16 bytes); stage
// c = p / KB of angle group g holds two B blocks (masked probes, supports)
// of NB rows (angle within the group) x KB bytes in the canonical layout:
//   bops[((g * n_chunks + c) * 2 + blk) * B_BYTES + canon(angle, p % KB)].
__global__ void probe_rotate_kernel(const uint8_t* __restrict__ base, int m, int kr, int na,
                                    const double* __restrict__ cs, const double* __restrict__ sn,
                                    uint8_t* __restrict__ bops, long long* __restrict__ stats) {
    const int a = blockIdx.x;
    const double c = cs[a], s = sn[a], ns = -sn[a];
    const double cx = __ddiv_rn((double)(m - 1), 2.0), cy = cx;
    const int group = a / MAX_GROUP_ANGLES, ag = a % MAX_GROUP_ANGLES;
    const long long n_chunks = n_stages_of(m);
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
        const long long blk = ((long long)group * n_chunks + p / KB) * 2;
        const int off = canon(ag, (int)(p % KB));
        bops[blk * B_BYTES + off] = (uint8_t)b;
        bops[(blk + 1) * B_BYTES + off] = (uint8_t)sel;
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

// 16 bytes at an arbitrary address: the two aligned 16-byte blocks that
// hold them, words wo .. wo + 4 selected, then funnel-shifted by the byte offset
__device__ __forceinline__ uint4 ld16_unaligned(const uint8_t* p) {
    const uintptr_t u = reinterpret_cast<uintptr_t>(p);
    const uint4* q = reinterpret_cast<const uint4*>(u & ~(uintptr_t)15);
    const uint4 a = __ldg(q), b = __ldg(q + 1);
    const unsigned off = (unsigned)(u & 15), sh = (off & 3) * 8;
    const bool w2 = off & 8, w1 = off & 4;
    const unsigned t0 = w2 ? a.z : a.x, t1 = w2 ? a.w : a.y, t2 = w2 ? b.x : a.z, t3 = w2 ? b.y : a.w,
                   t4 = w2 ? b.z : b.x, t5 = w2 ? b.w : b.y;
    const unsigned s0 = w1 ? t1 : t0, s1 = w1 ? t2 : t1, s2 = w1 ? t3 : t2, s3 = w1 ? t4 : t3, s4 = w1 ? t5 : t4;
    return make_uint4(__funnelshift_r(s0, s1, sh), __funnelshift_r(s1, s2, sh), __funnelshift_r(s2, s3, sh),
                      __funnelshift_r(s3, s4, sh));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// shared-memory matrix descriptor: canonical K-major, no swizzle, LBO = 128
// bytes (the next 16 bytes of K), SBO = CM_SBO (the next 8 rows), version 1
__device__ __forceinline__ unsigned long long umma_desc(unsigned saddr) {
    return (unsigned long long)((saddr >> 4) & 0x3fffu) | ((unsigned long long)(128 >> 4) << 16) |
           ((unsigned long long)(CM_SBO >> 4) << 32) | (1ull << 46);
}
// instruction descriptor, kind::i8: D s32 (bits 4-5 = 2), A and B unsigned 8-bit,
// both K-major, N = NB (bits 17-22 = N >> 3), M = TM (bits 24-28 = M >> 4)
constexpr unsigned IDESC = (2u << 4) | ((unsigned)(NB >> 3) << 17) | ((unsigned)(TM >> 4) << 24);

__device__ __forceinline__ void umma_u8(unsigned tmem_d, unsigned long long da, unsigned long long db, bool acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(IDESC), "r"((unsigned)acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit(unsigned long long* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// 8 consecutive 32-bit TMEM columns of this thread's lane (32x32b shape: warp w reads lanes 32w..32w+31)
__device__ __forceinline__ void tmem_ld8(unsigned taddr, unsigned (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

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

// One CTA of 256 threads per TM candidates.  Stage c covers K bytes
// [c KB, (c + 1) KB) of the windows: every thread gathers 6 of the 3 x 128 x 4
// 16-byte pieces of the three A planes (4 consecutive threads per candidate,
// so a warp reads 8 candidates' contiguous row segments; each piece lies in
// one window row) and up to 2 of the 384 16-byte pieces of the stage's B
// blocks; after a proxy fence and a barrier thread 0 issues 2 k-steps x 4
// UMMAs and commits them to the stage's mbarrier, which the threads wait on
// before refilling that stage NSTAGE stages later.  flush_rows > 0: every
// flush_rows window rows each thread adds its I x P columns (24 of its
// candidate's 48) into int64 registers and the accumulator restarts.
__global__ void __launch_bounds__(THREADS, 1) fused_kernel(
    const uint8_t* __restrict__ planes, long long pitch, long long plane_stride, const int* __restrict__ rows,
    int row_cols, long long first, long long count, int m, int kr, const uint8_t* __restrict__ bops, int na_g,
    int a0, const long long* __restrict__ stats, int flush_rows, int tl, double* __restrict__ part_score,
    long long* __restrict__ part_idx) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tm = 1 << tl;  // candidates of this CTA (rows tm.. of the tile are unused)
    __shared__ __align__(8) unsigned long long mma_bar[NSTAGE];
    __shared__ unsigned tmem_base_sh;
    __shared__ long long orig[TM];
    const int tid = threadIdx.x, warp = tid >> 5;
    const int quad = warp & 3, half = warp >> 2;  // TMEM lanes 32 quad .., column half
    const int lo = (m - 1) / 2;
    if (tid < TM) {
        const long long ci = (long long)blockIdx.x * tm + (tid < tm ? tid : 0);
        const long long r = first + (ci < count ? ci : 0);
        orig[tid] = (long long)(rows[r * row_cols + 1] - lo) * pitch + (rows[r * row_cols] - lo);
    }
    if (tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) mbar_init(&mma_bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "n"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const unsigned tmem = tmem_base_sh;
    const unsigned sbase = smem_u32(smem);
    const unsigned trow = tmem + ((unsigned)(quad * 32) << 16);
    const int row = quad * 32 + (tid & 31);  // this thread's candidate row in the epilogue
    constexpr int HALF_COLS = NB / 2;        // 24 I x P columns per thread
    long long ipacc[HALF_COLS];
#pragma unroll
    for (int e = 0; e < HALF_COLS; ++e) ipacc[e] = 0;
    const long long kwin = (long long)m * kr;  // K bytes of one window
    const int n_chunks = (int)n_stages_of(m);
    const int kc = tid & 3;  // this thread's 16-byte piece of every row segment
    bool ip_acc = false;
    for (int c = 0; c < n_chunks; ++c) {
        const int s = c % NSTAGE;
        if (c >= NSTAGE) mbar_wait(&mma_bar[s], (unsigned)((c / NSTAGE) - 1) & 1u);
        uint8_t* st = smem + s * STAGE_BYTES;
        const long long k0 = (long long)c * KB + kc * 16;
        const bool live = k0 < kwin;
        const int r = live ? (int)(k0 / kr) : 0;
        const long long roff = (long long)r * pitch + (k0 - (long long)r * kr);
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            const int q = tid + THREADS * i;
            const int p = q >> (tl + 2), cand = (q >> 2) & (tm - 1);
            if (p < 3) {
                uint4 v = make_uint4(0u, 0u, 0u, 0u);
                if (live) v = ld16_unaligned(planes + p * plane_stride + orig[cand] + roff);
                *reinterpret_cast<uint4*>(st + p * A_BYTES + canon(cand, kc * 16)) = v;
            }
        }
        const uint4* bsrc = reinterpret_cast<const uint4*>(bops + (size_t)c * 2 * B_BYTES);
        uint4* bdst = reinterpret_cast<uint4*>(st + 3 * A_BYTES);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int q = tid + THREADS * i;
            if (q < 2 * B_BYTES / 16) bdst[q] = __ldg(bsrc + q);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> tensor core
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const unsigned sa = sbase + s * STAGE_BYTES;
#pragma unroll
            for (int ks = 0; ks < KB / 32; ++ks) {
                const unsigned k = ks * 256;  // 32 bytes of K = two core matrices
                const unsigned long long dbp = umma_desc(sa + 3 * A_BYTES + k);
                const unsigned long long dbm = umma_desc(sa + 3 * A_BYTES + B_BYTES + k);
                const bool acc = c > 0 || ks > 0;
                umma_u8(tmem + 0, umma_desc(sa + k), dbp, ip_acc || ks > 0);
                umma_u8(tmem + NB, umma_desc(sa + k), dbm, acc);
                umma_u8(tmem + 2 * NB, umma_desc(sa + A_BYTES + k), dbm, acc);
                umma_u8(tmem + 3 * NB, umma_desc(sa + 2 * A_BYTES + k), dbm, acc);
            }
            umma_commit(&mma_bar[s]);
        }
        ip_acc = true;
        // the window row the next stage starts in
        const long long k_next = (long long)(c + 1) * KB;
        if (flush_rows > 0 && k_next < kwin && (k_next / kr) / flush_rows != ((long long)c * KB / kr) / flush_rows) {
            // drain I x P (< 2^31 so far) into int64 and restart it
            mbar_wait(&mma_bar[s], (unsigned)(c / NSTAGE) & 1u);
            tc_fence_after();
#pragma unroll
            for (int j = 0; j < HALF_COLS / 8; ++j) {
                unsigned v[8];
                tmem_ld8(trow + HALF_COLS * half + 8 * j, v);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 8; ++e) ipacc[8 * j + e] += (long long)v[e];
            }
            tc_fence_before();
            __syncthreads();
            ip_acc = false;
        }
    }
    {
        const int cl = n_chunks - 1;
        mbar_wait(&mma_bar[cl % NSTAGE], (unsigned)(cl / NSTAGE) & 1u);
    }
    tc_fence_after();
    // epilogue: this thread = candidate `row` (TMEM lane), angles [24 half, 24 half + 24)
    double* sc = reinterpret_cast<double*>(smem);  // [TM][MAX_GROUP_ANGLES]: the stages are idle now
    const long long ci = row < tm ? (long long)blockIdx.x * tm + row : count;
#pragma unroll
    for (int j = 0; j < HALF_COLS / 8; ++j) {
        const int col = HALF_COLS * half + 8 * j;
        if (col >= MAX_GROUP_ANGLES) break;
        unsigned ip[8], im[8], hi[8], lw[8];
        tmem_ld8(trow + col, ip);
        tmem_ld8(trow + NB + col, im);
        tmem_ld8(trow + 2 * NB + col, hi);
        tmem_ld8(trow + 3 * NB + col, lw);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int ag = col + e;
            const long long vip = (long long)ip[e] + ipacc[8 * j + e];
            double score = -1.0 / 0.0;
            if (ag < na_g && ci < count)
                score = ncc_score(vip, (long long)im[e], 256LL * hi[e] + lw[e], stats + (a0 + ag) * 3);
            sc[row * MAX_GROUP_ANGLES + ag] = score;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS) : "memory");
    }
    // best per angle over this CTA's candidates (np.argmax: the first on ties)
    for (int ag = tid; ag < na_g; ag += THREADS) {
        Best b{-1.0 / 0.0, -1};
        for (int rr = 0; rr < tm; ++rr) {
            const long long cr = (long long)blockIdx.x * tm + rr;
            if (cr >= count) break;
            const Best cb{sc[rr * MAX_GROUP_ANGLES + ag], cr};
            if (b.idx < 0 || better(cb, b)) b = cb;
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
    const int64_t groups = (n_angles + ss::MAX_GROUP_ANGLES - 1) / ss::MAX_GROUP_ANGLES;
    return (size_t)groups * (size_t)ss::n_stages_of(m) * 2 * ss::B_BYTES;
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
    ss::probe_rotate_kernel<<<(unsigned)n_angles, 256, 0, s>>>(d_base, m, ss::row_bytes(m), n_angles, d_cos, d_sin,
                                                              d_bfrag, d_stats);
    ss::note_launch();
    return ss::check_launch("probe_rotate_kernel");
}

int64_t ss_match_parts(int64_t count) {
    const int64_t tm = 1LL << ss::tile_log2(count);
    return (count + tm - 1) / tm;
}

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
    const int kr = ss::row_bytes(m);
    const int a0 = group * ss::MAX_GROUP_ANGLES, na_g = std::min(ss::MAX_GROUP_ANGLES, (int)n_angles - a0);
    const uint8_t* bops = d_bfrag + (size_t)group * ss::n_stages_of(m) * 2 * ss::B_BYTES;
    // window rows whose I x P sums fit int32 (255^2 per pixel); a stage can
    // straddle a flush boundary by part of one row (kr >= 192 when flushing)
    const long long rows_fit = 2147483647LL / (65025LL * m);
    const int flush_rows = rows_fit >= m ? 0 : (int)std::max<long long>(1, rows_fit - 1);
    const size_t smem = (size_t)ss::NSTAGE * ss::STAGE_BYTES;
    cudaFuncSetAttribute(ss::fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long parts = ss_match_parts(count);
    ss::fused_kernel<<<(unsigned)parts, ss::THREADS, smem, s>>>(d_planes, pitch, pitch * H, d_rows, row_cols, first,
                                                              count, m, kr, bops, na_g, a0, d_stats, flush_rows,
                                                              ss::tile_log2(count), d_part_score, d_part_idx);
    ss::note_launch();
    if (int e = ss::check_launch("fused_kernel")) return e;
    ss::reduce_kernel<<<(unsigned)na_g, 256, 0, s>>>(d_part_score, d_part_idx, parts, na_g, d_best_score + a0,
                                                    d_best_idx + a0);
    ss::note_launch();
    return ss::check_launch("reduce_kernel");
}

}  // extern "C"
