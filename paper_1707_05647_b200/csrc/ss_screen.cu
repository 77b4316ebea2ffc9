// ss_screen.cu -- K3: star features + quantize + membership + ballot mask.
//
// Replaces _scan_size (screening.py:418-471) for one ladder size: the ring
// features of _ring_maps_rect / _octagon_maps (screening.py:380-415,
// features.py:322-382), _quantize_arr (screening.py:86-87), _pack_cells
// (:90-97), _member_mask (:173-178) and the nonzero / mask bookkeeping.
//
// Bit-exactness: compiled with -fmad=false; every fp64 op is one IEEE-
// rounded operation in the reference's NumPy order.
// Divisions by the per-size constants (pixel counts, L1 masses, quantizer
// steps) use a precomputed y = RN(1/b) and two FMA remainder corrections
// (div_rn): by Markstein's theorem that is the correctly rounded quotient,
// i.e. identical to IEEE division (ss_selftest_div checks it against
// __ddiv_rn on the device; the parity tests check the whole path).
//
// Work decomposition: a warp owns a 256-centre segment of one row (8 chunks
// of 32).  Stage 1 of ring 0 -- the mean cell, from the PLAIN planes only --
// runs on all lanes.  A centre can only be a member if its mean cell is in
// the ring's mean projection, so only those centres are pushed into a
// per-warp shared-memory queue and finished (std stage on the SQUARED
// planes, gradient stage on the X/Y planes, then rings >= 1) 32 at a time
// with full lanes.  The decision is unchanged -- the projection tests are
// implied by full membership -- but the X/Y/SQ planes and most fp64 work are
// skipped for most centres and lane divergence stays bounded.  Membership
// tests use dense bitmaps of the key bounding box in shared memory (binary
// search over the sorted keys when the box is too large).
#include <algorithm>
#include <climits>
#include <cmath>

#include "ss_common.cuh"

namespace ss {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WARPS = 8;   // rows per CTA
constexpr int CHUNKS = 8;  // 32-centre chunks per warp
constexpr int SEG = 32 * CHUNKS;
constexpr int QCAP = 64;
constexpr int SMEM_BITMAP_WORDS = 12 * 1024;  // 48 KiB of membership bitmaps per CTA

struct RingDev {
    int n, d;
    int sa, sb, sc, sd;  // SAT corners rel. to [cy][cx]: [+n+1][+n+1] [+n+1][-n+1] [-n+1][+n+1] [-n+1][-n+1]
    int ea, ed;          // E corners: [+d+1][+1], [-d][+1]
    int ob, oc;          // O corners: [0][-d], [0][+d+1]
    double cnt_sq, rcp_sq, cnt_di, rcp_di, w1_sq, rw1_sq, w1_di, rw1_di;
    int cm_lo, cm_n, cs_lo, cs_n, cg_lo, cg_n;
    int bm;        // shared-memory word offset of [m | ms | full] bits; -1: binary search
    int wm, wms;   // words of the m and ms bitmaps
    int bsrc;      // uint32 index of the bit section in the device blob (-1: zero fill)
    int bwords;    // words to stage
    int off_m, n_m, off_ms, n_ms, off_k, n_k;
};

struct ScreenArgs {
    const long long* planes;
    long long pitch, ps;  // row pitch, plane stride (elements)
    int W, H, y_origin, y_begin, y_end, stride, lo, hi, n_rings;
    double qm, qs, qg, rqm, rqs, rqg;
    const long long* blob;
    unsigned* mask;
    long long mask_pitch;
    unsigned* row_counts;
    unsigned long long* stage_counts;
    RingDev ring[SS_MAX_RINGS];
};

// Correctly rounded a / b given y = RN(1 / b) (Markstein): the first FMA pair
// brings q within one ulp of a/b, the second rounds it exactly.
__device__ __forceinline__ double div_rn(double a, double b, double y) {
    double q = __dmul_rn(a, y);
    double r = __fma_rn(-b, q, a);
    q = __fma_rn(r, y, q);
    r = __fma_rn(-b, q, a);
    return __fma_rn(r, y, q);
}

// screening.py:86-87 floor(f / q + 0.5)
__device__ __forceinline__ int quant(double f, double q, double rq) {
    return (int)floor(__dadd_rn(div_rn(f, q, rq), 0.5));
}

__device__ __forceinline__ bool bsearch_eq(const long long* __restrict__ a, int n, long long key) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < key) lo = mid + 1; else hi = mid;
    }
    return lo < n && __ldg(a + lo) == key;
}

__device__ __forceinline__ bool bit(const unsigned* s, int idx) { return (s[idx >> 5] >> (idx & 31)) & 1u; }

__device__ __forceinline__ bool member_m(const ScreenArgs& a, const RingDev& R, const unsigned* sb, int cm) {
    if (R.bm >= 0) {
        const unsigned i = (unsigned)(cm - R.cm_lo);
        return i < (unsigned)R.cm_n && bit(sb + R.bm, (int)i);
    }
    return bsearch_eq(a.blob + R.off_m, R.n_m, cm);
}
__device__ __forceinline__ bool member_ms(const ScreenArgs& a, const RingDev& R, const unsigned* sb, int cm, int cs) {
    if (R.bm >= 0) {
        const unsigned j = (unsigned)(cs - R.cs_lo);
        return j < (unsigned)R.cs_n && bit(sb + R.bm + R.wm, (cm - R.cm_lo) * R.cs_n + (int)j);
    }
    return bsearch_eq(a.blob + R.off_ms, R.n_ms, (long long)cm * SS_KEY_BASE + cs);
}
__device__ __forceinline__ bool member_k(const ScreenArgs& a, const RingDev& R, const unsigned* sb, int cm, int cs,
                                         int cg) {
    if (R.bm >= 0) {
        const unsigned k = (unsigned)(cg - R.cg_lo);
        return k < (unsigned)R.cg_n &&
               bit(sb + R.bm + R.wm + R.wms, ((cm - R.cm_lo) * R.cs_n + (cs - R.cs_lo)) * R.cg_n + (int)k);
    }
    return bsearch_eq(a.blob + R.off_k, R.n_k, ((long long)cm * SS_KEY_BASE + cs) * SS_KEY_BASE + cg);
}

__device__ __forceinline__ long long ld(const long long* p) { return __ldg(p); }

// The 8 corner elements of one kind for ring R (4 SAT, 2 E, 2 O), loaded
// together so a single memory round trip covers them.
struct Corners {
    long long q[4], e[2], o[2];
};
__device__ __forceinline__ void load_corners(const ScreenArgs& a, const RingDev& R, const long long* pc, int kind,
                                             Corners& c) {
    const long long* pq = pc + (long long)kind * a.ps;
    const long long* pe = pc + (long long)(4 + kind) * a.ps;
    const long long* po = pc + (long long)(8 + kind) * a.ps;
    c.q[0] = ld(pq + R.sa);
    c.q[1] = ld(pq + R.sb);
    c.q[2] = ld(pq + R.sc);
    c.q[3] = ld(pq + R.sd);
    c.e[0] = ld(pe + R.ea);
    c.e[1] = ld(pe + R.ed);
    c.o[0] = ld(po + R.ob);
    c.o[1] = ld(po + R.oc);
}
__device__ __forceinline__ long long sq_of(const Corners& c) { return c.q[0] - c.q[1] - c.q[2] + c.q[3]; }
__device__ __forceinline__ long long di_of(const Corners& c) { return c.e[0] - c.o[0] - c.o[1] + c.e[1]; }

struct Stage1 {
    long long s1q, s1d;
    double mq, md;
    int cm;
};

// Stage 1 (mean cell) of ring R from its PLAIN corners.
__device__ __forceinline__ Stage1 stage1_of(const ScreenArgs& a, const RingDev& R, const Corners& c) {
    Stage1 s;
    s.s1q = sq_of(c);
    s.s1d = di_of(c);
    s.mq = div_rn((double)s.s1q, R.cnt_sq, R.rcp_sq);                   // features.py:325
    s.md = div_rn((double)s.s1d, R.cnt_di, R.rcp_di);                   // features.py:349
    s.cm = quant(__dmul_rn(__dadd_rn(s.mq, s.md), 0.5), a.qm, a.rqm);  // features.py:365
    return s;
}

// Stages 2 (std) and 3 (gradient) of ring R from its SQUARED, X and Y corners.
__device__ __forceinline__ bool finish_of(const ScreenArgs& a, const RingDev& R, const unsigned* sb, int cx, int cy,
                                         const Stage1& s, const Corners& c2, const Corners& cx_, const Corners& cy_,
                                         bool& grad) {
    const long long s2q = sq_of(c2), s2d = di_of(c2);
    // features.py:326, 350: sqrt(max(s2/count - mean*mean, 0))
    const double vq = __dsub_rn(div_rn((double)s2q, R.cnt_sq, R.rcp_sq), __dmul_rn(s.mq, s.mq));
    const double vd = __dsub_rn(div_rn((double)s2d, R.cnt_di, R.rcp_di), __dmul_rn(s.md, s.md));
    const double sd = __dmul_rn(__dadd_rn(__dsqrt_rn(vq > 0.0 ? vq : 0.0), __dsqrt_rn(vd > 0.0 ? vd : 0.0)), 0.5);
    const int cs = quant(sd, a.qs, a.rqs);
    if (!member_ms(a, R, sb, s.cm, cs)) return false;
    grad = true;
    const double fq = (double)s.s1q, fd = (double)s.s1d;
    // features.py:328-329, 351-352: (s - (c + off) * s1) / w1; product and difference are exact
    const double gxq = div_rn(__dsub_rn((double)sq_of(cx_), __dmul_rn(__dadd_rn((double)cx, 1.5), fq)), R.w1_sq, R.rw1_sq);
    const double gyq = div_rn(__dsub_rn((double)sq_of(cy_), __dmul_rn(__dadd_rn((double)cy, 1.5), fq)), R.w1_sq, R.rw1_sq);
    const double gxd = div_rn(__dsub_rn((double)di_of(cx_), __dmul_rn(__dadd_rn((double)cx, 1.0), fd)), R.w1_di, R.rw1_di);
    const double gyd = div_rn(__dsub_rn((double)di_of(cy_), __dmul_rn(__dadd_rn((double)cy, 1.0), fd)), R.w1_di, R.rw1_di);
    const double gx = __dmul_rn(__dadd_rn(gxq, gxd), 0.5);  // features.py:367-369
    const double gy = __dmul_rn(__dadd_rn(gyq, gyd), 0.5);
    const double gm = __dsqrt_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)));
    const int cg = quant(gm, a.qg, a.rqg);
    return member_k(a, R, sb, s.cm, cs, cg);
}

__global__ void __launch_bounds__(WARPS * 32) screen_kernel(const ScreenArgs a) {
    extern __shared__ unsigned sbits[];
    // Q1: ring-0 stage-1 passers with their stage-1 state; QN: (x, ring) pairs for rings >= 1
    __shared__ int q_x[WARPS][QCAP];
    __shared__ int q_cm[WARPS][QCAP];
    __shared__ double q_mq[WARPS][QCAP], q_md[WARPS][QCAP];
    __shared__ long long q_s1q[WARPS][QCAP], q_s1d[WARPS][QCAP];
    __shared__ int qn_x[WARPS][QCAP];
    __shared__ unsigned char qn_r[WARPS][QCAP];
    __shared__ unsigned s_mask[WARPS][CHUNKS];

    // stage the rings' membership bitmaps
    const int tid = threadIdx.y * 32 + threadIdx.x;
    const unsigned* blob32 = reinterpret_cast<const unsigned*>(a.blob);
    for (int r = 0; r < a.n_rings; ++r) {
        const RingDev& R = a.ring[r];
        if (R.bm < 0) continue;
        for (int i = tid; i < R.bwords; i += WARPS * 32) sbits[R.bm + i] = R.bsrc >= 0 ? __ldg(blob32 + R.bsrc + i) : 0u;
    }
    __syncthreads();

    const int lane = threadIdx.x, warp = threadIdx.y;
    const int y = a.y_begin + blockIdx.y * WARPS + warp;
    if (y >= a.y_end) return;  // warp-uniform; no block barriers below
    const int x0 = blockIdx.x * SEG;
    const int cy = y - a.y_origin;  // table-local row: features are frame-invariant
    const bool row_grid = (y % a.stride) == 0;
    const bool row_int = row_grid && y >= a.lo && y <= a.H - 1 - a.hi;
    const long long* rowp = a.planes + (long long)cy * a.pitch;
    const RingDev& R0 = a.ring[0];
    const unsigned lt = (1u << lane) - 1u;
    const bool inst = a.stage_counts != nullptr;

    int n1 = 0, nn = 0;  // queue lengths
    unsigned surv_count = 0;
    unsigned long long st0 = 0, st1 = 0, st2 = 0, st3 = 0;

    auto survive = [&](bool keep, int x) {
        if (keep) {
            const int off = x - x0;
            atomicOr(&s_mask[warp][off >> 5], 1u << (off & 31));
        }
        surv_count += __popc(__ballot_sync(FULL, keep));
    };
    auto push_next = [&](bool push, int x, int r) {
        const unsigned b = __ballot_sync(FULL, push);
        if (push) {
            const int e = nn + __popc(b & lt);
            qn_x[warp][e] = x;
            qn_r[warp][e] = (unsigned char)r;
        }
        nn += __popc(b);
        __syncwarp();
    };
    // ring-0 stages 2-3 for Q1 entries [n1 - cnt, n1)
    auto drain1 = [&](int cnt) {
        bool keep = false, more = false;
        int x = 0;
        if (lane < cnt) {
            const int e = n1 - cnt + lane;
            x = q_x[warp][e];
            Stage1 s;
            s.cm = q_cm[warp][e];
            s.mq = q_mq[warp][e];
            s.md = q_md[warp][e];
            s.s1q = q_s1q[warp][e];
            s.s1d = q_s1d[warp][e];
            const long long* pc = rowp + x;
            Corners c2, cxk, cyk;
            load_corners(a, R0, pc, 3, c2);
            load_corners(a, R0, pc, 1, cxk);
            load_corners(a, R0, pc, 2, cyk);
            bool grad = false;
            const bool pass = finish_of(a, R0, sbits, x, cy, s, c2, cxk, cyk, grad);
            st2 += grad;
            keep = pass && a.n_rings == 1;
            more = pass && a.n_rings > 1;
        }
        n1 -= cnt;
        __syncwarp();
        survive(keep, x);
        push_next(more, x, 1);
    };
    // one full ring evaluation for QN entries [nn - cnt, nn)
    auto drainN = [&](int cnt) {
        bool keep = false, more = false;
        int x = 0, r = 0;
        if (lane < cnt) {
            const int e = nn - cnt + lane;
            x = qn_x[warp][e];
            r = qn_r[warp][e];
        }
        nn -= cnt;
        __syncwarp();
        if (lane < cnt) {
            const RingDev& R = a.ring[r];
            const long long* pc = rowp + x;
            Corners c0, c2, cxk, cyk;
            load_corners(a, R, pc, 0, c0);
            load_corners(a, R, pc, 3, c2);
            load_corners(a, R, pc, 1, cxk);
            load_corners(a, R, pc, 2, cyk);
            ++st3;
            const Stage1 t = stage1_of(a, R, c0);
            bool grad = false;
            const bool pass = member_m(a, R, sbits, t.cm) && finish_of(a, R, sbits, x, cy, t, c2, cxk, cyk, grad);
            keep = pass && r + 1 == a.n_rings;
            more = pass && r + 1 < a.n_rings;
        }
        survive(keep, x);
        push_next(more, x, r + 1);
    };

    // stage 1 of ring 0 over the segment, software-pipelined one chunk ahead
    // (only centres inside the evaluable interior are loaded: their corners are in bounds)
    auto in_interior = [&](int xx) { return row_int && xx >= a.lo && xx <= a.W - 1 - a.hi; };
    Corners cur, nxt;
    if (in_interior(x0 + lane)) load_corners(a, R0, rowp + x0 + lane, 0, cur);
#pragma unroll 1
    for (int c = 0; c < CHUNKS; ++c) {
        const int x = x0 + c * 32 + lane;
        if (c + 1 < CHUNKS && in_interior(x + 32)) load_corners(a, R0, rowp + x + 32, 0, nxt);
        const bool on_grid = row_grid && x < a.W && (x % a.stride) == 0;
        const bool interior = row_int && on_grid && x >= a.lo && x <= a.W - 1 - a.hi;
        const unsigned border = __ballot_sync(FULL, on_grid && !interior);
        if (lane == 0) s_mask[warp][c] = border;
        bool pass = false;
        Stage1 s;
        if (interior) {
            s = stage1_of(a, R0, cur);
            pass = member_m(a, R0, sbits, s.cm);
        }
        const unsigned pb = __ballot_sync(FULL, pass);
        if (inst) {
            st0 += __popc(__ballot_sync(FULL, interior));
            st1 += __popc(pb);
        }
        if (pass) {
            const int e = n1 + __popc(pb & lt);
            q_x[warp][e] = x;
            q_cm[warp][e] = s.cm;
            q_mq[warp][e] = s.mq;
            q_md[warp][e] = s.md;
            q_s1q[warp][e] = s.s1q;
            q_s1d[warp][e] = s.s1d;
        }
        n1 += __popc(pb);
        __syncwarp();
        if (n1 >= 32) drain1(32);
        while (nn >= 32) drainN(32);
        cur = nxt;
    }
    if (n1 > 0) drain1(n1);
    while (nn > 0) drainN(nn < 32 ? nn : 32);
    __syncwarp();
    const long long row = y - a.y_begin;
    if (lane < CHUNKS) {
        const int w = blockIdx.x * CHUNKS + lane;
        if (w * 32 < a.W) a.mask[row * a.mask_pitch + w] = s_mask[warp][lane];
    }
    if (lane == 0 && surv_count) atomicAdd(a.row_counts + row, surv_count);
    if (inst) {
        unsigned long long v[4] = {st0, st1, st2, st3};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            unsigned long long t = (i < 2) ? (lane == 0 ? v[i] : 0ull) : v[i];  // st0/st1 are warp totals
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) t += __shfl_down_sync(FULL, t, d);
            if (lane == 0 && t) atomicAdd(a.stage_counts + i, t);
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

// div_rn vs IEEE division on n operands of a family (mode), divisor b.
__global__ void selftest_div_kernel(unsigned long long n, unsigned long long seed, double b, int mode,
                                    unsigned long long* bad) {
    const double y = __drcp_rn(b);
    unsigned long long local = 0;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        unsigned long long h = (i + seed) * 0x9E3779B97F4A7C15ull;
        h ^= h >> 31;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 27;
        double a;
        if (mode == 0) a = (double)(long long)(i + seed);                       // consecutive integers
        else if (mode == 1) a = (double)(long long)(h >> 21);                   // integers < 2^43
        else if (mode == 2) a = __longlong_as_double((long long)((h >> 4) | 0x3800000000000000ull));  // wide doubles
        else a = (double)(long long)(h >> 22) * 0.5 - 1099511627776.0;          // half-integers, both signs
        if (div_rn(a, b, y) != __ddiv_rn(a, b)) ++local;
    }
    if (local) atomicAdd(bad, local);
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
    if (W > (1 << 30) || H > (1 << 30)) { set_error("image too large"); return SS_EINVAL; }
    if (y_begin < 0 || y_end > H || y_begin > y_end) { set_error("bad row range"); return SS_EINVAL; }
    if (m < 2 * 4 || stride < 1) { set_error("bad size/stride"); return SS_EINVAL; }
    if (n_rings < 1 || n_rings > SS_MAX_RINGS) { set_error("n_rings out of range"); return SS_EINVAL; }
    if (pitch != plane_pitch(w)) { set_error("plane pitch mismatch"); return SS_EINVAL; }
    if (mask_pitch < (W + 31) / 32) { set_error("mask pitch too small"); return SS_EINVAL; }
    const int lo = (m - 1) / 2, hi = m / 2;
    const int64_t ylo = std::max<int64_t>(y_begin, lo), yhi = std::min<int64_t>(y_end - 1, H - 1 - hi);
    if (ylo <= yhi && (ylo - lo < y_origin || yhi + hi > y_origin + h - 1)) {
        set_error("table band [%lld, %lld) does not cover rows [%lld, %lld] with margins", (long long)y_origin,
                  (long long)(y_origin + h), (long long)ylo, (long long)yhi);
        return SS_EINVAL;
    }
    if (!h_blob || h_blob[0] != n_rings) { set_error("key blob does not match n_rings"); return SS_EINVAL; }
    if ((int64_t)(m / 2 + 2) * pitch + m > (int64_t)INT32_MAX) {
        set_error("patch offsets exceed 32 bits");
        return SS_EINVAL;
    }

    ScreenArgs a;
    a.planes = reinterpret_cast<const long long*>(d_planes);
    a.pitch = pitch;
    a.ps = (h + 1) * pitch;
    a.W = (int)W;
    a.H = (int)H;
    a.y_origin = (int)y_origin;
    a.y_begin = (int)y_begin;
    a.y_end = (int)y_end;
    a.stride = stride;
    a.lo = lo;
    a.hi = hi;
    a.n_rings = n_rings;
    a.qm = qm;
    a.qs = qs;
    a.qg = qg;
    a.rqm = 1.0 / qm;
    a.rqs = 1.0 / qs;
    a.rqg = 1.0 / qg;
    a.blob = reinterpret_cast<const long long*>(d_blob);
    a.mask = d_mask;
    a.mask_pitch = mask_pitch;
    a.row_counts = d_row_counts;
    a.stage_counts = d_stage_counts;
    int smem_words = 0;
    const long long P = pitch;
    for (int r = 0; r < n_rings; ++r) {
        RingDev& R = a.ring[r];
        const int n = ring_n[r], d = ring_d[r];
        if (n < 1 || d < 1 || n > hi || d > lo) {
            set_error("ring (%d,%d) does not fit m=%d", n, d, m);
            return SS_EINVAL;
        }
        R.n = n;
        R.d = d;
        R.sa = (int)((n + 1) * P + (n + 1));
        R.sb = (int)((n + 1) * P + (1 - n));
        R.sc = (int)((1 - n) * P + (n + 1));
        R.sd = (int)((1 - n) * P + (1 - n));
        R.ea = (int)((d + 1) * P + 1);
        R.ed = (int)(-(long long)d * P + 1);
        R.ob = -d;
        R.oc = d + 1;
        R.cnt_sq = (double)(4LL * n * n);                                            // features.py:323
        R.w1_sq = (double)(2LL * n * n * n);                                         // features.py:324
        R.cnt_di = (double)(2LL * d * d + 2LL * d + 1);                              // integral.py:189-191
        R.w1_di = (double)(2LL * d * d + (long long)d * (d - 1) * (2 * d - 1) / 3);  // features.py:341-343
        R.rcp_sq = 1.0 / R.cnt_sq;  // host IEEE division: RN(1/b)
        R.rcp_di = 1.0 / R.cnt_di;
        R.rw1_sq = 1.0 / R.w1_sq;
        R.rw1_di = 1.0 / R.w1_di;
        const int64_t* hd = h_blob + 1 + SS_BLOB_HDR * r;
        R.off_m = (int)hd[0];
        R.n_m = (int)hd[1];
        R.off_ms = (int)hd[2];
        R.n_ms = (int)hd[3];
        R.off_k = (int)hd[4];
        R.n_k = (int)hd[5];
        R.cm_lo = (int)hd[6];
        R.cm_n = (int)hd[7];
        R.cs_lo = (int)hd[8];
        R.cs_n = (int)hd[9];
        R.cg_lo = (int)hd[10];
        R.cg_n = (int)hd[11];
        R.bm = -1;
        R.wm = R.wms = 0;
        R.bsrc = -1;
        R.bwords = 0;
        if (R.n_k == 0) {  // empty ring: nothing passes
            R.bm = smem_words;
            R.cm_n = 0;
            R.bwords = 1;
            smem_words += 1;
        } else if (hd[12] >= 0) {
            const int64_t words = hd[13] + hd[14] + hd[15];
            if (smem_words + words <= SMEM_BITMAP_WORDS) {
                R.bm = smem_words;
                R.wm = (int)hd[13];
                R.wms = (int)hd[14];
                R.bsrc = (int)(hd[12] * 2);
                R.bwords = (int)words;
                smem_words += (int)words;
            }
        }
    }
    cudaStream_t s = as_stream(stream);
    const int64_t rows = y_end - y_begin;
    if (rows == 0) return SS_OK;
    if (cudaMemsetAsync(d_row_counts, 0, rows * sizeof(uint32_t), s) != cudaSuccess) return check_launch("memset");
    const size_t smem = (size_t)std::max(smem_words, 1) * 4;
    if (smem > 32 * 1024) cudaFuncSetAttribute(screen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((unsigned)((W + SEG - 1) / SEG), (unsigned)((rows + WARPS - 1) / WARPS));
    screen_kernel<<<grid, dim3(32, WARPS), smem, s>>>(a);
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

int selftest_div(uint64_t n, uint64_t seed, double b, int mode, unsigned long long* d_bad, void* stream) {
    if (b <= 0.0 || mode < 0 || mode > 3) { set_error("bad selftest arguments"); return SS_EINVAL; }
    selftest_div_kernel<<<148 * 16, 256, 0, as_stream(stream)>>>(n, seed, b, mode, d_bad);
    note_launch();
    return check_launch("selftest_div_kernel");
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
int ss_selftest_div(uint64_t n, uint64_t seed, double divisor, int32_t mode, unsigned long long* d_mismatches,
                    void* stream) {
    return ss::selftest_div(n, seed, divisor, mode, d_mismatches, stream);
}
}
