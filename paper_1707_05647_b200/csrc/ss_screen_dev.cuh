// ss_screen_dev.cuh -- device helpers shared by the per-size screen
// (ss_screen.cu) and the fused ladder screen (ss_ladder_screen.cu): ring
// parameters, the exact fp64 feature / quantize / membership sequence
// (SURVEY.md App. A), TMA + mbarrier wrappers, stage-1 tile geometry.
// Internal: included only by translation units compiled with -fmad=false.
#pragma once

#ifndef EVAL_TWO_PHASE
#define EVAL_TWO_PHASE 1  // eval_ring_fast: X / Y corners loaded after the std test (63 registers: 4 CTAs / SM)
#endif
#ifndef FUSED_RINGS_MINB
#define FUSED_RINGS_MINB 2  // 2 CTAs x 16 warps: 63 registers (X / Y loaded after the std test); config 1 K3 -3.4%, config 4 -12% vs one-phase loads at 24 warps / SM
#endif
#include <cuda.h>

#include <atomic>
#include <cmath>
#include <type_traits>
#include <map>
#include <mutex>
#include <set>
#include <tuple>

#include "ss_common.cuh"

namespace ss {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WARPS = 16;  // stage-1 consumer warps per CTA (one tile row each)
constexpr int SMEM_BITMAP_WORDS = 12 * 1024;  // 48 KiB of membership bitmaps per CTA

// Fields grouped in 16-byte blocks in the order the fused rings read them
// (per-lane loads from shared memory become LDS.128).
struct __align__(16) RingDev {
    int sa, sb, sc, sd;  // SAT corners rel. to [cy][cx]: [+n+1][+n+1] [+n+1][-n+1] [-n+1][+n+1] [-n+1][-n+1]
    int ea, ed;          // E corners: [+d+1][+1], [-d][+1]
    int ob, oc;          // O corners: [0][-d], [0][+d+1]
    float fa, fb;  // RN32(1 / (2 cnt qm)) of the square / diamond: fp32 estimate of the mean cell
    int icq, icd;  // pixel counts 4n^2, 2d^2+2d+1 (exact integer variances)
    float rcq, rcd, rw2q, rw1d;  // RN32 of 1/icq, 1/icd, 1/(2 w1_sq), 1/w1_di (fp32 estimates of std / gradient)
    int cm_lo, cm_n, cs_lo, cs_n;
    int cg_lo, cg_n, bm, wm;  // bm: shared-memory word offset of [m | ms | full] bits (-1: binary search)
    int wms;     // words of the m / ms bitmaps: wm (above), wms
    int bsrc;    // uint32 index of the bit section in the device blob (-1: zero fill)
    int bwords;  // words to stage
    int n, d;
    int off_m, n_m, off_ms, n_ms, off_k, n_k;
    double cnt_sq, rcp_sq, cnt_di, rcp_di, w1_sq, rw1_sq, w1_di, rw1_di;
};

struct ScreenArgs {
    const void* planes;   // 12 planes of int64, or of uint32 (cells mod 2^32)
    long long pitch, ps;  // row pitch, plane stride (elements)
    int W, H, y_origin, y_begin, y_end, stride, lo, hi, n_rings;
    int sums_in_list;  // ring-0 PLAIN sums fit 32 bits: list entries carry them (rings skip 8 gathers)
    double qm, qs, qg, rqm, rqs, rqg;
    int qpow2;  // bit c: quantizer step c (mean, std, grad) is a power of two
    float rqs_f, rqg_f, band_s;  // RN32(1/qs), RN32(1/qg), 1e-5 / qs (eval_ring_fast)
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
// With q a power of two (pow2, uniform), f / q is exact and equals f * rq.
__device__ __forceinline__ int quant(double f, double q, double rq, bool pow2) {
    return (int)floor(__dadd_rn(pow2 ? __dmul_rn(f, rq) : div_rn(f, q, rq), 0.5));
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

template <class A>
__device__ __forceinline__ bool member_m(const A& a, const RingDev& R, const unsigned* sb, int cm) {
    if (R.bm >= 0) {
        const unsigned i = (unsigned)(cm - R.cm_lo);
        return i < (unsigned)R.cm_n && bit(sb + R.bm, (int)i);
    }
    return bsearch_eq(a.blob + R.off_m, R.n_m, cm);
}
template <class A>
__device__ __forceinline__ bool member_ms(const A& a, const RingDev& R, const unsigned* sb, int cm, int cs) {
    if (R.bm >= 0) {
        const unsigned j = (unsigned)(cs - R.cs_lo);
        return j < (unsigned)R.cs_n && bit(sb + R.bm + R.wm, (cm - R.cm_lo) * R.cs_n + (int)j);
    }
    return bsearch_eq(a.blob + R.off_ms, R.n_ms, (long long)cm * SS_KEY_BASE + cs);
}
template <class A>
__device__ __forceinline__ bool member_k(const A& a, const RingDev& R, const unsigned* sb, int cm, int cs,
                                         int cg) {
    if (R.bm >= 0) {
        const unsigned k = (unsigned)(cg - R.cg_lo);
        return k < (unsigned)R.cg_n &&
               bit(sb + R.bm + R.wm + R.wms, ((cm - R.cm_lo) * R.cs_n + (cs - R.cs_lo)) * R.cg_n + (int)k);
    }
    return bsearch_eq(a.blob + R.off_k, R.n_k, ((long long)cm * SS_KEY_BASE + cs) * SS_KEY_BASE + cg);
}

// Plane elements: exact int64 cells, or the same cells mod 2^32 (u32).  A
// region sum is a +-+- combination of four cells; with u32 planes it is
// computed mod 2^32 and recovered exactly because the host only takes the u32
// path when every ring's sums are known to fit (fits32()):
//   PLAIN / SQUARED sums are non-negative and < 2^32;
//   X / Y sums are (c + 1) * S1 + D with D = sum (x - c) v, |D| < 2^31, so
//   D = (int32)(sum - (c + 1) * S1 mod 2^32).
template <typename T> struct Corners {
    T q[4], e[2], o[2];
};
// Per-centre plane pointers: the SAT / E / O planes of kind PLAIN at the
// centre, kinds `ks` elements apart (3 ks < 2^31, checked on the host), so
// every corner address is one 32-bit offset on a 64-bit pointer (IMAD.WIDE).
template <typename T> struct PlanePtrs {
    const T *q, *e, *o;
    int ks;
};
template <typename T, class A>
__device__ __forceinline__ PlanePtrs<T> plane_ptrs(const A& a, int cy, int x) {
    const T* p = static_cast<const T*>(a.planes) + ((long long)cy * a.pitch + x);
    return PlanePtrs<T>{p, p + 4 * a.ps, p + 8 * a.ps, (int)a.ps};
}
// One read-only load at a 32-bit element offset from a 64-bit pointer:
// address = p + sext(off) * sizeof(T) in one mad.wide (IMAD.WIDE); left to
// itself the compiler re-associates these into 64-bit index arithmetic and
// spends 3-4 integer instructions per corner.
__device__ __forceinline__ unsigned ldg_at(const unsigned* p, int off) {
    unsigned v;
    asm("{\n\t.reg .u64 ad;\n\tmad.wide.s32 ad, %2, 4, %1;\n\tld.global.nc.u32 %0, [ad];\n\t}"
        : "=r"(v) : "l"(p), "r"(off));
    return v;
}
__device__ __forceinline__ long long ldg_at(const long long* p, int off) {
    long long v;
    asm("{\n\t.reg .u64 ad;\n\tmad.wide.s32 ad, %2, 8, %1;\n\tld.global.nc.s64 %0, [ad];\n\t}"
        : "=l"(v) : "l"(p), "r"(off));
    return v;
}
// Wide cells: the 32-bit planes plus the hi16 planes (bits 32..47) give every
// cell mod 2^48; region sums of the rings' sizes stay below 2^48 (checked on
// the host), so A - B - C + D mod 2^48 is the exact sum.  6 bytes per cell
// instead of the int64 planes' 8.
using wide48 = unsigned long long;
constexpr unsigned long long M48 = (1ull << 48) - 1;
template <> struct PlanePtrs<wide48> {
    const unsigned *q, *e, *o;
    const unsigned short *qh, *eh, *oh;
    int ks;
};
template <typename T, class A>
__device__ __forceinline__ typename std::enable_if<std::is_same<T, wide48>::value, PlanePtrs<wide48>>::type
plane_ptrs_w(const A& a, int cy, int x) {
    const long long o = (long long)cy * a.pitch + x;
    const unsigned* p = a.planes32 + o;
    const unsigned short* h = a.hi16 + o;
    return PlanePtrs<wide48>{p, p + 4 * a.ps, p + 8 * a.ps, h, h + 4 * a.ps, h + 8 * a.ps, (int)a.ps};
}
__device__ __forceinline__ unsigned ldg_u16_at(const unsigned short* p, int off) {
    unsigned short v;
    asm("{\n\t.reg .u64 ad;\n\tmad.wide.s32 ad, %2, 2, %1;\n\tld.global.nc.u16 %0, [ad];\n\t}"
        : "=h"(v) : "l"(p), "r"(off));
    return v;
}
__device__ __forceinline__ wide48 cell48(const unsigned* lo, const unsigned short* hi, int off) {
    return (wide48)ldg_at(lo, off) | ((wide48)ldg_u16_at(hi, off) << 32);
}
__device__ __forceinline__ void load_corners(const PlanePtrs<wide48>& P, const RingDev& R, int kind,
                                             Corners<wide48>& c) {
    const int ko = kind * P.ks;
    if (kind == 0) {  // PLAIN: ring sums < 2^32, the 32-bit cells alone (no hi16 plane; plain_sum)
        c.q[0] = ldg_at(P.q, ko + R.sa);
        c.q[1] = ldg_at(P.q, ko + R.sb);
        c.q[2] = ldg_at(P.q, ko + R.sc);
        c.q[3] = ldg_at(P.q, ko + R.sd);
        c.e[0] = ldg_at(P.e, ko + R.ea);
        c.e[1] = ldg_at(P.e, ko + R.ed);
        c.o[0] = ldg_at(P.o, ko + R.ob);
        c.o[1] = ldg_at(P.o, ko + R.oc);
        return;
    }
    c.q[0] = cell48(P.q, P.qh, ko + R.sa);
    c.q[1] = cell48(P.q, P.qh, ko + R.sb);
    c.q[2] = cell48(P.q, P.qh, ko + R.sc);
    c.q[3] = cell48(P.q, P.qh, ko + R.sd);
    c.e[0] = cell48(P.e, P.eh, ko + R.ea);
    c.e[1] = cell48(P.e, P.eh, ko + R.ed);
    c.o[0] = cell48(P.o, P.oh, ko + R.ob);
    c.o[1] = cell48(P.o, P.oh, ko + R.oc);
}
// Corner loads from per-(plane type, kind) bases -- uniform across the warp,
// so they live in uniform registers -- plus one 32-bit byte offset per corner
// shared by all kinds: address = base + (u32) offset is two integer ops per
// load (a plane is < 4 GB: ps * sizeof(cell) < 2^32, checked on the host).
// pos = cy * pitch + cx.
template <typename T>
__device__ __forceinline__ T ld_plane(const void* base, unsigned byte_off) {
    return __ldg(reinterpret_cast<const T*>(static_cast<const char*>(base) + byte_off));
}
template <typename T, class A>
__device__ __forceinline__ void load_corners_u(const A& a, int pos, const RingDev& R, int kind, Corners<T>& c) {
    constexpr unsigned B = sizeof(T) == 8 && !std::is_same<T, wide48>::value ? 8u : 4u;  // lo-cell bytes
    const char* lo = static_cast<const char*>(std::is_same<T, wide48>::value ? static_cast<const void*>(a.planes32)
                                                                             : a.planes);
    const long long ps = a.ps;
    const char* bq = lo + (0 * 4 + kind) * ps * B;
    const char* be = lo + (1 * 4 + kind) * ps * B;
    const char* bo = lo + (2 * 4 + kind) * ps * B;
    const unsigned o[8] = {(unsigned)(pos + R.sa), (unsigned)(pos + R.sb), (unsigned)(pos + R.sc),
                           (unsigned)(pos + R.sd), (unsigned)(pos + R.ea), (unsigned)(pos + R.ed),
                           (unsigned)(pos + R.ob), (unsigned)(pos + R.oc)};
    using L = typename std::conditional<B == 8, long long, unsigned>::type;
    T v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (T)ld_plane<L>(j < 4 ? bq : (j < 6 ? be : bo), o[j] * B);
    if constexpr (std::is_same<T, wide48>::value) {  // bits 32..47 from the hi16 planes
        const char* h = reinterpret_cast<const char*>(a.hi16);
        const char* hq = h + (0 * 4 + kind) * ps * 2;
        const char* he = h + (1 * 4 + kind) * ps * 2;
        const char* ho = h + (2 * 4 + kind) * ps * 2;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            v[j] |= (wide48)ld_plane<unsigned short>(j < 4 ? hq : (j < 6 ? he : ho), o[j] * 2u) << 32;
    }
    c.q[0] = v[0];
    c.q[1] = v[1];
    c.q[2] = v[2];
    c.q[3] = v[3];
    c.e[0] = v[4];
    c.e[1] = v[5];
    c.o[0] = v[6];
    c.o[1] = v[7];
}
template <typename T>
__device__ __forceinline__ void load_corners(const PlanePtrs<T>& P, const RingDev& R, int kind, Corners<T>& c) {
    const int ko = kind * P.ks;
    SS_CHECK(kind >= 0 && kind < 4);
    c.q[0] = ldg_at(P.q, ko + R.sa);
    c.q[1] = ldg_at(P.q, ko + R.sb);
    c.q[2] = ldg_at(P.q, ko + R.sc);
    c.q[3] = ldg_at(P.q, ko + R.sd);
    c.e[0] = ldg_at(P.e, ko + R.ea);
    c.e[1] = ldg_at(P.e, ko + R.ed);
    c.o[0] = ldg_at(P.o, ko + R.ob);
    c.o[1] = ldg_at(P.o, ko + R.oc);
}
template <typename T> __device__ __forceinline__ T sq_of(const Corners<T>& c) { return c.q[0] - c.q[1] - c.q[2] + c.q[3]; }
template <typename T> __device__ __forceinline__ T di_of(const Corners<T>& c) { return c.e[0] - c.o[0] - c.o[1] + c.e[1]; }

// exact non-negative region sum (PLAIN, SQUARED)
__device__ __forceinline__ long long unsigned_sum(long long v) { return v; }
__device__ __forceinline__ long long unsigned_sum(unsigned v) { return (long long)v; }
__device__ __forceinline__ long long unsigned_sum(wide48 v) { return (long long)(v & M48); }
// the PLAIN (kind 0) sum of a ring: < 2^32 for every plane width (the wide
// path reads kind 0 from the 32-bit planes only, so it is recovered mod 2^32)
__device__ __forceinline__ long long plain_sum(unsigned v) { return (long long)v; }
__device__ __forceinline__ long long plain_sum(long long v) { return v; }
__device__ __forceinline__ long long plain_sum(wide48 v) { return (long long)(unsigned)v; }
// exact weighted region sum with weight (c + 1) at the centre column/row c
__device__ __forceinline__ long long weighted_sum(long long v, long long, long long) { return v; }
__device__ __forceinline__ long long weighted_sum(unsigned v, long long c1, long long s1) {
    const long long base = c1 * s1;
    return base + (long long)(int)(v - (unsigned)base);
}

// RN conversion of an exact non-negative region sum to fp32 (rel. error <= 2^-24)
__device__ __forceinline__ float to_f32(long long v) { return __ll2float_rn(v); }
__device__ __forceinline__ float to_f32(unsigned v) { return __uint2float_rn(v); }

// Mean cell floor(t), t = ((s1q/cq + s1d/cd) * 0.5) / qm + 0.5 (features.py:97, 349, 365;
// screening.py:86-87), from exact non-negative PLAIN sums.  The fp32 estimate tf is
// within 4e-7 (tf + 1) of the fp64 t (six roundings of 2^-24 on non-negative terms), so
// when [tf - dl, tf + dl] holds no integer, floor(t) = floor(tf) exactly; only centres
// whose mean lies within ~4e-6 of a cell boundary take the fp64 op sequence.
// The fp64 mean cell of ring R (features.py:97, 349, 365; screening.py:86-87).
template <typename S, class A>
__device__ __forceinline__ int mean_cell_exact(const A& a, const RingDev& R, S s1q, S s1d) {
    const double mq = div_rn((double)s1q, R.cnt_sq, R.rcp_sq);
    const double md = div_rn((double)s1d, R.cnt_di, R.rcp_di);
    return quant(__dmul_rn(__dadd_rn(mq, md), 0.5), a.qm, a.rqm, a.qpow2 & 1);
}
template <typename S, class A>
__device__ __forceinline__ int mean_cell(const A& a, const RingDev& R, S s1q, S s1d) {
    const float tf = fmaf(to_f32(s1q), R.fa, fmaf(to_f32(s1d), R.fb, 0.5f));
    const float dl = fmaf(tf, 4e-6f, 4e-6f);
    int cm = (int)floorf(tf - dl);
    if (cm != (int)floorf(tf + dl)) {
        const double mq = div_rn((double)s1q, R.cnt_sq, R.rcp_sq);  // features.py:97
        const double md = div_rn((double)s1d, R.cnt_di, R.rcp_di);  // features.py:121
        cm = quant(__dmul_rn(__dadd_rn(mq, md), 0.5), a.qm, a.rqm, a.qpow2 & 1);
    }
    return cm;
}

#ifndef RINGS_FAST_CM
#define RINGS_FAST_CM 0  // the rings need the fp64 means anyway; the exact cell is a short chain on top
#endif
#ifndef STAGE1_FAST_CM
#define STAGE1_FAST_CM 1
#endif

struct Stage1 {
    long long s1q, s1d;
    double mq, md;
    int cm;
};

// Stage 1 of ring R from its exact PLAIN sums: means and mean cell.
template <class A>
__device__ __forceinline__ Stage1 stage1_from(const A& a, const RingDev& R, long long s1q, long long s1d) {
    Stage1 s;
    s.s1q = s1q;
    s.s1d = s1d;
    s.mq = div_rn((double)s.s1q, R.cnt_sq, R.rcp_sq);  // features.py:97
    s.md = div_rn((double)s.s1d, R.cnt_di, R.rcp_di);  // features.py:121
#if RINGS_FAST_CM
    s.cm = mean_cell(a, R, s1q, s1d);  // features.py:137
#else
    s.cm = quant(__dmul_rn(__dadd_rn(s.mq, s.md), 0.5), a.qm, a.rqm, a.qpow2 & 1);  // features.py:137
#endif
    return s;
}

// Stages 2 (std) and 3 (gradient) of ring R from its SQUARED, X and Y corners.
// The fp64 std cell (features.py:98, 350, 366; screening.py:86-87):
// sqrt(max(s2/count - mean*mean, 0)) of both parts, averaged, quantized.
template <class A>
__device__ __forceinline__ int std_cell_exact(const A& a, const RingDev& R, double mq, double md, long long s2q,
                                              long long s2d) {
    const double vq = __dsub_rn(div_rn((double)s2q, R.cnt_sq, R.rcp_sq), __dmul_rn(mq, mq));
    const double vd = __dsub_rn(div_rn((double)s2d, R.cnt_di, R.rcp_di), __dmul_rn(md, md));
    const double sd = __dmul_rn(__dadd_rn(__dsqrt_rn(vq > 0.0 ? vq : 0.0), __dsqrt_rn(vd > 0.0 ? vd : 0.0)), 0.5);
    return quant(sd, a.qs, a.rqs, (a.qpow2 >> 1) & 1);
}
// The fp64 gradient-magnitude cell (features.py:100-101, 351-352, 367-371)
// from the exact first moments sx*, sy* (weights x+1 / y+1) and PLAIN sums:
// (s - (c + off) * s1) / w1 -- product and difference exact -- averaged,
// hypot as sqrt(gx*gx + gy*gy), quantized.
template <class A>
__device__ __forceinline__ int grad_cell_exact(const A& a, const RingDev& R, int cx, int cy, long long s1q,
                                               long long s1d, long long sxq, long long syq, long long sxd,
                                               long long syd) {
    const double fq = (double)s1q, fd = (double)s1d;
    const double gxq = div_rn(__dsub_rn((double)sxq, __dmul_rn(__dadd_rn((double)cx, 1.5), fq)), R.w1_sq, R.rw1_sq);
    const double gyq = div_rn(__dsub_rn((double)syq, __dmul_rn(__dadd_rn((double)cy, 1.5), fq)), R.w1_sq, R.rw1_sq);
    const double gxd = div_rn(__dsub_rn((double)sxd, __dmul_rn(__dadd_rn((double)cx, 1.0), fd)), R.w1_di, R.rw1_di);
    const double gyd = div_rn(__dsub_rn((double)syd, __dmul_rn(__dadd_rn((double)cy, 1.0), fd)), R.w1_di, R.rw1_di);
    const double gx = __dmul_rn(__dadd_rn(gxq, gxd), 0.5);
    const double gy = __dmul_rn(__dadd_rn(gyq, gyd), 0.5);
    const double gm = __dsqrt_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)));
    return quant(gm, a.qg, a.rqg, (a.qpow2 >> 2) & 1);
}

// Stages 2 (std) and 3 (gradient) of ring R from its SQUARED, X and Y corners.
template <typename T, class A>
__device__ __forceinline__ bool finish_of(const A& a, const RingDev& R, const unsigned* sb, int cx, int cy,
                                         const Stage1& s, const Corners<T>& c2, const Corners<T>& cx_,
                                         const Corners<T>& cy_) {
    const long long s2q = unsigned_sum(sq_of(c2)), s2d = unsigned_sum(di_of(c2));
    const int cs = std_cell_exact(a, R, s.mq, s.md, s2q, s2d);
    if (!member_ms(a, R, sb, s.cm, cs)) return false;
    const long long sxq = weighted_sum(sq_of(cx_), cx + 1, s.s1q), syq = weighted_sum(sq_of(cy_), cy + 1, s.s1q);
    const long long sxd = weighted_sum(di_of(cx_), cx + 1, s.s1d), syd = weighted_sum(di_of(cy_), cy + 1, s.s1d);
    const int cg = grad_cell_exact(a, R, cx, cy, s.s1q, s.s1d, sxq, syq, sxd, syd);
    return member_k(a, R, sb, s.cm, cs, cg);
}

// Centred first moment D = sum (x - c) v of a region from its weighted sum
// (weights c + 1 at the centre column / row c) and PLAIN sum s1, exact:
// 32-bit planes hold the weighted sum mod 2^32 and |D| < 2^31 (fits32).
__device__ __forceinline__ long long centred(unsigned v, int c1, long long s1) {
    return (long long)(int)(v - (unsigned)c1 * (unsigned)s1);
}
__device__ __forceinline__ long long centred(long long v, int c1, long long s1) { return v - (long long)c1 * s1; }
__device__ __forceinline__ long long centred(wide48 v, int c1, long long s1) {
    return (long long)(v & M48) - (long long)c1 * s1;
}

// fp32 square root of the estimates: sqrt.approx (MUFU; relative error
// < 2^-21 assumed in the bands below, which the self-test ss_selftest_cells
// checks against the fp64 sequence with boundary-aimed sums) unless
// FAST_SQRT=0 selects the correctly rounded one.
#ifndef FAST_SQRT
#define FAST_SQRT 1
#endif
__device__ __forceinline__ float est_sqrt(float x) {
#if FAST_SQRT
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
#else
    return __fsqrt_rn(x);
#endif
}
constexpr float EST_STD_REL = FAST_SQRT ? 2e-6f : 1e-6f;      // std band per (t + 1)
constexpr float EST_GRAD_REL = FAST_SQRT ? 1.6e-6f : 6e-7f;   // gradient band per (|parts| + gm) / qg

// A cell floor(t) from an fp32 estimate tf with |tf - t| <= band: exact
// unless [tf - band, tf + band] straddles an integer (returns false then).
#ifndef CELL_BAND_SCALE
#define CELL_BAND_SCALE 1.0f  // test hook: 0 disables the fp64 fallback (the self-test must then fail)
#endif
__device__ __forceinline__ bool cell_of(float tf, float band, int& cell) {
    band *= CELL_BAND_SCALE;
    cell = (int)floorf(tf - band);
    return cell == (int)floorf(tf + band);
}

// std cell from the exact integer variances V = s2 * count - s1^2 (>= 0):
// fp32 estimate, the fp64 reference sequence only within its error band of a
// boundary (bounds: eval_ring_fast).
// NARROW: the PLAIN / SQUARED sums are < 2^32 (32-bit planes, fits32), so the
// variance products are single 32 x 32 -> 64-bit multiplies.
template <bool NARROW = false, class A>
__device__ __forceinline__ int std_cell_fast(const A& a, const RingDev& R, long long s1q, long long s1d, long long s2q,
                                             long long s2d) {
    long long vq, vd;
    if constexpr (NARROW) {
        vq = (long long)((unsigned long long)(unsigned)s2q * (unsigned)R.icq -
                         (unsigned long long)(unsigned)s1q * (unsigned)s1q);
        vd = (long long)((unsigned long long)(unsigned)s2d * (unsigned)R.icd -
                         (unsigned long long)(unsigned)s1d * (unsigned)s1d);
    } else {
        vq = s2q * R.icq - s1q * s1q;
        vd = s2d * R.icd - s1d * s1d;
    }
    const float sdf = __fmul_rn(__fadd_rn(__fmul_rn(est_sqrt(__ll2float_rn(vq)), R.rcq),
                                          __fmul_rn(est_sqrt(__ll2float_rn(vd)), R.rcd)),
                                0.5f);
    const float ts = __fmaf_rn(sdf, a.rqs_f, 0.5f);
    int cs;
    if (!cell_of(ts, __fmaf_rn(ts, EST_STD_REL, EST_STD_REL) + a.band_s, cs)) {
        const double mq = div_rn((double)s1q, R.cnt_sq, R.rcp_sq), md = div_rn((double)s1d, R.cnt_di, R.rcp_di);
        cs = std_cell_exact(a, R, mq, md, s2q, s2d);
    }
    return cs;
}
// gradient-magnitude cell from the exact centred moments D (square offset
// c + 1.5 => numerator 2D - s1 over 2 w1; diamond offset c + 1 => D / w1).
template <class A>
__device__ __forceinline__ int grad_cell_fast(const A& a, const RingDev& R, int cx, int cy, long long s1q,
                                              long long s1d, long long dxq, long long dyq, long long dxd,
                                              long long dyd) {
    const float gxq = __fmul_rn(__ll2float_rn(2 * dxq - s1q), R.rw2q), gyq = __fmul_rn(__ll2float_rn(2 * dyq - s1q), R.rw2q);
    const float gxd = __fmul_rn(__ll2float_rn(dxd), R.rw1d), gyd = __fmul_rn(__ll2float_rn(dyd), R.rw1d);
    const float gx = __fmul_rn(__fadd_rn(gxq, gxd), 0.5f), gy = __fmul_rn(__fadd_rn(gyq, gyd), 0.5f);
    const float gm = est_sqrt(__fmaf_rn(gx, gx, __fmul_rn(gy, gy)));
    const float tg = __fmaf_rn(gm, a.rqg_f, 0.5f);
    const float sum = __fadd_rn(__fadd_rn(fabsf(gxq), fabsf(gxd)), __fadd_rn(fabsf(gyq), fabsf(gyd)));
    const float bg =
        __fmaf_rn(__fmul_rn(__fadd_rn(sum, gm), EST_GRAD_REL), a.rqg_f, __fmaf_rn(tg, 4e-7f, 4e-7f));
    int cg;
    if (!cell_of(tg, bg, cg)) {
        cg = grad_cell_exact(a, R, cx, cy, s1q, s1d, (long long)(cx + 1) * s1q + dxq, (long long)(cy + 1) * s1q + dyq,
                             (long long)(cx + 1) * s1d + dxd, (long long)(cy + 1) * s1d + dyd);
    }
    return cg;
}

// Ring R at table-local centre (cx, cy), decided from fp32 estimates of the
// three cells built on exact integer region sums -- the variances
// s2*count - s1^2 and the centred moments are exact integers, so each
// estimate is within a few 2^-24 relative (plus, for the std, the fp64
// reference's own cancellation error near zero variance) of the value the
// reference's fp64 sequence produces -- and the fp64 sequence itself only
// for a lane whose estimate lies within that error band of a cell boundary.
// Same decisions as stage1_from + finish_of (the parity tests compare the
// fused path, which uses this, with the oracle); the error bands:
//   mean: mean_cell (4e-6 (t + 1));
//   std:  |sqrt(V)/c| in fp32 <= 2.7e-7 rel (+ 4.8e-7 with sqrt.approx),
//         t <= 4.5e-7 (t + 1) (+ 4.8e-7); fp64 var error <= 4 * 2^-53 *
//         65025 => std error <= 5.4e-6 absolute; band EST_STD_REL (t + 1)
//         + 1e-5 / qs;
//   grad: |gx_f - gx| <= 2.5e-7 (|gxq| + |gxd|) (likewise y), hypot is
//         1-Lipschitz, + 2.5e-7 rel (+ 4.8e-7 with sqrt.approx); band
//         EST_GRAD_REL (sum + gm) / qg plus 4e-7 (t + 1).
//   have_s1: ring R's PLAIN sums s1q_in / s1d_in are given (stage 1 carried
//   them in the candidate list: exact u32), so its 8 PLAIN corners are not read.
template <typename T, class A>
__device__ __forceinline__ bool eval_ring_fast(const A& a, const RingDev& R, const unsigned* sb, int level, int cx,
                                               int cy, bool have_s1 = false, unsigned s1q_in = 0,
                                               unsigned s1d_in = 0) {
    // every corner of the ring inside the table band (rows 0..h, columns 0..W)
    SS_CHECK(cy - (R.n - 1 > R.d ? R.n - 1 : R.d) >= 0 && cy + (R.n > R.d ? R.n : R.d) + 1 <= a.ps / a.pitch - 1 &&
             cx - (R.n - 1 > R.d ? R.n - 1 : R.d) >= 0 && cx + (R.n > R.d ? R.n : R.d) + 1 <= a.W);
    // (load_corners_u -- per-kind uniform bases + 32-bit byte offsets -- measured
    // slower here: config 1 K3 0.482 -> 0.499 ms; per-centre plane pointers kept)
    PlanePtrs<T> P;
    if constexpr (std::is_same<T, wide48>::value) {
        P = plane_ptrs_w<T>(a, cy, cx);
    } else {
        P = plane_ptrs<T>(a, cy, cx);
    }
    Corners<T> c0, c2, ckx, cky;
    long long s1q, s1d;
    if (have_s1) {
        s1q = s1q_in;
        s1d = s1d_in;
    } else {
        load_corners(P, R, 0, c0);
        s1q = plain_sum(sq_of(c0));
        s1d = plain_sum(di_of(c0));
    }
    load_corners(P, R, 3, c2);
#if !EVAL_TWO_PHASE
    load_corners(P, R, 1, ckx);
    load_corners(P, R, 2, cky);
#endif
    const int cm = mean_cell(a, R, s1q, s1d);  // features.py:137 (level 0 entries passed this test in stage 1)
#if RINGS_STATS
    atomicAdd(a.stage_counts + 4 + 4 * level, 1ull);
#endif
    // level 0 too: the coarse stage 1 passes centres it could not decide
    // (ladder_stage1_coarse_kernel); for the others this repeats its test
    if (!member_m(a, R, sb, cm)) return false;
#if RINGS_STATS
    atomicAdd(a.stage_counts + 5 + 4 * level, 1ull);
#endif
    const long long s2q = unsigned_sum(sq_of(c2)), s2d = unsigned_sum(di_of(c2));
    const int cs = std_cell_fast<sizeof(T) == 4>(a, R, s1q, s1d, s2q, s2d);
    if (!member_ms(a, R, sb, cm, cs)) return false;
#if RINGS_STATS
    atomicAdd(a.stage_counts + 6 + 4 * level, 1ull);
#endif
#if EVAL_TWO_PHASE
    load_corners(P, R, 1, ckx);  // X / Y planes only for (mean, std) members
    load_corners(P, R, 2, cky);
#endif
    // gradient from the exact centred moments
    const long long dxq = centred(sq_of(ckx), cx + 1, s1q), dyq = centred(sq_of(cky), cy + 1, s1q);
    const long long dxd = centred(di_of(ckx), cx + 1, s1d), dyd = centred(di_of(cky), cy + 1, s1d);
    const int cg = grad_cell_fast(a, R, cx, cy, s1q, s1d, dxq, dyq, dxd, dyd);
    return member_k(a, R, sb, cm, cs, cg);
}

// Host: bit c set when quantizer step c (mean, std, grad) is a power of two
// (then f / q == f * (1 / q) exactly and quant skips the division).
inline int quant_pow2_bits(double qm, double qs, double qg) {
    auto p2 = [](double q) {
        int e = 0;
        return q > 0.0 && std::frexp(q, &e) == 0.5;
    };
    return (p2(qm) ? 1 : 0) | (p2(qs) ? 2 : 0) | (p2(qg) ? 4 : 0);
}

// Host: the device parameters of ring (n, d) of patch side m (features.py:
// 94-142 constants, corner offsets at row pitch P, the key blob header hd of
// ss_keyset_blob with its offsets rebased by blob_base slots) and its
// membership bitmap's place in the shared-memory budget (rings are packed in
// the order they are filled; a ring that does not fit uses binary search).
inline int fill_ring(RingDev& R, int n, int d, int m, long long P, double qm, const int64_t* hd, long long blob_base,
                     int& bm_words, int budget) {
    const int lo = (m - 1) / 2, hi = m / 2;
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
    R.cnt_sq = (double)(4LL * n * n);                                            // features.py:95
    R.w1_sq = (double)(2LL * n * n * n);                                         // features.py:96
    R.cnt_di = (double)(2LL * d * d + 2LL * d + 1);                              // integral.py:189-191
    R.w1_di = (double)(2LL * d * d + (long long)d * (d - 1) * (2 * d - 1) / 3);  // features.py:113-115
    R.rcp_sq = 1.0 / R.cnt_sq;  // host IEEE division: RN(1/b)
    R.rcp_di = 1.0 / R.cnt_di;
    R.rw1_sq = 1.0 / R.w1_sq;
    R.rw1_di = 1.0 / R.w1_di;
    R.fa = (float)(1.0 / (2.0 * R.cnt_sq * qm));
    R.fb = (float)(1.0 / (2.0 * R.cnt_di * qm));
    R.icq = (int)(4LL * n * n);
    R.icd = (int)(2LL * d * d + 2LL * d + 1);
    R.rcq = (float)(1.0 / R.cnt_sq);
    R.rcd = (float)(1.0 / R.cnt_di);
    R.rw2q = (float)(1.0 / (2.0 * R.w1_sq));
    R.rw1d = (float)(1.0 / R.w1_di);
    R.off_m = (int)(hd[0] + blob_base);
    R.n_m = (int)hd[1];
    R.off_ms = (int)(hd[2] + blob_base);
    R.n_ms = (int)hd[3];
    R.off_k = (int)(hd[4] + blob_base);
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
        if (bm_words + 1 <= budget) {
            R.bm = bm_words;
            R.cm_n = 0;
            R.bwords = 1;
            bm_words += 1;
        } else {
            R.n_m = 0;  // binary search over nothing: never a member
        }
    } else if (hd[12] >= 0) {
        const int64_t words = hd[13] + hd[14] + hd[15];
        if (bm_words + words <= budget) {
            R.bm = bm_words;
            R.wm = (int)hd[13];
            R.wms = (int)hd[14];
            R.bsrc = (int)((hd[12] + blob_base) * 2);
            R.bwords = (int)words;
            bm_words += (int)words;
        }
    }
    return SS_OK;
}

// atomicAdd from one lane whose result is consumed later (a reservation taken
// one step ahead): the builtin is warp-aggregated by the compiler, whose
// broadcast of the returned value waits for the atomic right away and
// defeats the look-ahead; the plain PTX atom leaves the latency hidden.
__device__ __forceinline__ unsigned atom_add_ahead(unsigned* p, unsigned v) {
    unsigned r;
    asm volatile("atom.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
    return r;
}

// ── TMA / mbarrier helpers (sm_90+ PTX, used on sm_100a) ──────────────────
__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(smem_addr(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_addr(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar))
        : "memory");
}

struct TmaMaps {
    CUtensorMap sat, e, o;  // PLAIN SAT / E / O planes: 2-D (cols, rows) of T
};

// Stage-1 tile geometry: TY rows (one per consumer warp) x TX columns; the 8
// ring-0 PLAIN corner boxes of a tile are staged by TMA into one pipeline
// stage.  Measured on B200 + driver 580: a tile-mode TMA box must start at a
// 16-byte aligned inner coordinate (an odd int64 column raises "illegal
// instruction"), so each box starts at the ALIGN-column boundary at or below
// the corner and is BW = TX + ALIGN columns wide; readers skip the offset.
constexpr int TY = WARPS;     // tile rows
#ifndef S1_CPW
#define S1_CPW 2
#endif
#ifndef S1_STAGES32
#define S1_STAGES32 4
#endif
constexpr int CPW = S1_CPW;   // 32-centre chunks per warp per tile
constexpr int TX = 32 * CPW;  // tile columns
constexpr int NBOX = 8;
constexpr int TILE_POS = TX * TY;  // centres per tile
// Candidate lists, two modes picked per size on the host (see screen_size):
// * small sizes: one list, entries (x, y);
// * large sizes (>= LARGE_TILES tiles): `parts` sub-lists -- stage-1 CTA b
//   serves partition b % parts (tiles p, p + parts, ...) and appends to its
//   own sub-list and counter, so no single counter serialises a long grid --
//   and entries (x, y, s1q, s1d) that carry the ring-0 PLAIN sums (the rings
//   kernel skips those 8 gathers).
// Either way the lists follow the strip-major tile order.
constexpr int MAX_PARTS = 8;
constexpr int TILE_CTRS = MAX_PARTS;  // stage-1 tile counters (partition p's CTAs use counter p)
// List slots a stage-1 warp reserves per atomic (a multiple of 32): fewer
// atomics on the list counter vs. the padding of each warp's last blocks.
// Re-measured at the end of round 2 (row steps emit whole groups of rows at
// once): single list 64 / 128 / 256 -> config 1 step 0.617 / 0.597 / 0.595 ms,
// config 3 16.9 / 16.35 / 16.4; partitioned lists 128 / 256 / 512 / 1024 /
// 2048 -> config 4 step 18.48 / 17.97 / 17.78 / 17.72 / 17.85 ms.
#ifndef RESERVE_SMALL_MACRO
#define RESERVE_SMALL_MACRO 128
#endif
#ifndef RESERVE_LARGE_MACRO
#define RESERVE_LARGE_MACRO 1024
#endif
constexpr int RESERVE_SMALL = RESERVE_SMALL_MACRO, RESERVE_LARGE = RESERVE_LARGE_MACRO,
              RESERVE_MAX = RESERVE_SMALL > RESERVE_LARGE ? RESERVE_SMALL : RESERVE_LARGE;
// the per-size kernels (ss_screen.cu) keep their round-1 reservations (their
// workspace is the floor of every ladder workspace)
constexpr int PS_RESERVE_SMALL = 64, PS_RESERVE_LARGE = 128, PS_RESERVE_MAX = 128;
#ifndef GROUP_CTRS
#define GROUP_CTRS 8u  // rings group counters per partition
#endif
constexpr int CTR_STRIDE = 32;  // words between counters (one 128-B line each)
template <typename E> __device__ __forceinline__ E make_entry(int x, int y, unsigned sq, unsigned sd);
template <> __device__ __forceinline__ int4 make_entry<int4>(int x, int y, unsigned sq, unsigned sd) {
    return make_int4(x, y, (int)sq, (int)sd);
}
template <> __device__ __forceinline__ int2 make_entry<int2>(int x, int y, unsigned, unsigned) {
    return make_int2(x, y);
}
__device__ __forceinline__ int4 widen(int4 e) { return e; }
__device__ __forceinline__ int4 widen(int2 e) { return make_int4(e.x, e.y, 0, 0); }
template <typename T> struct Geo {
    static constexpr int STAGES = sizeof(T) == 4 ? S1_STAGES32 : 3;  // pipeline depth (u32: 35 KB, int64: 68 KB a stage)
    static constexpr int ALIGN = 16 / (int)sizeof(T);
    static constexpr int BW = TX + ALIGN;  // staged box width (elements)
    static constexpr int BOX_ELEMS = BW * TY;
    static constexpr int BOX_BYTES = BOX_ELEMS * (int)sizeof(T);
    static constexpr int STAGE_BYTES = NBOX * BOX_BYTES;
    __device__ static int floor_al(int c) { return c & ~(ALIGN - 1); }  // two's complement
    __device__ static int rem(int c) { return c & (ALIGN - 1); }
};

struct TileMap {
    int n_tx, n_ty;  // tiles along x, y
    int strip;       // tiles per column strip (L2 locality for wide images)
    long long n_tiles;
};

__device__ __forceinline__ void tile_coords(const TileMap& t, long long idx, int& tx, int& ty) {
    // strip-major: strips of `strip` tile columns, row-blocks within a strip, x fastest
    const unsigned per_strip = (unsigned)t.strip * (unsigned)t.n_ty;
    const unsigned i = (unsigned)idx;
    const unsigned s = i / per_strip;
    const int s0 = (int)(s * (unsigned)t.strip);
    const unsigned width = (unsigned)min(t.strip, t.n_tx - s0);
    const unsigned r = i - s * per_strip;
    const unsigned q = r / width;
    ty = (int)q;
    tx = s0 + (int)(r - q * width);
}

// Copy the rings' membership bitmaps into shared memory (all threads);
// m_only: just the mean-projection words (all stage 1 tests).
__device__ __forceinline__ void stage_bitmaps(const ScreenArgs& a, unsigned* sbits, int r_lo, int r_hi,
                                              bool m_only = false) {
    const unsigned* blob32 = reinterpret_cast<const unsigned*>(a.blob);
    for (int r = r_lo; r < r_hi; ++r) {
        const RingDev& R = a.ring[r];
        if (R.bm < 0) continue;
        const int words = m_only ? max(R.wm, 1) : R.bwords;
        for (int i = threadIdx.x; i < words; i += blockDim.x)
            sbits[R.bm + i] = R.bsrc >= 0 ? __ldg(blob32 + R.bsrc + i) : 0u;
    }
}

#ifndef RK_WARPS_MACRO
#define RK_WARPS_MACRO 16  // rings warps per CTA (measured: 16 x 2 CTAs ~ 8 x 4 CTAs, slightly ahead)
#endif
constexpr int RK_WARPS = RK_WARPS_MACRO;
#ifndef QCAP_MACRO
#define QCAP_MACRO 64
#endif
constexpr int QCAP = QCAP_MACRO;
#ifndef RINGS_MINB
#define RINGS_MINB 3  // resident CTAs per SM the register budget is sized for
#endif

#ifndef RINGS_GROUP
#define RINGS_GROUP 64  // list entries a warp takes per grab (measured: 64 beats 128 / 96 on configs 1 and 4)
#endif

inline int device_sms() {
    static std::atomic<int> cached[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && cached[dev].load(std::memory_order_relaxed) > 0) return cached[dev].load();
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (dev >= 0 && dev < 64) cached[dev].store(sms);
    return sms;
}

// Resident CTAs per SM of kernel `fn` at `smem` dynamic bytes.  The first use
// of a kernel on a device raises its dynamic shared-memory limit to the
// maximum; results are cached per (kernel, block, smem, device) -- these
// queries cost more host time than a launch, and a ladder makes 2 per size.
inline int occupancy(const void* fn, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, size_t, int>, int> cache;
    static std::set<std::pair<const void*, int>> raised;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_tuple(fn, threads, smem, dev);
    const auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    if (raised.insert({fn, dev}).second) {
        // the opt-in limit covers static + dynamic shared memory
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, fn);
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
    per_sm = std::max(per_sm, 1);
    cache[key] = per_sm;
    return per_sm;
}
// 2-D TMA descriptor of one plane (int64 or u32 elements): dims (W+1 columns,
// h+1 rows), box BW x TY.
// row_step > 1: the 3-D view (column, row mod row_step, row / row_step) of the
// plane; a box of box_h rows at (x, r % row_step, r / row_step) holds rows r,
// r + row_step, ...  Rows of the last (partial) group past the plane's end lie
// in the next plane or in the padding ss_coarse_bytes adds.
inline int encode_plane_map(CUtensorMap* map, const void* plane, int elem_bytes, int box_w, int64_t W, int64_t h,
                            int64_t pitch, int box_h = TY, int row_step = 1) {
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
            set_error("cuTensorMapEncodeTiled unavailable");
            return SS_ECUDA;
        }
        encode = reinterpret_cast<EncodeFn>(fn);
    }
    const bool v3 = row_step > 1;
    const cuuint64_t dims[3] = {(cuuint64_t)(W + 1), v3 ? (cuuint64_t)row_step : (cuuint64_t)(h + 1),
                                (cuuint64_t)((h + row_step) / row_step)};
    const cuuint64_t strides[2] = {(cuuint64_t)pitch * (cuuint64_t)elem_bytes,
                                   (cuuint64_t)pitch * (cuuint64_t)elem_bytes * (cuuint64_t)row_step};
    const cuuint32_t box[3] = {(cuuint32_t)box_w, v3 ? 1u : (cuuint32_t)box_h, (cuuint32_t)box_h};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    if (const char* e = getenv("SS_TMA_PROMO")) promo = (CUtensorMapL2promotion)atoi(e);  // experiment hook
    const CUtensorMapDataType dt = elem_bytes == 8   ? CU_TENSOR_MAP_DATA_TYPE_INT64
                                   : elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                                                     : CU_TENSOR_MAP_DATA_TYPE_UINT16;
    const CUresult r = encode(map, dt, v3 ? 3 : 2,
                              const_cast<void*>(plane), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
        return SS_ECUDA;
    }
    return SS_OK;
}


}  // namespace
}  // namespace ss
