// ss_build.cu -- K1/K2: the twelve int64 integral planes in one tiled sweep.
//
// Replaces build_tables (integral.py:211-228): 4 x build_sat (:109-117, two
// cumsums) and 4 x build_rsat (:120-141, scatter + cumsum(u) + reverse
// cumsum(v) over a (W+H)^2 grid).  Instead of the rotated grid we keep two
// pixel-grid planes E, O per kind (see include/starscreen_b200.h) and use the
// row recurrences:
//
//   P_y(x)  = sum_{i<=x} v(i,y)                      row prefix
//   S_y(x)  = S_{y-1}(x)   + P_y(x)                  SAT
//   FF_y(x) = FF_{y-1}(x+1) + P_y(x)                 anti-diagonal carry
//   GG_y(x) = GG_{y-1}(x-1) + P_y(x-1)               diagonal carry
//   E(x,y)  = FF_y(x) - GG_y(x),   O(x,y) = FF_y(x+1) - GG_y(x)
//
// The image is cut into bands of Rb rows and column chunks of Cw plane
// columns; a 128-thread CTA owns one (band, chunk) tile plus an Rb-column
// halo on each side (4 consecutive columns per thread).  The only
// dependency between tiles is the row state (S, FF, GG) at the row above the
// band, so the build is three data-parallel passes:
//   pass 1  every tile computes its band's end state with a zero carry;
//   pass 2  a scan over bands turns local end states into true ones
//           (FF shifts left by Rb per band, GG right, S not at all);
//   pass 3  every tile recomputes its rows with the true carry and streams
//           the 12 planes out with 16-byte stores.
// All sums are exact int64 (integral.py:114,134,139).
#include <algorithm>

#include "ss_common.cuh"

namespace ss {
namespace {

constexpr int TPB = 128;  // threads per tile
constexpr int COLS = 4;   // consecutive columns per thread
constexpr int TILE = TPB * COLS;
static_assert(TILE == kTileCols && TPB == kBuildThreads, "tile geometry");
constexpr unsigned FULL = 0xffffffffu;

struct BuildArgs {
    const uint8_t* img;
    int64_t W, H, img_pitch;
    long long* planes;   // 12 int64 planes (nullable)
    unsigned* planes32;  // 12 planes mod 2^32, same pitch (nullable)
    int64_t pitch, plane_stride;
    const long long* rowpre;  // [H][G+1][3]
    int64_t G;
    long long* state;  // [B-1][4 kinds][3 types][state_len]
    int64_t slen;
    int64_t n_chunks;
    // coarse PLAIN planes for stage 1 (nullable): for shift c, the SAT / E /
    // O PLAIN cells as u16 bit slices (cell >> shift[c]) & 0xffff, planes
    // (c * 3 + type) * plane_stride apart (same pitch as the full planes)
    unsigned short* coarse;
    int n_coarse;
    int shift[SS_MAX_COARSE];
    // bits 32..47 of every exact cell (nullable; 12 u16 planes, same layout
    // as the 32-bit planes): with those, a cell is known mod 2^48 and every
    // region sum of the 12 planes below 2^48 is exact (the rings' wide path)
    unsigned short* hi16;
    int64_t band0;  // first band of this launch (row-range builds: ss_build_tables_rows)
};

__device__ __forceinline__ long long shfl_down64(long long v, int d) {
    return (long long)__shfl_down_sync(FULL, (unsigned long long)v, d);
}
__device__ __forceinline__ long long shfl_up64(long long v, int d) {
    return (long long)__shfl_up_sync(FULL, (unsigned long long)v, d);
}
__device__ __forceinline__ unsigned shfl_down64(unsigned v, int d) { return __shfl_down_sync(FULL, v, d); }
__device__ __forceinline__ unsigned shfl_up64(unsigned v, int d) { return __shfl_up_sync(FULL, v, d); }

__device__ __forceinline__ int64_t r_off(const BuildArgs& a, int64_t r) { return r * a.pitch; }

// state pointer: band b, kind k, type (0 S, 1 FF, 2 GG)
template <typename V>
__device__ __forceinline__ V* st_ptr(const BuildArgs& a, int64_t b, int k, int type) {
    return reinterpret_cast<V*>(a.state) + ((b * 4 + k) * 3 + type) * a.slen;
}

// row-prefix at group boundary g (sum over x < kGroup * g) for quantity q
__device__ __forceinline__ long long rowpre_at(const BuildArgs& a, int64_t y, int64_t g, int q) {
    if (g <= 0) return 0;
    if (g > a.G) g = a.G;
    return a.rowpre[(y * (a.G + 1) + g) * 3 + q];
}

// kMode 0: local end state (pass 1); kMode 1: final planes (pass 3).
// RB = rows per band; the tile owns CW plane columns plus RB+1 halo columns
// on each side; state index of x is x + OFF.
// V: the recurrences' element type -- long long (exact int64 cells; writes
// the int64 planes and, if requested, their low 32 bits) or unsigned (cells
// mod 2^32: every operation is + - x, so the low 32 bits of the exact cells
// follow from 32-bit arithmetic; writes the 32-bit planes only, with half the
// registers, shuffles and band-state traffic).
// NK = 4: one CTA runs all four kinds; NK = 2: blockIdx.z picks the kinds
// {0, 2} (PLAIN, Y) or {1, 3} (X, SQ) -- half the recurrence registers, so the
// int64 build keeps more warps resident (pass 3 at config 4 ran 3 CTAs / SM).
template <int kMode, int RB, typename V, int NK = 4>
#ifndef BAND_MINB64
#define BAND_MINB64 3  // 168 registers, no spills: 3 CTAs per SM (config 4 build 6.3 -> 5.6 ms); 4 spills and is slower
#endif
#ifndef BAND_MINB32
#define BAND_MINB32 5  // 96 registers, no spills (config 1 step 0.646 -> 0.629 ms, config 2 1.72 -> 1.70)
#endif
__global__ void __launch_bounds__(TPB, (kMode == 1 && sizeof(V) == 8 && NK == 4)   ? BAND_MINB64
                                       : (kMode == 1 && sizeof(V) == 4 && NK == 2) ? BAND_MINB32
                                                                                   : 1) band_kernel(BuildArgs a) {
    static_assert(NK == 4 || NK == 2, "kinds per CTA");
    const int kg = NK == 4 ? 0 : (int)blockIdx.z;
    auto KIND = [&](int kk) { return NK == 4 ? kk : kg + 2 * kk; };
    constexpr int CW = kTileCols - 2 * RB - 2;
    constexpr int OFF = RB + 1;
    static_assert(CW % kGroup == 0 && (RB + 1) % kGroup == 0, "XL+1 must be group aligned");
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t chunk = blockIdx.x, band = a.band0 + blockIdx.y;
    const int64_t c0 = chunk * CW;             // first owned plane column
    const int64_t XL = c0 - RB - 2;            // x of thread 0, column 0
    const int64_t xb = XL + (int64_t)t * COLS; // x of this thread's column 0
    const int64_t y0 = band * RB;
    const int64_t y1 = min(a.H, y0 + RB);
    const int64_t W = a.W;

    __shared__ int sTot[2][TPB / 32][4];              // warp totals of (v, xw, sq)
    __shared__ V sEdgeFF[2][TPB / 32][4][2];  // lane-0 FF_old[0..1] per kind
    __shared__ V sEdgeQ[2][TPB / 32][4];      // lane-31 GG_old[3]+P[3]
    __shared__ V sEdgeP[2][TPB / 32][4];      // lane-0 P[0]

    V S[NK][COLS], FF[NK][COLS], GG[NK][COLS];
    // carry: state at row y0-1
    if (kMode == 1 && band > 0) {
        for (int kk = 0; kk < NK; ++kk) {
            const int k = KIND(kk);
            const V* pS = st_ptr<V>(a, band - 1, k, 0);
            const V* pF = st_ptr<V>(a, band - 1, k, 1);
            const V* pG = st_ptr<V>(a, band - 1, k, 2);
            const V swk = pS[W - 1 + OFF];
#pragma unroll
            for (int j = 0; j < COLS; ++j) {
                const int64_t x = xb + j;
                S[kk][j] = (x < 0) ? 0 : (x > W - 1 ? swk : pS[x + OFF]);
                FF[kk][j] = (x >= W - 1) ? swk : (x < -OFF ? 0 : pF[x + OFF]);
                GG[kk][j] = (x <= 0 || x > W + RB) ? 0 : pG[x + OFF];
            }
        }
    } else {
#pragma unroll
        for (int kk = 0; kk < NK; ++kk)
#pragma unroll
            for (int j = 0; j < COLS; ++j) S[kk][j] = FF[kk][j] = GG[kk][j] = 0;
    }

    if (kMode == 1 && band == 0) {
        // plane row 0 (y = -1) is zero in all 12 planes
        const int64_t c = c0 - RB - 1 + (int64_t)t * COLS;
        if (c >= c0 && c < c0 + CW && c < a.pitch) {
            for (int p = 0; p < 12; ++p) {
                if (NK == 2 && (p & 1) != kg) continue;  // plane p holds kind p % 4
                if (sizeof(V) == 8 && a.planes) {
                    long long* dst = a.planes + p * a.plane_stride + c;
                    reinterpret_cast<longlong2*>(dst)[0] = make_longlong2(0, 0);
                    reinterpret_cast<longlong2*>(dst)[1] = make_longlong2(0, 0);
                }
                if (a.planes32) *reinterpret_cast<uint4*>(a.planes32 + p * a.plane_stride + c) = make_uint4(0, 0, 0, 0);
            }
            if (kg == 0)
                for (int p = 0; p < 3 * a.n_coarse; ++p)
                    *reinterpret_cast<uint2*>(a.coarse + p * a.plane_stride + c) = make_uint2(0, 0);
            if (a.hi16)
                for (int p = 0; p < 12; ++p)
                    if (NK == 4 || (p & 1) == kg) *reinterpret_cast<uint2*>(a.hi16 + p * a.plane_stride + c) = make_uint2(0, 0);
        }
    }

    const int64_t g0 = (XL + 1) / kGroup;  // P(XL) = rowpre(g0): x < XL+1
    // next row's pixels and row prefixes are fetched one row ahead
    int pv[COLS];
    long long pb[3];
    auto fetch = [&](int64_t y) {
        const uint8_t* row = a.img + y * a.img_pitch;
#pragma unroll
        for (int j = 0; j < COLS; ++j) {
            const int64_t x = xb + j;
            pv[j] = (x >= 0 && x < W) ? (int)__ldg(row + x) : 0;
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) pb[q] = rowpre_at(a, y, g0, q);
    };
    if (y0 < y1) fetch(y0);
    int buf = 0;
    for (int64_t y = y0; y < y1; ++y, buf ^= 1) {
        // ── A: pixels, thread-local scans, warp scans ────────────────────
        int lv[COLS], lx[COLS], lq[COLS];
        const long long bv = pb[0], bx = pb[1], bq = pb[2];
        int cv[COLS];
#pragma unroll
        for (int j = 0; j < COLS; ++j) cv[j] = pv[j];
        if (y + 1 < y1) fetch(y + 1);
#pragma unroll
        for (int j = 0; j < COLS; ++j) {
            const int64_t x = xb + j;
            int v = cv[j];
            if (t == 0 && j == 0) v = 0;  // column XL is inside rowpre(g0)
            const int wl = (int)(x - XL);  // local x weight: (x+1) - (XL+1)
            lv[j] = v;
            lx[j] = wl * v;
            lq[j] = v * v;
        }
#pragma unroll
        for (int j = 1; j < COLS; ++j) { lv[j] += lv[j - 1]; lx[j] += lx[j - 1]; lq[j] += lq[j - 1]; }
        int tv = lv[COLS - 1], tx = lx[COLS - 1], tq = lq[COLS - 1];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int ov = __shfl_up_sync(FULL, tv, d), ox = __shfl_up_sync(FULL, tx, d),
                      oq = __shfl_up_sync(FULL, tq, d);
            if (lane >= d) { tv += ov; tx += ox; tq += oq; }
        }
        if (lane == 31) { sTot[buf][warp][0] = tv; sTot[buf][warp][1] = tx; sTot[buf][warp][2] = tq; }
        if (lane == 0) {
#pragma unroll
            for (int kk = 0; kk < NK; ++kk) { sEdgeFF[buf][warp][kk][0] = FF[kk][0]; sEdgeFF[buf][warp][kk][1] = FF[kk][1]; }
        }
        // exclusive thread prefix within the warp
        int ev = __shfl_up_sync(FULL, tv, 1), ex = __shfl_up_sync(FULL, tx, 1), eq = __shfl_up_sync(FULL, tq, 1);
        if (lane == 0) { ev = ex = eq = 0; }
        __syncthreads();

        // ── B: full row prefixes P for the 4 kinds ───────────────────────
        for (int w = 0; w < warp; ++w) { ev += sTot[buf][w][0]; ex += sTot[buf][w][1]; eq += sTot[buf][w][2]; }
        V P[NK][COLS];
#pragma unroll
        for (int j = 0; j < COLS; ++j) {
            const V cv = (V)(ev + lv[j]);
            const V p0 = (V)bv + cv;
#pragma unroll
            for (int kk = 0; kk < NK; ++kk) {
                const int k = KIND(kk);
                P[kk][j] = k == 0 ? p0
                         : k == 1 ? (V)bx + (V)(ex + lx[j]) + (V)(XL + 1) * cv  // (i+1) = (i-XL) + (XL+1)
                         : k == 2 ? (V)(y + 1) * p0
                                  : (V)bq + (V)(eq + lq[j]);
            }
        }
        V Q[NK];
#pragma unroll
        for (int kk = 0; kk < NK; ++kk) Q[kk] = GG[kk][COLS - 1] + P[kk][COLS - 1];
        if (lane == 31) {
#pragma unroll
            for (int kk = 0; kk < NK; ++kk) sEdgeQ[buf][warp][kk] = Q[kk];
        }
        if (lane == 0) {
#pragma unroll
            for (int kk = 0; kk < NK; ++kk) sEdgeP[buf][warp][kk] = P[kk][0];
        }
        __syncthreads();

        // ── C: advance the recurrences, emit planes ──────────────────────
#pragma unroll
        for (int kk = 0; kk < NK; ++kk) {
            const int k = KIND(kk);
            // FF_new(x) = FF_old(x+1) + P(x)
            V nf0 = shfl_down64(FF[kk][0], 1);
            V nf1 = shfl_down64(FF[kk][1], 1);
            V np0 = shfl_down64(P[kk][0], 1);
            if (lane == 31) {
                if (warp + 1 < TPB / 32) {
                    nf0 = sEdgeFF[buf][warp + 1][kk][0];
                    nf1 = sEdgeFF[buf][warp + 1][kk][1];
                    np0 = sEdgeP[buf][warp + 1][kk];
                } else {
                    nf0 = nf1 = np0 = 0;
                }
            }
            // GG_new(x) = GG_old(x-1) + P(x-1)
            V pq = shfl_up64(Q[kk], 1);
            if (lane == 0) pq = (warp > 0) ? sEdgeQ[buf][warp - 1][kk] : 0;
            V Fn[COLS], Gn[COLS];
#pragma unroll
            for (int j = 0; j < COLS - 1; ++j) Fn[j] = FF[kk][j + 1] + P[kk][j];
            Fn[COLS - 1] = nf0 + P[kk][COLS - 1];
            Gn[0] = pq;
#pragma unroll
            for (int j = 1; j < COLS; ++j) Gn[j] = GG[kk][j - 1] + P[kk][j - 1];
            const V fnext = nf1 + np0;  // FF_new of the next thread's column 0
#pragma unroll
            for (int j = 0; j < COLS; ++j) {
                S[kk][j] += P[kk][j];
                FF[kk][j] = Fn[j];
                GG[kk][j] = Gn[j];
            }
            if (kMode == 1) {
                const int64_t c = c0 - RB - 1 + (int64_t)t * COLS;  // plane column of j = 0
                if (c >= c0 && c < c0 + CW && c < a.pitch) {
                    const int64_t off = r_off(a, y + 1) + c;
                    const V e0 = Fn[0] - Gn[0], e1 = Fn[1] - Gn[1], e2 = Fn[2] - Gn[2], e3 = Fn[3] - Gn[3];
                    const V o0 = Fn[1] - Gn[0], o1 = Fn[2] - Gn[1], o2 = Fn[3] - Gn[2], o3 = fnext - Gn[3];
                    if (sizeof(V) == 8 && a.planes) {
                        longlong2* vs = reinterpret_cast<longlong2*>(a.planes + (0 * 4 + k) * a.plane_stride + off);
                        longlong2* ve = reinterpret_cast<longlong2*>(a.planes + (1 * 4 + k) * a.plane_stride + off);
                        longlong2* vo = reinterpret_cast<longlong2*>(a.planes + (2 * 4 + k) * a.plane_stride + off);
                        vs[0] = make_longlong2((long long)S[kk][0], (long long)S[kk][1]);
                        vs[1] = make_longlong2((long long)S[kk][2], (long long)S[kk][3]);
                        ve[0] = make_longlong2((long long)e0, (long long)e1);
                        ve[1] = make_longlong2((long long)e2, (long long)e3);
                        vo[0] = make_longlong2((long long)o0, (long long)o1);
                        vo[1] = make_longlong2((long long)o2, (long long)o3);
                    }
                    if (k == 0 && a.coarse) {  // stage 1's u16 bit slices of the PLAIN cells (K3L)
                        const unsigned sv[3][4] = {{(unsigned)S[kk][0], (unsigned)S[kk][1], (unsigned)S[kk][2], (unsigned)S[kk][3]},
                                                   {(unsigned)e0, (unsigned)e1, (unsigned)e2, (unsigned)e3},
                                                   {(unsigned)o0, (unsigned)o1, (unsigned)o2, (unsigned)o3}};
                        for (int ci = 0; ci < a.n_coarse; ++ci) {
                            const int sh = a.shift[ci];
#pragma unroll
                            for (int ty = 0; ty < 3; ++ty) {
                                const unsigned lo = ((sv[ty][0] >> sh) & 0xffffu) | (((sv[ty][1] >> sh) & 0xffffu) << 16);
                                const unsigned hi = ((sv[ty][2] >> sh) & 0xffffu) | (((sv[ty][3] >> sh) & 0xffffu) << 16);
                                *reinterpret_cast<uint2*>(a.coarse + (ci * 3 + ty) * a.plane_stride + off) =
                                    make_uint2(lo, hi);
                            }
                        }
                    }
                    if (sizeof(V) == 8 && a.hi16 && k != 0) {  // PLAIN ring sums stay below 2^32: no hi16
                        auto hi = [](V v) { return (unsigned)(((unsigned long long)v >> 32) & 0xffffu); };
                        *reinterpret_cast<uint2*>(a.hi16 + (0 * 4 + k) * a.plane_stride + off) =
                            make_uint2(hi(S[kk][0]) | hi(S[kk][1]) << 16, hi(S[kk][2]) | hi(S[kk][3]) << 16);
                        *reinterpret_cast<uint2*>(a.hi16 + (1 * 4 + k) * a.plane_stride + off) =
                            make_uint2(hi(e0) | hi(e1) << 16, hi(e2) | hi(e3) << 16);
                        *reinterpret_cast<uint2*>(a.hi16 + (2 * 4 + k) * a.plane_stride + off) =
                            make_uint2(hi(o0) | hi(o1) << 16, hi(o2) | hi(o3) << 16);
                    }
                    if (a.planes32) {  // the same cells mod 2^32 (region sums are exact in 32 bits)
                        *reinterpret_cast<uint4*>(a.planes32 + (0 * 4 + k) * a.plane_stride + off) =
                            make_uint4((unsigned)S[kk][0], (unsigned)S[kk][1], (unsigned)S[kk][2], (unsigned)S[kk][3]);
                        *reinterpret_cast<uint4*>(a.planes32 + (1 * 4 + k) * a.plane_stride + off) =
                            make_uint4((unsigned)e0, (unsigned)e1, (unsigned)e2, (unsigned)e3);
                        *reinterpret_cast<uint4*>(a.planes32 + (2 * 4 + k) * a.plane_stride + off) =
                            make_uint4((unsigned)o0, (unsigned)o1, (unsigned)o2, (unsigned)o3);
                    }
                }
            }
        }
    }

    if (kMode == 0) {
        // local end state of the band (rows y0..y1-1, y1 - y0 == RB here)
        const bool first = (chunk == 0), last = (chunk == a.n_chunks - 1);
#pragma unroll
        for (int j = 0; j < COLS; ++j) {
            const int64_t x = xb + j;
            const int64_t c = x + 1;
            const bool owned = (c >= c0 && c < c0 + CW) || (first && c < c0) || (last && c >= c0 + CW);
            if (!owned) continue;
#pragma unroll
            for (int kk = 0; kk < NK; ++kk) {
                const int k = KIND(kk);
                if (x >= 0 && x <= W - 1) st_ptr<V>(a, band, k, 0)[x + OFF] = S[kk][j];
                if (x >= -OFF && x <= W - 2) st_ptr<V>(a, band, k, 1)[x + OFF] = FF[kk][j];
                if (x >= 1 && x <= W + RB) st_ptr<V>(a, band, k, 2)[x + OFF] = GG[kk][j];
            }
        }
    }
}

// Pass 1, direct form: a band's zero-carry end state without running the row
// recurrences.  Unrolling them over the band's rows y0..e (e = y0 + RB - 1):
//   S_e(x)  = sum_y P_y(x)
//   FF_e(x) = sum_y P_y(x + e - y)            (P_y(z) = P_y(W-1) for z >= W)
//   GG_e(x) = sum_y P_y(x - 1 - e + y)        (P_y(z) = 0 for z < 0)
// With a group-aligned base B <= every z a tile needs, P_y(z) = R_y +
// sum_{B <= i <= z} v(i,y) (R_y = rowpre_y(B)), so each state is sum_y R_y
// plus a prefix over x of line sums of the band's pixels: column sums C(p)
// for S, anti-diagonal sums A(u) = sum_y v(u + e - y, y) for FF, diagonal sums
// D(w) = sum_y v(w - 1 - e + y, y) for GG (pixels left of B count as zero).
// Per line three small sums (v, y_local v, v^2) give all four kinds; the
// image tile is staged in shared memory; one block scan per state.  Replaces
// band_kernel<0>'s RB row steps of 12 recurrences (config 4: 2.8 ms).
constexpr int P1_TPB = 256;
constexpr int P1_K = 3;  // line positions per thread
constexpr int P1_L = P1_TPB * P1_K;
// state columns owned per CTA: the positions also cover the halo P0 .. xa
// (at most 2 RB + 15 columns)
__host__ __device__ constexpr int p1_cw(int rb) { return P1_L - 2 * rb - 16; }
// tile columns: the L positions, RB on each side, and up to 15 of 16-byte alignment
__host__ __device__ constexpr int p1_tw(int rb) { return (P1_L + 2 * rb + 15 + 15) & ~15; }
__host__ __device__ constexpr size_t p1_smem(int rb) { return (size_t)rb * p1_tw(rb); }

template <int RB, typename V>
__global__ void __launch_bounds__(P1_TPB) band_state_kernel(BuildArgs a) {
    constexpr int L = P1_L, CW = p1_cw(RB), TW = p1_tw(RB);
    constexpr int OFF = RB + 1;
    extern __shared__ __align__(16) unsigned char p1_tile[];
    auto tile = reinterpret_cast<unsigned char(*)[TW]>(p1_tile);
    __shared__ V wtot[3][P1_TPB / 32][4];
    __shared__ V sR[4];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t W = a.W;
    const int64_t band = a.band0 + blockIdx.y;
    const int64_t y0 = band * RB;
    const int64_t xa = -OFF + (int64_t)blockIdx.x * CW;  // owned x in [xa, xa + CW)
    int64_t B = xa - RB - 1;
    B = B <= 0 ? 0 : (B / kGroup) * kGroup;
    const int64_t P0 = B - RB + 1 < xa ? B - RB + 1 : xa;  // first line position
    const int64_t T0 = (P0 - RB) & ~(int64_t)15;            // tile column 0 (16-aligned image column)
    const int OC = (int)(P0 - T0);                          // tile column of position P0 (RB .. RB + 15)
    // stage the band's pixels of columns [T0, T0 + TW): zero left of B and from W on
    const bool vec = ((reinterpret_cast<uintptr_t>(a.img) | (uintptr_t)a.img_pitch) & 15) == 0;
    for (int q = t; q < RB * (TW / 16); q += P1_TPB) {
        const int r = q / (TW / 16), c = (q - r * (TW / 16)) * 16;
        const int64_t i = T0 + c;
        const uint8_t* src = a.img + (y0 + r) * a.img_pitch + i;
        uint4 v;
        if (vec && i >= B && i + 16 <= W) {
            v = __ldg(reinterpret_cast<const uint4*>(src));
        } else {
            unsigned w[4] = {0, 0, 0, 0};
            for (int b = 0; b < 16; ++b)
                if (i + b >= B && i + b < W) w[b >> 2] |= (unsigned)__ldg(src + b) << (8 * (b & 3));
            v = make_uint4(w[0], w[1], w[2], w[3]);
        }
        *reinterpret_cast<uint4*>(&tile[r][c]) = v;
    }
    // sum_y R_y per kind (PLAIN, X, Y, SQ), R_y = rowpre_y(B): warp 0 over the band's rows
    if (warp == 0) {
        long long R[4] = {0, 0, 0, 0};
        const int64_t g = B / kGroup;
        for (int r = lane; r < RB; r += 32) {
            const long long r0 = rowpre_at(a, y0 + r, g, 0);
            R[0] += r0;
            R[1] += rowpre_at(a, y0 + r, g, 1);
            R[2] += (long long)(y0 + r + 1) * r0;
            R[3] += rowpre_at(a, y0 + r, g, 2);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) R[k] += shfl_down64(R[k], d);
            if (lane == 0) sR[k] = (V)R[k];
        }
    }
    __syncthreads();
    // type 0 (S): column lines (p, y); type 1 (FF): anti-diagonals (p + e - y, y);
    // type 2 (GG): diagonals (p - 1 - e + y, y) = (p - RB + r, y0 + r).
    // X weight of a pixel on the line of p: (p + xo) + dr r.
#pragma unroll 1
    for (int ty = 0; ty < 3; ++ty) {
        const int cb = OC + (ty == 0 ? 0 : (ty == 1 ? RB - 1 : -RB));
        const int dr = ty == 0 ? 0 : (ty == 1 ? -1 : 1);
        const V xo = (V)(ty == 0 ? 1 : (ty == 1 ? RB : 1 - RB));
        V inc[P1_K][4];
#pragma unroll
        for (int j = 0; j < P1_K; ++j) {
            const int pc = t * P1_K + j;  // p - P0
            const unsigned char* col = &tile[0][cb + pc];
            int sv = 0, sy = 0, sq = 0;
#pragma unroll 9
            for (int r = 0; r < RB; ++r) {
                const int v = col[r * (TW + dr)];
                sv += v;
                sy += r * v;
                sq += v * v;
            }
            const V p = (V)(P0 + pc);
            inc[j][0] = (V)sv;
            inc[j][1] = (p + xo) * (V)sv + (V)(dr * sy);
            inc[j][2] = (V)(y0 + 1) * (V)sv + (V)sy;
            inc[j][3] = (V)sq;
        }
        // inclusive prefix over positions: thread-local, warp, block
#pragma unroll
        for (int j = 1; j < P1_K; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k) inc[j][k] += inc[j - 1][k];
        V ex[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            V v = inc[P1_K - 1][k];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const V o = shfl_up64(v, d);
                if (lane >= d) v += o;
            }
            if (lane == 31) wtot[ty][warp][k] = v;
            ex[k] = v - inc[P1_K - 1][k] + sR[k];
        }
        __syncthreads();
        for (int w = 0; w < warp; ++w)
#pragma unroll
            for (int k = 0; k < 4; ++k) ex[k] += wtot[ty][w][k];
        const int64_t lo = ty == 0 ? 0 : (ty == 1 ? -OFF : 1), hi = ty == 0 ? W - 1 : (ty == 1 ? W - 2 : W + RB);
#pragma unroll
        for (int j = 0; j < P1_K; ++j) {
            const int64_t x = P0 + t * P1_K + j;
            if (x < xa || x >= xa + CW || x < lo || x > hi) continue;
#pragma unroll
            for (int k = 0; k < 4; ++k) st_ptr<V>(a, band, k, ty)[x + OFF] = ex[k] + inc[j][k];
        }
    }
}

// Row prefixes at group boundaries: rowpre[y][g] = sums over x < kGroup * g
// of (v, (x+1) v, v^2), g = 0..G.  One warp per row.
__global__ void rowpre_kernel(BuildArgs a, int64_t y0, int64_t y1) {
    const int64_t y = y0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (y >= y1) return;
    const uint8_t* row = a.img + y * a.img_pitch;
    long long* out = const_cast<long long*>(a.rowpre) + y * (a.G + 1) * 3;
    if (lane == 0) out[0] = out[1] = out[2] = 0;
    long long c0 = 0, c1 = 0, c2 = 0;
    for (int64_t gb = 0; gb < a.G; gb += 32) {
        const int64_t g = gb + lane;
        long long s0 = 0, s1 = 0, s2 = 0;
        if (g < a.G) {
            const int64_t xa = g * kGroup, xe = min(a.W, xa + kGroup);
            for (int64_t x = xa; x < xe; ++x) {
                const long long v = __ldg(row + x);
                s0 += v;
                s1 += (x + 1) * v;
                s2 += v * v;
            }
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long o0 = shfl_up64(s0, d), o1 = shfl_up64(s1, d), o2 = shfl_up64(s2, d);
            if (lane >= d) { s0 += o0; s1 += o1; s2 += o2; }
        }
        if (g < a.G) {
            out[(g + 1) * 3 + 0] = c0 + s0;
            out[(g + 1) * 3 + 1] = c1 + s1;
            out[(g + 1) * 3 + 2] = c2 + s2;
        }
        c0 += __shfl_sync(FULL, s0, 31);
        c1 += __shfl_sync(FULL, s1, 31);
        c2 += __shfl_sync(FULL, s2, 31);
    }
}

// Pass 2 loads a batch of band states into registers before the dependent
// running sum, so the serial chain is over adds, not memory round trips.
constexpr int SCAN_BATCH = 16;

// Pass 2a: inclusive band states of the SAT rows (in place).
// Scans cover bands [bb, nb) (row-range builds continue from band bb - 1's
// inclusive state; bb = 0 is the whole image).
template <typename V>
__global__ void band_scan_s_kernel(BuildArgs a, int64_t nb, int RB, int64_t bb) {
    const int OFF = RB + 1;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= 4 * a.W) return;
    const int k = (int)(gid / a.W);
    const int64_t x = gid % a.W;
    V acc = bb > 0 ? st_ptr<V>(a, bb - 1, k, 0)[x + OFF] : (V)0;
    for (int64_t b0 = bb; b0 < nb; b0 += SCAN_BATCH) {
        V v[SCAN_BATCH];
#pragma unroll
        for (int j = 0; j < SCAN_BATCH; ++j) v[j] = (b0 + j < nb) ? st_ptr<V>(a, b0 + j, k, 0)[x + OFF] : 0;
#pragma unroll
        for (int j = 0; j < SCAN_BATCH; ++j) {
            if (b0 + j < nb) {
                acc += v[j];
                st_ptr<V>(a, b0 + j, k, 0)[x + OFF] = acc;
            }
        }
    }
}

// Pass 2b: inclusive FF / GG band states.  FF paths move left by RB per band
// (clamped to S(W-1) beyond the right edge), GG paths move right (zero at
// x <= 0).  Each stored element is read and written by exactly one thread.
template <typename V>
__global__ void band_scan_fg_kernel(BuildArgs a, int64_t nb, int RB, int64_t bb) {
    const int OFF = RB + 1;
    const int64_t W = a.W;
    const int64_t nF = W - 1 + OFF + (nb - 1) * RB, nG = W + RB + (nb - 1) * RB;
    const int64_t per_kind = nF + nG;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= 4 * per_kind) return;
    const int k = (int)(gid / per_kind);
    const int64_t i = gid % per_kind;
    const bool ff = i < nF;
    // FF: p0 in [-OFF, W-2 + (nb-1) RB], p = p0 - b RB; GG: p0 in [1-(nb-1)RB, W+RB], p = p0 + b RB
    const int64_t p0 = ff ? (-OFF + i) : (1 - (nb - 1) * RB + (i - nF));
    const int64_t step = ff ? -RB : RB;
    V acc = 0;
    if (bb > 0) {  // the path's inclusive value at band bb - 1 (same clamp rules as below)
        const int64_t p = p0 + (bb - 1) * step;
        if (ff) {
            if (p < -OFF) return;  // the path left the stored range (moving left)
            acc = p >= W - 1 ? st_ptr<V>(a, bb - 1, k, 0)[W - 1 + OFF] : st_ptr<V>(a, bb - 1, k, 1)[p + OFF];
        } else {
            if (p > W + RB) return;  // moving right, beyond the stored range
            acc = p <= 0 ? (V)0 : st_ptr<V>(a, bb - 1, k, 2)[p + OFF];
        }
    }
    for (int64_t b0 = bb; b0 < nb; b0 += SCAN_BATCH) {
        V v[SCAN_BATCH];
        int kind[SCAN_BATCH];  // 0 skip/stop, 1 accumulate+store, 2 clamp (FF: acc = S(W-1); GG: acc = 0)
#pragma unroll
        for (int j = 0; j < SCAN_BATCH; ++j) {
            const int64_t b = b0 + j;
            const int64_t p = p0 + b * step;
            v[j] = 0;
            kind[j] = 0;
            if (b >= nb) continue;
            if (ff) {
                if (p < -OFF) continue;
                if (p >= W - 1) { kind[j] = 2; v[j] = st_ptr<V>(a, b, k, 0)[W - 1 + OFF]; }
                else { kind[j] = 1; v[j] = st_ptr<V>(a, b, k, 1)[p + OFF]; }
            } else {
                if (p > W + RB) continue;
                if (p <= 0) { kind[j] = 2; }
                else { kind[j] = 1; v[j] = st_ptr<V>(a, b, k, 2)[p + OFF]; }
            }
        }
#pragma unroll
        for (int j = 0; j < SCAN_BATCH; ++j) {
            if (kind[j] == 2) {
                acc = v[j];
            } else if (kind[j] == 1) {
                acc += v[j];
                const int64_t p = p0 + (b0 + j) * step;
                st_ptr<V>(a, b0 + j, k, ff ? 1 : 2)[p + OFF] = acc;
            }
        }
    }
}

}  // namespace

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

static size_t rowpre_bytes(int64_t W, int64_t H) { return align_up((size_t)H * (n_groups(W) + 1) * 3 * 8, 256); }
static size_t state_bytes(int64_t W, int64_t H) {
    size_t need = 0;
    for (bool wide : {true, false}) {  // either build geometry
        const int rb = pick_band_rows(W, H, wide);
        const int64_t nb = n_bands(H, rb) - 1;
        if (nb > 0) need = std::max(need, align_up((size_t)nb * 12 * state_len(W, rb) * 8, 256));
    }
    return need;
}

size_t build_workspace_bytes(int64_t W, int64_t H) { return rowpre_bytes(W, H) + state_bytes(W, H); }

// Bands [b_lo, b_hi) of an image of nbands bands: pass 1 and the scans for
// the bands among them whose end state is needed (all but the image's last),
// pass 3 for all of them.  Earlier bands' states must be final (a previous
// call over [0, b_lo)).
template <int RB, typename V>
static int launch_bands(BuildArgs& a, int64_t nbands, cudaStream_t s, int64_t b_lo = 0, int64_t b_hi = -1) {
    if (b_hi < 0) b_hi = nbands;
    const int64_t nb = nbands - 1, W = a.W;  // bands with an end state
    const int64_t s_hi = std::min(b_hi, nb);
    if (s_hi > b_lo) {
        a.band0 = b_lo;
        // SS_BUILD_PASS1=rec: the recurrence form of pass 1 (A/B and tests)
        static const bool rec = [] {
            const char* e = getenv("SS_BUILD_PASS1");
            return e && e[0] == 'r';
        }();
        if (rec) {
            band_kernel<0, RB, V><<<dim3((unsigned)a.n_chunks, (unsigned)(s_hi - b_lo)), TPB, 0, s>>>(a);
        } else {
            constexpr size_t smem = p1_smem(RB);
            if (smem > 48 * 1024) {
                static const cudaError_t attr = cudaFuncSetAttribute(
                    band_state_kernel<RB, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (attr != cudaSuccess) {
                    set_error("band_state_kernel smem attribute: %s", cudaGetErrorString(attr));
                    return SS_ECUDA;
                }
            }
            const int64_t span = W + 2 * (RB + 1);  // state x in [-(RB+1), W+RB]
            const unsigned nx = (unsigned)((span + p1_cw(RB) - 1) / p1_cw(RB));
            band_state_kernel<RB, V><<<dim3(nx, (unsigned)(s_hi - b_lo)), P1_TPB, smem, s>>>(a);
        }
        note_launch();
        if (int e = check_launch("band pass 1")) return e;
        band_scan_s_kernel<V><<<(unsigned)((4 * W + 255) / 256), 256, 0, s>>>(a, s_hi, RB, b_lo);
        note_launch();
        if (int e = check_launch("band_scan_s_kernel")) return e;
        const int64_t per_kind = (W - 1 + (RB + 1) + (s_hi - 1) * RB) + (W + RB + (s_hi - 1) * RB);
        band_scan_fg_kernel<V><<<(unsigned)((4 * per_kind + 255) / 256), 256, 0, s>>>(a, s_hi, RB, b_lo);
        note_launch();
        if (int e = check_launch("band_scan_fg_kernel")) return e;
    }
    a.band0 = b_lo;
    // the 32-bit build: two CTAs per tile, two kinds each (2048^2: 0.124 -> 0.117 ms,
    // 4096^2: 0.392 -> 0.372); the int64 / hi16 build keeps one CTA per tile
    // (config 4 split: 6.57 -> 7.50 ms).  SS_BUILD_KINDS=2|4 forces either.
    static const int kinds = [] {
        const char* e = getenv("SS_BUILD_KINDS");
        return e ? atoi(e) : 0;
    }();
    if (kinds == 2 || (kinds != 4 && sizeof(V) == 4))
        band_kernel<1, RB, V, 2><<<dim3((unsigned)a.n_chunks, (unsigned)(b_hi - b_lo), 2), TPB, 0, s>>>(a);
    else
        band_kernel<1, RB, V><<<dim3((unsigned)a.n_chunks, (unsigned)(b_hi - b_lo)), TPB, 0, s>>>(a);
    note_launch();
    return check_launch("band_kernel<final>");
}

int build_tables(const uint8_t* d_img, int64_t W, int64_t H, int64_t img_pitch, int64_t* d_planes, uint32_t* d_planes32,
                 int64_t plane_pitch_, void* d_ws, size_t ws_bytes, void* stream, uint16_t* d_coarse = nullptr,
                 int n_coarse = 0, const int32_t* h_shifts = nullptr, uint16_t* d_hi16 = nullptr, int64_t y0 = 0,
                 int64_t y1 = -1) {
    if (W < 1 || H < 1) { set_error("empty image"); return SS_EINVAL; }
    if (overflow_guard_fails(W, H)) {
        set_error("image %lldx%lld too large for 64-bit integral cells", (long long)W, (long long)H);
        return SS_EINVAL;
    }
    if (img_pitch < W) { set_error("img_pitch %lld < width %lld", (long long)img_pitch, (long long)W); return SS_EINVAL; }
    if (plane_pitch_ != plane_pitch(W)) {
        set_error("plane_pitch must be ss_plane_pitch(W) = %lld", (long long)plane_pitch(W));
        return SS_EINVAL;
    }
    if (!d_img || (!d_planes && !d_planes32) || (reinterpret_cast<uintptr_t>(d_planes) & 15) ||
        (reinterpret_cast<uintptr_t>(d_planes32) & 15)) {
        set_error("null or misaligned device pointer");
        return SS_EINVAL;
    }
    if (n_coarse < 0 || n_coarse > SS_MAX_COARSE || (n_coarse > 0 && (!d_coarse || !h_shifts)) ||
        (reinterpret_cast<uintptr_t>(d_coarse) & 15) || (reinterpret_cast<uintptr_t>(d_hi16) & 15) ||
        (d_hi16 && !d_planes32)) {
        set_error("bad coarse / hi16 planes");
        return SS_EINVAL;
    }
    for (int i = 0; i < n_coarse; ++i)
        if (h_shifts[i] < 0 || h_shifts[i] > 16) {  // bits [shift, shift + 16) of a cell known mod 2^32
            set_error("coarse shift %d outside [0, 16]", (int)h_shifts[i]);
            return SS_EINVAL;
        }
    const size_t need = build_workspace_bytes(W, H);
    if (ws_bytes < need || (need && !d_ws)) {
        set_error("build workspace too small: %zu < %zu", ws_bytes, need);
        return SS_EINVAL;
    }
    cudaStream_t s = as_stream(stream);
    const bool exact = d_planes || d_hi16;  // int64 recurrences (cells beyond 32 bits are written)
    const int rb = pick_band_rows(W, H, exact);
    BuildArgs a;
    a.img = d_img;
    a.W = W;
    a.H = H;
    a.img_pitch = img_pitch;
    a.planes = reinterpret_cast<long long*>(d_planes);
    a.planes32 = reinterpret_cast<unsigned*>(d_planes32);
    a.pitch = plane_pitch_;
    a.plane_stride = (H + 1) * plane_pitch_;
    a.G = n_groups(W);
    a.rowpre = reinterpret_cast<long long*>(d_ws);
    a.state = reinterpret_cast<long long*>(static_cast<char*>(d_ws) + rowpre_bytes(W, H));
    a.slen = state_len(W, rb);
    a.n_chunks = n_chunks(W, rb);
    a.hi16 = reinterpret_cast<unsigned short*>(d_hi16);
    a.coarse = reinterpret_cast<unsigned short*>(d_coarse);
    a.n_coarse = d_coarse ? n_coarse : 0;
    for (int i = 0; i < SS_MAX_COARSE; ++i) a.shift[i] = i < a.n_coarse ? (int)h_shifts[i] : 0;
    const int64_t nbands = n_bands(H, rb);
    // row range [y0, y1): whole bands (a later call continues from the state
    // of band y0 / rb - 1, which an earlier call over the rows above wrote)
    if (y1 < 0) y1 = H;
    if (y0 < 0 || y1 > H || y0 >= y1 || y0 % rb || (y1 % rb && y1 != H)) {
        set_error("row range [%lld, %lld) is not a run of whole %d-row bands", (long long)y0, (long long)y1, rb);
        return SS_EINVAL;
    }
    const int64_t b_lo = y0 / rb, b_hi = (y1 + rb - 1) / rb;
    a.band0 = 0;

    rowpre_kernel<<<(unsigned)(((y1 - y0) * 32 + 255) / 256), 256, 0, s>>>(a, y0, y1);
    note_launch();
    if (int e = check_launch("rowpre_kernel")) return e;
    // exact int64 recurrences when the int64 or hi16 planes are wanted, else mod 2^32
    if (exact) {
        switch (rb) {
        case 63: return launch_bands<63, long long>(a, nbands, s, b_lo, b_hi);
        case 31: return launch_bands<31, long long>(a, nbands, s, b_lo, b_hi);
        default: return launch_bands<15, long long>(a, nbands, s, b_lo, b_hi);
        }
    }
    switch (rb) {
    case 63: return launch_bands<63, unsigned>(a, nbands, s, b_lo, b_hi);
    case 31: return launch_bands<31, unsigned>(a, nbands, s, b_lo, b_hi);
    default: return launch_bands<15, unsigned>(a, nbands, s, b_lo, b_hi);
    }
}

}  // namespace ss

extern "C" {
int64_t ss_plane_pitch(int64_t W) { return ss::plane_pitch(W); }
size_t ss_tables_bytes(int64_t W, int64_t H) { return (size_t)12 * (size_t)(H + 1) * ss::plane_pitch(W) * 8; }
size_t ss_tables32_bytes(int64_t W, int64_t H) { return (size_t)12 * (size_t)(H + 1) * ss::plane_pitch(W) * 4; }
size_t ss_build_workspace_bytes(int64_t W, int64_t H) { return ss::build_workspace_bytes(W, H); }
int ss_build_tables(const uint8_t* d_img, int64_t W, int64_t H, int64_t img_pitch, int64_t* d_planes,
                    int64_t plane_pitch, void* d_workspace, size_t workspace_bytes, void* stream) {
    return ss::build_tables(d_img, W, H, img_pitch, d_planes, nullptr, plane_pitch, d_workspace, workspace_bytes,
                            stream);
}
int ss_build_tables2(const uint8_t* d_img, int64_t W, int64_t H, int64_t img_pitch, int64_t* d_planes,
                     uint32_t* d_planes32, int64_t plane_pitch, void* d_workspace, size_t workspace_bytes,
                     void* stream) {
    return ss::build_tables(d_img, W, H, img_pitch, d_planes, d_planes32, plane_pitch, d_workspace, workspace_bytes,
                            stream);
}
size_t ss_coarse_bytes(int64_t W, int64_t H, int32_t n_coarse) {
    // + 16 rows: stage 1's row-step TMA views (row mod step, row / step) address
    // whole groups of up to 16 rows, the last of which may end past row H
    return (size_t)3 * (size_t)n_coarse * (size_t)(H + 1) * ss::plane_pitch(W) * 2 + (size_t)16 * ss::plane_pitch(W) * 2;
}
int32_t ss_build_band_rows(int64_t W, int64_t H, int32_t exact) { return ss::pick_band_rows(W, H, exact != 0); }
int ss_build_tables_rows(const uint8_t* d_img, int64_t W, int64_t H, int64_t img_pitch, int64_t* d_planes,
                         uint32_t* d_planes32, uint16_t* d_hi16, int64_t plane_pitch, uint16_t* d_coarse,
                         int32_t n_coarse, const int32_t* h_shifts, int64_t y0, int64_t y1, void* d_workspace,
                         size_t workspace_bytes, void* stream) {
    return ss::build_tables(d_img, W, H, img_pitch, d_planes, d_planes32, plane_pitch, d_workspace, workspace_bytes,
                            stream, d_coarse, n_coarse, h_shifts, d_hi16, y0, y1);
}
size_t ss_tables_hi16_bytes(int64_t W, int64_t H) { return (size_t)12 * (size_t)(H + 1) * ss::plane_pitch(W) * 2; }
int ss_build_tables3(const uint8_t* d_img, int64_t W, int64_t H, int64_t img_pitch, int64_t* d_planes,
                     uint32_t* d_planes32, uint16_t* d_hi16, int64_t plane_pitch, uint16_t* d_coarse,
                     int32_t n_coarse, const int32_t* h_shifts, void* d_workspace, size_t workspace_bytes,
                     void* stream) {
    return ss::build_tables(d_img, W, H, img_pitch, d_planes, d_planes32, plane_pitch, d_workspace, workspace_bytes,
                            stream, d_coarse, n_coarse, h_shifts, d_hi16);
}
}
