// ss_ladder_screen.cu -- K3 for a whole ladder in lock-step (fused sizes).
//
// The per-size screen (ss_screen.cu) reads every plane once per ladder size:
// a 9-size ladder streams the 12 planes from HBM nine times, in 18 launches.
// Here all sizes that share a plane width advance through the image
// together, in two launches per row band:
//   * ladder_stage1_kernel -- the stage-1 tile space is (strip, tile row,
//     size, tile column): every size's tiles of one 16-row block are handed
//     out back to back, so the ring-0 PLAIN corner boxes of all sizes come
//     from the same rows while they sit in L2;
//   * ladder_rings_kernel -- consumes the single candidate list in that
//     order; each entry carries its size (y | size << TAG_SHIFT), each lane
//     reads its size's ring parameters from shared memory, and deeper rings
//     go through the same per-warp queues as in the per-size kernel.
// A plane row is therefore fetched from HBM about once per row band instead
// of once per size.  The decisions are the per-size kernels' (same device
// helpers, same fp64 op order): only the order of work changes.
//
// Replaces, for all sizes of screen()'s ladder loop at once (screening.py:
// 502-520), the per-size _scan_size (screening.py:418-471).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <type_traits>
#include <vector>

#include "ss_screen_dev.cuh"

namespace ss {
namespace {

constexpr int FMAX_SIZES = 64;  // sizes per fused group (larger groups are declined: per-size path); bounded by the 32 KB of kernel parameters
static_assert(FMAX_SIZES <= SS_MAX_SIZES, "fused group size");
constexpr int FMAX_RINGS = 104;  // rings over all fused sizes (kernel parameters <= 32 KB)
constexpr int TAG_SHIFT = 24;    // list entry .y = row | size << TAG_SHIFT
constexpr int YMASK = (1 << TAG_SHIFT) - 1;
constexpr int S1_BITS_WORDS = 4096;  // stage-1 mean-projection bits of all sizes

constexpr int S1_VIEWS = 5;                    // row steps 1, 2, 4, 8, 16
constexpr int S1_SUPER = 1 << (S1_VIEWS - 1);  // tile-row blocks per super row (= the largest step)

struct SizeDev {
    unsigned* mask;        // this size's mask; row 0 is global row mask_y0
    unsigned* row_counts;  // per mask row
    int lo, hi, n_rings, ring0;
    int bm1, wm1, bsrc1;  // stage-1 mean bits: smem word offset (-1: binary search), words, blob u32 index
    int c_sq, c_di;       // coarse stage 1: plane-set index of ring 0's square / diamond sums
    float fa_c, fb_c;     // coarse stage 1: 2^shift / (2 count q_mean) of the square / diamond
    float band_c;         // coarse stage 1: bound on |t_coarse - t| from the bit slices (K3L)
    float t0_c;           // coarse stage 1: 1/2 - fa_c - fb_c (estimate from the sums biased by one)
    int contig;           // ring 0's mean projection is one run of cells [B0, B1) (or empty): w* below apply
    // candidate window of the estimate per row-step view v (rows tested: one in
    // 1 << v): [B0, B1) widened by the estimate's bound and by the most t can
    // move inside a row group (ladder_stage1_coarse_kernel)
    float wlo[S1_VIEWS], whi[S1_VIEWS];
    int s1_views;         // views 0 .. s1_views - 1 are allowed for this size (>= 1)
};

struct FusedArgs {
    const void* planes;  // 12 planes of T
    const unsigned* planes32;  // the 32-bit planes
    const unsigned short* hi16;  // bits 32..47 of the cells (the rings' wide48 path)
    long long pitch, ps;
    int W, H, y_origin, y_begin, y_end, stride;  // [y_begin, y_end): rows decided by this pass
    int mask_y0;
    int n_sizes, n_rings, max_levels, bm_words, bm1_words;
    double qm, qs, qg, rqm, rqs, rqg;
    int qpow2;  // see ScreenArgs
    float rqs_f, rqg_f, band_s;
    const long long* blob;  // all sizes' key blobs (offsets in RingDev rebased)
    long long mask_pitch;
    unsigned long long* stage_counts;
    SizeDev size[FMAX_SIZES];
    RingDev ring[FMAX_RINGS];
};
// Stage 1 from coarse planes: per shift set c, the u16 bit slices (cell >>
// shift) & 0xffff of the SAT / E / O PLAIN cells (ss_build_tables3).
constexpr int CNK = SS_MAX_COARSE;
// Row-step views: view v takes every (1 << v)-th row -- a 3-D map (column, row
// mod step, row / step) of the same plane, so a 16-row box at (x, row mod
// step, row / step) holds rows row, row + step, ... (stage 1's row steps).
// View 0 (plain 2-D maps) travels in the kernel parameters; views 1.. live in
// device memory (CoarseViewMaps, written once per plane buffer).
struct CoarseMaps {
    CUtensorMap sat[CNK], e[CNK], o[CNK];
};
struct CoarseViewMaps {
    CUtensorMap sat[S1_VIEWS - 1][CNK], e[S1_VIEWS - 1][CNK], o[S1_VIEWS - 1][CNK];
};
#ifndef S1_SLACK_DEFAULT
#define S1_SLACK_DEFAULT 4.0
#endif
#ifndef S1_RATIO_DEFAULT
#define S1_RATIO_DEFAULT 13.0
#endif
// Stage 1's row steps, chosen on the device per call (ladder_plan_kernel).
struct S1Plan {
    int view[FMAX_SIZES];         // the chosen view (row step 1 << view) per size
    unsigned cnt[FMAX_SIZES][S1_VIEWS + 1];  // samples inside the window of each view; samples taken
    unsigned ticket;
    int pad[3];
};
static_assert(sizeof(FusedArgs) + sizeof(CoarseMaps) + 256 <= 32764, "fused ladder parameters exceed the kernel parameter limit");
static_assert(sizeof(RingDev) % 4 == 0, "RingDev is copied to shared memory by words");

// Candidate-list entries: (x, y | size << TAG_SHIFT), plus -- when stage 1
// runs on the 32-bit PLAIN planes, so ring 0's PLAIN sums are exact u32 -- the
// square and diamond PLAIN sums themselves: the rings kernel then skips ring
// 0's 8 PLAIN gathers (level 0 is most of its work).
#ifndef FUSED_SUMS
#define FUSED_SUMS 0  // measured slower: int4 entries cost more list traffic than the 8 gathers they save (config 1 K3 0.480 -> 0.510 ms, config 4 36.3 -> 38.1 ms)
#endif
template <typename T1> struct FEntryT { using type = int2; };
#if FUSED_SUMS
template <> struct FEntryT<unsigned> { using type = int4; };
#endif
template <typename T1> using FEntry = typename FEntryT<T1>::type;
__device__ __forceinline__ int2 entry_of(int x, int tag, unsigned, unsigned, int2*) { return make_int2(x, tag); }
__device__ __forceinline__ int4 entry_of(int x, int tag, unsigned sq, unsigned sd, int4*) {
    return make_int4(x, tag, (int)sq, (int)sd);
}
template <typename E> __device__ __forceinline__ E no_entry() {
    return entry_of(-1, -1, 0u, 0u, static_cast<E*>(nullptr));
}
constexpr int CAND_BUF = 64;  // per-warp staging of list entries (flushed 32 at a time)

struct TileMapF {
    int n_tx, n_ty, strip, n_sizes;
    long long n_tiles;  // n_tx * n_ty * n_sizes
    // float reciprocals of the divisors of tile_coords_fast (n_tiles < 2^24)
    float r_per_strip, r_strip, r_last, r_span, r_span_last;
};

// q = n / d for n < 2^24 from a float reciprocal rd ~ 1/d, corrected to exact.
__device__ __forceinline__ unsigned fdiv24(unsigned n, unsigned d, float rd) {
    unsigned q = __float2uint_rz(__uint2float_rn(n) * rd);
    const int r = (int)(n - q * d);
    if (r < 0) --q;
    else if (r >= (int)d) ++q;
    return q;
}
// tile_coords_f without integer divisions (n_tiles < 2^24, checked on the host)
__device__ __forceinline__ void tile_coords_fast(const TileMapF& t, unsigned i, int& tx, int& ty, int& s) {
    const unsigned per_strip = (unsigned)t.strip * (unsigned)t.n_ty * (unsigned)t.n_sizes;
    const unsigned st = fdiv24(i, per_strip, t.r_per_strip);
    const int s0 = (int)(st * (unsigned)t.strip);
    const bool last = s0 + t.strip > t.n_tx;
    const unsigned width = last ? (unsigned)(t.n_tx - s0) : (unsigned)t.strip;
    const unsigned r = i - st * per_strip;
    const unsigned span = width * (unsigned)t.n_sizes;
    const unsigned q = fdiv24(r, span, last ? t.r_span_last : t.r_span);
    const unsigned rem = r - q * span;
    const unsigned sz = fdiv24(rem, width, last ? t.r_last : t.r_strip);
    ty = (int)q;
    s = (int)sz;
    tx = s0 + (int)(rem - sz * width);
}

// Fused stage-1 tile geometry: 16 rows x 32*CPW columns; 32-bit planes take
// 128-column tiles (four independent centres per lane: the chains overlap),
// int64 planes 64 (three pipeline stages must fit shared memory).
#ifndef FUSED_CPW32
#define FUSED_CPW32 6  // 32-bit tiles: 32-column chunks per lane (measured: 6 x 2 stages beats 5 x 2, 4 x 3, 3 x 4, 2 x 5)
#endif
#ifndef FUSED_STAGES32
#define FUSED_STAGES32 2
#endif
template <typename T> struct GeoF {
    static constexpr int CPW = sizeof(T) == 4 ? FUSED_CPW32 : 2;
    static constexpr int TX = 32 * CPW;
    static constexpr int STAGES = sizeof(T) == 4 ? FUSED_STAGES32 : 3;
    static constexpr int ALIGN = 16 / (int)sizeof(T);
    static constexpr int BW = TX + ALIGN;
    static constexpr int BOX_ELEMS = BW * TY;
    static constexpr int BOX_BYTES = BOX_ELEMS * (int)sizeof(T);
    static constexpr int STAGE_BYTES = NBOX * BOX_BYTES;
    __device__ static int floor_al(int c) { return c & ~(ALIGN - 1); }
    __device__ static int rem(int c) { return c & (ALIGN - 1); }
};
constexpr int TXMAX = 32 * (FUSED_CPW32 > 2 ? FUSED_CPW32 : 2);  // widest fused tile (workspace sizing)

// A stage-1 tile and the constants of its size, written by the producer next
// to the tile's boxes (the consumers read 4 x 16 B instead of indexing the
// parameter block per tile).
struct __align__(16) TileConst {
    int tx, ty, sz, ylo;
    int yhi, xlo, xhi, bm1;  // bm1: smem word offset of the mean bits, -1: binary search, -2: `win` holds them
    int qr, ql, po0, po1;  // corner columns inside the staged boxes
    float fa, fb;
    int cm_lo, cm_n;
    unsigned win_lo, win_hi;  // ring-0 mean-projection bits of cells cm_lo .. cm_lo + 63 (when cm_n <= 64)
    int pad0, pad1;
};

// strip-major; inside a strip: tile row, then size, then tile column
__device__ __forceinline__ void tile_coords_f(const TileMapF& t, long long idx, int& tx, int& ty, int& s) {
    const unsigned per_strip = (unsigned)t.strip * (unsigned)t.n_ty * (unsigned)t.n_sizes;
    const unsigned i = (unsigned)idx;
    const unsigned st = i / per_strip;
    const int s0 = (int)(st * (unsigned)t.strip);
    const unsigned width = (unsigned)min(t.strip, t.n_tx - s0);
    const unsigned r = i - st * per_strip;
    const unsigned span = width * (unsigned)t.n_sizes;
    const unsigned q = r / span;
    const unsigned rem = r - q * span;
    const unsigned sz = rem / width;
    ty = (int)q;
    s = (int)sz;
    tx = s0 + (int)(rem - sz * width);
}

// Stage 1 of every fused size (interior centres; ladder_border_kernel wrote the
// border keeps): ring-0 mean cell
// from TMA-staged PLAIN corner boxes, mean-projection passers appended to the
// candidate list tagged with their size.  Persistent CTAs; warp WARPS is the
// producer.  Same pipeline as stage1_kernel (ss_screen.cu).
template <typename T>
__global__ void __launch_bounds__((WARPS + 1) * 32, 1)
    ladder_stage1_kernel(const __grid_constant__ FusedArgs a, const __grid_constant__ TmaMaps maps, const TileMapF tm,
                         int parts, int reserve, FEntry<T>* list_base, long long part_cap, unsigned* list_ctr,
                         unsigned* tile_ctr_base) {
    using G = GeoF<T>;
    using E = FEntry<T>;
    constexpr int STAGES = G::STAGES, CPW = G::CPW;
    extern __shared__ __align__(128) unsigned char dsmem[];
    unsigned char* stage_buf = dsmem;
    unsigned* sbits = reinterpret_cast<unsigned*>(dsmem + STAGES * G::STAGE_BYTES);
    __shared__ __align__(8) unsigned long long full_bar[STAGES], empty_bar[STAGES];
    __shared__ TileConst tile_info[STAGES];  // the tile in each stage and its size's constants
    __shared__ E cand_buf[WARPS][CAND_BUF];
    {
        const unsigned* blob32 = reinterpret_cast<const unsigned*>(a.blob);
        for (int s = threadIdx.x >> 5; s < a.n_sizes; s += blockDim.x >> 5) {  // a warp per size
            const SizeDev& S = a.size[s];
            if (S.bm1 < 0) continue;
            for (int i = threadIdx.x & 31; i < S.wm1; i += 32)
                sbits[S.bm1 + i] = S.bsrc1 >= 0 ? __ldg(blob32 + S.bsrc1 + i) : 0u;
        }
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int part = (int)(blockIdx.x % parts);

    if (warp == WARPS) {
        if (lane == 0) {
            const int tc = (int)(blockIdx.x % TILE_CTRS);
            unsigned* tile_ctr = tile_ctr_base + tc * CTR_STRIDE;
            unsigned t_next = atom_add_ahead(tile_ctr, 1u);
            for (int it = 0;; ++it) {
                const int s = it % STAGES;
                const long long t = (long long)t_next * TILE_CTRS + tc;
                if (t < tm.n_tiles) t_next = atom_add_ahead(tile_ctr, 1u);
                mbar_wait(&empty_bar[s], ((it / STAGES) & 1) ^ 1);
                if (t >= tm.n_tiles) {
                    tile_info[s].tx = -1;
                    mbar_arrive(&full_bar[s]);
                    break;
                }
                int tx, ty, sz;
                tile_coords_f(tm, t, tx, ty, sz);
                const SizeDev& S = a.size[sz];
                const RingDev& R0 = a.ring[S.ring0];
                {  // published to the consumers by the mbarrier arrive (complete_tx) below
                    TileConst& tcst = tile_info[s];
                    tcst.tx = tx;
                    tcst.ty = ty;
                    tcst.sz = sz;
                    tcst.ylo = S.lo;
                    tcst.yhi = a.H - 1 - S.hi;
                    tcst.xlo = S.lo;
                    tcst.xhi = a.W - 1 - S.hi;
                    // cm_n <= 64 (every 8-level mean quantizer): the whole
                    // mean projection rides in two registers of the tile
                    if (S.bm1 >= 0 && R0.cm_n <= 64) {
                        tcst.bm1 = -2;
                        tcst.win_lo = sbits[S.bm1];
                        tcst.win_hi = S.wm1 > 1 ? sbits[S.bm1 + 1] : 0u;
                    } else {
                        tcst.bm1 = S.bm1;
                    }
                    tcst.qr = G::rem(R0.n + 1);
                    tcst.ql = G::rem(1 - R0.n);
                    tcst.po0 = G::rem(-R0.d);
                    tcst.po1 = G::rem(R0.d + 1);
                    tcst.fa = R0.fa;
                    tcst.fb = R0.fb;
                    tcst.cm_lo = R0.cm_lo;
                    tcst.cm_n = R0.cm_n;
                }
                const int x0 = tx * G::TX;
                const int cy0 = a.y_begin + ty * TY - a.y_origin;
                unsigned char* dst = stage_buf + s * G::STAGE_BYTES;
                mbar_expect_tx(&full_bar[s], G::STAGE_BYTES);
                const int n = R0.n, d = R0.d;
                tma_load_2d(dst + 0 * G::BOX_BYTES, &maps.sat, G::floor_al(x0 + n + 1), cy0 + n + 1, &full_bar[s]);
                tma_load_2d(dst + 1 * G::BOX_BYTES, &maps.sat, G::floor_al(x0 - n + 1), cy0 + n + 1, &full_bar[s]);
                tma_load_2d(dst + 2 * G::BOX_BYTES, &maps.sat, G::floor_al(x0 + n + 1), cy0 - n + 1, &full_bar[s]);
                tma_load_2d(dst + 3 * G::BOX_BYTES, &maps.sat, G::floor_al(x0 - n + 1), cy0 - n + 1, &full_bar[s]);
                tma_load_2d(dst + 4 * G::BOX_BYTES, &maps.e, G::floor_al(x0 + 1), cy0 + d + 1, &full_bar[s]);
                tma_load_2d(dst + 5 * G::BOX_BYTES, &maps.e, G::floor_al(x0 + 1), cy0 - d, &full_bar[s]);
                tma_load_2d(dst + 6 * G::BOX_BYTES, &maps.o, G::floor_al(x0 - d), cy0, &full_bar[s]);
                tma_load_2d(dst + 7 * G::BOX_BYTES, &maps.o, G::floor_al(x0 + d + 1), cy0, &full_bar[s]);
            }
        }
        return;
    }

    const unsigned lt = (1u << lane) - 1u;
    E* list0 = list_base + part * part_cap;
    unsigned* count0 = list_ctr + part * CTR_STRIDE;
    E* buf = cand_buf[warp];
    int nbuf = 0;
    unsigned res = 0;
    bool have_res = false;
    unsigned res_base = 0, res_left = 0;
    unsigned n_int = 0, n_pass = 0;  // per warp: < 2^32
    const bool unit_stride = a.stride == 1;
    for (int it = 0;; ++it) {
        const int s = it % STAGES;
        mbar_wait(&full_bar[s], (it / STAGES) & 1);
        const TileConst tc = tile_info[s];
        if (tc.tx < 0) break;
        const int tx = tc.tx, ty = tc.ty, sz = tc.sz;
        const int y = a.y_begin + ty * TY + warp;
        // border keeps are already in the masks (ladder_border_kernel); only
        // interior centres of interior grid rows are evaluated here
        const bool row_int = y < a.y_end && y >= tc.ylo && y <= tc.yhi && (unit_stride || (y % a.stride) == 0);
        T s1q[CPW], s1d[CPW];  // exact PLAIN region sums
        if (row_int) {
            const int qr = tc.qr, ql = tc.ql, pe = 1, po0 = tc.po0, po1 = tc.po1;
            const T* box = reinterpret_cast<const T*>(stage_buf + s * G::STAGE_BYTES) + warp * G::BW + lane;
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                const T* b = box + 32 * c;
                constexpr int E = G::BOX_ELEMS;
                s1q[c] = (T)(b[0 * E + qr] - b[1 * E + ql] - b[2 * E + qr] + b[3 * E + ql]);
                s1d[c] = (T)(b[4 * E + pe] - b[6 * E + po0] - b[7 * E + po1] + b[5 * E + pe]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);
        if (!row_int) continue;
        // mean cells of all chunks (fp32 estimate, exact unless within ~4e-6
        // of a cell boundary: see mean_cell), then the rare exact fallback
        int cm[CPW];
        unsigned amb = 0;
#pragma unroll
        for (int c = 0; c < CPW; ++c) {
            const float tf = fmaf(to_f32(s1q[c]), tc.fa, fmaf(to_f32(s1d[c]), tc.fb, 0.5f));
            const float dl = fmaf(tf, 4e-6f, 4e-6f);
            cm[c] = (int)floorf(tf - dl);
            amb |= (unsigned)(cm[c] != (int)floorf(tf + dl)) << c;
        }
        if (__any_sync(FULL, amb != 0)) {
            const RingDev& R0 = a.ring[a.size[sz].ring0];
#pragma unroll
            for (int c = 0; c < CPW; ++c)
                if ((amb >> c) & 1u) cm[c] = mean_cell_exact(a, R0, s1q[c], s1d[c]);
        }
        const int xlo = tc.xlo, xhi = tc.xhi;
        const int tag = y | (sz << TAG_SHIFT);
        const int xt = tx * G::TX;
        const bool full = unit_stride && xt >= xlo && xt + G::TX - 1 <= xhi;  // warp-uniform: no per-lane tests
        unsigned pm = 0;  // bit c: chunk c's centre passes
        if (tc.bm1 == -2) {
            // bits cm_lo..cm_lo+63 in two registers; bits at and above cm_n are 0
            const int cm_lo = tc.cm_lo;
            const unsigned wl = tc.win_lo, wh = tc.win_hi;
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                const unsigned i = (unsigned)(cm[c] - cm_lo);
                const unsigned w = (i & 32u) ? wh : wl;
                pm |= (unsigned)(i < 64u && ((w >> (i & 31u)) & 1u)) << c;
            }
        } else if (tc.bm1 >= 0) {
            const int cm_lo = tc.cm_lo;
            const unsigned cm_n = (unsigned)tc.cm_n;
            const unsigned* bits = sbits + tc.bm1;
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                const unsigned i = (unsigned)(cm[c] - cm_lo);
                pm |= (unsigned)(i < cm_n && bit(bits, (int)i)) << c;
            }
        } else {
            const RingDev& R0 = a.ring[a.size[sz].ring0];
#pragma unroll
            for (int c = 0; c < CPW; ++c) pm |= (unsigned)bsearch_eq(a.blob + R0.off_m, R0.n_m, cm[c]) << c;
        }
        if (!full) {
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                const int x = xt + 32 * c + lane;
                const bool interior = x >= xlo && x <= xhi && (unit_stride || (x % a.stride) == 0);
                if (!interior) pm &= ~(1u << c);
                if (a.stage_counts) n_int += __popc(__ballot_sync(FULL, interior));
            }
        } else if (a.stage_counts) {
            n_int += 32 * CPW;
        }
        if (!__any_sync(FULL, pm != 0u)) continue;  // most warp rows of a tile have no passer
#pragma unroll
        for (int c = 0; c < CPW; ++c) {
            const bool p = (pm >> c) & 1u;
            const unsigned pb = __ballot_sync(FULL, p);
            if (p) buf[nbuf + __popc(pb & lt)] = entry_of(xt + 32 * c + lane, tag, (unsigned)s1q[c], (unsigned)s1d[c], buf);
            nbuf += __popc(pb);
            n_pass += __popc(pb);
            if (nbuf >= 32) {  // < 64 staged: flush the newest 32 (list order is free)
                __syncwarp();
                if (res_left == 0) {
                    if (!have_res && lane == 0) res = atom_add_ahead(count0, (unsigned)reserve);
                    res_base = __shfl_sync(FULL, res, 0);
                    res_left = reserve;
                    if (lane == 0) res = atom_add_ahead(count0, (unsigned)reserve);
                    have_res = true;
                }
                SS_CHECK(res_base + lane < (unsigned)part_cap && nbuf - 32 + lane < CAND_BUF);
                if (res_base + lane < (unsigned)part_cap) list0[res_base + lane] = buf[nbuf - 32 + lane];
                res_base += 32;
                res_left -= 32;
                nbuf -= 32;
                __syncwarp();
            }
        }
    }
    __syncwarp();
    if (have_res) {
        unsigned base = res_base, left = res_left;
        if (left == 0) {
            base = __shfl_sync(FULL, res, 0);
            left = reserve;
        } else {
            const unsigned ahead = __shfl_sync(FULL, res, 0);
            for (unsigned i = lane; i < (unsigned)reserve; i += 32)
                if (ahead + i < (unsigned)part_cap) list0[ahead + i] = no_entry<E>();
        }
        for (unsigned i = lane; i < left; i += 32)
            if (base + i < (unsigned)part_cap) list0[base + i] = i < (unsigned)nbuf ? buf[i] : no_entry<E>();
    } else if (nbuf > 0) {
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(count0, (unsigned)nbuf);
        base = __shfl_sync(FULL, base, 0);
        if (lane < nbuf && base + lane < (unsigned)part_cap) list0[base + lane] = buf[lane];
    }
    if (a.stage_counts && lane == 0) {
        atomicAdd(a.stage_counts + 0, (unsigned long long)n_int);
        atomicAdd(a.stage_counts + 1, (unsigned long long)n_pass);
    }
}

// Coarse stage-1 tiles: 16 rows x TX columns of u16 bit slices, CW consumer
// warps (CW / 16 per tile row, CPW 32-column chunks each).  Boxes are
// 16 x (TX + 8): measured on B200 with tools/tma_probe, 16 x 248-256 u16 boxes
// stream at ~40 B/clk/SM, 16 x 192-200 at ~16, u32 16 x 196 at ~32.
#ifndef COARSE_WARPS
#define COARSE_WARPS 16
#endif
#ifndef COARSE_CPW
#define COARSE_CPW 7
#endif
#ifndef COARSE_STAGES
#define COARSE_STAGES 3
#endif
constexpr int S1_MAX_WARPS = 32;  // consumer warps a stage-1 kernel may have (a CTA holds <= 32 warps)
#ifndef COARSE_TY
#define COARSE_TY 16
#endif
template <int CW_, int CPW_, int STAGES_, int TY_ = COARSE_TY> struct GeoCT {
    static constexpr int CW = CW_;
    static constexpr int TYC = TY_;      // tile rows
    static constexpr int WPR = CW / TYC;  // warps per tile row
    static_assert(WPR * TYC == CW && CW <= S1_MAX_WARPS, "consumer warps tile the rows");
    static constexpr int CPW = CPW_;
    static constexpr int TX = WPR * 32 * CPW;
    static constexpr int STAGES = STAGES_;
    static constexpr int ALIGN = 8;  // 16-byte aligned box starts
#ifdef COARSE_BW
    static constexpr int BW = COARSE_BW;
#else
    static constexpr int BW = TX + ALIGN;
#endif
    static_assert(BW <= 256 && BW >= TX + ALIGN - 1, "box must cover the tile at any alignment (TMA box <= 256)");
    static constexpr int BOX_ELEMS = BW * TYC;
    static constexpr int BOX_BYTES = BOX_ELEMS * 2;
    static_assert(BOX_BYTES % 128 == 0, "TMA destinations stay 128-byte aligned");
    static constexpr int STAGE_BYTES = NBOX * BOX_BYTES;
    __device__ static int floor_al(int c) { return c & ~(ALIGN - 1); }
    __device__ static int rem(int c) { return c & (ALIGN - 1); }
};
using GeoC = GeoCT<COARSE_WARPS, COARSE_CPW, COARSE_STAGES>;

struct __align__(16) TileConstC {
    int tx, ty, sz, ylo;
    int yhi, xlo, xhi, bm1;  // bm1 as TileConst
    int qr, ql, po0, po1;
    float fa, fb, band;  // coarse factors of the size and its error bound
    int cm_lo;
    int cm_n;
    unsigned win_lo, win_hi;
    int contig;  // SizeDev::contig and its windows
    float w0lo, w0hi, w1lo, w1hi;
    float t0;    // 1/2 - fa - fb: the estimate from the biased sums J = I + 1
    int pad[2];
};

// Row steps of the coarse stage 1, chosen per size from a sample of the image
// (ladder_plan_kernel -> S1Plan, read by ladder_stage1_coarse_kernel; no host
// round trip, so the ladder stays one graph-capturable chain).  A size at view
// v tests one centre row per group of 1 << v rows against the window widened
// by the most the ring-0 mean can move inside the group, and sends every row
// of a passing column to the rings kernel: stage 1 costs 1 / step per centre,
// but centres inside the widened window and outside the plain one become
// false candidates (each decided exactly, and rejected, by the rings kernel's
// level 0).  The kernel evaluates ring 0's mean on a lattice of <= PLAN_N x
// PLAN_N centres per size from the 32-bit PLAIN planes, counts the samples in
// each view's window, and picks the view minimising
//     1 / step + ratio * (P_view - P_0),
// ratio = cost of a false candidate in the rings kernel / cost of a stage-1
// centre (measured ~13 on B200: ~28 ps against ~2 ps).
constexpr int PLAN_N = 64;  // lattice points per axis and size (each sample costs 8 sectors: config 4 plans 24 bands x 33 sizes)
constexpr int PLAN_BLOCKS = 8;  // blocks per size (two samples per thread)
// below this many positions x sizes per call the plan cannot repay its launch
// (config 1: stage 1 is 0.15 ms): every size keeps row step 1
constexpr long long PLAN_MIN_WORK = 100000000LL;
__global__ void __launch_bounds__(256) ladder_plan_kernel(const __grid_constant__ FusedArgs a, S1Plan* plan, int y_lo,
                                                          int y_hi, float ratio, int force) {
    const int sz = blockIdx.x / PLAN_BLOCKS, part = blockIdx.x % PLAN_BLOCKS;
    const SizeDev& S = a.size[sz];
    const RingDev& R0 = a.ring[S.ring0];
    __shared__ unsigned c_sh[S1_VIEWS + 1];
    __shared__ bool last_sh;
    if (threadIdx.x <= S1_VIEWS) c_sh[threadIdx.x] = 0;
    __syncthreads();
    const int xlo = S.lo, xhi = a.W - 1 - S.hi;
    const int ylo = max(y_lo, S.lo), yhi = min(y_hi - 1, a.H - 1 - S.hi);
    if (S.s1_views > 1 && !force && xlo <= xhi && ylo <= yhi) {
        const int wx = xhi - xlo + 1, wy = yhi - ylo + 1;
        const int nx = min(PLAN_N, wx), ny = min(PLAN_N, wy);
        const unsigned* P = a.planes32;  // plane type * 4 + kind: PLAIN SAT 0, E 4, O 8
        const long long ps = a.ps, pitch = a.pitch;
        const int n = R0.n, d = R0.d;
        const float fa = (float)(0.5 / ((double)(4LL * n * n) * a.qm));
        const float fb = (float)(0.5 / ((double)(2LL * d * d + 2LL * d + 1) * a.qm));
        unsigned c[S1_VIEWS + 1];
#pragma unroll
        for (int v = 0; v <= S1_VIEWS; ++v) c[v] = 0;
#pragma unroll 2
        for (int i = part * 256 + threadIdx.x; i < nx * ny; i += PLAN_BLOCKS * 256) {
            const int iy = i / nx, ix = i - iy * nx;
            const int cx = xlo + (int)(((long long)(2 * ix + 1) * wx) / (2 * nx));
            const int cy = ylo + (int)(((long long)(2 * iy + 1) * wy) / (2 * ny));
            const long long r = cy - a.y_origin;  // table row of image row cy - 1
            const unsigned* sat = P;
            const unsigned* e = P + 4 * ps;
            const unsigned* o = P + 8 * ps;
            const unsigned sq = __ldg(sat + (r + n + 1) * pitch + cx + n + 1) - __ldg(sat + (r + n + 1) * pitch + cx - n + 1) -
                                __ldg(sat + (r - n + 1) * pitch + cx + n + 1) + __ldg(sat + (r - n + 1) * pitch + cx - n + 1);
            const unsigned di = __ldg(e + (r + d + 1) * pitch + cx + 1) - __ldg(o + r * pitch + cx - d) -
                                __ldg(o + r * pitch + cx + d + 1) + __ldg(e + (r - d) * pitch + cx + 1);
            const float t = fmaf((float)sq, fa, fmaf((float)di, fb, 0.5f));
            ++c[S1_VIEWS];
#pragma unroll
            for (int v = 0; v < S1_VIEWS; ++v) c[v] += v < S.s1_views && t >= S.wlo[v] && t <= S.whi[v];
        }
#pragma unroll
        for (int v = 0; v <= S1_VIEWS; ++v)
            if (c[v]) atomicAdd(&c_sh[v], c[v]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 0; k <= S1_VIEWS; ++k)
            if (c_sh[k]) atomicAdd(&plan->cnt[sz][k], c_sh[k]);
        __threadfence();
        last_sh = atomicAdd(&plan->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last_sh) return;
    __threadfence();
    for (int j = threadIdx.x; j < a.n_sizes; j += blockDim.x) {
        const SizeDev& Sj = a.size[j];
        const volatile unsigned* c = plan->cnt[j];
        int best = 0;
        if (force) {
            best = Sj.s1_views - 1;
        } else if (Sj.s1_views > 1 && c[S1_VIEWS] > 0) {
            const float inv = 1.0f / (float)c[S1_VIEWS];
            float cost = 1.0f;
            for (int v = 1; v < Sj.s1_views; ++v) {
                const float cv = 1.0f / (float)(1 << v) + ratio * (float)(c[v] - c[0]) * inv;
                if (cv < cost) {
                    cost = cv;
                    best = v;
                }
            }
        }
        plan->view[j] = best;
    }
}

// Stage 1 of every fused size from the coarse planes.  A region sum S of
// `count` pixels whose slices have shift k is recovered as the integer I with
// |S - I 2^k| < 2^(k+1) (four floors of cell / 2^k; no wrap since
// 255 count < (2^16 - 4) 2^k, ss_coarse_shift), so the mean-cell estimate
// t = I_sq fa + I_di fb + 1/2 is within band (+ the fp32 terms of mean_cell)
// of the reference's t.  A centre is decided from the estimate unless t lies
// within that bound of a cell boundary whose two cells differ in ring-0
// membership; those centres are passed on as candidates and the rings
// kernel's level 0 decides them from the exact sums (eval_ring_fast tests
// ring 0's mean cell again).  The survivors equal ladder_stage1_kernel's; the
// candidate list is a (slightly larger) superset; half the TMA bytes per
// centre.
__global__ void __launch_bounds__((GeoC::CW + 1) * 32, 1)
    ladder_stage1_coarse_kernel(const __grid_constant__ FusedArgs a, const __grid_constant__ CoarseMaps maps,
                                const CoarseViewMaps* __restrict__ vmaps, const TileMapF tm_in, int parts, int reserve, int2* list_base, long long part_cap,
                                unsigned* list_ctr, unsigned* tile_ctr_base, const S1Plan* plan) {
    using G = GeoC;
    constexpr int STAGES = G::STAGES, CPW = G::CPW, CW = G::CW;
    extern __shared__ __align__(128) unsigned char dsmem[];
    unsigned char* stage_buf = dsmem;
    unsigned* sbits = reinterpret_cast<unsigned*>(dsmem + STAGES * G::STAGE_BYTES);
    __shared__ __align__(8) unsigned long long full_bar[STAGES], empty_bar[STAGES];
    __shared__ int4 slot[STAGES];               // the tile in each stage: (tx, ty, size, -)
    __shared__ TileConstC size_info[FMAX_SIZES];  // per-size constants, filled once
    __shared__ int4 size_tma[FMAX_SIZES];         // per-size (n, d, square plane set | view << 8, diamond plane set)
    __shared__ unsigned short entries[S1_SUPER * FMAX_SIZES];  // tile-row entries of a super row: size | sub-block << 8
    __shared__ TileMapF tm;  // tm_in with the entry count of the plan's row steps
    __shared__ int2 cand_buf[CW][CAND_BUF];
    {
        const unsigned* blob32 = reinterpret_cast<const unsigned*>(a.blob);
        for (int s = threadIdx.x >> 5; s < a.n_sizes; s += blockDim.x >> 5) {  // a warp per size
            const SizeDev& S = a.size[s];
            if (S.bm1 < 0) continue;
            for (int i = threadIdx.x & 31; i < S.wm1; i += 32)
                sbits[S.bm1 + i] = S.bsrc1 >= 0 ? __ldg(blob32 + S.bsrc1 + i) : 0u;
        }
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    for (int sz = threadIdx.x; sz < a.n_sizes; sz += blockDim.x) {
        const SizeDev& S = a.size[sz];
        const RingDev& R0 = a.ring[S.ring0];
        {
                    TileConstC& tcst = size_info[sz];
                    tcst.tx = 0;
                    tcst.ty = 0;
                    tcst.sz = sz;
                    tcst.ylo = S.lo;
                    tcst.yhi = a.H - 1 - S.hi;
                    tcst.xlo = S.lo;
                    tcst.xhi = a.W - 1 - S.hi;
                    if (S.bm1 >= 0 && R0.cm_n <= 64) {
                        tcst.bm1 = -2;
                        tcst.win_lo = sbits[S.bm1];
                        tcst.win_hi = S.wm1 > 1 ? sbits[S.bm1 + 1] : 0u;
                    } else {
                        tcst.bm1 = S.bm1;
                    }
                    tcst.qr = G::rem(R0.n + 1);
                    tcst.ql = G::rem(1 - R0.n);
                    tcst.po0 = G::rem(-R0.d);
                    tcst.po1 = G::rem(R0.d + 1);
                    tcst.fa = S.fa_c;
                    tcst.fb = S.fb_c;
                    tcst.band = S.band_c;
                    tcst.cm_lo = R0.cm_lo;
                    tcst.cm_n = R0.cm_n;
                    tcst.contig = S.contig;
                    const int view = plan ? min(max(__ldg(&plan->view[sz]), 0), S.s1_views - 1) : 0;
                    tcst.w0lo = S.wlo[view];
                    tcst.w0hi = S.wlo[view];
                    tcst.w1lo = S.whi[view];
                    tcst.w1hi = S.whi[view];
                    tcst.t0 = S.t0_c;
                    size_tma[sz] = make_int4(R0.n, R0.d, S.c_sq | (view << 8), S.c_di);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // a super row is S1_SUPER tile rows of 16 image rows; a size of row
        // step s covers it with S1_SUPER / s tiles of 16 s rows each
        int ne = 0;
        for (int sz = 0; sz < a.n_sizes; ++sz) {
            const int st = 1 << (size_tma[sz].z >> 8);
            for (int sub = 0; sub < S1_SUPER / st; ++sub) entries[ne++] = (unsigned short)(sz | (sub << 8));
        }
        tm = tm_in;
        tm.n_sizes = ne;
        tm.n_tiles = (long long)tm.n_tx * tm.n_ty * ne;
        const int last_w = tm.n_tx - (tm.n_tx - 1) / tm.strip * tm.strip;
        tm.r_per_strip = (float)(1.0 / ((double)tm.strip * tm.n_ty * ne));
        tm.r_span = (float)(1.0 / ((double)tm.strip * ne));
        tm.r_span_last = (float)(1.0 / ((double)last_w * ne));
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int part = (int)(blockIdx.x % parts);

    if (warp == CW) {
        if (lane < NBOX) {
            // tiles are uniform work: static round robin over the persistent
            // CTAs (strip-major order kept: the tiles in flight stay contiguous).
            // Lane b issues box b of every tile (measured with tools/tma_probe:
            // 8 issuing lanes stream these u16 boxes at ~53 B/clk/SM, one lane
            // at ~34).
            const bool fast = tm.n_tiles < (1LL << 24);
            const unsigned pmask = (1u << NBOX) - 1u;
            for (int it = 0, k = 0;; ++it) {
                const int s = k % STAGES;
                const long long t = (long long)blockIdx.x + (long long)it * gridDim.x;
                if (t >= tm.n_tiles) {
                    mbar_wait(&empty_bar[s], ((k / STAGES) & 1) ^ 1);
                    if (lane == 0) {
                        slot[s] = make_int4(-1, 0, 0, 0);
                        mbar_arrive(&full_bar[s]);
                    }
                    break;
                }
                int tx, ty, en;
                if (fast) tile_coords_fast(tm, (unsigned)t, tx, ty, en);
                else tile_coords_f(tm, t, tx, ty, en);
                const int ent = entries[en];
                const int sz = ent & 0xff, sub = ent >> 8;
                const int4 st = size_tma[sz];
                const int view = st.z >> 8, csq = st.z & 0xff, step = 1 << view;
                // the tile: 16 groups of `step` rows from image row y_begin + r0
                const int r0 = (ty * S1_SUPER + sub * step) * G::TYC;
                if (a.y_begin + r0 >= a.y_end) continue;  // past the band's last row
                mbar_wait(&empty_bar[s], ((k / STAGES) & 1) ^ 1);
                ++k;
                if (lane == 0) {
                    slot[s] = make_int4(tx, r0, sz, step);  // published by the arrive (complete_tx) below
                    mbar_expect_tx(&full_bar[s], G::STAGE_BYTES);
                }
                __syncwarp(pmask);  // expect_tx before any of the boxes lands
                SS_CHECK(sz >= 0 && sz < a.n_sizes && csq >= 0 && csq < CNK && st.w >= 0 && st.w < CNK && view < S1_VIEWS);
                const int n = st.x, d = st.y, b = lane;
                // box b: SAT (+-n+1 columns, +-n+1 rows), E (+1, d+1 / -d), O (-d / d+1, 0)
                const int xo = b < 4 ? ((b & 1) ? 1 - n : n + 1) : (b < 6 ? 1 : (b == 6 ? -d : d + 1));
                const int yo = b < 4 ? ((b & 2) ? 1 - n : n + 1) : (b == 4 ? d + 1 : (b == 5 ? -d : 0));
                const CUtensorMap* m =
                    view == 0 ? (b < 4 ? &maps.sat[csq] : (b < 6 ? &maps.e[st.w] : &maps.o[st.w]))
                              : (b < 4 ? &vmaps->sat[view - 1][csq]
                                       : (b < 6 ? &vmaps->e[view - 1][st.w] : &vmaps->o[view - 1][st.w]));
                const int x0 = tx * G::TX;
                // tile row j tests the centre row y_begin + r0 + j step + step / 2 for its group of `step` rows
                const int cy0 = a.y_begin + r0 + (step >> 1) - a.y_origin;
                void* dst = stage_buf + s * G::STAGE_BYTES + b * G::BOX_BYTES;
                const int row = cy0 + yo;
                if (view == 0) tma_load_2d(dst, m, G::floor_al(x0 + xo), row, &full_bar[s]);
                else tma_load_3d(dst, m, G::floor_al(x0 + xo), row & (step - 1), row >> view, &full_bar[s]);
            }
        }
        return;
    }

    const unsigned lt = (1u << lane) - 1u;
    int2* list0 = list_base + part * part_cap;
    unsigned* count0 = list_ctr + part * CTR_STRIDE;
    int2* buf = cand_buf[warp];
    int nbuf = 0;
    unsigned res = 0;
    bool have_res = false;
    unsigned res_base = 0, res_left = 0;
    unsigned n_int = 0, n_pass = 0;
    const bool unit_stride = a.stride == 1;
    for (int it = 0;; ++it) {
        const int s = it % STAGES;
        mbar_wait(&full_bar[s], (it / STAGES) & 1);
        const int4 sl = slot[s];
        if (sl.x < 0) break;
        const int tx = sl.x, sz = sl.z, step = sl.w;
        const TileConstC& tc = size_info[sz];
        const int row = warp / G::WPR, half = warp - row * G::WPR;  // tile row, column block of this warp
        // this warp's group of `step` rows [g0, g0 + step) and the row it tests
        const int g0 = a.y_begin + sl.y + row * step;
        const int y = g0 + (step >> 1);
        const int gv0 = max(g0, tc.ylo), gv1 = min(min(g0 + step - 1, tc.yhi), a.y_end - 1);  // the group's interior rows
        const bool grp_int = gv0 <= gv1 && (step > 1 || unit_stride || (g0 % a.stride) == 0);
        const bool row_int = grp_int && y >= gv0 && y <= gv1;  // the tested row is interior itself
        // coarse sums biased by one: J = I + 1 in [0, 2^16 - 2], where
        // |S - I 2^k| < 2^(k+1) (the -1 is folded into the estimate's constant)
        unsigned jq[CPW], jd[CPW];
        if (row_int) {
            const int qr = tc.qr, ql = tc.ql, pe = 1, po0 = tc.po0, po1 = tc.po1;
            const unsigned short* box =
                reinterpret_cast<const unsigned short*>(stage_buf + s * G::STAGE_BYTES) + row * G::BW + half * 32 * CPW +
                lane;
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                const unsigned short* b = box + 32 * c;
                constexpr int E = G::BOX_ELEMS;
                jq[c] = ((unsigned)b[0 * E + qr] - b[1 * E + ql] - b[2 * E + qr] + b[3 * E + ql] + 1u) & 0xffffu;
                jd[c] = ((unsigned)b[4 * E + pe] - b[6 * E + po0] - b[7 * E + po1] + b[5 * E + pe] + 1u) & 0xffffu;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);
#ifdef COARSE_NOCOMPUTE  // experiment: the producer / TMA rate alone
        if (row_int && jq[0] == 0x12345u) list0[0] = make_int2((int)jd[1], 0);
        continue;
#endif
        if (!grp_int) continue;
        const int cm_lo = tc.cm_lo;
        auto member = [&](int cm) -> bool {
            if (tc.bm1 == -2) {
                const unsigned i = (unsigned)(cm - cm_lo);
                const unsigned w = (i & 32u) ? tc.win_hi : tc.win_lo;
                return i < 64u && ((w >> (i & 31u)) & 1u);
            }
            if (tc.bm1 >= 0) {
                const unsigned i = (unsigned)(cm - cm_lo);
                return i < (unsigned)tc.cm_n && bit(sbits + tc.bm1, (int)i);
            }
            const RingDev& R0 = a.ring[a.size[sz].ring0];
            return bsearch_eq(a.blob + R0.off_m, R0.n_m, cm);
        };
        const int xt = tx * G::TX + half * 32 * CPW;  // this warp's first column
        unsigned pm = 0, amb = 0;
        if (!row_int) {
            // the tested row lies outside the interior (first / last rows of a
            // size, band ends): every centre of the group's rows is a candidate
            pm = (1u << CPW) - 1u;
        } else if (tc.contig) {
            // one run of member cells [B0, B1): a centre is a candidate unless t
            // lies below B0 or above B1 by more than the error bound -- those
            // within the bound of B0 or B1 are decided by the rings kernel
            // (windows precomputed on the host; t0 = 1/2 - fa - fb)
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                const float tf = fmaf((float)jq[c], tc.fa, fmaf((float)jd[c], tc.fb, tc.t0));
                pm |= (unsigned)(tf >= tc.w0lo && tf <= tc.w1hi) << c;
            }
        } else {
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                const float tf = fmaf((float)jq[c], tc.fa, fmaf((float)jd[c], tc.fb, tc.t0));
                const float dl = tc.band + fmaf(tf, 4e-6f, 4e-6f);
                const float fl = floorf(tf);
                const int cm = (int)fl;
                const float fr = tf - fl;
                const bool p = member(cm);
                pm |= (unsigned)p << c;
                if (fr < dl || fr > 1.0f - dl) {  // the true cell may be the neighbour
                    if (member(fr < dl ? cm - 1 : cm + 1) != p) amb |= 1u << c;
                }
            }
        }
        const int xlo = tc.xlo, xhi = tc.xhi;
        const bool full = unit_stride && xt >= xlo && xt + 32 * CPW - 1 <= xhi;
        if (!full) {
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                const int x = xt + 32 * c + lane;
                const bool interior = x >= xlo && x <= xhi && (unit_stride || (x % a.stride) == 0);
                if (!interior) {
                    pm &= ~(1u << c);
                    amb &= ~(1u << c);
                }
                if (a.stage_counts) n_int += (unsigned)(gv1 - gv0 + 1) * __popc(__ballot_sync(FULL, interior));
            }
        } else if (a.stage_counts) {
            n_int += 32 * CPW * (gv1 - gv0 + 1);
        }
        // undecided centres go to the rings kernel as candidates: its level 0
        // recomputes ring 0's exact mean cell and tests it (eval_ring_fast)
        pm |= amb;
        if (!__any_sync(FULL, pm != 0u)) continue;
        // a passing column is a candidate on every interior row of the group:
        // the columns' places in the staging buffer are found once (one ballot
        // per 32-column chunk), then each row appends its entries
        unsigned long long cnt6 = 0;  // per-chunk counts (<= 32), 6 bits each
        int off[CPW];
#pragma unroll
        for (int c = 0; c < CPW; ++c) {
            const unsigned pb = __ballot_sync(FULL, (pm >> c) & 1u);
            off[c] = __popc(pb & lt);
            cnt6 |= (unsigned long long)__popc(pb) << (6 * c);
        }
        for (int yg = gv0; yg <= gv1; ++yg) {
            const int tag = yg | (sz << TAG_SHIFT);
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                const int cc = (int)((cnt6 >> (6 * c)) & 63ull);
                if (cc == 0) continue;  // warp-uniform
                if ((pm >> c) & 1u) buf[nbuf + off[c]] = make_int2(xt + 32 * c + lane, tag);
                nbuf += cc;
                n_pass += cc;
                if (nbuf >= 32) {
                    __syncwarp();
                    if (res_left == 0) {
                        if (!have_res && lane == 0) res = atom_add_ahead(count0, (unsigned)reserve);
                        res_base = __shfl_sync(FULL, res, 0);
                        res_left = reserve;
                        if (lane == 0) res = atom_add_ahead(count0, (unsigned)reserve);
                        have_res = true;
                    }
                    SS_CHECK(res_base + lane < (unsigned)part_cap && nbuf - 32 + lane < CAND_BUF);
                    if (res_base + lane < (unsigned)part_cap) list0[res_base + lane] = buf[nbuf - 32 + lane];
                    res_base += 32;
                    res_left -= 32;
                    nbuf -= 32;
                    __syncwarp();
                }
            }
        }
    }
    __syncwarp();
    if (have_res) {
        unsigned base = res_base, left = res_left;
        if (left == 0) {
            base = __shfl_sync(FULL, res, 0);
            left = reserve;
        } else {
            const unsigned ahead = __shfl_sync(FULL, res, 0);
            for (unsigned i = lane; i < (unsigned)reserve; i += 32)
                if (ahead + i < (unsigned)part_cap) list0[ahead + i] = make_int2(-1, -1);
        }
        for (unsigned i = lane; i < left; i += 32)
            if (base + i < (unsigned)part_cap) list0[base + i] = i < (unsigned)nbuf ? buf[i] : make_int2(-1, -1);
    } else if (nbuf > 0) {
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(count0, (unsigned)nbuf);
        base = __shfl_sync(FULL, base, 0);
        if (lane < nbuf && base + lane < (unsigned)part_cap) list0[base + lane] = buf[lane];
    }
    if (a.stage_counts && lane == 0) {
        atomicAdd(a.stage_counts + 0, (unsigned long long)n_int);
        atomicAdd(a.stage_counts + 1, (unsigned long long)n_pass);
    }
}

// Border keeps of every fused size (screening.py:438-442): rows [y_begin,
// y_end) of each mask get the grid centres outside the size's interior; the
// interior bits start at 0 and the rings kernel ORs its survivors in.
__global__ void __launch_bounds__(256) ladder_border_kernel(const __grid_constant__ FusedArgs a, unsigned* ctrs,
                                                             int ctr_words) {
    // grid (row blocks, sizes): a block writes whole mask rows of one size,
    // its threads striding over the row's words (coalesced stores)
    const int words = (a.W + 31) >> 5;
    const SizeDev& S = a.size[blockIdx.y];
    const int xlo = S.lo, xhi = a.W - 1 - S.hi;
    if (blockIdx.x == 0 && blockIdx.y == 0)  // the band's tile / list / group counters
        for (int i = threadIdx.x; i < ctr_words; i += blockDim.x) ctrs[i] = 0u;
    const int rows = a.y_end - a.y_begin;
    auto word = [&](int y, int w) -> unsigned {
        const bool row_grid = a.stride == 1 || y % a.stride == 0;
        const int x0 = w * 32;
        const int nb = min(32, a.W - x0);
        if (!row_grid || nb <= 0) return 0u;
        unsigned grid = 0;
        if (a.stride == 1) {
            grid = nb == 32 ? FULL : (1u << nb) - 1u;
        } else {
            for (int b = 0; b < nb; ++b)
                if ((x0 + b) % a.stride == 0) grid |= 1u << b;
        }
        unsigned inter = 0;
        if (y >= S.lo && y <= a.H - 1 - S.hi) {
            const int lb = max(xlo - x0, 0), hb = min(xhi - x0, 31);
            if (lb <= hb) inter = (hb == 31 ? FULL : (1u << (hb + 1)) - 1u) & ~((1u << lb) - 1u);
        }
        return grid & ~inter;
    };
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nthr = gridDim.x * blockDim.x;
    for (int r = tid; r < rows; r += nthr) S.row_counts[a.y_begin + r - a.mask_y0] = 0u;
    unsigned* base = S.mask + (long long)(a.y_begin - a.mask_y0) * a.mask_pitch;
    SS_CHECK(a.y_begin >= a.mask_y0 && a.y_end <= a.H);
    const int qpr = (words + 3) >> 2;  // 16-byte pieces per row (the masks are ~1 GB per step at config 4)
    if ((reinterpret_cast<uintptr_t>(base) & 15) == 0 && (a.mask_pitch & 3) == 0 && 4LL * qpr <= a.mask_pitch) {
        // every thread of the grid stores 16 bytes per turn, rows x pieces flattened
        const long long total = (long long)rows * qpr;
        if (total < (1LL << 31)) {  // 32-bit index arithmetic (a 64-bit division per store is ~100 instructions)
            for (unsigned i = (unsigned)tid; i < (unsigned)total; i += (unsigned)nthr) {
                const int r = (int)(i / (unsigned)qpr), q = (int)(i - (unsigned)r * (unsigned)qpr);
                const int y = a.y_begin + r;
                reinterpret_cast<uint4*>(base + (long long)r * a.mask_pitch)[q] =
                    make_uint4(word(y, 4 * q), word(y, 4 * q + 1), word(y, 4 * q + 2), word(y, 4 * q + 3));
            }
        } else {
            for (long long i = tid; i < total; i += nthr) {
                const int r = (int)(i / qpr), q = (int)(i - (long long)r * qpr);
                const int y = a.y_begin + r;
                reinterpret_cast<uint4*>(base + (long long)r * a.mask_pitch)[q] =
                    make_uint4(word(y, 4 * q), word(y, 4 * q + 1), word(y, 4 * q + 2), word(y, 4 * q + 3));
            }
        }
    } else {
        const long long total = (long long)rows * words;
        for (long long i = tid; i < total; i += nthr) {
            const int r = (int)(i / words), w = (int)(i - (long long)r * words);
            base[(long long)r * a.mask_pitch + w] = word(a.y_begin + r, w);
        }
    }
}

struct SizeSm {
    unsigned* mask;
    unsigned* row_counts;
    int ring0, n_rings;
};

// Every ring of every fused size over the stage-1 list (see rings_kernel in
// ss_screen.cu for the batching / queue scheme); lanes of one batch may
// belong to different sizes: each reads its size's ring from shared memory.
template <typename T, typename E>
__global__ void __launch_bounds__(RK_WARPS * 32, FUSED_RINGS_MINB)
    ladder_rings_kernel(const __grid_constant__ FusedArgs a, int parts, const E* list_base, long long part_cap,
                        const unsigned* list_ctr, unsigned* group_ctr) {
    constexpr bool SUMS = sizeof(E) == sizeof(int4);  // level-0 entries carry ring 0's PLAIN sums
    extern __shared__ __align__(16) unsigned char rsm[];
    RingDev* sring = reinterpret_cast<RingDev*>(rsm);
    SizeSm* ssize = reinterpret_cast<SizeSm*>(rsm + (size_t)a.n_rings * sizeof(RingDev));
    unsigned* sbits = reinterpret_cast<unsigned*>(ssize + a.n_sizes);
    {
        const int* src = reinterpret_cast<const int*>(a.ring);
        int* dst = reinterpret_cast<int*>(sring);
        const int words = a.n_rings * (int)(sizeof(RingDev) / 4);
        for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
        for (int s = threadIdx.x; s < a.n_sizes; s += blockDim.x)
            ssize[s] = SizeSm{a.size[s].mask, a.size[s].row_counts, a.size[s].ring0, a.size[s].n_rings};
        // a warp per ring: the rings' bitmap loads go out together (one ring
        // after another, each copy waited out a global-load round trip -- ~75
        // in a row per CTA and launch at config 4)
        const unsigned* blob32 = reinterpret_cast<const unsigned*>(a.blob);
        for (int r = threadIdx.x >> 5; r < a.n_rings; r += blockDim.x >> 5) {
            const RingDev& R = a.ring[r];
            if (R.bm < 0) continue;
            for (int i = threadIdx.x & 31; i < R.bwords; i += 32)
                sbits[R.bm + i] = R.bsrc >= 0 ? __ldg(blob32 + R.bsrc + i) : 0u;
        }
    }
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int levels = a.max_levels;
    int2* queues = reinterpret_cast<int2*>(sbits + ((a.bm_words + 1) & ~1)) + (size_t)warp * levels * QCAP;
    // per-level queue fill counts, 8 bits each, warp-uniform in a register (levels <= 8)
    unsigned long long qc = 0;
    auto qget = [&](int l) { return (int)((qc >> (8 * l)) & 255ull); };
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    unsigned long long n_pass0 = 0, n_surv = 0;
    constexpr unsigned RG = RINGS_GROUP;
    const unsigned wid = blockIdx.x * RK_WARPS + warp;
    int q = (int)(wid % parts), visited = 1;
    const unsigned gc = (wid / parts) % GROUP_CTRS;
    // A list never extends past its partition (stage 1 does not store what
    // would not fit); a partition that did overflow -- impossible with a
    // workspace of ss_ladder_workspace_bytes unless the tile hand-out were
    // skewed beyond its 1/16 headroom on an image where every centre is a
    // candidate -- must not yield a silently incomplete screen: trap, so the
    // caller's next synchronisation reports a CUDA error.
    auto list_len = [&](int part_i) -> unsigned {
        const unsigned c = __ldg(list_ctr + part_i * CTR_STRIDE);
        if (c > (unsigned)part_cap) asm volatile("trap;");
        return c;
    };
    unsigned cnt_q = list_len(q);
    const E* in = list_base + q * part_cap;
    unsigned g_raw = 0;
    if (lane == 0) g_raw = atom_add_ahead(group_ctr + (q * GROUP_CTRS + gc) * CTR_STRIDE, 1u);
    unsigned cur = 0, k = 0;
    bool have_input = true;
    auto grab = [&]() {
        for (;;) {
            cur = (__shfl_sync(FULL, g_raw, 0) * GROUP_CTRS + gc) * RG;
            if (cur < cnt_q) {
                if (lane == 0) g_raw = atom_add_ahead(group_ctr + (q * GROUP_CTRS + gc) * CTR_STRIDE, 1u);
                return;
            }
            if (visited == parts) {
                have_input = false;
                return;
            }
            ++visited;
            q = q + 1 == parts ? 0 : q + 1;
            cnt_q = list_len(q);
            in = list_base + q * part_cap;
            if (lane == 0) g_raw = atom_add_ahead(group_ctr + (q * GROUP_CTRS + gc) * CTR_STRIDE, 1u);
        }
    };
    auto fetch = [&]() -> E {
        const unsigned slot = cur + 32 * k + lane;
        SS_CHECK(!(have_input && slot < cnt_q) || slot < (unsigned)part_cap);
        return (have_input && slot < cnt_q) ? in[slot] : no_entry<E>();
    };
    grab();
    E next = fetch();
    for (;;) {
        int level = -1;
        for (int l = levels - 1; l >= 1; --l)
            if (qget(l) >= 32) { level = l; break; }
        int2 e;
        unsigned s1q0 = 0, s1d0 = 0;  // level 0 (SUMS): ring 0's PLAIN sums from stage 1
        if (level < 0 && have_input) {
            level = 0;
            e = make_int2(next.x, next.y);
            if constexpr (SUMS) {
                s1q0 = (unsigned)reinterpret_cast<const int4&>(next).z;
                s1d0 = (unsigned)reinterpret_cast<const int4&>(next).w;
            }
            if (++k == RG / 32 || cur + 32 * k >= cnt_q) {
                k = 0;
                grab();
            }
            next = fetch();
        } else {
            if (level < 0) {
                for (int l = levels - 1; l >= 1; --l)
                    if (qget(l) > 0) { level = l; break; }
                if (level < 0) break;
            }
            const int c = qget(level), take = min(c, 32);
            const int2* qq = queues + level * QCAP;
            e = ((int)lane < take) ? qq[c - take + lane] : make_int2(-1, -1);
            qc -= (unsigned long long)take << (8 * level);
            __syncwarp();  // the slots just read may be refilled by the next push
        }
        const bool valid = e.x >= 0;
        const int sz = valid ? (e.y >> TAG_SHIFT) : 0, y = e.y & YMASK;
        const SizeSm S = ssize[sz];
        const bool pass = valid && eval_ring_fast<T>(a, sring[S.ring0 + level], sbits, level, e.x, y - a.y_origin,
                                                     SUMS && level == 0, s1q0, s1d0);
#if RINGS_STATS
        if (valid && pass) atomicAdd(a.stage_counts + 7 + 4 * level, 1ull);
        if (valid && level == 0) {  // would the means of all deeper rings pass?
            bool all = true;
            const PlanePtrs<T> P = plane_ptrs<T>(a, y - a.y_origin, e.x);
            for (int l = 1; l < S.n_rings && all; ++l) {
                const RingDev& Rl = sring[S.ring0 + l];
                Corners<T> c0;
                load_corners(P, Rl, 0, c0);
                all = member_m(a, Rl, sbits, mean_cell(a, Rl, plain_sum(sq_of(c0)), plain_sum(di_of(c0))));
            }
            if (all) atomicAdd(a.stage_counts + 20, 1ull);
            if (all && pass) atomicAdd(a.stage_counts + 21, 1ull);
        }
#endif
        const bool last = level + 1 == S.n_rings;
        const unsigned pb = __ballot_sync(FULL, pass);
        if (level == 0) n_pass0 += __popc(pb);
        const unsigned sb = __ballot_sync(FULL, pass && last);
        n_surv += __popc(sb);
        if (pass && last) {
            const long long row = y - a.mask_y0;
            SS_CHECK(row >= 0 && row < a.y_end - a.mask_y0 && e.x >= 0 && e.x < a.W);
            atomicOr(S.mask + row * a.mask_pitch + (e.x >> 5), 1u << (e.x & 31));
            atomicAdd(S.row_counts + row, 1u);
        }
        const unsigned qb = pb & ~sb;
        if (qb) {
            const int c = qget(level + 1);
            SS_CHECK(level + 1 < levels && c + __popc(qb) <= QCAP);
            if (pass && !last) queues[(level + 1) * QCAP + c + __popc(qb & lt)] = e;
            qc += (unsigned long long)__popc(qb) << (8 * (level + 1));
            __syncwarp();  // the entries are visible to the lanes that pop them
        }
    }
    if (a.stage_counts && lane == 0) {
        if (n_pass0) atomicAdd(a.stage_counts + 2, n_pass0);
        if (n_surv) atomicAdd(a.stage_counts + 3, n_surv);
    }
}

constexpr size_t FCTR_BYTES = (2 + GROUP_CTRS) * MAX_PARTS * CTR_STRIDE * 4;
constexpr size_t PLAN_BYTES = (sizeof(S1Plan) + 255) / 256 * 256;  // after the counters (the border kernel zeroes those per band)
#ifndef FUSED_LARGE_TILES_MACRO
#define FUSED_LARGE_TILES_MACRO 32768
#endif
constexpr long long FUSED_LARGE_TILES = FUSED_LARGE_TILES_MACRO;  // partitioned lists from this many tiles per pass
// 16 GiB: config 4 runs 8 + 2 row bands per step instead of 16 + 8 at 4 GiB
// (every band costs a plan, a border, a stage-1 and a rings launch with their
// prologues and pipeline ramps: step 19.04 -> 18.46 ms; 32 GiB: 18.42)
#ifndef FUSED_WS_CAP_SHIFT
#define FUSED_WS_CAP_SHIFT 30
#endif
constexpr size_t FUSED_WS_CAP = (size_t)(2 * sizeof(FEntry<unsigned>)) << FUSED_WS_CAP_SHIFT;  // ss_ladder_workspace_bytes: row bands beyond this

// capacity in tiles of TXMAX x TY centres (covers either fused tile width)
long long tiles_of(int64_t W, int64_t rows) {
    return ((std::max<int64_t>(W, 1) + TXMAX - 1) / TXMAX) * ((std::max<int64_t>(rows, 1) + TY - 1) / TY);
}
int parts_for(int64_t W, int64_t rows, int n_sizes) {
    return tiles_of(W, rows) * n_sizes >= FUSED_LARGE_TILES ? MAX_PARTS : 1;
}
long long fused_part_cap(int64_t W, int64_t rows, int n_sizes, int sms, int parts) {
    const long long ctas = (2LL * sms + parts - 1) / parts;
    constexpr int s1_warps = WARPS > GeoC::CW ? WARPS : GeoC::CW;  // list reservation slack per stage-1 warp
    // partitioned lists: 1/16 headroom for the uneven shares of a round-robin
    // hand-out (148 CTAs over 8 partitions, tiles of 1 / 2 / 4 row steps)
    const long long share = (tiles_of(W, rows) * n_sizes + parts - 1) / parts;
    return (share + (parts > 1 ? share / 16 + 64 : 0)) * (TXMAX * TY) +
           ctas * s1_warps * 2 * (parts > 1 ? RESERVE_LARGE : RESERVE_SMALL);
}
size_t fused_ws_bytes(int64_t W, int64_t rows, int n_sizes, int sms, size_t entry = sizeof(FEntry<unsigned>)) {
    const int parts = parts_for(W, rows, n_sizes);
    return FCTR_BYTES + PLAN_BYTES + (size_t)parts * (size_t)fused_part_cap(W, rows, n_sizes, sms, parts) * entry;
}

// The three PLAIN-plane TMA descriptors (SAT / E / O) of a plane buffer,
// cached per (buffer, geometry): an engine screens from the same planes every
// call, and encoding costs host time on the critical path of screen().
int plane_maps_cached(TmaMaps& maps, const void* planes, int eb, int bw, int64_t W, int64_t h, int64_t pitch,
                      long long ps) {
    using Key = std::tuple<const void*, int, int, int64_t, int64_t, int64_t, int>;
    static std::mutex mu;
    static std::map<Key, TmaMaps> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const Key key{planes, eb, bw, W, h, pitch, dev};
    {
        std::lock_guard<std::mutex> lock(mu);
        const auto it = cache.find(key);
        if (it != cache.end()) {
            maps = it->second;
            return SS_OK;
        }
    }
    const char* base = static_cast<const char*>(planes);
    const size_t pb = (size_t)ps * eb;
    if (int e = encode_plane_map(&maps.sat, base, eb, bw, W, h, pitch)) return e;
    if (int e = encode_plane_map(&maps.e, base + 4 * pb, eb, bw, W, h, pitch)) return e;
    if (int e = encode_plane_map(&maps.o, base + 8 * pb, eb, bw, W, h, pitch)) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (cache.size() > 256) cache.clear();  // buffers come and go with engines; bound the cache
    cache[key] = maps;
    return SS_OK;
}

// The coarse TMA descriptors (u16 SAT / E / O bit-slice planes of every
// shift set), cached like plane_maps_cached.
int coarse_maps_cached(CoarseMaps& maps, const CoarseViewMaps*& d_vmaps, const uint16_t* coarse, int n_coarse, int64_t W,
                       int64_t h, int64_t pitch, long long ps) {
    using Key = std::tuple<const void*, int, int64_t, int64_t, int64_t, int>;
    struct Val {
        CoarseMaps maps;
        CoarseViewMaps* d_views;
    };
    static std::mutex mu;
    static std::map<Key, Val> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const Key key{coarse, n_coarse, W, h, pitch, dev};
    {
        std::lock_guard<std::mutex> lock(mu);
        const auto it = cache.find(key);
        if (it != cache.end()) {
            maps = it->second.maps;
            d_vmaps = it->second.d_views;
            return SS_OK;
        }
    }
    std::memset(&maps, 0, sizeof(maps));
    std::vector<CoarseViewMaps> hv(1);
    std::memset(hv.data(), 0, sizeof(CoarseViewMaps));
    for (int v = 0; v < S1_VIEWS; ++v)
        for (int c = 0; c < n_coarse; ++c) {
            const uint16_t* base = coarse + (size_t)c * 3 * (size_t)ps;
            CUtensorMap* ms = v ? &hv[0].sat[v - 1][c] : &maps.sat[c];
            CUtensorMap* me = v ? &hv[0].e[v - 1][c] : &maps.e[c];
            CUtensorMap* mo = v ? &hv[0].o[v - 1][c] : &maps.o[c];
            if (int e = encode_plane_map(ms, base, 2, GeoC::BW, W, h, pitch, GeoC::TYC, 1 << v)) return e;
            if (int e = encode_plane_map(me, base + ps, 2, GeoC::BW, W, h, pitch, GeoC::TYC, 1 << v)) return e;
            if (int e = encode_plane_map(mo, base + 2 * ps, 2, GeoC::BW, W, h, pitch, GeoC::TYC, 1 << v)) return e;
        }
    // the row-step views go to device memory once per plane buffer (a blocking
    // copy: the first screen from a buffer, never inside a graph capture that
    // replays an already cached buffer)
    CoarseViewMaps* d_views = nullptr;
    if (cudaMalloc(&d_views, sizeof(CoarseViewMaps)) != cudaSuccess ||
        cudaMemcpy(d_views, hv.data(), sizeof(CoarseViewMaps), cudaMemcpyHostToDevice) != cudaSuccess) {
        set_error("row-step TMA views: %s", cudaGetErrorString(cudaGetLastError()));
        if (d_views) cudaFree(d_views);
        return SS_ECUDA;
    }
    d_vmaps = d_views;
    std::lock_guard<std::mutex> lock(mu);
    if (cache.size() > 256) {
        for (auto& kv : cache) cudaFree(kv.second.d_views);
        cache.clear();
    }
    cache[key] = Val{maps, d_views};
    return SS_OK;
}

}  // namespace

// The coarse shift of a region of `count` pixels (ss_coarse_shift): the
// smallest of 1, 4, 7, ... 16 with 255 count < (2^16 - 4) 2^shift, so its u16
// slice sum never wraps; -1 when none.  Consecutive grid shifts keep
// 2^shift / count <= 4 x 510 / 65532 (the estimate's error, K3L).
int coarse_shift(long long count) {
    for (int k = 1; k <= 16; k += 3)
        if (255LL * count < (65532LL << k)) return k;
    return -1;
}

size_t screen_workspace_bytes(int64_t W, int64_t rows);  // ss_screen.cu

// Half a row band, on whole super rows of the coarse stage 1 (16 x 16 rows)
// while that still shrinks it, else on whole tile rows.
int64_t halve_band(int64_t band) {
    constexpr int AL = TY * S1_SUPER;
    const int64_t b = (band / 2 + AL - 1) / AL * AL;
    return b < band ? b : (band / 2 + TY - 1) / TY * TY;
}

// Workspace of the fused ladder for `n_sizes` sizes: one row band up to
// FUSED_WS_CAP (taller images run in several bands), and never less than the
// per-size screen needs (the fallback shares it).
size_t ladder_workspace_bytes(int64_t W, int64_t rows, int32_t n_sizes) {
    const int sms = device_sms();
    const int64_t S = std::max<int32_t>(n_sizes, 1);
    int64_t band = std::max<int64_t>(rows, 1);
    while (band > 4 * TY && fused_ws_bytes(W, band, (int)S, sms) > FUSED_WS_CAP) band = halve_band(band);
    return std::max(fused_ws_bytes(W, band, (int)S, sms), screen_workspace_bytes(W, std::max<int64_t>(rows, 1)));
}

// K3 for the sizes ks[0..n) of a ladder, all screened from planes of one
// width (eb = 4: 32-bit cells, 8: int64), in row bands of as many rows as the
// workspace holds.  Returns SS_DECLINED (nothing enqueued) when the sizes do
// not fit the fused parameter block or the workspace is too small for a
// useful band; the caller then screens them one by one.
int screen_ladder_fused(const void* planes, int eb, const void* planes32_s1, int64_t h, int64_t pitch, int64_t W,
                        int64_t H, int64_t y_origin, int64_t y_begin, int64_t y_end, int32_t stride, int n,
                        const int* ks, const int32_t* h_m,
                        const int32_t* h_n_rings, const int32_t* h_ring_n, const int32_t* h_ring_d,
                        const int64_t* d_blobs, const int64_t* h_blobs, const int64_t* h_blob_off, double qm,
                        double qs, double qg, uint32_t* d_masks, int64_t mask_pitch, int64_t size_stride,
                        uint32_t* d_row_counts, int64_t rc_stride, unsigned long long* d_stage_counts, void* d_ws,
                        size_t ws_bytes, cudaStream_t s, const uint16_t* d_coarse, int n_coarse,
                        const int32_t* h_shifts, const uint16_t* d_hi16) {
    if (n < 1 || n > FMAX_SIZES || H >= (1LL << TAG_SHIFT) || W > (1 << 30) || stride < 1) return SS_DECLINED;
    if (pitch != plane_pitch(W)) { set_error("plane pitch mismatch"); return SS_EINVAL; }
    if (mask_pitch < (W + 31) / 32) { set_error("mask pitch too small"); return SS_EINVAL; }
    if (y_begin < 0 || y_end > H || y_begin > y_end || y_origin < 0 || y_origin + h > H) {
        set_error("bad row range");
        return SS_EINVAL;
    }
    const int64_t rows = y_end - y_begin;
    if (rows == 0) return SS_OK;
    std::vector<unsigned char> hostbuf(sizeof(FusedArgs), 0);
    FusedArgs& a = *reinterpret_cast<FusedArgs*>(hostbuf.data());
    a.planes = planes;
    a.planes32 = static_cast<const unsigned*>(eb == 4 ? planes : planes32_s1);
    a.hi16 = reinterpret_cast<const unsigned short*>(d_hi16);
    // int64 group without int64 planes: the rings read 32-bit + hi16 cells
    // (mod 2^48), valid while every ring sum stays below 2^48
    const bool wide = eb == 8 && !planes;
    if (wide && (!d_hi16 || !planes32_s1)) {
        set_error("ladder needs the int64 planes or the 32-bit + hi16 planes");
        return SS_EINVAL;
    }
    a.pitch = pitch;
    a.ps = (h + 1) * pitch;
    if (3 * a.ps >= (long long)INT32_MAX) return SS_DECLINED;  // PlanePtrs: 32-bit kind offsets
    a.W = (int)W;
    a.H = (int)H;
    a.y_origin = (int)y_origin;
    a.stride = stride;
    a.mask_y0 = (int)y_begin;
    a.n_sizes = n;
    a.qm = qm;
    a.qs = qs;
    a.qg = qg;
    a.rqm = 1.0 / qm;
    a.rqs = 1.0 / qs;
    a.rqg = 1.0 / qg;
    a.qpow2 = quant_pow2_bits(qm, qs, qg);
    a.rqs_f = (float)(1.0 / qs);
    a.rqg_f = (float)(1.0 / qg);
    a.band_s = (float)(1e-5 / qs);
    a.blob = reinterpret_cast<const long long*>(d_blobs);
    a.mask_pitch = mask_pitch;
    a.stage_counts = d_stage_counts;
    int n_rings = 0, bm_words = 0, bm1 = 0, max_m = 0;
    for (int j = 0; j < n; ++j) {
        const int k = ks[j], m = h_m[k], nr = h_n_rings[k];
        const int64_t* hb = h_blobs + h_blob_off[k];
        if (m < 8 || nr < 1 || nr > SS_MAX_RINGS || hb[0] != nr) {
            set_error("bad fused ladder size %d (m=%d)", k, m);
            return SS_EINVAL;
        }
        if (n_rings + nr > FMAX_RINGS) return SS_DECLINED;
        const int lo = (m - 1) / 2, hi = m / 2;
        const int64_t ylo = std::max<int64_t>(y_begin, lo), yhi = std::min<int64_t>(y_end - 1, H - 1 - hi);
        if (ylo <= yhi && (ylo - lo < y_origin || yhi + hi > y_origin + h - 1)) {
            set_error("table band [%lld, %lld) does not cover rows [%lld, %lld] with margins", (long long)y_origin,
                      (long long)(y_origin + h), (long long)ylo, (long long)yhi);
            return SS_EINVAL;
        }
        if ((int64_t)(m / 2 + 2) * pitch + m > (int64_t)INT32_MAX) {
            set_error("patch offsets exceed 32 bits");
            return SS_EINVAL;
        }
        SizeDev& S = a.size[j];
        S.mask = d_masks + (size_t)k * (size_t)size_stride;
        S.row_counts = d_row_counts + (size_t)k * (size_t)rc_stride;
        S.lo = lo;
        S.hi = hi;
        S.n_rings = nr;
        S.ring0 = n_rings;
        for (int r = 0; r < nr; ++r)
            if (int e = fill_ring(a.ring[n_rings + r], h_ring_n[(size_t)k * SS_MAX_RINGS + r],
                                  h_ring_d[(size_t)k * SS_MAX_RINGS + r], m, pitch, qm, hb + 1 + SS_BLOB_HDR * r,
                                  h_blob_off[k], bm_words, SMEM_BITMAP_WORDS))
                return e;
        if (wide)
            for (int r = 0; r < nr; ++r) {
                const long long rn = h_ring_n[(size_t)k * SS_MAX_RINGS + r], rd = h_ring_d[(size_t)k * SS_MAX_RINGS + r];
                const long long cnt = std::max(4 * rn * rn, 2 * rd * rd + 2 * rd + 1);
                if ((double)255 * (double)cnt * (double)(std::max(W, H) + 1) >= 281474976710656.0) {
                    set_error("ring sums reach 2^48: the int64 planes are needed");
                    return SS_EINVAL;
                }
            }
        // stage 1's copy of ring 0's mean-projection bits
        const int64_t* hd = hb + 1;
        S.bm1 = -1;
        S.wm1 = 0;
        S.bsrc1 = -1;
        if (hd[5] == 0) {  // empty ring 0: cm_n == 0, nothing passes
            if (bm1 + 1 <= S1_BITS_WORDS) { S.bm1 = bm1; S.wm1 = 1; bm1 += 1; }
        } else if (hd[12] >= 0 && bm1 + hd[13] <= S1_BITS_WORDS) {
            S.bm1 = bm1;
            S.wm1 = (int)hd[13];
            S.bsrc1 = (int)((hd[12] + h_blob_off[k]) * 2);
            bm1 += (int)hd[13];
        }
        a.max_levels = std::max(a.max_levels, nr);
        max_m = std::max(max_m, m);
        n_rings += nr;
    }
    if (a.max_levels > 8) return SS_DECLINED;  // the rings' queue counts are 8 x 8 bits
    // Coarse stage 1 (ladder_stage1_coarse_kernel) when every size's ring-0
    // square and diamond have a built shift and the estimate's error bound
    // stays well inside a cell; SS_COARSE=0 forces the 32-bit stage 1.
    bool coarse = d_coarse && n_coarse > 0 && h_shifts && a.planes32;
    if (const char* e = getenv("SS_COARSE")) coarse = coarse && atoi(e) != 0;
    // SS_S1_SLACK: the most cells ring 0's mean may move inside a row group for a
    // row-step view to be allowed (0: every row is tested); SS_S1_RATIO: the
    // plan's cost ratio; SS_S1_FORCE=1: the largest allowed view (tests)
    double s1_slack = S1_SLACK_DEFAULT, s1_ratio = S1_RATIO_DEFAULT;
    int s1_force = 0;
    if (const char* e = getenv("SS_S1_SLACK")) s1_slack = atof(e);
    if (const char* e = getenv("SS_S1_RATIO")) s1_ratio = atof(e);
    if (const char* e = getenv("SS_S1_FORCE")) s1_force = atoi(e);
    long long s1_min_work = PLAN_MIN_WORK;
    if (const char* e = getenv("SS_S1_MIN_WORK")) s1_min_work = atoll(e);
    for (int j = 0; j < n && coarse; ++j) {
        SizeDev& S = a.size[j];
        const RingDev& R0 = a.ring[S.ring0];
        const long long cq = 4LL * R0.n * R0.n, cd = 2LL * R0.d * R0.d + 2LL * R0.d + 1;
        const int kq = coarse_shift(cq), kd = coarse_shift(cd);
        S.c_sq = S.c_di = -1;
        for (int i = 0; i < n_coarse; ++i) {
            if (h_shifts[i] == kq) S.c_sq = i;
            if (h_shifts[i] == kd) S.c_di = i;
        }
        const double band = (std::ldexp(1.0, kq) / (double)cq + std::ldexp(1.0, kd) / (double)cd) / qm;
        if (kq < 0 || kd < 0 || S.c_sq < 0 || S.c_di < 0 || !(band < 0.2)) {
            coarse = false;
            break;
        }
        S.fa_c = (float)(std::ldexp(1.0, kq) / (2.0 * (double)cq * qm));
        S.fb_c = (float)(std::ldexp(1.0, kd) / (2.0 * (double)cd * qm));
        S.band_c = (float)(band * (1.0 + 1e-5));
        S.t0_c = (float)(0.5 - (double)S.fa_c - (double)S.fb_c);
        // ring 0's mean projection as one run of cells [B0, B1) when its
        // keys are consecutive (n_m == cm_n) or empty; windows = B -+ the
        // estimate's bound (band + mean_cell's fp32 term), rounded outwards
        const int64_t* hd = h_blobs + h_blob_off[ks[j]] + 1;
        const int64_t n_m = hd[1], cm_lo = hd[6], cm_n = hd[7];
        S.contig = 0;
        S.s1_views = 1;
        for (int v = 0; v < S1_VIEWS; ++v) S.wlo[v] = S.whi[v] = 0.0f;
        if (n_m == 0 || n_m == cm_n) {
            const double B0 = n_m ? (double)cm_lo : 1e30, B1 = n_m ? (double)(cm_lo + cm_n) : 1e30;
            auto dn = [](double v) { return std::nextafter((float)v, -INFINITY); };
            auto up = [](double v) { return std::nextafter((float)v, INFINITY); };
            // Row steps: moving a centre by one row swaps one row of the square
            // (2n pixels) and the 2d + 1 boundary pixels of the diamond, so
            // |S_sq(y+1) - S_sq(y)| <= 255 * 2n and |S_di(y+1) - S_di(y)| <=
            // 255 (2d + 1), i.e. the mean cell coordinate t moves by at most
            // lip = (255 * 2n / c_sq + 255 (2d + 1) / c_di) / (2 q_mean) per row.
            // View v tests the row at offset step / 2 of each group of step =
            // 1 << v rows, at most step / 2 rows from any row of the group:
            // its window is [B0, B1) widened by the estimate's bound and by
            // (step / 2) lip.  Views whose widening stays within s1_slack
            // cells are allowed; ladder_plan_kernel picks among them.
            const double lip = (255.0 * 2.0 * R0.n / (double)cq + 255.0 * (2.0 * R0.d + 1.0) / (double)cd) / (2.0 * qm);
            S.contig = 1;
            for (int v = 0; v < S1_VIEWS; ++v) {
                const double extra = v ? (double)(1 << (v - 1)) * lip * (1.0 + 1e-6) : 0.0;
                if (v && !(stride == 1 && extra <= s1_slack)) break;
                const double d0 = (band + 4e-6 * (B0 + 1.0 + band)) * (1.0 + 1e-5) + 1e-7 + extra;
                const double d1 = (band + 4e-6 * (B1 + 1.0 + band)) * (1.0 + 1e-5) + 1e-7 + extra;
                S.wlo[v] = dn(B0 - d0);
                S.whi[v] = up(B1 + d1);
                S.s1_views = v + 1;
            }
        }
    }
    a.n_rings = n_rings;
    a.bm_words = bm_words;
    a.bm1_words = bm1;

    const int sms = device_sms();
    // row bands: as many rows per pass as the workspace holds
    int64_t band = rows;
    while (band > 4 * TY && fused_ws_bytes(W, band, n, sms) > ws_bytes) band = halve_band(band);
    if (!d_ws || fused_ws_bytes(W, band, n, sms) > ws_bytes) return SS_DECLINED;

    // Stage 1 reads only the ring-0 PLAIN sums: when they fit 32 bits for
    // every size (255 x pixels < 2^32, n <= 2048), an int64 group's stage 1
    // runs on the 32-bit PLAIN planes (half the TMA bytes, 128-column tiles)
    // and only its rings read the int64 planes.
    bool s1_u32 = eb == 4;
    if (eb == 8 && planes32_s1) {
        s1_u32 = true;
        for (int j = 0; j < n && s1_u32; ++j) {
            const RingDev& R0 = a.ring[a.size[j].ring0];
            s1_u32 = 255LL * 4 * R0.n * R0.n < (1LL << 32) && 255LL * (2LL * R0.d * R0.d + 2LL * R0.d + 1) < (1LL << 32);
        }
    }
    // (row counts and workspace counters are zeroed by ladder_border_kernel)
    TmaMaps maps;
    CoarseMaps cmaps;
    const CoarseViewMaps* d_vmaps = nullptr;
    if (coarse) {
        if (int e = coarse_maps_cached(cmaps, d_vmaps, d_coarse, n_coarse, W, h, pitch, a.ps)) return e;
    } else if (int e = s1_u32 ? plane_maps_cached(maps, eb == 4 ? planes : planes32_s1, 4, GeoF<unsigned>::BW, W, h,
                                                  pitch, a.ps)
                              : plane_maps_cached(maps, planes, 8, GeoF<long long>::BW, W, h, pitch, a.ps)) {
        return e;
    }
    unsigned* tile_ctr = static_cast<unsigned*>(d_ws);
    unsigned* list_ctr = tile_ctr + MAX_PARTS * CTR_STRIDE;
    unsigned* group_ctr = list_ctr + MAX_PARTS * CTR_STRIDE;
    S1Plan* plan = reinterpret_cast<S1Plan*>(static_cast<char*>(d_ws) + FCTR_BYTES);
    void* list_raw = static_cast<char*>(d_ws) + FCTR_BYTES + PLAN_BYTES;
    bool any_views = false;
    for (int j = 0; j < n; ++j) any_views = any_views || a.size[j].s1_views > 1;
    if (!coarse || !any_views || (!s1_force && (long long)rows * W * n < s1_min_work)) plan = nullptr;
    // stage 1's row steps, planned per row band (the candidate density varies
    // along an image: config 4's last 3 of 16 bands hold 60% of the rings' work)
    auto plan_rows = [&](int64_t yb, int64_t ye) -> int {
        if (cudaMemsetAsync(plan, 0, sizeof(S1Plan), s) != cudaSuccess) {
            set_error("plan memset failed");
            return SS_ECUDA;
        }
        ladder_plan_kernel<<<n * PLAN_BLOCKS, 256, 0, s>>>(a, plan, (int)yb, (int)ye, (float)s1_ratio, s1_force);
        note_launch();
        if (int e = check_launch("ladder_plan_kernel")) return e;
        if (getenv("SS_S1_DEBUG")) {  // experiments: print the plan (blocks the stream)
            S1Plan hp;
            cudaStreamSynchronize(s);
            cudaMemcpy(&hp, plan, sizeof(hp), cudaMemcpyDeviceToHost);
            for (int j = 0; j < n; ++j) {
                const RingDev& R0 = a.ring[a.size[j].ring0];
                std::fprintf(stderr, "[s1 plan] rows [%lld, %lld) size %d n=%d d=%d views=%d -> step %d; samples %u in-window",
                             (long long)yb, (long long)ye, j, R0.n, R0.d, a.size[j].s1_views, 1 << hp.view[j],
                             hp.cnt[j][S1_VIEWS]);
                for (int v = 0; v < a.size[j].s1_views; ++v) std::fprintf(stderr, " %u", hp.cnt[j][v]);
                std::fprintf(stderr, "\n");
            }
        }
        return SS_OK;
    };

    auto launch = [&](auto tag, auto tag1) -> int {
        using T = decltype(tag);    // the rings' planes
        using T1 = decltype(tag1);  // stage 1's PLAIN planes
        using G = GeoF<T1>;
        using E = FEntry<T1>;
        E* list = static_cast<E*>(list_raw);
        auto s1 = ladder_stage1_kernel<T1>;
        auto s1c = ladder_stage1_coarse_kernel;
        auto rk = ladder_rings_kernel<T, E>;
        const int tile_x = coarse ? GeoC::TX : G::TX;
        const size_t s1_smem = (size_t)(coarse ? GeoC::STAGES * GeoC::STAGE_BYTES : G::STAGES * G::STAGE_BYTES) +
                               (size_t)std::max(bm1, 1) * 4;
        const void* s1_fn = coarse ? reinterpret_cast<const void*>(s1c) : reinterpret_cast<const void*>(s1);
        const int s1_threads = ((coarse ? GeoC::CW : WARPS) + 1) * 32;
        const int s1_per_sm = std::min(occupancy(s1_fn, s1_threads, s1_smem), 2);
        const size_t rk_smem = (size_t)n_rings * sizeof(RingDev) + (size_t)n * sizeof(SizeSm) +
                               (size_t)((bm_words + 1) & ~1) * 4 + (size_t)RK_WARPS * a.max_levels * QCAP * sizeof(int2);
        const int rk_per_sm = std::max(occupancy(reinterpret_cast<const void*>(rk), RK_WARPS * 32, rk_smem), 1);
        for (int64_t yb = y_begin; yb < y_end; yb += band) {
            const int64_t ye = std::min<int64_t>(y_end, yb + band), brows = ye - yb;
            a.y_begin = (int)yb;
            a.y_end = (int)ye;
            if (plan)
                if (int e = plan_rows(yb, ye)) return e;
            TileMapF tm;
            tm.n_tx = (int)((W + tile_x - 1) / tile_x);
            const int tile_y = coarse ? GeoC::TYC : TY;
            tm.n_ty = (int)((brows + tile_y - 1) / tile_y);
            tm.n_sizes = n;
            if (coarse) {
                // super rows of S1_SUPER tile rows; a size of row step s has S1_SUPER / s tile-row entries in each
                tm.n_ty = (int)((brows + tile_y * S1_SUPER - 1) / (tile_y * S1_SUPER));
                tm.n_sizes = n * S1_SUPER;  // every size at row step 1: the kernel recounts from the plan
            }
            const int n_ent = tm.n_sizes;
            tm.n_tiles = (long long)tm.n_tx * tm.n_ty * n_ent;
            // column strips: the widest whose working set -- (max_m + rows in
            // flight) x (strip + max_m) columns of all 12 planes -- fits the L2
            // budget (the rings that follow touch every plane of those rows)
            {
                int64_t budget = 96ll << 20;  // measured: 96 MB beats 48 MB on configs 2 and 4, equal on 1 and 3
                if (const char* e = getenv("SS_FUSED_STRIP_BUDGET_MB")) budget = (int64_t)atoi(e) << 20;
                const int64_t in_flight = (int64_t)sms * s1_per_sm * G::STAGES;
                tm.strip = 1;
                for (int strip = tm.n_tx; strip >= 1; strip = (strip > 8) ? strip * 3 / 4 : strip - 1) {
                    const int64_t rws = (in_flight + (int64_t)strip * n_ent - 1) / ((int64_t)strip * n_ent) * tile_y *
                                        (coarse ? S1_SUPER : 1);
                    const int64_t ws = (max_m + 2 + rws) * ((int64_t)strip * tile_x + max_m + 2) * 12 * eb;
                    if (ws <= budget) {
                        tm.strip = strip;
                        break;
                    }
                }
                const int last_w = tm.n_tx - (tm.n_tx - 1) / tm.strip * tm.strip;
                tm.r_per_strip = (float)(1.0 / ((double)tm.strip * tm.n_ty * n_ent));
                tm.r_strip = (float)(1.0 / tm.strip);
                tm.r_last = (float)(1.0 / last_w);
                tm.r_span = (float)(1.0 / ((double)tm.strip * n_ent));
                tm.r_span_last = (float)(1.0 / ((double)last_w * n_ent));
            }
            const int parts = parts_for(W, brows, n);
            const long long part_cap = fused_part_cap(W, brows, n, sms, parts);
            {
                // 16 bytes per thread and turn over (rows x row pieces) of each size
                const long long pieces = brows * ((((W + 31) >> 5) + 3) >> 2);
                const dim3 bg((unsigned)std::max<long long>(1, std::min<long long>((pieces + 255) / 256, 16LL * sms / n + 1)),
                              (unsigned)n);
                ladder_border_kernel<<<bg, 256, 0, s>>>(a, static_cast<unsigned*>(d_ws), (int)(FCTR_BYTES / 4));
                note_launch();
                if (int e = check_launch("ladder_border_kernel")) return e;
            }
            const long long grid = std::max<long long>(std::min<long long>(tm.n_tiles, (long long)sms * s1_per_sm),
                                                       (long long)TILE_CTRS);
            if (coarse) {
                if constexpr (std::is_same<E, int2>::value) {
                    s1c<<<(unsigned)grid, s1_threads, s1_smem, s>>>(a, cmaps, d_vmaps, tm, parts,
                                                                          parts > 1 ? RESERVE_LARGE : RESERVE_SMALL,
                                                                          list, part_cap, list_ctr, tile_ctr, plan);
                }
            } else {
                s1<<<(unsigned)grid, (WARPS + 1) * 32, s1_smem, s>>>(a, maps, tm, parts,
                                                                     parts > 1 ? RESERVE_LARGE : RESERVE_SMALL, list,
                                                                     part_cap, list_ctr, tile_ctr);
            }
            note_launch();
            if (int e = check_launch("ladder_stage1_kernel")) return e;
            rk<<<(unsigned)(sms * rk_per_sm), RK_WARPS * 32, rk_smem, s>>>(a, parts, list, part_cap, list_ctr,
                                                                          group_ctr);
            note_launch();
            if (int e = check_launch("ladder_rings_kernel")) return e;
        }
        return SS_OK;
    };
    if (eb == 4) return launch((unsigned)0, (unsigned)0);
    if (wide) {
        if (!s1_u32) {
            set_error("ring-0 PLAIN sums reach 2^32: the int64 planes are needed");
            return SS_EINVAL;
        }
        return launch((wide48)0, (unsigned)0);
    }
    return s1_u32 ? launch((long long)0, (unsigned)0) : launch((long long)0, (long long)0);
}

}  // namespace ss

extern "C" int32_t ss_coarse_shift(int64_t count) { return ss::coarse_shift(count); }

extern "C" size_t ss_ladder_workspace_bytes(int64_t W, int64_t rows, int32_t n_sizes) {
    return ss::ladder_workspace_bytes(W, rows, n_sizes);
}
