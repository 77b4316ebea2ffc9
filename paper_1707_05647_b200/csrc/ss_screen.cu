// ss_screen.cu -- K3: star features + quantize + membership + ballot mask.
//
// Replaces _scan_size (screening.py:418-471) for one ladder size: the ring
// features of _ring_maps_rect / _octagon_maps (screening.py:380-415,
// features.py:94-154), _quantize_arr (screening.py:86-87), _pack_cells
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
// Work decomposition (per ladder size, all on one stream):
//   K3a stage1_kernel -- persistent CTAs; a producer warp streams the 8 ring-0
//       PLAIN corner boxes of each 8 x 32 centre tile into shared memory with
//       TMA (mbarrier pipeline); consumer warps write the border keeps into
//       the mask, compute the ring-0 mean cell and append the centres whose
//       mean cell is in the ring's mean projection to a candidate list.
//   K3b rings_kernel -- one launch for all rings, one candidate per thread:
//       gathers all 32 corners of a ring at once, finishes the cascade (mean,
//       std, gradient membership); members of ring r wait in per-warp shared
//       queues for ring r+1 (full 32-lane batches, same L2 neighbourhood); the
//       last ring ORs survivors into the mask.
// The projection tests are implied by full membership, so the decision is
// the reference's; the SQUARED/X/Y planes and most fp64 work are only
// touched for candidates, and every gather kernel runs with full lanes and
// full occupancy.  Membership tests use dense bitmaps of the key bounding
// box in shared memory (binary search over the sorted keys when the box is
// too large).
#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <vector>

#include <cuda.h>

#include "ss_common.cuh"
#include "ss_screen_dev.cuh"

namespace ss {
namespace {

constexpr int RK_WARPS_PS = 8;  // per-size rings kernel: warps per CTA (RINGS_MINB CTAs per SM)


// K3a: every grid centre of the decided rows -- border keeps into the mask,
// ring-0 mean cell from TMA-staged PLAIN corner boxes, mean-projection
// passers appended to list0.  Persistent CTAs: warp WARPS is the producer.
template <typename T, typename Entry>
__global__ void __launch_bounds__((WARPS + 1) * 32, 1) stage1_kernel(const ScreenArgs a, const __grid_constant__ TmaMaps maps,
                                                                  const TileMap tm, int parts, int reserve, Entry* list_base, long long part_cap,
                                                                  unsigned* list_ctr, unsigned* tile_ctr_base) {
    using G = Geo<T>;
    constexpr int STAGES = G::STAGES;
    extern __shared__ __align__(128) unsigned char dsmem[];
    unsigned char* stage_buf = dsmem;
    unsigned* sbits = reinterpret_cast<unsigned*>(dsmem + STAGES * G::STAGE_BYTES);
    __shared__ __align__(8) unsigned long long full_bar[STAGES], empty_bar[STAGES];
    __shared__ int2 tile_xy[STAGES];  // (tx, ty) of the tile in each stage, written by the producer
    __shared__ Entry cand_buf[WARPS][32 * (CPW + 1)];
    stage_bitmaps(a, sbits, 0, 1, true);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const RingDev& R0 = a.ring[0];
    const int part = (int)(blockIdx.x % parts);

    if (warp == WARPS) {
        // ── producer: one lane streams the tiles' corner boxes ──────────────
        if (lane == 0) {
            // Tiles are handed out by a global counter so every CTA works near
            // the same point of the strip-major order: the L2 working set is
            // the rows in flight, not the spread of CTAs that drift apart.
            // TILE_CTRS interleaved tile counters (counter c: tiles c, c +
            // TILE_CTRS, ...): one address for the whole grid serialised the
            // producers.  With partitioned lists, counter == partition.
            const int tc = (int)(blockIdx.x % TILE_CTRS);
            unsigned* tile_ctr = tile_ctr_base + tc * CTR_STRIDE;
            unsigned t_next = atom_add_ahead(tile_ctr, 1u);
            for (int it = 0;; ++it) {
                const int s = it % STAGES;
                const long long t = (long long)t_next * TILE_CTRS + tc;
                if (t < tm.n_tiles) t_next = atom_add_ahead(tile_ctr, 1u);  // one tile ahead: hides the atomic
                mbar_wait(&empty_bar[s], ((it / STAGES) & 1) ^ 1);
                if (t >= tm.n_tiles) {
                    tile_xy[s] = make_int2(-1, -1);
                    mbar_arrive(&full_bar[s]);
                    break;
                }
                int tx, ty;
                tile_coords(tm, t, tx, ty);
                tile_xy[s] = make_int2(tx, ty);  // published by the mbarrier arrive below
                const int x0 = tx * TX;
                const int cy0 = a.y_begin + ty * TY - a.y_origin;  // table-local first row
                unsigned char* dst = stage_buf + s * G::STAGE_BYTES;
                mbar_expect_tx(&full_bar[s], G::STAGE_BYTES);
                // plane coordinates are (col = x + 1, row = y + 1) of the corner (include/starscreen_b200.h)
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

    // ── consumers: warp w takes row w of each tile, CPW chunks of 32 ────────
    const int ylo = a.lo, yhi = a.H - 1 - a.hi, xlo = a.lo, xhi = a.W - 1 - a.hi;
    // offsets of the corner column inside each box (x0 is a multiple of ALIGN)
    const int qr = G::rem(R0.n + 1), ql = G::rem(1 - R0.n), pe = 1, po0 = G::rem(-R0.d), po1 = G::rem(R0.d + 1);
    const unsigned lt = (1u << lane) - 1u;
    Entry* list0 = list_base + part * part_cap;
    unsigned* count0 = list_ctr + part * CTR_STRIDE;
    Entry* buf = cand_buf[warp];  // passers are staged per warp and flushed 32 at a time
    int nbuf = 0;
    unsigned res = 0;       // lane 0: base of the next reserved block of `reserve` list slots
    bool have_res = false;  // warp-uniform
    unsigned res_base = 0, res_left = 0;  // warp-uniform: the block being filled
    unsigned long long n_int = 0, n_pass = 0;
    const bool unit_stride = a.stride == 1;
    for (int it = 0;; ++it) {
        const int s = it % STAGES;
        mbar_wait(&full_bar[s], (it / STAGES) & 1);
        const int2 txy = tile_xy[s];
        if (txy.x < 0) break;  // producer ran out of tiles
        const int tx = txy.x, ty = txy.y;
        const int y = a.y_begin + ty * TY + warp;
        const T* box = reinterpret_cast<const T*>(stage_buf + s * G::STAGE_BYTES) + warp * G::BW + lane;
        T s1q[CPW], s1d[CPW];  // exact PLAIN region sums (u32 planes: sums < 2^32, see weighted_sum)
#pragma unroll
        for (int c = 0; c < CPW; ++c) {
            const T* b = box + 32 * c;
            constexpr int E = G::BOX_ELEMS;
            s1q[c] = (T)(b[0 * E + qr] - b[1 * E + ql] - b[2 * E + qr] + b[3 * E + ql]);
            s1d[c] = (T)(b[4 * E + pe] - b[6 * E + po0] - b[7 * E + po1] + b[5 * E + pe]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);
        if (y >= a.y_end) continue;  // warp-uniform (past the last row)
        const bool row_grid = unit_stride || (y % a.stride) == 0;
        const bool row_int = row_grid && y >= ylo && y <= yhi;
#pragma unroll
        for (int c = 0; c < CPW; ++c) {
            const int x = tx * TX + 32 * c + lane;
            const bool on_grid = row_grid && x < a.W && (unit_stride || (x % a.stride) == 0);
            const bool interior = row_int && on_grid && x >= xlo && x <= xhi;
            const unsigned border = __ballot_sync(FULL, on_grid && !interior);
            const int word = tx * CPW + c;
            if (lane == 0 && word * 32 < a.W) a.mask[(long long)(y - a.y_begin) * a.mask_pitch + word] = border;
            bool pass = false;
#if STAGE1_FAST_CM
            if (interior) pass = member_m(a, R0, sbits, mean_cell(a, R0, s1q[c], s1d[c]));
#else
            if (interior) {
                const double mq = div_rn((double)s1q[c], R0.cnt_sq, R0.rcp_sq);  // features.py:97
                const double md = div_rn((double)s1d[c], R0.cnt_di, R0.rcp_di);  // features.py:121
                pass = member_m(a, R0, sbits, quant(__dmul_rn(__dadd_rn(mq, md), 0.5), a.qm, a.rqm, a.qpow2 & 1));
            }
#endif
            const unsigned pb = __ballot_sync(FULL, pass);
            n_int += __popc(__ballot_sync(FULL, interior));
            n_pass += __popc(pb);
            if (pass) buf[nbuf + __popc(pb & lt)] = make_entry<Entry>(x, y, (unsigned)s1q[c], (unsigned)s1d[c]);
            nbuf += __popc(pb);
        }
        // Full batches of 32 go to list slots reserved `reserve` at a time,
        // one reservation ahead (the atomic's round trip overlaps the next
        // tiles); the rest of the warp's last reservations is padded with
        // x = -1, which the rings kernel skips.
        while (nbuf >= 32) {
            __syncwarp();
            if (res_left == 0) {
                if (!have_res && lane == 0) res = atom_add_ahead(count0, (unsigned)reserve);
                res_base = __shfl_sync(FULL, res, 0);
                res_left = reserve;
                if (lane == 0) res = atom_add_ahead(count0, (unsigned)reserve);
                have_res = true;
            }
            list0[res_base + lane] = buf[nbuf - 32 + lane];
            res_base += 32;
            res_left -= 32;
            nbuf -= 32;
            __syncwarp();
        }
    }
    __syncwarp();
    if (have_res) {
        // finish the current block, then the one reserved ahead
        unsigned base = res_base, left = res_left;
        if (left == 0) {
            base = __shfl_sync(FULL, res, 0);
            left = reserve;
        } else {
            const unsigned ahead = __shfl_sync(FULL, res, 0);
            for (unsigned i = lane; i < (unsigned)reserve; i += 32) list0[ahead + i] = make_entry<Entry>(-1, -1, 0, 0);
        }
        for (unsigned i = lane; i < left; i += 32) list0[base + i] = i < (unsigned)nbuf ? buf[i] : make_entry<Entry>(-1, -1, 0, 0);
    } else if (nbuf > 0) {
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(count0, (unsigned)nbuf);
        base = __shfl_sync(FULL, base, 0);
        if (lane < nbuf) list0[base + lane] = buf[lane];
    }
    if (a.stage_counts && lane == 0) {
        atomicAdd(a.stage_counts + 0, n_int);
        atomicAdd(a.stage_counts + 1, n_pass);
    }
}

// K3b: every ring of the cascade over the ring-0 candidate list, one launch
// per size.  Each warp evaluates 32 entries of one ring level at a time with
// full lanes: a level-0 batch comes from the list, deeper levels from the
// warp's own shared-memory queues of the previous level's members (deepest
// full queue first, so each holds < 64).  Ring r >= 1 is therefore evaluated
// shortly after ring r-1 on centres the warp has just touched -- their planes'
// rows are still in L2 -- instead of in a later pass over the whole image.
// Ring 0 recomputes its (passed) mean cell and finishes std and gradient;
// deeper rings run the whole cascade; last-ring members are OR'ed into the
// mask and the per-row survivor counts.
// Ring `level` at centre e = (x, y, s1q, s1d): level 0 entries come from the
// stage-1 list and passed the mean test (with a.sums_in_list they carry the
// ring-0 PLAIN sums, so those 8 gathers are skipped); deeper levels start
// with the mean test.
template <typename T, bool SUMS>
__device__ __forceinline__ bool eval_ring(const ScreenArgs& a, const RingDev& R, const unsigned* sbits, int level,
                                          int4 e) {
    const int cy = e.y - a.y_origin;
    const PlanePtrs<T> pc = plane_ptrs<T>(a, cy, e.x);
    Corners<T> c2, cxk, cyk;
    long long s1q, s1d;
    if (SUMS && level == 0 && a.sums_in_list) {
        s1q = (unsigned)e.z;
        s1d = (unsigned)e.w;
    } else {
        Corners<T> c0;
        load_corners(pc, R, 0, c0);
        s1q = unsigned_sum(sq_of(c0));
        s1d = unsigned_sum(di_of(c0));
    }
    load_corners(pc, R, 3, c2);
    load_corners(pc, R, 1, cxk);
    load_corners(pc, R, 2, cyk);
    const Stage1 s = stage1_from(a, R, s1q, s1d);
    return (level == 0 || member_m(a, R, sbits, s.cm)) && finish_of(a, R, sbits, e.x, cy, s, c2, cxk, cyk);
}

template <typename T, typename Entry>
__global__ void __launch_bounds__(RK_WARPS_PS * 32, RINGS_MINB) rings_kernel(const ScreenArgs a, int parts, const Entry* list_base,
                                                                 long long part_cap, const unsigned* list_ctr,
                                                                 unsigned* group_ctr, int bitmap_words) {
    extern __shared__ unsigned sbits[];  // [all rings' bitmaps][queues: warp x level x QCAP int2]
    __shared__ int qcnt[RK_WARPS_PS][SS_MAX_RINGS];
    stage_bitmaps(a, sbits, 0, a.n_rings);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int levels = a.n_rings;
    int2* queues = reinterpret_cast<int2*>(sbits + ((bitmap_words + 1) & ~1)) + (size_t)warp * levels * QCAP;
    if (lane < SS_MAX_RINGS) qcnt[warp][lane] = 0;
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    unsigned long long n_pass0 = 0, n_surv = 0;
    // Level-0 entries come in groups of RG list entries, in list (tile) order:
    // warp w starts on partition w % parts and moves on to the next
    // partition when its own is used up.  Each partition's groups are handed
    // out by GROUP_CTRS interleaved counters (counter c: groups c, c +
    // GROUP_CTRS, ...) so no single address serialises the grabs.  The next
    // group's number waits in lane 0 (one atomic ahead) and the next batch is
    // loaded one batch ahead.
    constexpr unsigned RG = RINGS_GROUP;
    const unsigned wid = blockIdx.x * RK_WARPS_PS + warp;
    int q = (int)(wid % parts), visited = 1;
    const unsigned gc = (wid / parts) % GROUP_CTRS;
    unsigned cnt_q = __ldg(list_ctr + q * CTR_STRIDE);
    const Entry* in = list_base + q * part_cap;
    unsigned g_raw = 0;
    if (lane == 0) g_raw = atom_add_ahead(group_ctr + (q * GROUP_CTRS + gc) * CTR_STRIDE, 1u);
    unsigned cur = 0, k = 0;
    bool have_input = true;
    // next group of the current partition (a group number at or past the end
    // means the partition is used up: later ones are too, so the prefetched
    // number can be dropped)
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
            cnt_q = __ldg(list_ctr + q * CTR_STRIDE);
            in = list_base + q * part_cap;
            if (lane == 0) g_raw = atom_add_ahead(group_ctr + (q * GROUP_CTRS + gc) * CTR_STRIDE, 1u);
        }
    };
    auto fetch = [&]() -> int4 {  // this lane's entry of batch k of the current group
        const unsigned slot = cur + 32 * k + lane;
        return (have_input && slot < cnt_q) ? widen(in[slot]) : make_int4(-1, -1, 0, 0);
    };
    grab();
    int4 next = fetch();
    for (;;) {
        // pick the batch: deepest queue holding >= 32, else the list, else drain
        int level = -1;
        for (int l = levels - 1; l >= 1; --l)
            if (qcnt[warp][l] >= 32) { level = l; break; }
        int4 e;
        if (level < 0 && have_input) {
            level = 0;
            e = next;
            if (++k == RG / 32 || cur + 32 * k >= cnt_q) {
                k = 0;
                grab();
            }
            next = fetch();
        } else {
            if (level < 0) {
                for (int l = levels - 1; l >= 1; --l)
                    if (qcnt[warp][l] > 0) { level = l; break; }
                if (level < 0) break;  // list and queues empty
            }
            const int c = qcnt[warp][level], take = min(c, 32);
            const int2* q = queues + level * QCAP;
            const int2 qe = ((int)lane < take) ? q[c - take + lane] : make_int2(-1, -1);
            e = make_int4(qe.x, qe.y, 0, 0);
            __syncwarp();
            if (lane == 0) qcnt[warp][level] = c - take;
            __syncwarp();
        }
        const bool pass = e.x >= 0 && eval_ring<T, sizeof(Entry) == sizeof(int4)>(a, a.ring[level], sbits, level, e);
        const unsigned pb = __ballot_sync(FULL, pass);
        if (level == 0) n_pass0 += __popc(pb);
        if (level + 1 == levels) {
            n_surv += __popc(pb);
            if (pass) {
                const long long row = e.y - a.y_begin;
                atomicOr(a.mask + row * a.mask_pitch + (e.x >> 5), 1u << (e.x & 31));
                atomicAdd(a.row_counts + row, 1u);
            }
        } else if (pb) {
            const int c = qcnt[warp][level + 1];
            if (pass) queues[(level + 1) * QCAP + c + __popc(pb & lt)] = make_int2(e.x, e.y);
            __syncwarp();
            if (lane == 0) qcnt[warp][level + 1] = c + __popc(pb);
            __syncwarp();
        }
    }
    if (a.stage_counts && lane == 0) {
        if (n_pass0) atomicAdd(a.stage_counts + 2, n_pass0);
        if (n_surv) atomicAdd(a.stage_counts + 3, n_surv);
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

// The fused rings' fp32-estimate cells (std_cell_fast, grad_cell_fast) vs
// the fp64 reference sequence (std_cell_exact, grad_cell_exact) on random
// region sums an 8-bit image can produce (0 <= s1 <= 255 count, s1^2 / count
// <= s2 <= 255 s1), most of them aimed at a std / gradient cell boundary:
// counts[0] std mismatches, counts[1] gradient mismatches.
__device__ __forceinline__ unsigned long long mix64(unsigned long long h) {
    h ^= h >> 31;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 27;
    h *= 0x94D049BB133111EBull;
    return h ^ (h >> 31);
}
__global__ void selftest_cells_kernel(unsigned long long n, unsigned long long seed, const ScreenArgs a,
                                      unsigned long long* counts) {
    const RingDev& R = a.ring[0];
    unsigned long long bad_s = 0, bad_g = 0;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        unsigned long long h = mix64((i + 1) * 0x9E3779B97F4A7C15ull + seed);
        auto uni = [&]() {  // uniform in [0, 1)
            h = mix64(h + 0x9E3779B97F4A7C15ull);
            return (double)(h >> 11) * 0x1.0p-53;
        };
        const bool aim = (i & 3) != 0;  // 3 in 4 samples aimed at a boundary
        // means and a std split around a target
        const double mq = 255.0 * uni(), md = fmin(255.0, fmax(0.0, mq + 40.0 * (uni() - 0.5)));
        double sq_t = 60.0 * uni(), sd_t = 60.0 * uni();
        if (aim) {  // (sq + sd) / 2 near qs (k - 1/2), k = 1..8
            const double target = a.qs * (double)(1 + (int)(8.0 * uni()) - 0.5) * (1.0 + 1e-6 * (uni() - 0.5));
            const double split = uni();
            sq_t = 2.0 * target * split;
            sd_t = 2.0 * target * (1.0 - split);
        }
        auto sums = [&](int cnt, double mean, double sdev, long long& s1, long long& s2) {
            s1 = llrint(mean * cnt);
            s1 = s1 < 0 ? 0 : (s1 > 255LL * cnt ? 255LL * cnt : s1);
            long long lo = (s1 * s1 + cnt - 1) / cnt, hi = 255 * s1;
            long long v = llrint((double)cnt * ((double)s1 / cnt * ((double)s1 / cnt) + sdev * sdev));
            s2 = v < lo ? lo : (v > hi ? hi : v);
        };
        long long s1q, s2q, s1d, s2d;
        sums(R.icq, mq, sq_t, s1q, s2q);
        sums(R.icd, md, sd_t, s1d, s2d);
        const int cs_ref =
            std_cell_exact(a, R, div_rn((double)s1q, R.cnt_sq, R.rcp_sq), div_rn((double)s1d, R.cnt_di, R.rcp_di), s2q, s2d);
        if (std_cell_fast(a, R, s1q, s1d, s2q, s2d) != cs_ref) ++bad_s;
        // the 32 x 32-bit variance products of the 32-bit-plane path, wherever its sums fit
        if (s2q < (1LL << 32) && s2d < (1LL << 32) && std_cell_fast<true>(a, R, s1q, s1d, s2q, s2d) != cs_ref) ++bad_s;
        // gradient: components of a target magnitude split between square and diamond
        double gm_t = 200.0 * uni();
        if (aim) gm_t = a.qg * (double)(1 + (int)(8.0 * uni()) - 0.5) * (1.0 + 1e-6 * (uni() - 0.5));
        const double th = 6.283185307179586 * uni(), dx = 30.0 * (uni() - 0.5), dy = 30.0 * (uni() - 0.5);
        const double gx = gm_t * cos(th), gy = gm_t * sin(th);
        const int cx = (int)(16384.0 * uni()), cy = (int)(16384.0 * uni());
        const long long dxq = llrint(((gx + dx) * 2.0 * R.w1_sq + (double)s1q) * 0.5);
        const long long dyq = llrint(((gy + dy) * 2.0 * R.w1_sq + (double)s1q) * 0.5);
        const long long dxd = llrint((gx - dx) * R.w1_di), dyd = llrint((gy - dy) * R.w1_di);
        if (grad_cell_fast(a, R, cx, cy, s1q, s1d, dxq, dyq, dxd, dyd) !=
            grad_cell_exact(a, R, cx, cy, s1q, s1d, (long long)(cx + 1) * s1q + dxq, (long long)(cy + 1) * s1q + dyq,
                            (long long)(cx + 1) * s1d + dxd, (long long)(cy + 1) * s1d + dyd))
            ++bad_g;
    }
    if (bad_s) atomicAdd(counts + 0, bad_s);
    if (bad_g) atomicAdd(counts + 1, bad_g);
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

// Workspace: [counters: 3 x MAX_PARTS lines] [`parts` candidate sub-lists of
// part_cap entries].  A partition serves ceil(tiles / parts) tiles (<=
// TILE_POS passers each) plus the padding of its warps' last reserved blocks
// (< 32 per stage-1 consumer warp; at most 2 CTAs per SM).
constexpr size_t CTR_BYTES = (2 + GROUP_CTRS) * MAX_PARTS * CTR_STRIDE * 4;
constexpr long long LARGE_TILES = 32768;  // sizes with at least this many tiles use the large-list mode
static long long n_tiles_of(int64_t W, int64_t rows) {
    return ((std::max<int64_t>(W, 1) + TX - 1) / TX) * ((std::max<int64_t>(rows, 1) + TY - 1) / TY);
}
static long long part_cap_of(int64_t W, int64_t rows, int sms, int parts) {
    const long long ctas = (2LL * sms + parts - 1) / parts;
    return (n_tiles_of(W, rows) + parts - 1) / parts * TILE_POS + ctas * WARPS * 2 * PS_RESERVE_MAX;
}
static size_t list_bytes(int64_t W, int64_t rows, int sms, bool large) {
    return large ? (size_t)MAX_PARTS * part_cap_of(W, rows, sms, MAX_PARTS) * sizeof(int4)
                 : (size_t)part_cap_of(W, rows, sms, 1) * sizeof(int2);
}
size_t screen_workspace_bytes(int64_t W, int64_t rows) {
    const int sms = device_sms();
    return CTR_BYTES + std::max(list_bytes(W, rows, sms, false), list_bytes(W, rows, sms, true));
}

// True when every region sum of ring (n, d) is recoverable from planes mod
// 2^32 (see weighted_sum): PLAIN/SQUARED sums of the square (4n^2 pixels)
// and the diamond (2d^2+2d+1 pixels) are < 2^32, and the centred first
// moments |sum (x - c) v| of both are < 2^31.
bool ring_fits32(int64_t n, int64_t d) {
    const int64_t lim_u = (int64_t)1 << 32, lim_s = (int64_t)1 << 31;
    if (65025 * 4 * n * n >= lim_u) return false;
    if (65025 * (2 * d * d + 2 * d + 1) >= lim_u) return false;
    if (255 * 2 * n * n * n >= lim_s) return false;  // sum |x - c| over the square <= 2 n^3
    int64_t mom = 0;                                 // sum |dx| over the diamond
    for (int64_t k = 1; k <= d; ++k) mom += 2 * k * (2 * (d - k) + 1);
    return 255 * mom < lim_s;
}

struct K3Launch {
    ScreenArgs a;
    TmaMaps maps;
    TileMap tm;
    int m, eb, sms, bm_words;
    void* list;
    unsigned *list_ctr, *tile_ctr, *group_ctr;
    cudaStream_t s;
};

// K3a stage1_kernel then K3b rings_kernel of one size, with planes of T and
// list entries of E in `parts` sub-lists.
template <typename T, typename E>
static int launch_k3(K3Launch& L, int parts) {
    using G = Geo<T>;
    const ScreenArgs& a = L.a;
    TileMap& tm = L.tm;
    const long long part_cap = part_cap_of(a.W, a.y_end - a.y_begin, L.sms, parts);
    E* list = static_cast<E*>(L.list);
    // K3a: the mask rows are (re)initialised here; survivors are OR'ed in by K3b
    auto s1 = stage1_kernel<T, E>;
    const size_t s1_smem_all = (size_t)G::STAGES * G::STAGE_BYTES + (size_t)std::max(a.ring[0].wm, 1) * 4;
    const int s1_per_sm = std::min(occupancy(reinterpret_cast<const void*>(s1), (WARPS + 1) * 32, s1_smem_all),
                                   2);  // part_cap_of budgets <= 2 CTAs per SM
    // Column strips: a SAT element is used by four centres at the corners of
    // a 2n x 2n square, so it is read from HBM once only if the rows between
    // them (vertical reuse) and the columns between them (horizontal reuse)
    // are still in L2.  The widest strip whose working set -- (m + rows in
    // flight) x (strip + m) x 3 planes of PLAIN SAT/E/O -- fits the budget keeps
    // both; narrower strips re-read (strip + m) / strip of the columns.
    {
        int64_t budget = 40ll << 20, planes = 3;
        if (const char* e = getenv("SS_STRIP_BUDGET_MB")) budget = (int64_t)atoi(e) << 20;  // experiment hooks
        if (const char* e = getenv("SS_STRIP_PLANES")) planes = atoi(e);
        const int64_t in_flight = (int64_t)L.sms * s1_per_sm * G::STAGES;
        tm.strip = 1;
        for (int strip = tm.n_tx; strip >= 1; strip = (strip > 8) ? strip * 3 / 4 : strip - 1) {
            const int64_t rows = (in_flight + strip - 1) / strip * TY;
            const int64_t ws = (L.m + 2 + rows) * ((int64_t)strip * TX + L.m + 2) * planes * L.eb;
            if (ws <= budget) {
                tm.strip = strip;
                break;
            }
        }
    }
    if (const char* e = getenv("SS_STRIP")) tm.strip = std::max(1, std::min(tm.n_tx, atoi(e)));  // experiment hook
    {
        // every tile counter / partition needs a CTA (CTAs without tiles exit at once)
        const long long grid = std::max<long long>(std::min<long long>(tm.n_tiles, (long long)L.sms * s1_per_sm),
                                                   (long long)TILE_CTRS);
        s1<<<(unsigned)grid, (WARPS + 1) * 32, s1_smem_all, L.s>>>(a, L.maps, tm, parts,
                                                                  parts > 1 ? PS_RESERVE_LARGE : PS_RESERVE_SMALL, list, part_cap, L.list_ctr,
                                                                  L.tile_ctr);
        note_launch();
        if (int e = check_launch("stage1_kernel")) return e;
    }
    // K3b: all rings over the stage-1 sub-lists; survivors into the mask
    {
        const size_t smem = (size_t)((L.bm_words + 1) & ~1) * 4 + (size_t)RK_WARPS_PS * a.n_rings * QCAP * sizeof(int2);
        auto rk = rings_kernel<T, E>;
        const int per_sm = occupancy(reinterpret_cast<const void*>(rk), RK_WARPS_PS * 32, smem);
        rk<<<(unsigned)(L.sms * std::max(per_sm, 1)), RK_WARPS_PS * 32, smem, L.s>>>(a, parts, list, part_cap, L.list_ctr,
                                                                                L.group_ctr, L.bm_words);
        note_launch();
        if (int e = check_launch("rings_kernel")) return e;
    }
    return SS_OK;
}

int screen_size(const int64_t* d_planes, const uint32_t* d_planes32, int64_t w, int64_t h, int64_t pitch, int64_t W,
                int64_t H, int64_t y_origin,
                int64_t y_begin, int64_t y_end, int32_t m, int32_t stride, int32_t n_rings, const int32_t* ring_n,
                const int32_t* ring_d, const int64_t* d_blob, const int64_t* h_blob, double qm, double qs, double qg,
                uint32_t* d_mask, int64_t mask_pitch, uint32_t* d_row_counts, unsigned long long* d_stage_counts,
                void* d_ws, size_t ws_bytes, void* stream) {
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
    a.pitch = pitch;
    a.ps = (h + 1) * pitch;
    if (3 * a.ps >= (long long)INT32_MAX) {  // kinds of one plane type are 32-bit offsets apart (PlanePtrs)
        set_error("table too large: 3 planes exceed 2^31 elements");
        return SS_EINVAL;
    }
    a.W = (int)W;
    a.H = (int)H;
    a.y_origin = (int)y_origin;
    a.y_begin = (int)y_begin;
    a.y_end = (int)y_end;
    a.stride = stride;
    a.lo = lo;
    a.hi = hi;
    a.n_rings = n_rings;
    {
        // ring-0 PLAIN sums (square 4n^2, diamond 2d^2+2d+1 pixels of <= 255) below 2^32
        const int64_t n0 = ring_n[0], d0 = ring_d[0];
        a.sums_in_list = (255 * 4 * n0 * n0 < ((int64_t)1 << 32)) && (255 * (2 * d0 * d0 + 2 * d0 + 1) < ((int64_t)1 << 32));
    }
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
    a.blob = reinterpret_cast<const long long*>(d_blob);
    a.mask = d_mask;
    a.mask_pitch = mask_pitch;
    a.row_counts = d_row_counts;
    a.stage_counts = d_stage_counts;
    const long long P = pitch;
    int bm_words = 0;
    for (int r = 0; r < n_rings; ++r)
        if (int e = fill_ring(a.ring[r], ring_n[r], ring_d[r], m, P, qm, h_blob + 1 + SS_BLOB_HDR * r, 0, bm_words,
                              SMEM_BITMAP_WORDS))
            return e;
    bool use32 = d_planes32 != nullptr;
    for (int r = 0; r < n_rings && use32; ++r) use32 = ring_fits32(ring_n[r], ring_d[r]);
    if (!use32 && !d_planes) {
        set_error("size m=%d needs the int64 planes (ring sums exceed 32 bits)", m);
        return SS_EINVAL;
    }
    a.planes = use32 ? static_cast<const void*>(d_planes32) : static_cast<const void*>(d_planes);
    const int eb = use32 ? 4 : 8;
    cudaStream_t s = as_stream(stream);
    const int64_t rows = y_end - y_begin;
    if (rows == 0) return SS_OK;
    const size_t need = screen_workspace_bytes(W, rows);
    if (!d_ws || ws_bytes < need) {
        set_error("screen workspace too small: %zu < %zu", ws_bytes, need);
        return SS_EINVAL;
    }
    // workspace counters (one 128-B line each): stage-1 tile counters, list
    // counters, rings group counters -- MAX_PARTS of each
    unsigned* tile_ctr = static_cast<unsigned*>(d_ws);
    unsigned* list_ctr = tile_ctr + MAX_PARTS * CTR_STRIDE;
    unsigned* group_ctr = list_ctr + MAX_PARTS * CTR_STRIDE;
    const int sms = device_sms();
    void* list_a = static_cast<char*>(d_ws) + CTR_BYTES;
    if (cudaMemsetAsync(d_row_counts, 0, rows * sizeof(uint32_t), s) != cudaSuccess) return check_launch("memset");
    if (cudaMemsetAsync(tile_ctr, 0, CTR_BYTES, s) != cudaSuccess) return check_launch("memset");

    TmaMaps maps;  // PLAIN SAT / E / O planes for the stage-1 TMA boxes
    {
        const char* base = static_cast<const char*>(a.planes);
        const int bw = use32 ? Geo<unsigned>::BW : Geo<long long>::BW;
        const size_t pb = (size_t)a.ps * eb;
        if (int e = encode_plane_map(&maps.sat, base, eb, bw, W, h, pitch)) return e;
        if (int e = encode_plane_map(&maps.e, base + 4 * pb, eb, bw, W, h, pitch)) return e;
        if (int e = encode_plane_map(&maps.o, base + 8 * pb, eb, bw, W, h, pitch)) return e;
    }
    TileMap tm;
    tm.n_tx = (int)((W + TX - 1) / TX);
    tm.n_ty = (int)((rows + TY - 1) / TY);
    tm.n_tiles = (long long)tm.n_tx * tm.n_ty;
    tm.strip = 1;
    bool large = tm.n_tiles >= LARGE_TILES;
    if (const char* e = getenv("SS_LIST_MODE")) large = atoi(e) != 0;  // experiment hook
    K3Launch L{a, maps, tm, m, eb, sms, bm_words, list_a, list_ctr, tile_ctr, group_ctr, s};
    if (large) {
        L.a.sums_in_list = a.sums_in_list;
        return use32 ? launch_k3<unsigned, int4>(L, MAX_PARTS) : launch_k3<long long, int4>(L, MAX_PARTS);
    }
    L.a.sums_in_list = 0;
    return use32 ? launch_k3<unsigned, int2>(L, 1) : launch_k3<long long, int2>(L, 1);
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

int selftest_cells(uint64_t n, uint64_t seed, int32_t ring_n, int32_t ring_d, double qm, double qs, double qg,
                   unsigned long long* d_counts, void* stream) {
    if (ring_n < 1 || ring_d < 1 || ring_n > 1024 || ring_d > 1448 || !(qm > 0) || !(qs > 0) || !(qg > 0) || !d_counts) {
        set_error("bad selftest arguments");
        return SS_EINVAL;
    }
    std::vector<unsigned char> buf(sizeof(ScreenArgs), 0);
    ScreenArgs& a = *reinterpret_cast<ScreenArgs*>(buf.data());
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
    // ring constants only (no key blob): a one-ring header with no keys
    int64_t hd[SS_BLOB_HDR] = {};
    hd[12] = -1;
    int bm_words = 0;
    const int m = 2 * std::max<int>(ring_n, ring_d + 1) + 2;
    if (int e = fill_ring(a.ring[0], ring_n, ring_d, m, 1 << 20, qm, hd, 0, bm_words, 0)) return e;
    selftest_cells_kernel<<<148 * 8, 256, 0, as_stream(stream)>>>(n, seed, a, d_counts);
    note_launch();
    return check_launch("selftest_cells_kernel");
}

int selftest_div(uint64_t n, uint64_t seed, double b, int mode, unsigned long long* d_bad, void* stream) {
    if (b <= 0.0 || mode < 0 || mode > 3) { set_error("bad selftest arguments"); return SS_EINVAL; }
    selftest_div_kernel<<<148 * 16, 256, 0, as_stream(stream)>>>(n, seed, b, mode, d_bad);
    note_launch();
    return check_launch("selftest_div_kernel");
}

}  // namespace ss

extern "C" {
int ss_screen_size(const int64_t* d_planes, const uint32_t* d_planes32, int64_t w, int64_t h, int64_t plane_pitch,
                   int64_t W, int64_t H, int64_t y_origin, int64_t y_begin, int64_t y_end, int32_t m, int32_t stride,
                   int32_t n_rings, const int32_t* h_ring_n, const int32_t* h_ring_d, const int64_t* d_blob,
                   const int64_t* h_blob, double q_mean, double q_std, double q_grad, uint32_t* d_mask,
                   int64_t mask_pitch_words, uint32_t* d_row_counts, unsigned long long* d_stage_counts,
                   void* d_workspace, size_t workspace_bytes, void* stream) {
    return ss::screen_size(d_planes, d_planes32, w, h, plane_pitch, W, H, y_origin, y_begin, y_end, m, stride, n_rings,
                           h_ring_n, h_ring_d, d_blob, h_blob, q_mean, q_std, q_grad, d_mask, mask_pitch_words,
                           d_row_counts, d_stage_counts, d_workspace, workspace_bytes, stream);
}
int ss_screen_fits32(int32_t n_rings, const int32_t* h_ring_n, const int32_t* h_ring_d) {
    if (n_rings < 1 || !h_ring_n || !h_ring_d) return 0;
    for (int r = 0; r < n_rings; ++r)
        if (!ss::ring_fits32(h_ring_n[r], h_ring_d[r])) return 0;
    return 1;
}
size_t ss_screen_workspace_bytes(int64_t W, int64_t rows) { return ss::screen_workspace_bytes(W, rows); }
int ss_fill_grid(int64_t W, int64_t y_begin, int64_t y_end, int32_t stride, uint32_t* d_mask,
                 int64_t mask_pitch_words, uint32_t* d_row_counts, void* stream) {
    return ss::fill_grid(W, y_begin, y_end, stride, d_mask, mask_pitch_words, d_row_counts, stream);
}
int ss_selftest_cells(uint64_t n, uint64_t seed, int32_t ring_n, int32_t ring_d, double q_mean, double q_std,
                      double q_grad, unsigned long long* d_counts, void* stream) {
    return ss::selftest_cells(n, seed, ring_n, ring_d, q_mean, q_std, q_grad, d_counts, stream);
}
int ss_selftest_div(uint64_t n, uint64_t seed, double divisor, int32_t mode, unsigned long long* d_mismatches,
                    void* stream) {
    return ss::selftest_div(n, seed, divisor, mode, d_mismatches, stream);
}
}
