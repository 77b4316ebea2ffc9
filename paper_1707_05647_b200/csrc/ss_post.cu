// ss_post.cu -- K4 survivor compaction, K5 kept-region mask, popcount.
//
// K4 replaces the np.nonzero + list building of _scan_size / screen()
// (screening.py:455-470, 512-516): survivors come out row-major per size and
// sizes are appended in ladder order, which is the candidates order.
// K5 replaces _footprint_union (screening.py:316-330): the union of the m x m
// footprints [c-lo, c+hi] of the evaluated survivors, as a separable box
// dilation of the bit-packed survivor mask (van Herk/Gil-Werman along
// columns, word-parallel; log-step shift-OR doubling along rows).
#include <algorithm>
#include <vector>

#include "ss_common.cuh"

namespace ss {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned interior_bits(long long word, int x_lo, int x_hi) {
    // bits of word `word` whose column lies in [x_lo, x_hi]
    const long long a = word * 32, b = a + 31;
    if (x_hi < x_lo || b < x_lo || a > x_hi) return 0u;
    const int s = (int)max(0LL, (long long)x_lo - a);
    const int e = (int)min(31LL, (long long)x_hi - a);
    const unsigned hi_mask = (e == 31) ? FULL : ((1u << (e + 1)) - 1u);
    const unsigned lo_mask = FULL << s;
    return hi_mask & lo_mask;
}

// Exclusive scan of row counts (one CTA), offset by *total; advances *total.
__global__ void __launch_bounds__(1024) scan_rows_kernel(const unsigned* counts, long long rows,
                                                         unsigned long long* row_off, unsigned long long* total,
                                                         unsigned long long* size_count) {
    __shared__ unsigned long long warp_sums[32];
    __shared__ unsigned long long carry;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) carry = *total;
    __syncthreads();
    for (long long base = 0; base < rows; base += 1024) {
        const long long i = base + t;
        const unsigned long long v = (i < rows) ? counts[i] : 0ull;
        unsigned long long s = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long o = __shfl_up_sync(FULL, s, d);
            if (lane >= d) s += o;
        }
        if (lane == 31) warp_sums[warp] = s;
        __syncthreads();
        if (warp == 0) {
            unsigned long long w = warp_sums[lane];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned long long o = __shfl_up_sync(FULL, w, d);
                if (lane >= d) w += o;
            }
            warp_sums[lane] = w;
        }
        __syncthreads();
        const unsigned long long before = carry + (warp ? warp_sums[warp - 1] : 0ull) + s - v;
        if (i < rows) row_off[i] = before;
        __syncthreads();
        if (t == 1023) carry = before + v;
        __syncthreads();
    }
    if (t == 0) {
        if (size_count) *size_count = carry - *total;
        *total = carry;
    }
}

// One warp per mask row: write (cx, cy) of every interior survivor.
__global__ void write_xy_kernel(const unsigned* mask, long long mask_pitch, int W, int y_begin, long long rows, int x_lo,
                                int x_hi, const unsigned* counts, const unsigned long long* row_off, int* xy,
                                long long capacity) {
    const long long row = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows || counts[row] == 0) return;  // warp-uniform
    const unsigned* mrow = mask + row * mask_pitch;
    const long long words = (W + 31) / 32;
    unsigned long long pos = row_off[row];
    const int y = y_begin + (int)row;
    for (long long wb = 0; wb < words; wb += 32) {
        const long long w = wb + lane;
        unsigned bits = (w < words) ? (mrow[w] & interior_bits(w, x_lo, x_hi)) : 0u;
        const int c = __popc(bits);
        int incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int o = __shfl_up_sync(FULL, incl, d);
            if (lane >= d) incl += o;
        }
        unsigned long long p = pos + (unsigned long long)(incl - c);
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            if (p < (unsigned long long)capacity) {
                xy[2 * p] = (int)(w * 32 + b);
                xy[2 * p + 1] = y;
            }
            ++p;
        }
        pos += (unsigned long long)__shfl_sync(FULL, incl, 31);
    }
}

__device__ __forceinline__ unsigned get_word(const unsigned* row, long long i, long long words) {
    return (i >= 0 && i < words) ? row[i] : 0u;
}
// word i of F(x + s), s >= 0 (shift toward lower x)
__device__ __forceinline__ unsigned shifted_lo(const unsigned* row, long long i, long long words, int s) {
    const long long q = s >> 5;
    const int r = s & 31;
    const unsigned a = get_word(row, i + q, words);
    if (r == 0) return a;
    return (a >> r) | (get_word(row, i + q + 1, words) << (32 - r));
}
// word i of F(x - s), s >= 0 (shift toward higher x)
__device__ __forceinline__ unsigned shifted_hi(const unsigned* row, long long i, long long words, int s) {
    const long long q = s >> 5;
    const int r = s & 31;
    const unsigned a = get_word(row, i - q, words);
    if (r == 0) return a;
    return (a << r) | (get_word(row, i - q - 1, words) >> (32 - r));
}

// Column pass of the footprint dilation: V(y) = OR_{r in [y-hi, y+lo]} S(r)
// = F_L(y - hi) with F_l(r) = OR S[r, r+l-1], by shift-OR doubling over the
// rows of one 32-column word held in shared memory (padded by P >= L rows on
// both sides so F at r < 0 is kept).  One CTA per word column.
__global__ void vdilate_kernel(const unsigned* mask, long long mask_pitch, long long words, int H, int L, int hi,
                               long long P, int x_lo, int x_hi, int y_lo, int y_hi, unsigned* V) {
    extern __shared__ unsigned smem[];
    const long long ext = (long long)H + 2 * P;
    unsigned* A = smem;
    unsigned* B = smem + ext;
    const long long w = blockIdx.x;
    const unsigned cm = interior_bits(w, x_lo, x_hi);
    int any = 0;
    for (long long i = threadIdx.x; i < ext; i += blockDim.x) {
        const long long r = i - P;
        const unsigned v = (r >= y_lo && r <= y_hi) ? (mask[r * mask_pitch + w] & cm) : 0u;
        A[i] = v;
        any |= (v != 0u);
    }
    if (!__syncthreads_or(any)) {
        for (long long y = threadIdx.x; y < H; y += blockDim.x) V[y * words + w] = 0u;
        return;
    }
    int l = 1;
    while (2 * l <= L) {
        for (long long i = threadIdx.x; i < ext; i += blockDim.x) B[i] = A[i] | (i + l < ext ? A[i + l] : 0u);
        __syncthreads();
        unsigned* t = A; A = B; B = t;
        l *= 2;
    }
    if (l < L) {
        const int s = L - l;
        for (long long i = threadIdx.x; i < ext; i += blockDim.x) B[i] = A[i] | (i + s < ext ? A[i + s] : 0u);
        __syncthreads();
        unsigned* t = A; A = B; B = t;
    }
    for (long long y = threadIdx.x; y < H; y += blockDim.x) V[y * words + w] = A[y - hi + P];
}

// Row pass: R(x) = OR_{c in [x-hi, x+lo]} V(c) = F_L(x - hi) with F_l(x) = OR V[x, x+l-1]
// built by shift-OR doubling in shared memory, OR'ed into the region row.
// The row is padded by P words on both sides so F at x < 0 is kept.  One CTA
// per row.
__global__ void hdilate_rows_kernel(const unsigned* V, long long words, long long P, int W, int L, int hi,
                                    unsigned* region, long long region_pitch) {
    extern __shared__ unsigned smem[];
    const long long ext = words + 2 * P;
    unsigned* A = smem;
    unsigned* B = smem + ext;
    const int y = blockIdx.x;
    int any = 0;
    for (long long i = threadIdx.x; i < ext; i += blockDim.x) {
        const long long wi = i - P;
        const unsigned v = (wi >= 0 && wi < words) ? V[(long long)y * words + wi] : 0u;
        A[i] = v;
        any |= (v != 0u);
    }
    if (!__syncthreads_or(any)) return;
    int l = 1;
    while (2 * l <= L) {  // F_{2l}(x) = F_l(x) | F_l(x + l)
        for (long long i = threadIdx.x; i < ext; i += blockDim.x) B[i] = A[i] | shifted_lo(A, i, ext, l);
        __syncthreads();
        unsigned* tmp = A; A = B; B = tmp;
        l *= 2;
    }
    if (l < L) {  // F_L(x) = F_l(x) | F_l(x + L - l), L - l < l
        for (long long i = threadIdx.x; i < ext; i += blockDim.x) B[i] = A[i] | shifted_lo(A, i, ext, L - l);
        __syncthreads();
        unsigned* tmp = A; A = B; B = tmp;
    }
    const unsigned last_mask = (W % 32) ? ((1u << (W % 32)) - 1u) : FULL;
    for (long long i = threadIdx.x; i < words; i += blockDim.x) {
        unsigned r = shifted_hi(A, i + P, ext, hi);  // F_L(x - hi)
        if (i == words - 1) r &= last_mask;
        if (r) region[(long long)y * region_pitch + i] |= r;
    }
}

__global__ void popcount_kernel(const unsigned* bits, long long pitch, long long words, int W, long long H,
                                unsigned long long* count) {
    const unsigned last_mask = (W % 32) ? ((1u << (W % 32)) - 1u) : FULL;
    unsigned long long local = 0;
    const long long n = words * H;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / words, w = i % words;
        unsigned v = bits[r * pitch + w];
        if (w == words - 1) v &= last_mask;
        local += __popc(v);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) local += __shfl_down_sync(FULL, local, d);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

// ── whole-ladder variants: one launch per kernel for every size ───────────

struct Ladder {
    int L;
    int m[SS_MAX_SIZES];
};

// One CTA per size: relative exclusive scan of the size's row counts.
__global__ void __launch_bounds__(1024) scan_sizes_kernel(const unsigned* counts, long long rows,
                                                          unsigned long long* row_off, unsigned long long* size_counts) {
    __shared__ unsigned long long warp_sums[32];
    __shared__ unsigned long long carry;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int k = blockIdx.x;
    const unsigned* c = counts + (long long)k * rows;
    unsigned long long* off = row_off + (long long)k * rows;
    if (t == 0) carry = 0;
    __syncthreads();
    for (long long base = 0; base < rows; base += 1024) {
        const long long i = base + t;
        const unsigned long long v = (i < rows) ? c[i] : 0ull;
        unsigned long long s = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long o = __shfl_up_sync(FULL, s, d);
            if (lane >= d) s += o;
        }
        if (lane == 31) warp_sums[warp] = s;
        __syncthreads();
        if (warp == 0) {
            unsigned long long w = warp_sums[lane];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned long long o = __shfl_up_sync(FULL, w, d);
                if (lane >= d) w += o;
            }
            warp_sums[lane] = w;
        }
        __syncthreads();
        const unsigned long long before = carry + (warp ? warp_sums[warp - 1] : 0ull) + s - v;
        if (i < rows) off[i] = before;
        __syncthreads();
        if (t == 1023) carry = before + v;
        __syncthreads();
    }
    if (t == 0) size_counts[k] = carry;
}

// grid (row blocks, sizes): one warp per mask row writes its survivors at
// base(size) + row offset, base = survivors of the earlier ladder sizes.
__global__ void write_xy_all_kernel(const unsigned* masks, long long mask_pitch, long long size_stride, int W, int H,
                                    int y_begin, long long rows, int stride, const Ladder lad, const unsigned* counts,
                                    const unsigned long long* row_off, const unsigned long long* size_counts, int* xy,
                                    int cols, long long capacity, unsigned long long* total) {
    const int k = blockIdx.y;
    if (blockIdx.x == 0 && k == 0 && threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int j = 0; j < lad.L; ++j) s += size_counts[j];
        *total = s;
    }
    const int m = lad.m[k];
    if (m < 8) return;
    const long long row = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows || counts[(long long)k * rows + row] == 0) return;  // warp-uniform
    unsigned long long base = 0;
    for (int j = 0; j < k; ++j) base += size_counts[j];
    const int lo = (m - 1) / 2, hi = m / 2;
    const int x_lo = lo, x_hi = W - 1 - hi;
    const unsigned* mrow = masks + (long long)k * size_stride + row * mask_pitch;
    const long long words = (W + 31) / 32;
    unsigned long long pos = base + row_off[(long long)k * rows + row];
    const int y = y_begin + (int)row;
    for (long long wb = 0; wb < words; wb += 32) {
        const long long w = wb + lane;
        unsigned bits = (w < words) ? (mrow[w] & interior_bits(w, x_lo, x_hi)) : 0u;
        const int c = __popc(bits);
        int incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int o = __shfl_up_sync(FULL, incl, d);
            if (lane >= d) incl += o;
        }
        unsigned long long p = pos + (unsigned long long)(incl - c);
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            if (p < (unsigned long long)capacity) {
                int* o = xy + (long long)cols * (long long)p;
                o[0] = (int)(w * 32 + b);
                o[1] = y;
                if (cols == 3) o[2] = m;
            }
            ++p;
        }
        pos += (unsigned long long)__shfl_sync(FULL, incl, 31);
    }
    (void)stride;
    (void)H;
}

// K5 (ladder form), pass 1 -- row dilation of every size: H_k(y) bit x =
// OR of size k's evaluated survivors (interior bits of its mask) in columns
// [x - hi, x + lo], i.e. the footprint columns (screening.py:316-330).  One
// warp per (size, row): the row sits in shared memory, F_L(x) = OR S[x,
// x+L-1] by shift-OR doubling (ping-pong buffers, __syncwarp between steps),
// then H(x) = F_L(x - hi).  Rows outside the size's interior are zero.
constexpr int RP_WARPS = 8;
__global__ void __launch_bounds__(RP_WARPS * 32) region_rows_kernel(const unsigned* masks, long long mask_pitch,
                                                                    long long size_stride, int W, int H,
                                                                    long long words, long long P,
                                                                    const Ladder lad, unsigned* Hb,
                                                                    unsigned* region, long long region_pitch,
                                                                    int y0, int Hg, unsigned char* live_rows,
                                                                    const unsigned* row_counts, long long rc_stride) {
    extern __shared__ unsigned rsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long task = (long long)blockIdx.x * RP_WARPS + warp;
    if (task >= (long long)lad.L * H) return;
    const int k = (int)(task / H), y = (int)(task % H);
    if (k == 0)  // the region is written (not accumulated): the column pass ORs into cleared rows
        for (long long i = lane; i < words; i += 32) region[(long long)y * region_pitch + i] = 0u;
    const int m = lad.m[k];
    const int lo = (m - 1) / 2, hi = m / 2;
    // K3's per-row survivor counts, when the caller has them: a row without
    // an interior survivor is flagged dead without reading its mask row
    if (row_counts && row_counts[(long long)k * rc_stride + y] == 0u) {
        if (lane == 0) live_rows[(long long)k * H + y] = 0;
        return;
    }
    unsigned* out = Hb + ((long long)k * H + y) * words;
    const unsigned* mrow = masks + (long long)k * size_stride + (long long)y * mask_pitch;
    // F is needed at x - hi >= -hi: the row sits at word offset P of a
    // left-padded buffer (padding = 0 = no survivors)
    const long long ext = words + P;
    unsigned* A = rsm + (size_t)warp * 2 * ext;
    unsigned* B = A + ext;
    const int gy = y0 + y;  // global row: interior status is decided in image coordinates
    const bool live = m >= 8 && gy >= lo && gy <= Hg - 1 - hi;
    unsigned any = 0;
    for (long long i = lane; i < ext; i += 32) {
        const long long wi = i - P;
        const unsigned v = (live && wi >= 0) ? (mrow[wi] & interior_bits(wi, lo, W - 1 - hi)) : 0u;
        A[i] = v;
        any |= v;
    }
    // rows without a survivor (3 in 4 at config 4) are only flagged: the column
    // pass reads live_rows and never touches their H_k row
    const bool has = __any_sync(FULL, any != 0u);
    if (lane == 0) live_rows[(long long)k * H + y] = has ? 1 : 0;
    if (!has) return;
    __syncwarp();
    const int L = m;
    int l = 1;
    while (2 * l <= L) {
        for (long long i = lane; i < ext; i += 32) B[i] = A[i] | shifted_lo(A, i, ext, l);
        __syncwarp();
        unsigned* t = A; A = B; B = t;
        l *= 2;
    }
    if (l < L) {
        for (long long i = lane; i < ext; i += 32) B[i] = A[i] | shifted_lo(A, i, ext, L - l);
        __syncwarp();
        unsigned* t = A; A = B; B = t;
    }
    const unsigned last_mask = (W % 32) ? ((1u << (W % 32)) - 1u) : FULL;
    for (long long i = lane; i < words; i += 32) {
        unsigned r = shifted_hi(A, i + P, ext, hi);
        if (i == words - 1) r &= last_mask;
        out[i] = r;
    }
}

// K5 pass 2 -- column dilation of H_k over rows [y - hi, y + lo], OR'ed into
// the region.  One thread per (size, chunk of C rows, word column): the C
// windows [r0 + c - hi, r0 + c - hi + L - 1] all contain row b = r0 - hi +
// L - 1 when L >= C, so each is a suffix-OR of rows [.., b] (computed
// backwards) | a prefix-OR of rows [b + 1, ..] (forwards): L + C - 1 loads
// for C outputs (van Herk / Gil-Werman).  Sizes with L < C take every window
// directly.
template <int C>
__global__ void __launch_bounds__(128) region_cols_kernel(const unsigned* Hb, int H, long long words, long long wblocks,
                                                          long long chunks, const Ladder lad, unsigned* region,
                                                          long long region_pitch, const unsigned char* live_rows) {
    // a block: 128 word columns of one (size, row chunk); the live flags of
    // the rows its windows cover are staged once, and a block none of whose
    // rows holds a survivor leaves at once
    const long long t = blockIdx.x;
    const long long wb = t % wblocks, ch = (t / wblocks) % chunks;
    const int k = (int)(t / (wblocks * chunks));
    const int m = lad.m[k];
    if (m < 8) return;
    const int lo = (m - 1) / 2, hi = m / 2, L = m;
    const int r0 = (int)(ch * C);
    const int a0 = r0 - hi, span = L + C - 1;  // rows a0 .. a0 + span - 1
    extern __shared__ unsigned char live_sh[];
    const unsigned char* lv = live_rows + (long long)k * H;
    int any = 0;
    for (int i = threadIdx.x; i < span; i += blockDim.x) {
        const int j = a0 + i;
        const unsigned char f = (j >= 0 && j < H) ? lv[j] : 0;
        live_sh[i] = f;
        any |= f;
    }
    if (!__syncthreads_or(any)) return;
    const long long w = wb * 128 + threadIdx.x;
    if (w >= words) return;
    const unsigned* col = Hb + (long long)k * H * words + w;
    auto ld = [&](int j) -> unsigned { return live_sh[j - a0] ? __ldg(col + (long long)j * words) : 0u; };
    unsigned out[C];
    if (L >= C) {
        const int b = a0 + L - 1;
        unsigned s = 0;
#pragma unroll 16
        for (int j = b; j >= a0 + C; --j) s |= ld(j);  // independent loads: 16 in flight
#pragma unroll
        for (int c = C - 1; c >= 0; --c) {
            s |= ld(a0 + c);
            out[c] = s;
        }
        unsigned p = 0;
#pragma unroll
        for (int c = 1; c < C; ++c) {
            p |= ld(b + c);
            out[c] |= p;
        }
    } else {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            unsigned v = 0;
            for (int j = r0 + c - hi; j <= r0 + c + lo; ++j) v |= ld(j);
            out[c] = v;
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c)
        if (out[c] && r0 + c < H) atomicOr(region + (long long)(r0 + c) * region_pitch + w, out[c]);
}

// K5, chained form (full image): the region is the union over sizes of each
// size's interior survivors dilated by its footprint [-lo_k, hi_k] in x and y
// (screening.py:316-330).  With the sizes in descending order and
// J_k = [-(lo_{k-1} - lo_k), hi_{k-1} - hi_k] the footprints telescope:
//   R_1 = S_1,  R_k = (R_{k-1} (+) J_k) | S_k,  region = R_n (+) [-lo_n, hi_n],
// so every step dilates by a small box (the ladder's consecutive margin gaps,
// cut to <= 31 each way) over the whole bitmap: one streaming pass per step
// instead of one full-size dilation per size.
// dilate_step_kernel: dst(p) = OR of src over rows / columns [p - b, p + a]
// (| the interior survivors of `mask`, when given).  A CTA owns a tile of
// DS_TR rows x DS_TW words: the tile plus its halo (b rows above, a below,
// one word each side) sits in shared memory; the vertical and then the
// horizontal window OR are shift-OR doublings.
constexpr int DS_TR = 64, DS_TW = 32, DS_HALO = 31;
__global__ void __launch_bounds__(256) dilate_step_kernel(const unsigned* src, const unsigned* mask, long long mask_pitch,
                                                         int lo_k, int hi_k, unsigned* dst, long long dst_pitch, int W,
                                                         int H, int words, int a, int b) {
    extern __shared__ unsigned dsm[];
    // tile words [w0 - 1, w0 + DS_TW + 3): one word left (the output's shift
    // by b < 32), three right (the window's a + b + 1 <= 63 bits past the
    // last output bit)
    constexpr int NW = DS_TW + 4;
    const int nr = DS_TR + a + b, L = a + b + 1;
    unsigned* A = dsm;
    unsigned* B = dsm + nr * NW;
    const int r0 = blockIdx.y * DS_TR, w0 = blockIdx.x * DS_TW;
    // load src rows [r0 - b, r0 + DS_TR + a), words [w0 - 1, w0 + DS_TW + 3)
    for (int i = threadIdx.x; i < nr * NW; i += blockDim.x) {
        const int t = i / NW, u = i - t * NW;
        const int gy = r0 - b + t, gw = w0 - 1 + u;
        A[i] = (src && gy >= 0 && gy < H && gw >= 0 && gw < words) ? __ldg(src + (long long)gy * words + gw) : 0u;
    }
    __syncthreads();
    // vertical: F_len(t) = OR A[t .. t + len - 1] (rows past the tile read as 0)
    int l = 1;
    while (l < L) {
        const int step = min(l, L - l);
        for (int i = threadIdx.x; i < nr * NW; i += blockDim.x) {
            const int t = i / NW;
            B[i] = A[i] | (t + step < nr ? A[i + step * NW] : 0u);
        }
        __syncthreads();
        unsigned* tmp = A; A = B; B = tmp;
        l += step;
    }
    // rows t in [0, DS_TR) of A now hold V(r0 + t) = OR src rows [r0 + t - b, r0 + t + a]
    // horizontal, per row, on bits: G_len(x) = OR V[x .. x + len - 1]
    l = 1;
    while (l < L) {
        const int step = min(l, L - l);
        for (int i = threadIdx.x; i < DS_TR * NW; i += blockDim.x) {
            const int t = i / NW, u = i - t * NW;
            const unsigned* row = A + t * NW;
            const unsigned lo = row[u], hi = u + 1 < NW ? row[u + 1] : 0u;
            B[i] = lo | ((lo >> step) | (hi << (32 - step)));  // step < 32
        }
        __syncthreads();
        unsigned* tmp = A; A = B; B = tmp;
        l += step;
    }
    // out(x) = G_L(x - b); | the interior survivors of this size
    const unsigned last_mask = (W & 31) ? ((1u << (W & 31)) - 1u) : 0xffffffffu;
    for (int i = threadIdx.x; i < DS_TR * DS_TW; i += blockDim.x) {
        const int t = i / DS_TW, u = i - t * DS_TW;
        const int gy = r0 + t, gw = w0 + u;
        if (gy >= H || gw >= words) continue;
        const unsigned* row = A + t * NW;
        const unsigned cur = row[u + 1], prev = row[u];
        unsigned v = b == 0 ? cur : ((cur << b) | (prev >> (32 - b)));  // b < 32
        if (mask && gy >= lo_k && gy <= H - 1 - hi_k)
            v |= __ldg(mask + (long long)gy * mask_pitch + gw) & interior_bits(gw, lo_k, W - 1 - hi_k);
        if (gw == words - 1) v &= last_mask;
        dst[(long long)gy * dst_pitch + gw] = v;
    }
}

// f4: bit-packed mask rows -> one byte per pixel, 255 kept / 0 not
// (cli.py:97-98 _mask_to_pgm), the PGM raster.  A thread per output 16 B:
// one 16-bit slice of a mask word, coalesced stores.
__global__ void bits_to_bytes_kernel(const unsigned* bits, long long pitch, int W, long long H, uint8_t* out) {
    const long long per_row = (W + 15) / 16;
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= per_row * H) return;
    const long long y = gid / per_row, c = gid % per_row;
    const unsigned wv = bits[y * pitch + (c >> 1)] >> ((c & 1) * 16);
    uint8_t v[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) v[b] = ((wv >> b) & 1u) ? 255 : 0;
    uint8_t* o = out + y * (long long)W + c * 16;
    const long long rem = (long long)W - c * 16;
    const int n = rem < 16 ? (int)rem : 16;
    if (n == 16 && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
        *reinterpret_cast<uint4*>(o) = *reinterpret_cast<const uint4*>(v);
    } else {
        for (int b = 0; b < n; ++b) o[b] = v[b];
    }
}

}  // namespace

size_t compact_workspace_bytes(int64_t rows) { return (size_t)std::max<int64_t>(rows, 1) * 8; }

int compact(const uint32_t* d_mask, int64_t mask_pitch, int64_t W, int64_t H, int64_t y_begin, int64_t y_end, int32_t m,
            int32_t stride, const uint32_t* d_row_counts, int32_t* d_xy, int64_t capacity, unsigned long long* d_total,
            unsigned long long* d_size_count, void* d_ws, size_t ws_bytes, void* stream) {
    const int64_t rows = y_end - y_begin;
    if (rows < 0 || W < 1 || m < 1 || stride < 1) { set_error("bad compact arguments"); return SS_EINVAL; }
    if (rows == 0) {
        if (d_size_count) cudaMemsetAsync(d_size_count, 0, sizeof(unsigned long long), as_stream(stream));
        return SS_OK;
    }
    if (ws_bytes < compact_workspace_bytes(rows) || !d_ws) { set_error("compact workspace too small"); return SS_EINVAL; }
    cudaStream_t s = as_stream(stream);
    auto* row_off = static_cast<unsigned long long*>(d_ws);
    scan_rows_kernel<<<1, 1024, 0, s>>>(d_row_counts, rows, row_off, d_total, d_size_count);
    note_launch();
    if (int e = check_launch("scan_rows_kernel")) return e;
    const int lo = (m - 1) / 2, hi = m / 2;
    write_xy_kernel<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, s>>>(
        d_mask, mask_pitch, (int)W, (int)y_begin, rows, lo, (int)(W - 1 - hi), d_row_counts, row_off, d_xy, capacity);
    note_launch();
    return check_launch("write_xy_kernel");
}

size_t region_workspace_bytes(int64_t W, int64_t H, int32_t m_max) {
    (void)m_max;
    return (size_t)H * ((W + 31) / 32) * 4;
}

int region_accumulate(const uint32_t* d_mask, int64_t mask_pitch, int64_t W, int64_t H, int32_t m, int32_t stride,
                      uint32_t* d_region, void* d_ws, size_t ws_bytes, void* stream) {
    if (W < 1 || H < 1 || m < 1 || stride < 1) { set_error("bad region arguments"); return SS_EINVAL; }
    if (ws_bytes < region_workspace_bytes(W, H, m) || !d_ws) { set_error("region workspace too small"); return SS_EINVAL; }
    const int lo = (m - 1) / 2, hi = m / 2, L = m;
    const int x_lo = lo, x_hi = (int)(W - 1 - hi), y_lo = lo, y_hi = (int)(H - 1 - hi);
    if (x_hi < x_lo || y_hi < y_lo) return SS_OK;  // no evaluated centres
    const int64_t words = (W + 31) / 32;
    unsigned* V = static_cast<unsigned*>(d_ws);
    cudaStream_t s = as_stream(stream);
    {
        const int64_t P = L;
        const size_t smem = (size_t)2 * (H + 2 * P) * 4;
        if (smem > 227 * 1024) { set_error("image too tall for the region pass"); return SS_EINVAL; }
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(vdilate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        vdilate_kernel<<<(unsigned)words, 1024, smem, s>>>(d_mask, mask_pitch, words, (int)H, L, hi, P, x_lo, x_hi, y_lo,
                                                           y_hi, V);
        note_launch();
        if (int e = check_launch("vdilate_kernel")) return e;
    }
    const int64_t P = (L + 31) / 32 + 1;
    const int threads = (int)std::min<int64_t>(1024, ((words + 2 * P + 31) / 32) * 32);
    const size_t smem = (size_t)2 * (words + 2 * P) * 4;
    if (smem > 48 * 1024) cudaFuncSetAttribute(hdilate_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    hdilate_rows_kernel<<<(unsigned)H, threads, smem, s>>>(V, words, P, (int)W, L, hi, d_region, mask_pitch);
    note_launch();
    return check_launch("hdilate_rows_kernel");
}

static int fill_ladder(Ladder& lad, int32_t L, const int32_t* h_m) {
    if (L < 1 || L > SS_MAX_SIZES || !h_m) {
        set_error("ladder length %d out of range", (int)L);
        return SS_EINVAL;
    }
    lad.L = L;
    for (int k = 0; k < L; ++k) lad.m[k] = h_m[k];
    return SS_OK;
}

size_t compact_ladder_workspace_bytes(int64_t rows, int32_t L) {
    return (size_t)std::max<int64_t>(rows, 1) * std::max<int32_t>(L, 1) * 8 + 256 + (size_t)SS_MAX_SIZES * 8;
}

int compact_ladder(const uint32_t* d_masks, int64_t mask_pitch, int64_t size_stride, int64_t W, int64_t H,
                   int64_t y_begin, int64_t y_end, int32_t L, const int32_t* h_m, int32_t stride,
                   const uint32_t* d_row_counts, int32_t* d_xy, int32_t cols, int64_t capacity,
                   unsigned long long* d_total, unsigned long long* d_size_counts, void* d_ws, size_t ws_bytes,
                   void* stream) {
    Ladder lad;
    if (int e = fill_ladder(lad, L, h_m)) return e;
    const int64_t rows = y_end - y_begin;
    if (rows < 0 || W < 1 || stride < 1) { set_error("bad compact arguments"); return SS_EINVAL; }
    if (cols != 2 && cols != 3) { set_error("xy_columns must be 2 or 3"); return SS_EINVAL; }
    cudaStream_t s = as_stream(stream);
    if (rows == 0) {
        cudaMemsetAsync(d_size_counts, 0, sizeof(unsigned long long) * L, s);
        cudaMemsetAsync(d_total, 0, sizeof(unsigned long long), s);
        return SS_OK;
    }
    if (ws_bytes < compact_ladder_workspace_bytes(rows, L) || !d_ws) {
        set_error("compact workspace too small");
        return SS_EINVAL;
    }
    auto* row_off = static_cast<unsigned long long*>(d_ws);
    scan_sizes_kernel<<<(unsigned)L, 1024, 0, s>>>(d_row_counts, rows, row_off, d_size_counts);
    note_launch();
    if (int e = check_launch("scan_sizes_kernel")) return e;
    write_xy_all_kernel<<<dim3((unsigned)((rows * 32 + 255) / 256), (unsigned)L), 256, 0, s>>>(
        d_masks, mask_pitch, size_stride, (int)W, (int)H, (int)y_begin, rows, stride, lad, d_row_counts, row_off,
        d_size_counts, d_xy, cols, capacity, d_total);
    note_launch();
    return check_launch("write_xy_all_kernel");
}

size_t region_ladder_workspace_bytes(int64_t W, int64_t H, int32_t L) {
    // the row-pass buffer of every size (region_ladder_rows), >= the chained form's two bitmaps
    // + one live flag per (size, row)
    return (size_t)std::max<int32_t>(L, 2) * H * ((W + 31) / 32) * 4 + ((size_t)std::max<int32_t>(L, 2) * H + 255) / 256 * 256;
}

// K5 over a window of H mask rows whose row 0 is global row y0 of an Hg-row
// image (a row band plus the neighbours' halo rows, sharding.py): interior
// status in global rows; footprints clipped to the window, which holds every
// survivor that covers the rows the caller keeps.
int region_ladder_rows(const uint32_t* d_masks, int64_t mask_pitch, int64_t size_stride, int64_t W, int64_t H,
                       int64_t y0, int64_t Hg, int32_t L, const int32_t* h_m, int32_t stride, uint32_t* d_region,
                       void* d_ws, size_t ws_bytes, void* stream, const uint32_t* d_row_counts = nullptr,
                       int64_t rc_stride = 0) {
    Ladder lad;
    if (int e = fill_ladder(lad, L, h_m)) return e;
    if (W < 1 || H < 1 || stride < 1 || y0 < 0 || y0 + H > Hg) { set_error("bad region arguments"); return SS_EINVAL; }
    if (ws_bytes < region_ladder_workspace_bytes(W, H, L) || !d_ws) {
        set_error("region workspace too small");
        return SS_EINVAL;
    }
    int m_max = 1;
    for (int k = 0; k < L; ++k) m_max = std::max(m_max, (int)h_m[k]);
    const int64_t words = (W + 31) / 32;
    unsigned* Hb = static_cast<unsigned*>(d_ws);
    unsigned char* live_rows = reinterpret_cast<unsigned char*>(Hb + (size_t)std::max<int32_t>(L, 2) * H * words);
    cudaStream_t s = as_stream(stream);
    {
        const int64_t P = m_max / 32 + 2;  // left padding (words) >= ceil(hi / 32)
        const size_t smem = (size_t)RP_WARPS * 2 * (words + P) * 4;
        if (smem > 227 * 1024) { set_error("image too wide for the region pass"); return SS_EINVAL; }
        static std::atomic<size_t> raised{0};
        if (smem > 48 * 1024 && smem > raised.load()) {
            cudaFuncSetAttribute(region_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            raised.store(smem);
        }
        const long long tasks = (long long)L * H;
        region_rows_kernel<<<(unsigned)((tasks + RP_WARPS - 1) / RP_WARPS), RP_WARPS * 32, smem, s>>>(
            d_masks, mask_pitch, size_stride, (int)W, (int)H, words, P, lad, Hb, d_region, mask_pitch, (int)y0,
            (int)Hg, live_rows, d_row_counts, (long long)rc_stride);
        note_launch();
        if (int e = check_launch("region_rows_kernel")) return e;
    }
    // taller footprints take longer row chunks (loads per output (L + C - 1) / C)
    const bool tall = m_max >= 128;
    const int C = tall ? 32 : 16;
    const long long chunks = (H + C - 1) / C;
    const long long wblocks = (words + 127) / 128;
    const unsigned grid = (unsigned)((long long)L * chunks * wblocks);
    const size_t fl = (size_t)(m_max + C - 1 + 15) / 16 * 16;  // the live flags of a block's rows
    if (tall)
        region_cols_kernel<32><<<grid, 128, fl, s>>>(Hb, (int)H, words, wblocks, chunks, lad, d_region, mask_pitch,
                                                      live_rows);
    else
        region_cols_kernel<16><<<grid, 128, fl, s>>>(Hb, (int)H, words, wblocks, chunks, lad, d_region, mask_pitch,
                                                      live_rows);
    note_launch();
    return check_launch("region_cols_kernel");
}

int region_ladder(const uint32_t* d_masks, int64_t mask_pitch, int64_t size_stride, int64_t W, int64_t H, int32_t L,
                  const int32_t* h_m, int32_t stride, uint32_t* d_region, void* d_ws, size_t ws_bytes, void* stream,
                  const uint32_t* d_row_counts = nullptr, int64_t rc_stride = 0) {
    // the chained form is opt-in (SS_REGION_CHAIN=1): measured slower than the
    // per-size row / column passes -- config 4 step 35.7 -> 36.6 ms, config 1
    // 0.66 -> 0.75 ms (a full-bitmap pass per step, each smem-bound)
    const char* chain = getenv("SS_REGION_CHAIN");
    if (!chain || atoi(chain) == 0)
        return region_ladder_rows(d_masks, mask_pitch, size_stride, W, H, 0, H, L, h_m, stride, d_region, d_ws,
                                  ws_bytes, stream, d_row_counts, rc_stride);
    Ladder lad;
    if (int e = fill_ladder(lad, L, h_m)) return e;
    if (W < 1 || H < 1 || stride < 1) { set_error("bad region arguments"); return SS_EINVAL; }
    const int64_t words = (W + 31) / 32;
    if (ws_bytes < (size_t)2 * H * words * 4 || !d_ws) {
        set_error("region workspace too small");
        return SS_EINVAL;
    }
    // evaluated sizes in descending order (the ladder is descending; m < 8 keep no survivors)
    std::vector<int> ks;
    for (int k = 0; k < L; ++k)
        if (h_m[k] >= 8) ks.push_back(k);
    std::stable_sort(ks.begin(), ks.end(), [&](int x, int y) { return h_m[x] > h_m[y]; });
    cudaStream_t s = as_stream(stream);
    if (ks.empty()) return cudaMemsetAsync(d_region, 0, (size_t)H * mask_pitch * 4, s) == cudaSuccess ? SS_OK
                                                                                                     : check_launch("region");
    unsigned* buf[2] = {static_cast<unsigned*>(d_ws), static_cast<unsigned*>(d_ws) + H * words};
    int cur = -1;  // buffer holding R (-1: R = 0)
    static std::atomic<int> raised{0};
    auto step = [&](const unsigned* mask, int lo_k, int hi_k, int a, int b, unsigned* dst, long long dst_pitch) -> int {
        const size_t smem = (size_t)2 * (DS_TR + a + b) * (DS_TW + 4) * 4;
        if ((int)smem > raised.load()) {
            cudaFuncSetAttribute(dilate_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            raised.store((int)smem);
        }
        const dim3 grid((unsigned)((words + DS_TW - 1) / DS_TW), (unsigned)((H + DS_TR - 1) / DS_TR));
        dilate_step_kernel<<<grid, 256, smem, s>>>(cur < 0 ? nullptr : buf[cur], mask, mask_pitch, lo_k, hi_k, dst,
                                                   dst_pitch, (int)W, (int)H, (int)words, a, b);
        note_launch();
        return check_launch("dilate_step_kernel");
    };
    // a dilation by [-a, b] in pieces of <= DS_HALO each way; the last piece ORs `mask`
    auto dilate = [&](int a, int b, const unsigned* mask, int lo_k, int hi_k, bool final) -> int {
        do {
            const int pa = std::min(a, DS_HALO), pb = std::min(b, DS_HALO);
            a -= pa;
            b -= pb;
            const bool last = a == 0 && b == 0;
            const int nxt = cur == 0 ? 1 : 0;
            unsigned* dst = (last && final) ? d_region : buf[nxt];
            if (int e = step(last ? mask : nullptr, lo_k, hi_k, pa, pb, dst, (last && final) ? mask_pitch : words))
                return e;
            cur = (last && final) ? -2 : nxt;
        } while (a > 0 || b > 0);
        return SS_OK;
    };
    int plo = 0, phi = 0;
    for (size_t j = 0; j < ks.size(); ++j) {
        const int k = ks[j], m = h_m[k], lo = (m - 1) / 2, hi = m / 2;
        const unsigned* mk = d_masks + (size_t)k * size_stride;
        if (int e = dilate(j == 0 ? 0 : plo - lo, j == 0 ? 0 : phi - hi, mk, lo, hi, false)) return e;
        plo = lo;
        phi = hi;
    }
    return dilate(plo, phi, nullptr, 0, 0, true);  // region = R_n (+) [-lo_n, hi_n]
}

int bits_to_bytes(const uint32_t* d_bits, int64_t pitch, int64_t W, int64_t H, uint8_t* d_out, void* stream) {
    if (W < 1 || H < 1 || pitch < (W + 31) / 32 || !d_bits || !d_out) {
        set_error("bad bits_to_bytes arguments");
        return SS_EINVAL;
    }
    const long long n = (W + 15) / 16 * H;
    bits_to_bytes_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(d_bits, pitch, (int)W, H, d_out);
    note_launch();
    return check_launch("bits_to_bytes_kernel");
}

int popcount(const uint32_t* d_bits, int64_t pitch, int64_t W, int64_t H, unsigned long long* d_count, void* stream) {
    if (W < 1 || H < 0) { set_error("bad popcount arguments"); return SS_EINVAL; }
    if (H == 0) return SS_OK;
    const int64_t words = (W + 31) / 32;
    const int64_t n = words * H;
    const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
    if (cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), as_stream(stream)) != cudaSuccess)
        return check_launch("memset");
    popcount_kernel<<<blocks, 256, 0, as_stream(stream)>>>(d_bits, pitch, words, (int)W, H, d_count);
    note_launch();
    return check_launch("popcount_kernel");
}

}  // namespace ss

extern "C" {
size_t ss_compact_workspace_bytes(int64_t rows) { return ss::compact_workspace_bytes(rows); }
int ss_compact(const uint32_t* d_mask, int64_t mask_pitch_words, int64_t W, int64_t H, int64_t y_begin, int64_t y_end,
               int32_t m, int32_t stride, const uint32_t* d_row_counts, int32_t* d_xy, int64_t capacity,
               unsigned long long* d_total, unsigned long long* d_size_count, void* d_workspace,
               size_t workspace_bytes, void* stream) {
    return ss::compact(d_mask, mask_pitch_words, W, H, y_begin, y_end, m, stride, d_row_counts, d_xy, capacity, d_total,
                       d_size_count, d_workspace, workspace_bytes, stream);
}
size_t ss_region_workspace_bytes(int64_t W, int64_t H, int32_t m_max) { return ss::region_workspace_bytes(W, H, m_max); }
int ss_region_accumulate(const uint32_t* d_mask, int64_t mask_pitch_words, int64_t W, int64_t H, int32_t m,
                         int32_t stride, uint32_t* d_region, void* d_workspace, size_t workspace_bytes, void* stream) {
    return ss::region_accumulate(d_mask, mask_pitch_words, W, H, m, stride, d_region, d_workspace, workspace_bytes,
                                 stream);
}
size_t ss_compact_ladder_workspace_bytes(int64_t rows, int32_t n_sizes) {
    return ss::compact_ladder_workspace_bytes(rows, n_sizes);
}
int ss_compact_ladder(const uint32_t* d_masks, int64_t mask_pitch_words, int64_t size_stride_words, int64_t W,
                      int64_t H, int64_t y_begin, int64_t y_end, int32_t n_sizes, const int32_t* h_m, int32_t stride,
                      const uint32_t* d_row_counts, int32_t* d_xy, int32_t xy_columns, int64_t capacity,
                      unsigned long long* d_total, unsigned long long* d_size_counts, void* d_workspace,
                      size_t workspace_bytes, void* stream) {
    return ss::compact_ladder(d_masks, mask_pitch_words, size_stride_words, W, H, y_begin, y_end, n_sizes, h_m, stride,
                              d_row_counts, d_xy, xy_columns, capacity, d_total, d_size_counts, d_workspace,
                              workspace_bytes, stream);
}
size_t ss_region_ladder_workspace_bytes(int64_t W, int64_t H, int32_t n_sizes) {
    return ss::region_ladder_workspace_bytes(W, H, n_sizes);
}
int ss_region_ladder(const uint32_t* d_masks, int64_t mask_pitch_words, int64_t size_stride_words, int64_t W, int64_t H,
                     int32_t n_sizes, const int32_t* h_m, int32_t stride, uint32_t* d_region, void* d_workspace,
                     size_t workspace_bytes, void* stream) {
    return ss::region_ladder(d_masks, mask_pitch_words, size_stride_words, W, H, n_sizes, h_m, stride, d_region,
                             d_workspace, workspace_bytes, stream);
}
int ss_region_ladder2(const uint32_t* d_masks, int64_t mask_pitch_words, int64_t size_stride_words, int64_t W, int64_t H,
                      int32_t n_sizes, const int32_t* h_m, int32_t stride, const uint32_t* d_row_counts,
                      int64_t row_counts_stride, uint32_t* d_region, void* d_workspace, size_t workspace_bytes,
                      void* stream) {
    return ss::region_ladder(d_masks, mask_pitch_words, size_stride_words, W, H, n_sizes, h_m, stride, d_region,
                             d_workspace, workspace_bytes, stream, d_row_counts, row_counts_stride);
}
int ss_region_ladder_rows(const uint32_t* d_masks, int64_t mask_pitch_words, int64_t size_stride_words, int64_t W,
                          int64_t rows, int64_t y0, int64_t H, int32_t n_sizes, const int32_t* h_m, int32_t stride,
                          uint32_t* d_region, void* d_workspace, size_t workspace_bytes, void* stream) {
    return ss::region_ladder_rows(d_masks, mask_pitch_words, size_stride_words, W, rows, y0, H, n_sizes, h_m, stride,
                                  d_region, d_workspace, workspace_bytes, stream);
}
int ss_popcount(const uint32_t* d_bits, int64_t mask_pitch_words, int64_t W, int64_t H, unsigned long long* d_count,
                void* stream) {
    return ss::popcount(d_bits, mask_pitch_words, W, H, d_count, stream);
}
int ss_bits_to_bytes(const uint32_t* d_bits, int64_t mask_pitch_words, int64_t W, int64_t H, uint8_t* d_out,
                     void* stream) {
    return ss::bits_to_bytes(d_bits, mask_pitch_words, W, H, d_out, stream);
}
int ss_copy_rows_async(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch, int64_t row_bytes,
                       int64_t rows, void* stream) {
    if (rows < 0 || row_bytes < 0 || (rows > 0 && (!dst || !src || dst_pitch < row_bytes || src_pitch < row_bytes))) {
        ss::set_error("bad row copy");
        return SS_EINVAL;
    }
    if (rows == 0 || row_bytes == 0) return SS_OK;
    if (cudaMemcpy2DAsync(dst, (size_t)dst_pitch, src, (size_t)src_pitch, (size_t)row_bytes, (size_t)rows,
                          cudaMemcpyDefault, ss::as_stream(stream)) != cudaSuccess)
        return ss::check_launch("row copy");
    return SS_OK;
}
}
