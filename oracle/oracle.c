/*
 * oracle.c -- CPU restatement of the starscreen pre-screening hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * (paper_1707_05647_b200) never links, imports or calls anything here.
 *
 * Every function restates the reference algorithm in plain C, citing the
 * reference file:line it follows (paths relative to
 * /root/reference/pkg/src/starscreen/).  The layouts are the reference's
 * own: Sat.cells is (H+1)x(W+1), Rsat.table is (W+H)x(W+H) indexed
 * [u+1][v+H-1].  Floating point follows NumPy's op-by-op IEEE binary64
 * rounding; this file must be compiled with -ffp-contract=off (no FMA).
 *
 * Pinned against golden vectors generated from the reference itself
 * (tests/golden/make_golden.py writes tests/golden/ fixtures).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { K_PLAIN = 0, K_X = 1, K_Y = 2, K_SQ = 3 };

/* integral.py:44-56 weight_map: 1-based x/y weights, I*I for SQUARED. */
static inline int64_t or_weight(int kind, int64_t v, int64_t x, int64_t y) {
    switch (kind) {
    case K_PLAIN: return v;
    case K_X: return v * (x + 1);
    case K_Y: return v * (y + 1);
    default: return v * v;
    }
}

/* integral.py:59-63 _check_overflow: 255*max(w,h)*w*h < 2^62. */
int or_check_overflow(int64_t W, int64_t H) {
    __int128 bound = (__int128)255 * (W > H ? W : H) * W * H;
    return bound < ((__int128)1 << 62) ? 0 : 1;
}

/* integral.py:109-117 build_sat: cumsum over rows (axis 0), then columns. */
void or_build_sat(const uint8_t* img, int64_t W, int64_t H, int kind, int64_t* cells) {
    const int64_t P = W + 1;
    memset(cells, 0, sizeof(int64_t) * (size_t)P * (size_t)(H + 1));
    for (int64_t y = 0; y < H; ++y)
        for (int64_t x = 0; x < W; ++x)
            cells[(y + 1) * P + x + 1] =
                cells[y * P + x + 1] + or_weight(kind, img[y * W + x], x, y);
    for (int64_t y = 1; y <= H; ++y)
        for (int64_t x = 1; x <= W; ++x)
            cells[y * P + x] += cells[y * P + x - 1];
}

/* integral.py:120-141 build_rsat: scatter wm into diag[x+y, x-y+h-1]
 * (side = w+h-1), cumsum over u (axis 0), reverse cumsum over v (axis 1),
 * table[1:, :side] = diag with a zero row 0 and zero last column. */
void or_build_rsat(const uint8_t* img, int64_t W, int64_t H, int kind, int64_t* table) {
    const int64_t side = W + H - 1, T = W + H;
    memset(table, 0, sizeof(int64_t) * (size_t)T * (size_t)T);
    /* diag[u][v] lives at table[(u+1)*T + v] */
    for (int64_t y = 0; y < H; ++y)
        for (int64_t x = 0; x < W; ++x)
            table[(x + y + 1) * T + (x - y + H - 1)] = or_weight(kind, img[y * W + x], x, y);
    for (int64_t u = 1; u < side; ++u)
        for (int64_t v = 0; v < side; ++v)
            table[(u + 1) * T + v] += table[u * T + v];
    for (int64_t u = 0; u < side; ++u)
        for (int64_t v = side - 2; v >= 0; --v)
            table[(u + 1) * T + v] += table[(u + 1) * T + v + 1];
}

typedef struct {
    const int64_t* sat[4];  /* Sat.cells per kind, (H+1)x(W+1) */
    const int64_t* rsat[4]; /* Rsat.table per kind, (W+H)x(W+H) */
    int64_t W, H;
} or_tables;

/* integral.py:79-81 Sat.cell */
static inline int64_t sat_cell(const int64_t* c, int64_t W, int64_t x, int64_t y) {
    return c[(y + 1) * (W + 1) + (x + 1)];
}
/* integral.py:100-101 Rsat._h */
static inline int64_t rsat_h(const int64_t* t, int64_t W, int64_t H, int64_t u, int64_t v) {
    return t[(u + 1) * (W + H) + (v + H - 1)];
}

/* integral.py:144-162 square_region_sum (caller guarantees bounds). */
static inline int64_t or_square_sum(const int64_t* c, int64_t W, int64_t cx, int64_t cy, int64_t n) {
    return sat_cell(c, W, cx + n, cy + n) - sat_cell(c, W, cx - n, cy + n) -
           sat_cell(c, W, cx + n, cy - n) + sat_cell(c, W, cx - n, cy - n);
}
/* integral.py:165-186 diamond_region_sum (caller guarantees bounds). */
static inline int64_t or_diamond_sum(const int64_t* t, int64_t W, int64_t H, int64_t cx, int64_t cy, int64_t r) {
    const int64_t u = cx + cy, v = cx - cy;
    return rsat_h(t, W, H, u + r, v - r) - rsat_h(t, W, H, u - r - 1, v - r) -
           rsat_h(t, W, H, u + r, v + r + 1) + rsat_h(t, W, H, u - r - 1, v + r + 1);
}

/* features.py:94-102 _square_stats_from_sums: exact NumPy op order. */
static void or_square_stats(int64_t s1, int64_t sx, int64_t sy, int64_t s2, int64_t cx, int64_t cy,
                            int64_t n, double out[4]) {
    const double count = (double)(4 * n * n);
    const double w1 = (double)(2 * n * n * n);
    const double mean = (double)s1 / count;
    const double var = (double)s2 / count - mean * mean;
    out[0] = mean;
    out[1] = sqrt(var > 0.0 ? var : 0.0);
    out[2] = ((double)sx - ((double)cx + 1.5) * (double)s1) / w1;
    out[3] = ((double)sy - ((double)cy + 1.5) * (double)s1) / w1;
}

/* features.py:113-115 _ball_l1_mass; integral.py:189-191 diamond_pixel_count. */
static inline int64_t or_ball_l1_mass(int64_t r) { return 2 * r * r + r * (r - 1) * (2 * r - 1) / 3; }
static inline int64_t or_diamond_count(int64_t r) { return 2 * r * r + 2 * r + 1; }

/* features.py:118-125 _diamond_stats_from_sums. */
static void or_diamond_stats(int64_t s1, int64_t sx, int64_t sy, int64_t s2, int64_t cx, int64_t cy,
                             int64_t r, double out[4]) {
    const double count = (double)or_diamond_count(r);
    const double w1 = (double)or_ball_l1_mass(r);
    const double mean = (double)s1 / count;
    const double var = (double)s2 / count - mean * mean;
    out[0] = mean;
    out[1] = sqrt(var > 0.0 ? var : 0.0);
    out[2] = ((double)sx - ((double)cx + 1.0) * (double)s1) / w1;
    out[3] = ((double)sy - ((double)cy + 1.0) * (double)s1) / w1;
}

/* features.py:136-142 _octagon_from_parts. */
static void or_octagon_from_parts(const double sq[4], const double di[4], double out[3]) {
    const double gx = (sq[2] + di[2]) * 0.5;
    const double gy = (sq[3] + di[3]) * 0.5;
    out[0] = (sq[0] + di[0]) * 0.5;
    out[1] = (sq[1] + di[1]) * 0.5;
    out[2] = sqrt(gx * gx + gy * gy);
}

/* features.py:151-154 _octagon_maps for one center. */
static void or_octagon(const or_tables* t, int64_t cx, int64_t cy, int64_t n, int64_t d, double out[3]) {
    double sq[4], di[4];
    or_square_stats(or_square_sum(t->sat[K_PLAIN], t->W, cx, cy, n),
                    or_square_sum(t->sat[K_X], t->W, cx, cy, n),
                    or_square_sum(t->sat[K_Y], t->W, cx, cy, n),
                    or_square_sum(t->sat[K_SQ], t->W, cx, cy, n), cx, cy, n, sq);
    or_diamond_stats(or_diamond_sum(t->rsat[K_PLAIN], t->W, t->H, cx, cy, d),
                     or_diamond_sum(t->rsat[K_X], t->W, t->H, cx, cy, d),
                     or_diamond_sum(t->rsat[K_Y], t->W, t->H, cx, cy, d),
                     or_diamond_sum(t->rsat[K_SQ], t->W, t->H, cx, cy, d), cx, cy, d, di);
    or_octagon_from_parts(sq, di, out);
}

/* Exported single-center features (tests compare to golden ring maps). */
void or_ring_features(const int64_t* const* sats, const int64_t* const* rsats, int64_t W, int64_t H,
                      int64_t cx, int64_t cy, int64_t n_rings, const int32_t* ring_n,
                      const int32_t* ring_d, double* out /* n_rings*3 */) {
    or_tables t;
    for (int k = 0; k < 4; ++k) { t.sat[k] = sats[k]; t.rsat[k] = rsats[k]; }
    t.W = W; t.H = H;
    for (int64_t r = 0; r < n_rings; ++r) or_octagon(&t, cx, cy, ring_n[r], ring_d[r], out + 3 * r);
}

/* screening.py:81-87 quantize: floor(f / q + 0.5). */
static inline int64_t or_quantize(double f, double q) { return (int64_t)floor(f / q + 0.5); }

#define OR_KEY_BASE ((int64_t)1 << 21) /* screening.py:57 */

/* screening.py:90-97 _pack_cells; returns -1 when a cell is out of range
 * (the reference raises ValueError for the whole array in that case). */
static inline int64_t or_pack(int64_t cm, int64_t cs, int64_t cg) {
    if (cm < 0 || cs < 0 || cg < 0 || cm >= OR_KEY_BASE || cs >= OR_KEY_BASE || cg >= OR_KEY_BASE)
        return -1;
    return (cm * OR_KEY_BASE + cs) * OR_KEY_BASE + cg;
}

/* screening.py:173-178 _member_mask via searchsorted equality. */
static int or_member(const int64_t* keys, int64_t nkeys, int64_t key) {
    int64_t lo = 0, hi = nkeys; /* searchsorted 'left' */
    if (nkeys == 0) return 0;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < key) lo = mid + 1; else hi = mid;
    }
    if (lo > nkeys - 1) lo = nkeys - 1;
    return keys[lo] == key;
}

/* SURVEY.md 8(d) parity protocol: t = f/q + 1/2 lies within the 1e-6
 * relative band of a quantisation boundary, |t - round(t)| <= 1e-6 max(|t|, 1)
 * (exact boundaries included).  Only the checker uses this; it does not
 * change any decision. */
static inline int or_in_band(double f, double q) {
    const double t = f / q + 0.5;
    const double at = fabs(t);
    return fabs(t - nearbyint(t)) <= 1e-6 * (at > 1.0 ? at : 1.0);
}

/*
 * screening.py:418-471 _scan_size over one ladder size.
 *   mask: H*W bytes, set to 1 for kept grid centers (border keeps included)
 *   kept_xy: capacity 2*cap int32 (cx,cy) pairs, row-major order
 *   band: optional H*W bytes, 1 at interior centres that are band positions
 *         (or_in_band), else 0
 * Returns the number of evaluated survivors (or -1 if cap too small,
 * -2 on a pack-capacity error, the reference's ValueError).
 * *tested receives ix.size * iy.size.
 */
int64_t or_scan_size(const int64_t* const* sats, const int64_t* const* rsats, int64_t W, int64_t H,
                     int64_t m, int64_t stride, int64_t n_rings, const int32_t* ring_n,
                     const int32_t* ring_d, const int64_t* keys, const int64_t* key_off,
                     double qm, double qs, double qg, uint8_t* mask, int32_t* kept_xy,
                     int64_t cap, int64_t* tested, int nthreads, uint8_t* band) {
    or_tables t;
    for (int k = 0; k < 4; ++k) { t.sat[k] = sats[k]; t.rsat[k] = rsats[k]; }
    t.W = W; t.H = H;
    /* features.py:214-217 patch_center_margins */
    const int64_t lo = (m - 1) / 2, hi = m / 2;
    memset(mask, 0, (size_t)W * (size_t)H);
    if (band) memset(band, 0, (size_t)W * (size_t)H);
    int64_t nix = 0, niy = 0;
    for (int64_t y = 0; y < H; y += stride) {
        const int in_y = (y >= lo) && (y <= H - 1 - hi);
        niy += in_y;
        for (int64_t x = 0; x < W; x += stride) {
            const int in_x = (x >= lo) && (x <= W - 1 - hi);
            if (y == 0) nix += in_x;
            /* screening.py:438-442: every grid center outside the interior is kept */
            if (!in_x || !in_y) mask[y * W + x] = 1;
        }
    }
    *tested = nix * niy;
    if (nix == 0 || niy == 0) return 0;
    int err = 0;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(| : err)
#endif
    for (int64_t y = lo; y <= H - 1 - hi; ++y) {
        if (y % stride) continue;
        for (int64_t x = lo; x <= W - 1 - hi; ++x) {
            if (x % stride) continue;
            int ok = 1;
            for (int64_t r = 0; r < n_rings && ok; ++r) {
                double f[3];
                or_octagon(&t, x, y, ring_n[r], ring_d[r], f);
                /* band positions: any channel of any ring the reference evaluates here */
                if (band && (or_in_band(f[0], qm) || or_in_band(f[1], qs) || or_in_band(f[2], qg)))
                    band[y * W + x] = 1;
                const int64_t key = or_pack(or_quantize(f[0], qm), or_quantize(f[1], qs), or_quantize(f[2], qg));
                if (key < 0) { err = 1; ok = 0; break; }
                ok = or_member(keys + key_off[r], key_off[r + 1] - key_off[r], key);
            }
            if (ok) mask[y * W + x] = 1;
        }
    }
    if (err) return -2;
    int64_t nk = 0;
    for (int64_t y = lo; y <= H - 1 - hi; ++y) {
        if (y % stride) continue;
        for (int64_t x = lo; x <= W - 1 - hi; ++x) {
            if (x % stride) continue;
            if (mask[y * W + x]) {
                if (nk >= cap) return -1;
                kept_xy[2 * nk] = (int32_t)x;
                kept_xy[2 * nk + 1] = (int32_t)y;
                ++nk;
            }
        }
    }
    return nk;
}

/* image_io.py:131-161 _sample_bilinear + _quantize_levels for the
 * half-pixel-centred resize of image_io.py:164-178. */
void or_resize_bilinear(const uint8_t* img, int64_t w, int64_t h, int64_t out_w, int64_t out_h, uint8_t* out) {
    const double sx_ = (double)w / (double)out_w, sy_ = (double)h / (double)out_h;
    for (int64_t j = 0; j < out_h; ++j) {
        const double ys = ((double)j + 0.5) * sy_ - 0.5;
        const double y0f = floor(ys), fy = ys - y0f;
        int64_t y0 = (int64_t)y0f, y1 = y0 + 1;
        y0 = y0 < 0 ? 0 : (y0 > h - 1 ? h - 1 : y0);
        y1 = y1 < 0 ? 0 : (y1 > h - 1 ? h - 1 : y1);
        for (int64_t i = 0; i < out_w; ++i) {
            const double xs = ((double)i + 0.5) * sx_ - 0.5;
            const double x0f = floor(xs), fx = xs - x0f;
            int64_t x0 = (int64_t)x0f, x1 = x0 + 1;
            x0 = x0 < 0 ? 0 : (x0 > w - 1 ? w - 1 : x0);
            x1 = x1 < 0 ? 0 : (x1 > w - 1 ? w - 1 : x1);
            const double v00 = img[y0 * w + x0], v01 = img[y0 * w + x1];
            const double v10 = img[y1 * w + x0], v11 = img[y1 * w + x1];
            const double top = v00 + fx * (v01 - v00);
            const double bot = v10 + fx * (v11 - v10);
            double v = floor((top + fy * (bot - top)) + 0.5);
            v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
            out[j * out_w + i] = (uint8_t)v;
        }
    }
}

/*
 * screening.py:238-249 one iteration of build_feature_set: resize the n x n
 * template to k x k (image_io.py:164-178), crop the centred m x m window
 * (image_io.py:216-228), build its tables (integral.py:211-228) and take the
 * ring features at c = (m-1)//2 (features.py:220-224).  out: n_rings*3.
 */
void or_template_ring_features(const uint8_t* tpl, int64_t n, int64_t k, int64_t m, int64_t n_rings,
                               const int32_t* ring_n, const int32_t* ring_d, double* out) {
    uint8_t* scaled = (uint8_t*)malloc((size_t)(k * k));
    uint8_t* z = (uint8_t*)malloc((size_t)(m * m));
    or_resize_bilinear(tpl, n, n, k, k, scaled);
    const int64_t x0 = (k - m) / 2, y0 = (k - m) / 2;
    for (int64_t j = 0; j < m; ++j) memcpy(z + j * m, scaled + (y0 + j) * k + x0, (size_t)m);
    int64_t* sats[4];
    int64_t* rsats[4];
    for (int kk = 0; kk < 4; ++kk) {
        sats[kk] = (int64_t*)malloc(sizeof(int64_t) * (size_t)((m + 1) * (m + 1)));
        rsats[kk] = (int64_t*)malloc(sizeof(int64_t) * (size_t)((2 * m) * (2 * m)));
        or_build_sat(z, m, m, kk, sats[kk]);
        or_build_rsat(z, m, m, kk, rsats[kk]);
    }
    const int64_t c = (m - 1) / 2;
    or_ring_features((const int64_t* const*)sats, (const int64_t* const*)rsats, m, m, c, c, n_rings,
                     ring_n, ring_d, out);
    for (int kk = 0; kk < 4; ++kk) { free(sats[kk]); free(rsats[kk]); }
    free(scaled);
    free(z);
}
