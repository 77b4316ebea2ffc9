// ss_template.cpp -- host side of the screen: template feature sets and the
// device key blob.  Compiled with -ffp-contract=off: the resampling and the
// feature arithmetic reproduce NumPy's op-by-op binary64 rounding.
//
// Replaces build_feature_set (screening.py:222-250), FeatureSet.insert /
// _guard_cells / ring_keys (screening.py:122-155), resize_bilinear +
// _sample_bilinear + _quantize_levels (image_io.py:131-178), crop_center
// (image_io.py:216-228) and the patch-side ring features (features.py:
// 220-224 via :322-370).
#include <algorithm>
#include <array>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/starscreen_b200.h"

namespace ss {
void set_error(const char* fmt, ...);

namespace {

// image_io.py:131-178 -- half-pixel-centred bilinear resize, edge clamp,
// round half up, clip to [0, 255].
void resize_bilinear(const uint8_t* img, int64_t w, int64_t h, int64_t ow, int64_t oh, uint8_t* out) {
    const double fxs = (double)w / (double)ow, fys = (double)h / (double)oh;
    for (int64_t j = 0; j < oh; ++j) {
        const double ys = ((double)j + 0.5) * fys - 0.5;
        const double y0f = std::floor(ys), fy = ys - y0f;
        const int64_t y0 = std::min<int64_t>(std::max<int64_t>((int64_t)y0f, 0), h - 1);
        const int64_t y1 = std::min<int64_t>(std::max<int64_t>((int64_t)y0f + 1, 0), h - 1);
        for (int64_t i = 0; i < ow; ++i) {
            const double xs = ((double)i + 0.5) * fxs - 0.5;
            const double x0f = std::floor(xs), fx = xs - x0f;
            const int64_t x0 = std::min<int64_t>(std::max<int64_t>((int64_t)x0f, 0), w - 1);
            const int64_t x1 = std::min<int64_t>(std::max<int64_t>((int64_t)x0f + 1, 0), w - 1);
            const double v00 = img[y0 * w + x0], v01 = img[y0 * w + x1];
            const double v10 = img[y1 * w + x0], v11 = img[y1 * w + x1];
            const double top = v00 + fx * (v01 - v00);
            const double bot = v10 + fx * (v11 - v10);
            double v = std::floor((top + fy * (bot - top)) + 0.5);
            v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
            out[j * ow + i] = (uint8_t)v;
        }
    }
}

struct Sums {
    int64_t s1 = 0, sx = 0, sy = 0, s2 = 0;
};

// features.py:94-142 on exact integer sums of the m x m patch z, centre c.
void ring_features(const uint8_t* z, int64_t m, int32_t n_rings, const int32_t* rn, const int32_t* rd, double* out) {
    const int64_t c = (m - 1) / 2;
    for (int32_t r = 0; r < n_rings; ++r) {
        const int64_t n = rn[r], d = rd[r];
        Sums q, di;
        for (int64_t y = c - n + 1; y <= c + n; ++y)
            for (int64_t x = c - n + 1; x <= c + n; ++x) {
                const int64_t v = z[y * m + x];
                q.s1 += v;
                q.sx += (x + 1) * v;
                q.sy += (y + 1) * v;
                q.s2 += v * v;
            }
        for (int64_t y = c - d; y <= c + d; ++y) {
            const int64_t ry = d - (y > c ? y - c : c - y);
            for (int64_t x = c - ry; x <= c + ry; ++x) {
                const int64_t v = z[y * m + x];
                di.s1 += v;
                di.sx += (x + 1) * v;
                di.sy += (y + 1) * v;
                di.s2 += v * v;
            }
        }
        // _square_stats_from_sums
        const double cq = (double)(4 * n * n), wq = (double)(2 * n * n * n);
        const double mq = (double)q.s1 / cq;
        const double vq = (double)q.s2 / cq - mq * mq;
        const double sq = std::sqrt(vq > 0.0 ? vq : 0.0);
        const double gxq = ((double)q.sx - ((double)c + 1.5) * (double)q.s1) / wq;
        const double gyq = ((double)q.sy - ((double)c + 1.5) * (double)q.s1) / wq;
        // _diamond_stats_from_sums
        const double cd = (double)(2 * d * d + 2 * d + 1), wd = (double)(2 * d * d + d * (d - 1) * (2 * d - 1) / 3);
        const double md = (double)di.s1 / cd;
        const double vd = (double)di.s2 / cd - md * md;
        const double sd = std::sqrt(vd > 0.0 ? vd : 0.0);
        const double gxd = ((double)di.sx - ((double)c + 1.0) * (double)di.s1) / wd;
        const double gyd = ((double)di.sy - ((double)c + 1.0) * (double)di.s1) / wd;
        // _octagon_from_parts
        const double gx = (gxq + gxd) * 0.5, gy = (gyq + gyd) * 0.5;
        out[3 * r + 0] = (mq + md) * 0.5;
        out[3 * r + 1] = (sq + sd) * 0.5;
        out[3 * r + 2] = std::sqrt(gx * gx + gy * gy);
    }
}

// one rescale k: resize n x n -> k x k, crop centred m x m, ring features
void template_features(const uint8_t* tpl, int32_t n, int32_t k, int32_t m, int32_t n_rings, const int32_t* rn,
                       const int32_t* rd, double* out) {
    std::vector<uint8_t> scaled((size_t)k * k), z((size_t)m * m);
    resize_bilinear(tpl, n, n, k, k, scaled.data());
    const int64_t off = (k - m) / 2;  // crop_center: floor((size - out) / 2)
    for (int64_t j = 0; j < m; ++j) std::memcpy(&z[j * m], &scaled[(off + j) * k + off], (size_t)m);
    ring_features(z.data(), m, n_rings, rn, rd, out);
}

inline int64_t quantize(double v, double q) { return (int64_t)std::floor(v / q + 0.5); }

}  // namespace
}  // namespace ss

extern "C" {

int ss_template_ring_features(const uint8_t* h_template, int32_t n, int32_t k, int32_t m, int32_t n_rings,
                              const int32_t* h_ring_n, const int32_t* h_ring_d, double* h_out) {
    if (!h_template || n < 1 || k < m || m < 8 || n_rings < 1) {
        ss::set_error("bad template feature arguments");
        return SS_EINVAL;
    }
    ss::template_features(h_template, n, k, m, n_rings, h_ring_n, h_ring_d, h_out);
    return SS_OK;
}

int ss_feature_set_keys(const uint8_t* h_template, int32_t n, int32_t m, int32_t k_hi, int32_t n_rings,
                        const int32_t* h_ring_n, const int32_t* h_ring_d, double q_mean, double q_std, double q_grad,
                        int64_t* h_keys, int64_t* h_key_off) {
    if (!h_template || n < 1 || m < 8 || k_hi < m || n_rings < 1 || n_rings > SS_MAX_RINGS) {
        ss::set_error("bad feature-set arguments");
        return SS_EINVAL;
    }
    const int32_t nk = k_hi - m + 1;
    std::vector<double> feats((size_t)nk * n_rings * 3);
    // rescales are independent: spread them over host threads
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const int32_t nthreads = (int32_t)std::min<unsigned>(hw, (unsigned)((nk + 3) / 4));
    auto work = [&](int32_t tid) {
        for (int32_t i = tid; i < nk; i += nthreads)
            ss::template_features(h_template, n, m + i, m, n_rings, h_ring_n, h_ring_d, &feats[(size_t)i * n_rings * 3]);
    };
    if (nthreads <= 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (int32_t t = 0; t < nthreads; ++t) pool.emplace_back(work, t);
        for (auto& th : pool) th.join();
    }
    return ss_keys_from_features(feats.data(), nk, n_rings, q_mean, q_std, q_grad, h_keys, h_key_off);
}

int ss_keys_from_features(const double* h_feats, int32_t nk, int32_t n_rings, double q_mean, double q_std,
                          double q_grad, int64_t* h_keys, int64_t* h_key_off) {
    if (!h_feats || nk < 0 || n_rings < 1 || n_rings > SS_MAX_RINGS) {
        ss::set_error("bad feature-key arguments");
        return SS_EINVAL;
    }
    const double* feats_ = h_feats;
    // FeatureSet.insert in k order (screening.py:127-145)
    const double qs[3] = {q_mean, q_std, q_grad};
    // Per ring: the guard-banded keys of every instance (27 per instance,
    // heavily repeated across neighbouring rescales) deduplicated on insert
    // in a small open-addressing table, then the unique keys sorted -- the
    // set semantics of FeatureSet (screening.py:122-155).
    struct KeySet {
        std::vector<int64_t> slots, uniq;
        size_t mask = 0;
        void init(size_t expect) {
            size_t cap = 64;
            while (cap < 2 * expect) cap <<= 1;
            slots.assign(cap, -1);
            mask = cap - 1;
            uniq.clear();
        }
        void add(int64_t k) {  // keys are >= 0; -1 marks an empty slot
            size_t i = (size_t)(((uint64_t)k * 0x9E3779B97F4A7C15ull) >> 20) & mask;
            while (slots[i] != -1) {
                if (slots[i] == k) return;
                i = (i + 1) & mask;
            }
            slots[i] = k;
            uniq.push_back(k);
            if (2 * uniq.size() > slots.size()) rehash();
        }
        void rehash() {
            std::vector<int64_t> keep = uniq;
            init(2 * keep.size());
            for (int64_t k : keep) add(k);
        }
    };
    std::vector<KeySet> rings(n_rings);
    for (auto& r : rings) r.init(256);
    // an instance whose guard cells equal an earlier instance's (same ring)
    // adds the same 27 keys: skip it
    std::vector<std::vector<std::array<int64_t, 9>>> seen(n_rings);
    for (int32_t i = 0; i < nk; ++i) {
        for (int32_t r = 0; r < n_rings; ++r) {
            std::array<int64_t, 9> g;
            int nc[3];
            for (int ch = 0; ch < 3; ++ch) {
                const double v = feats_[((size_t)i * n_rings + r) * 3 + ch], q = qs[ch], half = q / 2.0;
                int64_t c3[3] = {ss::quantize(v - half, q), ss::quantize(v, q), ss::quantize(v + half, q)};
                std::sort(c3, c3 + 3);
                nc[ch] = (int)(std::unique(c3, c3 + 3) - c3);
                for (int j = 0; j < 3; ++j) g[(size_t)ch * 3 + j] = j < nc[ch] ? c3[j] : -1;
            }
            bool dup = false;
            for (const auto& t : seen[r])
                if (t == g) { dup = true; break; }
            if (dup) continue;
            seen[r].push_back(g);
            for (int a = 0; a < nc[0]; ++a)
                for (int b = 0; b < nc[1]; ++b)
                    for (int c = 0; c < nc[2]; ++c) {
                        const int64_t cm = g[a], cs = g[3 + b], cg = g[6 + c];
                        if (cm >= SS_KEY_BASE || cs >= SS_KEY_BASE || cg >= SS_KEY_BASE) {
                            ss::set_error("quantized cell exceeds key capacity, quantizer too fine");
                            return SS_ECAPACITY;
                        }
                        if (cm < 0 || cs < 0 || cg < 0) {
                            ss::set_error("negative quantized cell; features must be non-negative");
                            return SS_ECAPACITY;
                        }
                        rings[r].add((cm * SS_KEY_BASE + cs) * SS_KEY_BASE + cg);
                    }
        }
    }
    int64_t pos = 0;
    h_key_off[0] = 0;
    for (int32_t r = 0; r < n_rings; ++r) {
        auto& v = rings[r].uniq;
        std::sort(v.begin(), v.end());
        std::memcpy(h_keys + pos, v.data(), v.size() * sizeof(int64_t));
        pos += (int64_t)v.size();
        h_key_off[r + 1] = pos;
    }
    return SS_OK;
}

}  // extern "C"
namespace ss {
// The ss_keyset_blob layout built into `blob` (reused storage).
static int build_keyset_blob(const int64_t* h_keys, const int64_t* h_key_off, int32_t n_rings,
                             std::vector<int64_t>& blob);
}  // namespace ss
extern "C" {

int ss_keyset_blob(const int64_t* h_keys, const int64_t* h_key_off, int32_t n_rings, int64_t* h_blob,
                   size_t* blob_bytes) {
    if (!h_key_off || n_rings < 1 || n_rings > SS_MAX_RINGS || !blob_bytes) {
        ss::set_error("bad keyset arguments");
        return SS_EINVAL;
    }
    std::vector<int64_t> blob;
    if (int e = ss::build_keyset_blob(h_keys, h_key_off, n_rings, blob)) return e;
    const size_t need = blob.size() * sizeof(int64_t);
    if (h_blob) {
        if (*blob_bytes < need) {
            ss::set_error("key blob buffer too small: %zu < %zu", *blob_bytes, need);
            return SS_EINVAL;
        }
        std::memcpy(h_blob, blob.data(), need);
    }
    *blob_bytes = need;
    return SS_OK;
}

}  // extern "C"
namespace ss {
static int build_keyset_blob(const int64_t* h_keys, const int64_t* h_key_off, int32_t n_rings,
                             std::vector<int64_t>& blob) {
    // Layout (int64 slots): [0] n_rings; header of SS_BLOB_HDR slots per ring at
    // 1 + SS_BLOB_HDR * r:
    //   0 off_m  1 n_m  2 off_ms  3 n_ms  4 off_k  5 n_k        sorted arrays
    //   6 cm_lo  7 cm_n  8 cs_lo  9 cs_n  10 cg_lo  11 cg_n     key bounding box
    //   12 off_bits (-1: none)  13 words_m  14 words_ms  15 words_full
    // The bit section packs uint32 words [m | ms | full] two per slot; bit i of
    // ms is (cm-cm_lo)*cs_n + (cs-cs_lo), of full ((..)*cg_n + (cg-cg_lo)).
    const int H = SS_BLOB_HDR;
    blob.assign(1 + (size_t)H * n_rings, 0);
    blob[0] = n_rings;
    for (int32_t r = 0; r < n_rings; ++r) {
        const int64_t a = h_key_off[r], b = h_key_off[r + 1];
        std::vector<int64_t> km, kms;
        int64_t lo[3] = {INT64_MAX, INT64_MAX, INT64_MAX}, hi[3] = {-1, -1, -1};
        for (int64_t i = a; i < b; ++i) {
            if (i > a && h_keys[i] <= h_keys[i - 1]) {
                ss::set_error("ring keys must be sorted and unique");
                return SS_EINVAL;
            }
            const int64_t ms = h_keys[i] / SS_KEY_BASE, mm = ms / SS_KEY_BASE;
            const int64_t c3[3] = {mm, ms % SS_KEY_BASE, h_keys[i] % SS_KEY_BASE};
            for (int c = 0; c < 3; ++c) { lo[c] = std::min(lo[c], c3[c]); hi[c] = std::max(hi[c], c3[c]); }
            if (kms.empty() || kms.back() != ms) kms.push_back(ms);
            if (km.empty() || km.back() != mm) km.push_back(mm);
        }
        auto hd = [&](int i) -> int64_t& { return blob[1 + (size_t)H * r + i]; };
        hd(0) = (int64_t)blob.size();
        hd(1) = (int64_t)km.size();
        blob.insert(blob.end(), km.begin(), km.end());
        hd(2) = (int64_t)blob.size();
        hd(3) = (int64_t)kms.size();
        blob.insert(blob.end(), kms.begin(), kms.end());
        hd(4) = (int64_t)blob.size();
        hd(5) = b - a;
        blob.insert(blob.end(), h_keys + a, h_keys + b);
        const int64_t n[3] = {b > a ? hi[0] - lo[0] + 1 : 0, b > a ? hi[1] - lo[1] + 1 : 0,
                              b > a ? hi[2] - lo[2] + 1 : 0};
        for (int c = 0; c < 3; ++c) { hd(6 + 2 * c) = b > a ? lo[c] : 0; hd(7 + 2 * c) = n[c]; }
        hd(12) = -1;
        const int64_t bm = n[0], bms = n[0] * n[1], bfull = n[0] * n[1] * n[2];
        const int64_t wm = (bm + 31) / 32, wms = (bms + 31) / 32, wfull = (bfull + 31) / 32;
        if (b > a && wm + wms + wfull <= SS_BLOB_MAX_BITMAP_WORDS) {
            std::vector<uint32_t> words((size_t)(wm + wms + wfull), 0u);
            auto set = [&](int64_t base, int64_t bit) { words[(size_t)(base + bit / 32)] |= 1u << (bit % 32); };
            for (int64_t i = a; i < b; ++i) {
                const int64_t ms = h_keys[i] / SS_KEY_BASE, mm = ms / SS_KEY_BASE;
                const int64_t im = mm - lo[0], is = ms % SS_KEY_BASE - lo[1], ig = h_keys[i] % SS_KEY_BASE - lo[2];
                set(0, im);
                set(wm, im * n[1] + is);
                set(wm + wms, (im * n[1] + is) * n[2] + ig);
            }
            if (words.size() % 2) words.push_back(0u);
            hd(12) = (int64_t)blob.size();
            hd(13) = wm;
            hd(14) = wms;
            hd(15) = wfull;
            for (size_t i = 0; i < words.size(); i += 2)
                blob.push_back((int64_t)((uint64_t)words[i] | ((uint64_t)words[i + 1] << 32)));
        }
    }
    return SS_OK;
}
}  // namespace ss
extern "C" {


int ss_ladder_keysets(const double* h_feats, int32_t feat_ring_stride, int32_t n_sizes, const int32_t* h_nk,
                      const int32_t* h_n_rings, double q_mean, double q_std, double q_grad, int64_t* h_keys,
                      int64_t keys_cap, int64_t* h_key_off, int64_t* h_blobs, int64_t blobs_cap,
                      int64_t* h_blob_off) {
    if (!h_feats || n_sizes < 0 || n_sizes > SS_MAX_SIZES || !h_nk || !h_n_rings || !h_keys || !h_key_off ||
        !h_blobs || !h_blob_off || feat_ring_stride < 1 || feat_ring_stride > SS_MAX_RINGS) {
        ss::set_error("bad ladder keyset arguments");
        return SS_EINVAL;
    }
    int64_t key_pos = 0, blob_pos = 0, off_pos = 0, inst = 0;
    h_blob_off[0] = 0;
    std::vector<double> feats;
    std::vector<int64_t> blob;
    for (int32_t k = 0; k < n_sizes; ++k) {
        const int32_t nk = h_nk[k], nr = h_n_rings[k];
        if (nk < 0 || nr < 1 || nr > feat_ring_stride) {
            ss::set_error("bad ladder keyset size %d", k);
            return SS_EINVAL;
        }
        // this size's features, rings packed (ss_keys_from_features layout)
        feats.resize((size_t)nk * nr * 3);
        for (int32_t i = 0; i < nk; ++i)
            std::memcpy(&feats[(size_t)i * nr * 3], h_feats + (size_t)(inst + i) * feat_ring_stride * 3,
                        sizeof(double) * 3 * (size_t)nr);
        inst += nk;
        if (key_pos + (int64_t)nr * 27 * nk > keys_cap) {
            ss::set_error("ladder keyset key buffer too small");
            return SS_EINVAL;
        }
        int64_t* off = h_key_off + off_pos;  // nr + 1 offsets relative to this size's first key
        if (int e = ss_keys_from_features(feats.data(), nk, nr, q_mean, q_std, q_grad, h_keys + key_pos, off))
            return e;
        if (int e = ss::build_keyset_blob(h_keys + key_pos, off, nr, blob)) return e;
        const int64_t slots = (int64_t)blob.size();
        if (blob_pos + slots > blobs_cap) {
            ss::set_error("ladder keyset blob buffer too small");
            return SS_EINVAL;
        }
        std::memcpy(h_blobs + blob_pos, blob.data(), (size_t)slots * sizeof(int64_t));
        key_pos += off[nr];
        off_pos += nr + 1;
        blob_pos += slots;
        h_blob_off[k + 1] = blob_pos;
    }
    return SS_OK;
}

}  // extern "C"
