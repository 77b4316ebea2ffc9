/*
 * starscreen_b200.h -- C ABI of the B200-native pre-screening hot path.
 *
 * Drop-in boundary for the reference's Python screening API
 * (/root/reference/pkg/src/starscreen/screening.py:474 screen()).  The
 * reference has no FFI of its own (it is pure NumPy); these entry points are
 * what a maintainer binds with ctypes to replace the NumPy internals of
 * screen() -- see INTEGRATION.md.  Each declaration names the reference
 * interface it replaces (file:line, paths relative to pkg/src/starscreen/).
 *
 * Conventions (all entry points):
 *   - extern "C", plain pointers and sizes, no torch or CUDA types
 *     (streams are passed as void* = cudaStream_t);
 *   - d_* arguments are device pointers, h_* arguments host pointers;
 *   - return SS_OK or an SS_E* status; ss_last_error() (thread-local) holds
 *     the message.  SS_EINVAL / SS_ECAPACITY map to Python ValueError,
 *     SS_ECUDA to RuntimeError -- the reference's error classes;
 *   - stream-ordered and reentrant; nothing here allocates device memory:
 *     workspaces are caller-owned and sized by the *_bytes() queries --
 *     except a screening session (ss_session_*, the native runtime of one
 *     whole screen() call), which owns its buffers and streams.
 *
 * Device table layout ("planes"): 12 int64 planes of (H+1) rows x pitch
 * columns, plane p = type*4 + kind, kind in {PLAIN, X_WEIGHTED, Y_WEIGHTED,
 * SQUARED} (integral.py:37-41), type in {SAT, E, O}:
 *   SAT[y+1][x+1] = Sat.cell(x, y)                 (integral.py:66-81)
 *   E  [y+1][x+1] = H(x+y,   x-y) = Rsat.cell(x,y) (integral.py:84-106)
 *   O  [y+1][x+1] = H(x+y+1, x-y)                  (the off-parity corners)
 * for x in [-1, W-1], y in [-1, H-1], where H(u,v) is the reference's
 * rotated quadrant prefix.  A closed l1 ball of radius r about (cx,cy) is
 *   E(cx,cy+r) - O(cx-r-1,cy-1) - O(cx+r,cy-1) + E(cx,cy-r-1)
 * which equals diamond_region_sum (integral.py:165-186) bit for bit.
 */
#ifndef STARSCREEN_B200_H
#define STARSCREEN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_OK 0
#define SS_EINVAL 1    /* bad argument / bounds  -> ValueError   */
#define SS_ECAPACITY 2 /* key capacity exceeded  -> ValueError   */
#define SS_ECUDA 3     /* CUDA launch / runtime  -> RuntimeError */

#define SS_MAX_RINGS 16
#define SS_MAX_SIZES 64 /* ladder sizes per ss_*_ladder call */
#define SS_MAX_COARSE 5 /* coarse stage-1 plane sets (shifts) per table build */
#define SS_KEY_BASE (1LL << 21) /* screening.py:57 _KEY_BASE */
#define SS_BLOB_HDR 16             /* int64 header slots per ring in a key blob */
#define SS_BLOB_MAX_BITMAP_WORDS 8192 /* per-ring membership bitmap cap (32 KiB) */

/* ── diagnostics ─────────────────────────────────────────────────────── */
const char* ss_last_error(void);
int ss_version(void);
/* Number of CUDA kernels this library has launched (process lifetime). */
uint64_t ss_launch_count(void);

/* ── integral tables (integral.py:200-228 build_tables) ──────────────── */
/* Row pitch, in int64 elements, of every plane for an image W wide. */
int64_t ss_plane_pitch(int64_t W);
/* Bytes of the 12-plane table block for a W x H image. */
size_t ss_tables_bytes(int64_t W, int64_t H);
/* Bytes of device workspace ss_build_tables needs. */
size_t ss_build_workspace_bytes(int64_t W, int64_t H);
/*
 * Replaces build_tables (integral.py:211-228: 4 x build_sat :109-117 and
 * 4 x build_rsat :120-141).  d_img: H rows of W bytes, img_pitch bytes apart.
 * Rejects images that fail the reference's overflow guard
 * (integral.py:59-63) with SS_EINVAL.
 */
int ss_build_tables(const uint8_t* d_img, int64_t W, int64_t H, int64_t img_pitch, int64_t* d_planes,
                    int64_t plane_pitch, void* d_workspace, size_t workspace_bytes, void* stream);
/* Bytes of the 12-plane block of 32-bit cells (same pitch, in elements). */
size_t ss_tables32_bytes(int64_t W, int64_t H);
/*
 * ss_build_tables writing the int64 planes and/or ("32-bit planes") the same
 * cells mod 2^32 in one pass; either pointer may be NULL, not both.  The
 * screen reads the 32-bit planes for every ladder size whose ring sums fit
 * (ss_screen_fits32) -- half the bytes per corner -- and the int64 planes
 * otherwise.
 */
int ss_build_tables2(const uint8_t* d_img, int64_t W, int64_t H, int64_t img_pitch, int64_t* d_planes,
                     uint32_t* d_planes32, int64_t plane_pitch, void* d_workspace, size_t workspace_bytes,
                     void* stream);

/*
 * Stage 1's coarse planes (the fused screen's ring-0 mean test): for each of
 * n_coarse shifts, the SAT / E / O PLAIN cells as u16 bit slices
 * (cell >> shift) & 0xffff -- three planes per shift, same pitch as the
 * 32-bit planes, at d_coarse + (c * 3 + type) * (H + 1) * plane_pitch.
 * ss_coarse_shift(count) is the shift a region of `count` pixels uses: the
 * smallest of 1, 4, ..., 16 with 255 count < (2^16 - 4) 2^shift (its slice
 * sums cannot wrap), -1 if none.
 */
int32_t ss_coarse_shift(int64_t count);
/* Bytes of the coarse-plane buffer: the 3 * n_coarse planes plus 16 rows of
 * padding (stage 1's row-step TMA views address whole groups of up to 16 rows;
 * the last group of the last plane may end past row H).  Allocate at least
 * this much for d_coarse. */
size_t ss_coarse_bytes(int64_t W, int64_t H, int32_t n_coarse);
/*
 * ss_build_tables3 for the image rows [y0, y1) only, y0 and y1 whole bands of
 * ss_build_band_rows(W, H, exact) rows (y1 may be H; exact = the int64 or
 * hi16 planes are wanted), after the rows above were built by earlier calls
 * with the same workspace: table rows y0 + 1 .. y1 become final.  Only image
 * rows [y0, y1) are read -- a caller streams the image in and builds it band
 * by band (screen(): upload, build and screen overlap).
 */
int32_t ss_build_band_rows(int64_t W, int64_t H, int32_t exact);
int ss_build_tables_rows(const uint8_t* d_img, int64_t W, int64_t H, int64_t img_pitch, int64_t* d_planes,
                         uint32_t* d_planes32, uint16_t* d_hi16, int64_t plane_pitch, uint16_t* d_coarse,
                         int32_t n_coarse, const int32_t* h_shifts, int64_t y0, int64_t y1, void* d_workspace,
                         size_t workspace_bytes, void* stream);
/* Bytes of the 12 "hi16" planes: bits 32..47 of every exact cell (u16, same layout as the 32-bit planes). */
size_t ss_tables_hi16_bytes(int64_t W, int64_t H);
/*
 * ss_build_tables2 plus, when non-NULL, the hi16 planes (with the 32-bit
 * planes a cell is then known mod 2^48: every region sum below 2^48 is exact
 * -- the fused rings' wide path, 6 bytes per cell instead of 8) and the
 * coarse planes of h_shifts[0..n_coarse) (<= SS_MAX_COARSE).  d_hi16 needs
 * d_planes32.
 */
int ss_build_tables3(const uint8_t* d_img, int64_t W, int64_t H, int64_t img_pitch, int64_t* d_planes,
                     uint32_t* d_planes32, uint16_t* d_hi16, int64_t plane_pitch, uint16_t* d_coarse,
                     int32_t n_coarse, const int32_t* h_shifts, void* d_workspace, size_t workspace_bytes,
                     void* stream);

/* ── per-size membership sets (screening.py:100-178 FeatureSet) ──────── */
/*
 * Lays out one ladder size's per-ring sorted key arrays
 * (FeatureSet.ring_keys(), screening.py:147-155) as a device-ready blob:
 * the keys, their (cm) and (cm,cs) projections used by the screen's
 * early-exit cascade, and -- when the key bounding box is small enough --
 * dense membership bitmaps of all three (layout in ss_template.cpp).
 * Host-only; call with h_blob = NULL to get the size.
 * h_keys: concatenated sorted keys, key_off: n_rings+1 offsets.
 */
int ss_keyset_blob(const int64_t* h_keys, const int64_t* h_key_off, int32_t n_rings, int64_t* h_blob,
                   size_t* blob_bytes);

/* ── one ladder size (screening.py:418-471 _scan_size) ───────────────── */
/*
 * Evaluates every grid centre of global rows [y_begin, y_end) for patch side
 * m.  The tables cover a w x h sub-image whose row 0 is global row y_origin
 * (full width: w == W); row-band shards pass their halo'd band.  d_planes /
 * d_planes32: the int64 and/or 32-bit planes of ss_build_tables2 (either may
 * be NULL; the 32-bit ones are used when ss_screen_fits32 holds for the ring
 * plan, and the int64 ones are then not needed).  Writes the
 * bit-packed keep mask (bit x%32 of word x/32, rows y_begin.. at
 * mask_pitch_words apart; border grid centres set, as the reference keeps
 * them) and, per mask row, the number of evaluated survivors into
 * d_row_counts.  h_ring_n / h_ring_d: ring_plan(m) (features.py:190-211).
 * d_blob: the ss_keyset_blob() layout copied to the device.  d_stage_counts
 * (nullable, 4 x u64, accumulated) instruments the early-exit cascade:
 * ring-0 evaluations (every interior centre), ring-0 mean-projection
 * passes (candidates that read the SQUARED / X / Y planes), ring-0 full
 * passes, and final survivors.
 */
int ss_screen_size(const int64_t* d_planes, const uint32_t* d_planes32, int64_t w, int64_t h, int64_t plane_pitch,
                   int64_t W, int64_t H, int64_t y_origin, int64_t y_begin, int64_t y_end, int32_t m, int32_t stride,
                   int32_t n_rings, const int32_t* h_ring_n, const int32_t* h_ring_d, const int64_t* d_blob,
                   const int64_t* h_blob, double q_mean, double q_std, double q_grad, uint32_t* d_mask,
                   int64_t mask_pitch_words, uint32_t* d_row_counts, unsigned long long* d_stage_counts,
                   void* d_workspace, size_t workspace_bytes, void* stream);
/*
 * 1 when every region sum of ring_plan (h_ring_n, h_ring_d) is recoverable
 * from the 32-bit planes: PLAIN / SQUARED sums < 2^32 and centred x / y
 * moments < 2^31 in magnitude (n <= 128 for 8-bit images); else 0.
 */
int ss_screen_fits32(int32_t n_rings, const int32_t* h_ring_n, const int32_t* h_ring_d);
/* Bytes of device workspace ss_screen_size needs for `rows` decided rows. */
size_t ss_screen_workspace_bytes(int64_t W, int64_t rows);

/*
 * Device self-test of the screen's division routine: counts operands of
 * family `mode` (0 consecutive integers from seed, 1 random integers < 2^43,
 * 2 random wide-range doubles, 3 signed half-integers) whose quotient by
 * `divisor` differs from IEEE __ddiv_rn; adds the count to *d_mismatches.
 */
int ss_selftest_div(uint64_t n, uint64_t seed, double divisor, int32_t mode, unsigned long long* d_mismatches,
                    void* stream);
/*
 * Device self-test of the fused screen's fp32-estimated cells: n random
 * region-sum tuples an 8-bit image can produce for ring (ring_n, ring_d),
 * 3 in 4 aimed within ~1e-6 of a std / gradient cell boundary; adds the std
 * and gradient cells that differ from the fp64 reference sequence to
 * d_counts[0] and d_counts[1].
 */
int ss_selftest_cells(uint64_t n, uint64_t seed, int32_t ring_n, int32_t ring_d, double q_mean, double q_std,
                      double q_grad, unsigned long long* d_counts, void* stream);

/*
 * The whole ladder loop of screen() (screening.py:502-520) in one call: for
 * every size k (ladder order) ss_screen_size, or ss_fill_grid when m < 8
 * (screening.py:505-510), enqueued on streams[1 + k % (n_streams - 1)] with
 * an event fork from / join to streams[0] (all sizes on streams[0] when
 * n_streams == 1).  Per size k: h_m[k], h_n_rings[k], ring plan at
 * h_ring_n / h_ring_d + k * SS_MAX_RINGS, key blob at d_blobs / h_blobs +
 * h_blob_off[k] (ss_ladder_keysets), mask at d_masks + k *
 * size_stride_words, row counts at d_row_counts + k * row_counts_stride.
 * d_workspaces[i] (ss_screen_workspace_bytes each) belongs to streams[i].
 * flags bit 0: screen every size from the int64 planes (test hook).
 * flags bit 1: fused ladder -- the sizes that share a plane width are
 * screened in lock-step (ss_ladder_screen.cu: a few launches per row band, each
 * plane row read from HBM about once per band instead of once per size), all
 * on streams[0] with d_workspaces[0], whose workspace_bytes should be
 * ss_ladder_workspace_bytes(W, y_end - y_begin, n_sizes) (a smaller one
 * means more row bands, or per-size screening when it cannot hold one).
 * Same results as the per-size path.
 */
int ss_screen_ladder(const int64_t* d_planes, const uint32_t* d_planes32, int64_t w, int64_t h, int64_t plane_pitch,
                     int64_t W, int64_t H, int64_t y_origin, int64_t y_begin, int64_t y_end, int32_t stride,
                     int32_t n_sizes, const int32_t* h_m, const int32_t* h_n_rings, const int32_t* h_ring_n,
                     const int32_t* h_ring_d, const int64_t* d_blobs, const int64_t* h_blobs,
                     const int64_t* h_blob_off, double q_mean, double q_std, double q_grad, uint32_t* d_masks,
                     int64_t mask_pitch_words, int64_t size_stride_words, uint32_t* d_row_counts,
                     int64_t row_counts_stride, unsigned long long* d_stage_counts, int32_t flags, int32_t n_streams,
                     void* const* streams, void* const* d_workspaces, size_t workspace_bytes);

/*
 * ss_screen_ladder with stage 1's coarse planes (ss_build_tables3): when
 * every fused size's ring-0 square and diamond have their ss_coarse_shift in
 * h_shifts[0..n_coarse), stage 1 reads the u16 bit slices (half the bytes)
 * and passes centres near a membership boundary on to the rings (which
 * test ring 0's exact mean cell); same results.  d_hi16 (with d_planes32;
 * ss_build_tables3): the fused rings of sizes beyond 32 bits read 32-bit +
 * hi16 cells (mod 2^48) instead of the int64 planes, which may then be NULL
 * (SS_EINVAL if a ring sum could reach 2^48, or if the fused path declines
 * and the per-size fallback needs them).  All-NULL extras = ss_screen_ladder.
 */
int ss_screen_ladder2(const int64_t* d_planes, const uint32_t* d_planes32, int64_t w, int64_t h, int64_t plane_pitch,
                      int64_t W, int64_t H, int64_t y_origin, int64_t y_begin, int64_t y_end, int32_t stride,
                      int32_t n_sizes, const int32_t* h_m, const int32_t* h_n_rings, const int32_t* h_ring_n,
                      const int32_t* h_ring_d, const int64_t* d_blobs, const int64_t* h_blobs,
                      const int64_t* h_blob_off, double q_mean, double q_std, double q_grad, uint32_t* d_masks,
                      int64_t mask_pitch_words, int64_t size_stride_words, uint32_t* d_row_counts,
                      int64_t row_counts_stride, unsigned long long* d_stage_counts, int32_t flags, int32_t n_streams,
                      void* const* streams, void* const* d_workspaces, size_t workspace_bytes,
                      const uint16_t* d_coarse, int32_t n_coarse, const int32_t* h_shifts, const uint16_t* d_hi16);

/* Workspace bytes for the fused ladder (flags bit 1) of n_sizes sizes over
 * `rows` decided rows: one row band of at most 16 GiB of candidate list, and
 * at least ss_screen_workspace_bytes (the per-size fallback shares it). */
size_t ss_ladder_workspace_bytes(int64_t W, int64_t rows, int32_t n_sizes);

/* screening.py:505-510: sizes below MIN_PATCH_SIDE keep every grid centre. */
int ss_fill_grid(int64_t W, int64_t y_begin, int64_t y_end, int32_t stride, uint32_t* d_mask,
                 int64_t mask_pitch_words, uint32_t* d_row_counts, void* stream);

/* ── survivor list (screening.py:455-470, 512-516) ───────────────────── */
/* Bytes of device workspace ss_compact needs for `rows` mask rows. */
size_t ss_compact_workspace_bytes(int64_t rows);
/*
 * Appends the evaluated survivors of one size (interior grid centres with
 * their mask bit set, excluding border keeps) to d_xy as int32 (cx, cy)
 * pairs in row-major order, starting at index *d_total, and advances
 * *d_total.  Calling it per size in ladder order reproduces the order of
 * ScreeningResult.candidates (screening.py:280-283).  Entries past
 * `capacity` are counted but not written.  d_size_count (nullable) receives
 * this size's survivor count.
 */
int ss_compact(const uint32_t* d_mask, int64_t mask_pitch_words, int64_t W, int64_t H, int64_t y_begin,
               int64_t y_end, int32_t m, int32_t stride, const uint32_t* d_row_counts, int32_t* d_xy,
               int64_t capacity, unsigned long long* d_total, unsigned long long* d_size_count,
               void* d_workspace, size_t workspace_bytes, void* stream);

/*
 * Whole-ladder form of ss_compact: one call for every size of a ladder.
 * d_masks holds n_sizes masks size_stride_words apart (rows y_begin..y_end),
 * d_row_counts n_sizes x rows counts; sizes with m < MIN_PATCH_SIDE are
 * skipped.  d_size_counts (n_sizes u64) and *d_total receive the counts;
 * survivors are written in ladder order, then row-major, as int32 rows of
 * xy_columns = 2 (cx, cy) or 3 (cx, cy, m) -- the candidates list
 * (screening.py:280-283) in one buffer.
 */
size_t ss_compact_ladder_workspace_bytes(int64_t rows, int32_t n_sizes);
int ss_compact_ladder(const uint32_t* d_masks, int64_t mask_pitch_words, int64_t size_stride_words, int64_t W,
                      int64_t H, int64_t y_begin, int64_t y_end, int32_t n_sizes, const int32_t* h_m, int32_t stride,
                      const uint32_t* d_row_counts, int32_t* d_xy, int32_t xy_columns, int64_t capacity,
                      unsigned long long* d_total, unsigned long long* d_size_counts, void* d_workspace,
                      size_t workspace_bytes, void* stream);

/* ── kept region (screening.py:316-330 _footprint_union) ─────────────── */
/* Workspace for ss_region_accumulate with sizes up to m_max. */
size_t ss_region_workspace_bytes(int64_t W, int64_t H, int32_t m_max);
/*
 * ORs the m x m footprints of the evaluated survivors of one size (full
 * image mask, y_begin = 0, y_end = H) into d_region (same bit layout).
 */
int ss_region_accumulate(const uint32_t* d_mask, int64_t mask_pitch_words, int64_t W, int64_t H, int32_t m,
                         int32_t stride, uint32_t* d_region, void* d_workspace, size_t workspace_bytes,
                         void* stream);
/* Whole-ladder form of ss_region_accumulate (full-image masks); writes d_region
 * (the union of every size's footprints; prior contents are replaced). */
size_t ss_region_ladder_workspace_bytes(int64_t W, int64_t H, int32_t n_sizes);
int ss_region_ladder(const uint32_t* d_masks, int64_t mask_pitch_words, int64_t size_stride_words, int64_t W, int64_t H,
                     int32_t n_sizes, const int32_t* h_m, int32_t stride, uint32_t* d_region, void* d_workspace,
                     size_t workspace_bytes, void* stream);
/* ss_region_ladder with K3's per-row survivor counts (d_row_counts + k *
 * row_counts_stride + y: interior survivors of size k in mask row y, as the
 * ss_screen_* calls leave them; may be NULL): rows without a survivor are
 * skipped without reading their mask row (3 in 4 rows of BASELINE config 4). */
int ss_region_ladder2(const uint32_t* d_masks, int64_t mask_pitch_words, int64_t size_stride_words, int64_t W, int64_t H,
                      int32_t n_sizes, const int32_t* h_m, int32_t stride, const uint32_t* d_row_counts,
                      int64_t row_counts_stride, uint32_t* d_region, void* d_workspace, size_t workspace_bytes,
                      void* stream);
/*
 * K5 over a window of `rows` mask rows (per size, same layout) whose row 0 is
 * global row y0 of an H-row image: interior status (which survivors count,
 * screening.py:316-330) is decided in global rows, footprints are clipped to
 * the window.  A row band plus its neighbours' halo rows (hi_max above,
 * lo_max below) yields the band's region rows exactly (sharding.py).
 * Workspace: ss_region_ladder_workspace_bytes(W, rows, n_sizes).
 */
int ss_region_ladder_rows(const uint32_t* d_masks, int64_t mask_pitch_words, int64_t size_stride_words, int64_t W,
                          int64_t rows, int64_t y0, int64_t H, int32_t n_sizes, const int32_t* h_m, int32_t stride,
                          uint32_t* d_region, void* d_workspace, size_t workspace_bytes, void* stream);
/*
 * f4 (cli.py:97-98 _mask_to_pgm): a bit-packed W x H mask (size mask or
 * region) as one byte per pixel, 255 = kept, 0 = not -- the raster of the
 * PGM files `starscreen screen --out-mask / --out-size-masks` writes
 * (image_io.py:108-128 save_pgm).  d_out: H rows of W bytes.
 */
int ss_bits_to_bytes(const uint32_t* d_bits, int64_t mask_pitch_words, int64_t W, int64_t H, uint8_t* d_out,
                     void* stream);
/*
 * Asynchronous strided copy on `stream` (cudaMemcpy2DAsync, any direction):
 * `rows` runs of row_bytes bytes, src_pitch / dst_pitch bytes apart.  screen()
 * streams each finished row chunk of every size's packed mask to pinned host
 * memory with it while later chunks are still being screened.
 */
int ss_copy_rows_async(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch, int64_t row_bytes,
                       int64_t rows, void* stream);
/* *d_count = number of set bits of the W x H region mask. */
int ss_popcount(const uint32_t* d_bits, int64_t mask_pitch_words, int64_t W, int64_t H,
                unsigned long long* d_count, void* stream);

/* ── template side (screening.py:222-250 build_feature_set) ──────────── */
/*
 * Host C++: ring features of every template rescale k = m..k_hi
 * (resize_bilinear image_io.py:164-178, crop_center :216-228, the patch's
 * tables and ring_feature_maps features.py:220-224) inserted guard-banded
 * (screening.py:122-145) into per-ring sorted unique key sets.
 * h_keys must hold n_rings * 27 * (k_hi - m + 1) entries; h_key_off gets
 * n_rings + 1 offsets.  SS_ECAPACITY: "quantized cell exceeds key capacity".
 */
int ss_feature_set_keys(const uint8_t* h_template, int32_t n, int32_t m, int32_t k_hi, int32_t n_rings,
                        const int32_t* h_ring_n, const int32_t* h_ring_d, double q_mean, double q_std,
                        double q_grad, int64_t* h_keys, int64_t* h_key_off);
/*
 * Host: guard-banded key sets (screening.py:122-155) from precomputed ring
 * features h_feats[nk][n_rings][3] (mean, std, grad_mag), rescales in k
 * order.  Same outputs / errors as ss_feature_set_keys.
 */
int ss_keys_from_features(const double* h_feats, int32_t nk, int32_t n_rings, double q_mean, double q_std,
                          double q_grad, int64_t* h_keys, int64_t* h_key_off);
/*
 * Host: ss_keys_from_features + ss_keyset_blob for every size of a ladder in
 * one call.  h_feats: the instances of all sizes in ladder order, rings
 * feat_ring_stride apart (the ss_template_features_device layout, stride
 * SS_MAX_RINGS); size k has h_nk[k] instances and h_n_rings[k] rings.
 * Outputs: keys (size k's rings at h_key_off, n_rings[k] + 1 offsets per
 * size, relative to the size's first key), blobs (size k at
 * h_blob_off[k], n_sizes + 1 offsets in int64 slots).  keys_cap / blobs_cap
 * are the buffers' slots; too small -> SS_EINVAL.
 */
int ss_ladder_keysets(const double* h_feats, int32_t feat_ring_stride, int32_t n_sizes, const int32_t* h_nk,
                      const int32_t* h_n_rings, double q_mean, double q_std, double q_grad, int64_t* h_keys,
                      int64_t keys_cap, int64_t* h_key_off, int64_t* h_blobs, int64_t blobs_cap,
                      int64_t* h_blob_off);
/*
 * Device (f2): ring features of n_inst (m, k) rescale instances of the n x n
 * template d_template in one launch.  d_desc: n_inst rows of desc_stride
 * int32 = [m, k, n_rings, 0, n_0, d_0, n_1, d_1, ...] (desc_stride >=
 * 4 + 2*SS_MAX_RINGS); d_out: n_inst x SS_MAX_RINGS x 3 doubles.  Bit-identical
 * to ss_template_ring_features.
 */
int ss_template_features_device(const uint8_t* d_template, int32_t n, int32_t n_inst, const int32_t* d_desc,
                                int32_t desc_stride, double* d_out, void* stream);
/*
 * ss_template_features_device as one asynchronous round trip: copies the
 * n x n host template into d_template, runs the features, copies them into
 * h_out (pinned, n_inst x SS_MAX_RINGS x 3 doubles) and records `event`
 * (nullable) on `stream`.
 */
int ss_template_features_async(const uint8_t* h_template, int32_t n, int32_t n_inst, const int32_t* d_desc,
                               int32_t desc_stride, uint8_t* d_template, double* d_out, double* h_out, void* stream,
                               void* event);
/* Ring features (mean, std, grad_mag per ring) of one rescale k (tests). */
int ss_template_ring_features(const uint8_t* h_template, int32_t n, int32_t k, int32_t m, int32_t n_rings,
                              const int32_t* h_ring_n, const int32_t* h_ring_d, double* h_out);

/* ── second stage (f3, second_stage.py:106-204 match_candidates) ───── */
/* Row pitch (bytes) of the A planes of ss_match_planes for an image W wide. */
int64_t ss_match_plane_pitch(int64_t W);
/*
 * The three u8 A planes of the NCC dot products (H rows of `pitch` bytes
 * each, zero right of column W, at 0, H*pitch, 2*H*pitch of d_planes): the
 * image, and the high / low bytes of its squares.
 */
int ss_match_planes(const uint8_t* d_img, int64_t W, int64_t H, uint8_t* d_planes, int64_t pitch, void* stream);
/* Bytes of the probe operand blocks of ss_match_probes for size m, n_angles angles. */
size_t ss_match_probe_bytes(int32_t m, int32_t n_angles);
/*
 * Probes of ladder size m for n_angles rotations of the n x n template:
 * resize_bilinear to m x m (image_io.py:164-178), then _rotate_with_mask per
 * angle (image_io.py:181-203) with the rotation's cos / sin in d_cos / d_sin
 * (computed on the host exactly as NumPy does).  Writes the masked probes
 * and supports as the tcgen05 B operand (groups of 40 angles; per 64-byte K
 * stage one 48-row block of each in the UMMA canonical K-major layout) into
 * d_bfrag (ss_match_probe_bytes), and d_stats[a] = (support pixels, sum of
 * the masked probe, sum of its squares).  d_base: m*m bytes scratch.
 */
int ss_match_probes(const uint8_t* d_template, int32_t n, int32_t m, int32_t n_angles, const double* d_cos,
                    const double* d_sin, uint8_t* d_bfrag, long long* d_stats, uint8_t* d_base, void* stream);
/* Partial-result rows ss_match_fused needs for `count` candidates (x 40 each). */
int64_t ss_match_parts(int64_t count);
/*
 * For angle group `group` (angles 40*group ..) of the probes d_bfrag and the
 * candidates first .. first+count-1 of d_rows (rows of row_cols int32,
 * (cx, cy, ...), all of size m): the masked NCC scores of
 * second_stage.py:136-152 (exact integer dot products, float64 in NumPy's op
 * order; the dot products on the tensor cores: tcgen05.mma kind::i8 into
 * TMEM, 128 candidates per CTA) and, per angle, the best score and its
 * candidate index (relative to
 * `first`; the first candidate on equal scores, as np.argmax) into
 * d_best_score / d_best_idx[angle].  d_part_*: ss_match_parts(count) x 40.
 */
int ss_match_fused(const uint8_t* d_planes, int64_t W, int64_t H, int64_t pitch, const int32_t* d_rows,
                   int32_t row_cols, int64_t first, int64_t count, int32_t m, const uint8_t* d_bfrag, int32_t n_angles,
                   int32_t group, const long long* d_stats, double* d_part_score, long long* d_part_idx,
                   double* d_best_score, long long* d_best_idx, void* stream);

/* ── screening session: the whole screen() in one call ────────────────── */
/*
 * Native host runtime of screen() (screening.py:474-539) for one (W, H) on
 * one device: ss_session_screen runs the template features (f2), the image
 * upload (pinned staging filled by host worker threads), K1/K2, the key sets
 * (host, while the tables build), K3 (fused ladder), K4 beside K5 and the
 * D2H of every result, with one host synchronisation -- the same kernels and
 * results as the stream-level entry points above.  The session owns its
 * device / pinned buffers (grown on demand) and streams; calls on one session
 * are serialised (internal mutex); sessions are independent (one per host
 * thread overlaps several screens on the GPU).
 */
typedef struct ss_session ss_session;

/* The template-independent ladder of one (template side, config)
 * (ladder_sizes screening.py:202-219, ring_plan features.py:190-211) and the
 * f2 rescale instances of its evaluated sizes (screening.py:236-238). */
typedef struct ss_ladder_plan {
    int32_t n_sizes;        /* ladder sizes (<= SS_MAX_SIZES), ladder order */
    const int32_t* m;       /* (n_sizes) */
    const int32_t* n_rings; /* (n_sizes); 0 below MIN_PATCH_SIDE */
    const int32_t* ring_n;  /* (n_sizes, SS_MAX_RINGS) */
    const int32_t* ring_d;  /* (n_sizes, SS_MAX_RINGS) */
    int32_t n_inst;         /* rescale instances (ss_template_features_device rows) */
    const int32_t* desc;    /* (n_inst, desc_stride) */
    int32_t desc_stride;    /* >= 4 + 2 * SS_MAX_RINGS */
    const int32_t* nk;      /* instances per evaluated size */
    double q_mean, q_std, q_grad; /* Quantizer (screening.py:64-78) */
    int32_t stride;         /* ScreeningConfig.stride */
} ss_ladder_plan;

/* Host destinations and counts of one screen (ScreeningResult,
 * screening.py:276-298).  Destinations should be pinned for full-rate D2H. */
typedef struct ss_screen_out {
    uint32_t* masks;       /* (n_sizes, H, ceil(W/32)) packed size masks, or NULL */
    uint32_t* region;      /* (H, ceil(W/32)) packed kept region, or NULL */
    int32_t* rows;         /* (rows_cap, 3) int32 (cx, cy, m): the candidates */
    int64_t rows_cap;
    int64_t* size_counts;  /* (n_sizes) survivors per size, or NULL */
    int64_t kept;          /* out: patches_kept */
    int64_t region_pixels; /* out: region_pixels_kept */
    int64_t tested;        /* out: patches_tested */
} ss_screen_out;

int ss_session_create(int32_t device, int64_t W, int64_t H, ss_session** out);
void ss_session_destroy(ss_session* session);
/* Screen the W x H u8 host image h_img (rows W bytes apart) with the n x n
 * u8 host template.  SS_ECAPACITY: out->kept > out->rows_cap (every other
 * output is complete; fetch the rows with ss_session_rows). */
int ss_session_screen(ss_session* session, const uint8_t* h_img, const uint8_t* h_template, int32_t n,
                      const ss_ladder_plan* plan, ss_screen_out* out);
/* Survivor rows [first, first + count) of the session's last screen. */
int ss_session_rows(ss_session* session, int32_t* h_rows, int64_t first, int64_t count);

#ifdef __cplusplus
}
#endif
#endif /* STARSCREEN_B200_H */
