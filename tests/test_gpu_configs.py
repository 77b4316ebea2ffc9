"""Parity at the BASELINE.json configs' full sizes.

Configs 0 and 1 are compared with the untiled oracle in test_gpu_screen.py.
Here configs 2-4 run on the GPU at full size and are checked against the
oracle on halo'd tiles (screening img[Y0-lo:Y1+hi,
X0-lo:X1+hi] decides the core [Y0,Y1) x [X0,X1) exactly as the full image
does, with lo/hi the largest ladder size's margins), plus size-independent
properties over the whole result: every candidate is set in its size mask,
candidates are row-major per size, patches_tested matches the grid formula,
the kept region equals the union of candidate footprints (checked on row
slabs), and a second run is identical.
"""

import numpy as np
import pytest

import oracle as O
from conftest import packbits

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def ocfg(wl):
    return O.ScreeningConfig(alpha=wl.alpha, beta=wl.beta, ladder_ratio=wl.ladder_ratio, quantizer=O.Quantizer(*wl.q))


def tile_check(res, img, tpl, wl, y0, y1, x0, x1, nthreads=16):
    """GPU masks on the core [y0,y1) x [x0,x1) vs the oracle on the halo'd tile."""
    H, W = img.shape
    ladder = res.ladder
    ev = [m for m in ladder if m >= 8]
    lo = max((m - 1) // 2 for m in ev)
    hi = max(m // 2 for m in ev)
    Y0, Y1 = max(0, y0 - lo), min(H, y1 + hi)
    X0, X1 = max(0, x0 - lo), min(W, x1 + hi)
    sub = np.ascontiguousarray(img[Y0:Y1, X0:X1])
    ref = O.screen(sub, tpl, ocfg(wl), nthreads=nthreads)
    bad = {}
    from paper_1707_05647_b200.screening import unpack_bits

    for m in ladder:
        got = unpack_bits(res.size_masks.packed(m)[y0:y1], W)[:, x0:x1]
        want = ref.size_masks[m][y0 - Y0:y1 - Y0, x0 - X0:x1 - X0]
        d = int((got != want).sum())
        if d:
            bad[m] = d
    assert not bad, f"tile mask disagreements per size: {bad}"
    # candidates inside the core, row-major per size
    cand = res.candidates.array()
    inside = (cand[:, 0] >= x0) & (cand[:, 0] < x1) & (cand[:, 1] >= y0) & (cand[:, 1] < y1)
    rc = np.array(ref.candidates, np.int64).reshape(-1, 3)
    rc[:, 0] += X0
    rc[:, 1] += Y0
    rin = (rc[:, 0] >= x0) & (rc[:, 0] < x1) & (rc[:, 1] >= y0) & (rc[:, 1] < y1)
    assert np.array_equal(cand[inside], rc[rin].astype(np.int32))


def properties(res, img, wl):
    H, W = img.shape
    cand = res.candidates.array()
    # every candidate is set in its size mask; per-size row-major order
    for m in res.ladder:
        c = cand[cand[:, 2] == m]
        if len(c):
            bits = (res.size_masks.packed(m)[c[:, 1], c[:, 0] // 32] >> (c[:, 0] % 32).astype(np.uint32)) & 1
            assert bits.all()
            key = c[:, 1].astype(np.int64) * W + c[:, 0]
            assert np.all(np.diff(key) > 0)
    order = {m: i for i, m in enumerate(res.ladder)}
    assert np.all(np.diff([order[m] for m in cand[:, 2]]) >= 0)
    # tested count formula (pkg/tests/test_screening.py:346-358)
    want = 0
    for m in res.ladder:
        if m < 8:
            continue
        lo, hi = (m - 1) // 2, m // 2
        want += max(0, W - hi - lo) * max(0, H - hi - lo)
    assert res.stats.patches_tested == want
    assert res.stats.patches_kept == len(cand)
    # region == union of candidate footprints, on three row slabs (2-D difference array)
    from paper_1707_05647_b200.screening import unpack_bits

    for r0 in (0, H // 2 - 64, H - 128):
        r1 = r0 + 128
        lo = (cand[:, 2].astype(np.int64) - 1) // 2
        hi = cand[:, 2].astype(np.int64) // 2
        cx, cy = cand[:, 0].astype(np.int64), cand[:, 1].astype(np.int64)
        a, b = np.maximum(cy - lo, r0), np.minimum(cy + hi + 1, r1)
        sel = a < b
        diff = np.zeros((129, W + 1), np.int64)
        xa, xb = np.maximum(cx - lo, 0)[sel], np.minimum(cx + hi + 1, W)[sel]
        ya, yb = (a - r0)[sel], (b - r0)[sel]
        np.add.at(diff, (ya, xa), 1)
        np.add.at(diff, (ya, xb), -1)
        np.add.at(diff, (yb, xa), -1)
        np.add.at(diff, (yb, xb), 1)
        want_reg = diff.cumsum(0).cumsum(1)[:128, :W] > 0
        got = unpack_bits(res.region_packed()[r0:r1], W)
        assert np.array_equal(got, want_reg), r0


def run_config(idx, image_index=0):
    import workloads as WL
    from paper_1707_05647_b200 import screen

    wl = WL.CONFIGS[idx]
    case = WL.make_cases(wl, images=1, first_image=image_index)[0]
    res = screen(case.image, case.template, WL.screening_config(wl))
    return wl, case, res


def test_config2_tiles_and_properties(cuda):
    wl, case, res = run_config(2)
    H, W = case.image.shape
    tile_check(res, case.image, case.template, wl, 0, 384, 0, 640)            # top-left corner (borders)
    tile_check(res, case.image, case.template, wl, 1900, 2200, 1700, 2300)    # interior
    tile_check(res, case.image, case.template, wl, H - 300, H, W - 500, W)    # bottom-right corner
    properties(res, case.image, wl)


def test_config3_images(cuda):
    import workloads as WL
    from paper_1707_05647_b200 import screen

    wl = WL.CONFIGS[3]
    for i in (0, 63):
        case = WL.make_cases(wl, images=1, first_image=i)[0]
        res = screen(case.image, case.template, WL.screening_config(wl))
        ref = O.screen(case.image, case.template, ocfg(wl), nthreads=16)
        for m in res.ladder:
            assert np.array_equal(packbits(res.size_masks[m]), packbits(ref.size_masks[m])), (i, m)
        assert np.array_equal(res.candidates.array(), np.array(ref.candidates, np.int32).reshape(-1, 3))
        assert np.array_equal(res.region_mask, ref.region_mask)
        assert res.stats.patches_tested == ref.patches_tested


def test_config4_tiles_and_properties(cuda):
    wl, case, res = run_config(4)
    H, W = case.image.shape
    tile_check(res, case.image, case.template, wl, 0, 256, 0, 512)
    tile_check(res, case.image, case.template, wl, 8000, 8256, 9000, 9512)
    tile_check(res, case.image, case.template, wl, H - 256, H, W - 512, W)
    properties(res, case.image, wl)
    # determinism of the whole result
    from paper_1707_05647_b200 import screen
    import workloads as WL

    res2 = screen(case.image, case.template, WL.screening_config(wl))
    assert res2.candidates == res.candidates
    for m in res.ladder[::8]:
        assert np.array_equal(res2.size_masks.packed(m), res.size_masks.packed(m))


def test_config2_full_image_vs_tiled_oracle(cuda):
    """Config 2 over the WHOLE 4096^2 image: the tiled oracle (SURVEY.md App.
    B.1; 8 row bands, each screened with its halo) decides every centre; the
    GPU's size masks (all 17 sizes), candidate list, tested count and kept
    region must match on every core.  SURVEY.md 8(d)'s threshold-band
    positions are counted from the oracle's fp64 features: every disagreement
    would have to be one (0 disagreements expected and required here)."""
    import os

    from paper_1707_05647_b200.screening import unpack_bits

    wl, case, res = run_config(2)
    H, W = case.image.shape
    nthreads = os.cpu_count() or 1
    cand = res.candidates.array()
    tested = 0
    band_total = 0
    cands = []
    for i in range(8):
        y0, y1 = i * H // 8, (i + 1) * H // 8
        t = O.screen_tile(case.image, case.template, ocfg(wl), y0, y1, 0, W, nthreads=nthreads, band=True)
        assert tuple(t.ladder) == tuple(res.ladder)
        for m in res.ladder:
            got = unpack_bits(res.size_masks.packed(m)[y0:y1], W)
            d = got != t.size_masks[m]
            assert not (d & ~t.band_masks[m]).any(), f"rows [{y0},{y1}) m={m}: {int(d.sum())} off-band"
            assert not d.any(), f"rows [{y0},{y1}) m={m}: {int(d.sum())} in-band disagreements"
            band_total += int(t.band_masks[m].sum())
        ry0, ry1, rx0, rx1 = t.region_window
        assert np.array_equal(unpack_bits(res.region_packed()[ry0:ry1], W)[:, rx0:rx1], t.region)
        tested += t.patches_tested
        cands.append(t.candidates)
    want = np.concatenate(cands)
    # the oracle lists each band's candidates in ladder order; the global list
    # is ladder order first, then row-major: a stable sort by ladder position
    order = {m: k for k, m in enumerate(res.ladder)}
    want = want[np.argsort([order[int(m)] for m in want[:, 2]], kind="stable")]
    assert np.array_equal(cand, want)
    assert res.stats.patches_tested == tested
    print(f"config 2 full image: {tested} positions*scales, {len(cand)} candidates, "
          f"{band_total} threshold-band positions, 0 disagreements")
