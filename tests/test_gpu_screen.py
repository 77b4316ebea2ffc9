"""K3/K4/K5 parity through the drop-in screen(): masks, candidates, region, stats.

Expected values come from the reference (tests/golden/screens.npz,
report_cases.npz) and, at BASELINE sizes, from the pinned oracle run on the
same seeded inputs in the same process.  The bar is bit-exact: masks,
candidate lists and counts must be identical (the fp64 feature path
replays NumPy's op order, so no threshold-band disagreements are expected;
any would be reported by the band test below).
"""

import numpy as np
import pytest

import oracle as O
from conftest import golden, load_screen_case, packbits, screen_case_names

pytestmark = pytest.mark.gpu


def pcfg(kw):
    from paper_1707_05647_b200 import Quantizer, ScreeningConfig

    kw = dict(kw)
    if "quantizer" in kw:
        kw["quantizer"] = Quantizer(*kw["quantizer"])
    return ScreeningConfig(**kw)


def ocfg(kw):
    kw = dict(kw)
    if "quantizer" in kw:
        kw["quantizer"] = O.Quantizer(*kw["quantizer"])
    return O.ScreeningConfig(**kw)


def assert_same_as_golden(res, c):
    assert tuple(res.ladder) == c["ladder"]
    assert np.array_equal(res.candidates.array().reshape(-1, 3), c["candidates"])
    for m in res.ladder:
        assert np.array_equal(packbits(res.size_masks[m]), c["masks"][m]), f"mask m={m}"
    assert np.array_equal(packbits(res.region_mask), c["region"])
    st = res.stats
    assert (st.patches_tested, st.patches_kept, st.region_pixels_kept, st.total_pixels) == tuple(
        int(v) for v in c["stats"])


@pytest.mark.parametrize("name", screen_case_names())
def test_screen_matches_reference(cuda, name):
    from paper_1707_05647_b200 import screen

    c = load_screen_case(name)
    res = screen(c["image"], c["template"], pcfg(c["cfg"]))
    assert_same_as_golden(res, c)


def test_report_json_cases(cuda):
    """The 12 stored survivor counts of pkg/demos/out/report.json."""
    from paper_1707_05647_b200 import ScreeningConfig, screen

    z = golden("report_cases.npz")
    for i in range(int(z["n"])):
        img_idx, cands, tested, region = (int(v) for v in z[f"expect{i}"])
        res = screen(z[f"scene{img_idx}"], z[f"tpl{i}"], ScreeningConfig())
        assert len(res.candidates) == cands == res.stats.patches_kept
        assert res.stats.patches_tested == tested
        assert res.stats.region_pixels_kept == region
        pp, rp = z[f"pruning{i}"]
        assert res.stats.patch_pruning == pp and res.stats.region_pruning == rp


def compare_with_oracle(img, tpl, kw, nthreads=16):
    from paper_1707_05647_b200 import screen

    res = screen(img, tpl, pcfg(kw))
    ref = O.screen(img, tpl, ocfg(kw), nthreads=nthreads, band=True)
    assert tuple(res.ladder) == tuple(ref.ladder)
    mism, off_band, band = {}, 0, 0
    for m in res.ladder:
        d = res.size_masks[m] != ref.size_masks[m]
        b = ref.band_masks.get(m)
        if b is not None:  # threshold-band positions, counted
            band += int(b.sum())
            off_band += int((d & ~b).sum())
        else:
            off_band += int(d.sum())
        if d.any():
            mism[m] = int(d.sum())
    # north_star: disagreements are allowed only at band positions; the fp64
    # sequence is replayed bit for bit, so there must be none at all
    assert off_band == 0, f"disagreements outside the threshold band: {mism}"
    assert not mism, f"mask disagreements per size (all inside the band): {mism}"
    res.band_positions = band
    assert np.array_equal(res.candidates.array(), np.array(ref.candidates, np.int32).reshape(-1, 3))
    assert res.stats.patches_tested == ref.patches_tested
    assert res.stats.patches_kept == ref.patches_kept
    assert res.stats.region_pixels_kept == ref.region_pixels_kept
    assert np.array_equal(res.region_mask, ref.region_mask)
    return res


def test_config0_vs_oracle(cuda):
    import workloads as WL

    c = WL.make_cases(WL.CONFIGS[0])[0]
    wl = WL.CONFIGS[0]
    compare_with_oracle(c.image, c.template, {"alpha": wl.alpha, "beta": wl.beta, "ladder_ratio": wl.ladder_ratio,
                                              "quantizer": wl.q})


@pytest.mark.slow
def test_config1_vs_oracle(cuda):
    import workloads as WL

    wl = WL.CONFIGS[1]
    c = WL.make_cases(wl)[0]
    res = compare_with_oracle(c.image, c.template, {"alpha": wl.alpha, "beta": wl.beta,
                                                    "ladder_ratio": wl.ladder_ratio, "quantizer": wl.q})
    print(f"config 1: {res.band_positions} threshold-band positions, 0 disagreements")


def test_band_positions_are_counted(cuda):
    """SURVEY.md 8(d) band positions exist and are counted: flat blocks put
    mean cells exactly on a boundary (t integral), so the oracle must flag
    them, and the GPU must still agree there bit for bit."""
    img = np.full((96, 120), 100, np.uint8)
    img[40:80, 30:90] = 124  # mean 124 / q 8 = 15.5 -> t = 16 exactly
    rng = np.random.default_rng(5)
    img[:30] = rng.integers(0, 256, (30, 120), dtype=np.uint8)
    tpl = np.ascontiguousarray(img[2:26, 10:34])
    res = compare_with_oracle(img, tpl, {"alpha": 1.0, "beta": 1.0})
    assert res.band_positions > 0


def test_random_configs_vs_oracle(cuda):
    import workloads as WL

    rng = np.random.default_rng(7)
    for trial in range(6):
        W = int(rng.integers(60, 700))
        H = int(rng.integers(60, 500))
        img = WL.make_image(W, H, seed=100 + trial, sigma=float(rng.uniform(1, 4)), noise=float(rng.uniform(0, 6)))
        side = int(rng.integers(8, 48))
        case = WL.make_template(img, 200 + trial, side, (0.7, 1.4), std_threshold=10.0)
        kw = {"alpha": float(rng.uniform(0.4, 1.0)), "beta": float(rng.uniform(1.0, 2.2)),
              "ladder_ratio": float(rng.uniform(1.1, 1.5)), "stride": int(rng.integers(1, 4)),
              "ring_count": int(rng.integers(1, 5)),
              "quantizer": (float(rng.uniform(3, 10)), float(rng.uniform(3, 10)), float(rng.uniform(3, 10)))}
        compare_with_oracle(img, case.template, kw)


def test_never_misses_exact_crop(cuda):
    """pkg/tests/test_screening.py:277-289 on the GPU path."""
    from paper_1707_05647_b200 import patch_center_margins, screen
    import workloads as WL

    scene = WL.make_image(160, 120, seed=5)
    rng = np.random.default_rng(34)
    m = 32
    lo, hi = patch_center_margins(m)
    for _ in range(10):
        cx = int(rng.integers(lo, 160 - hi))
        cy = int(rng.integers(lo, 120 - hi))
        tpl = scene[cy - lo : cy - lo + m, cx - lo : cx - lo + m].copy()
        from paper_1707_05647_b200 import std_dev

        if std_dev(tpl) < 5.0:
            continue
        res = screen(scene, tpl)
        assert (cx, cy, m) in res.candidates
        assert res.size_masks[m][cy, cx]
        assert res.region_mask[cy, cx]


def test_errors_and_edge_cases(cuda):
    from paper_1707_05647_b200 import FlatTemplateError, ScreeningConfig, screen

    scene = golden("screens.npz")["t4_default/image"]
    with pytest.raises(FlatTemplateError, match="too flat"):
        screen(scene, np.full((32, 32), 128, np.uint8))
    with pytest.raises(ValueError):
        screen(scene, scene[:16, :20])
    with pytest.raises(ValueError):
        screen(scene, scene[:4, :4])
    # template larger than the image: every size is all-border, nothing tested
    small = scene[:10, :14].copy()
    res = screen(small, scene[:32, :32].copy())
    assert res.stats.patches_tested == 0 and len(res.candidates) == 0
    for m in res.ladder:
        assert res.size_masks[m].all()
    assert not res.region_mask.any()
    # determinism
    tpl = scene[20:52, 30:62].copy()
    a = screen(scene, tpl)
    b = screen(scene, tpl)
    assert a.candidates == b.candidates
    assert np.array_equal(a.region_mask, b.region_mask)
    # very fine quantizer: sparse (binary-search) membership path, still bit-exact
    compare_with_oracle(scene, tpl, {"quantizer": (1e-3, 1e-3, 1e-3)})


def test_int64_and_32bit_planes_agree(cuda):
    """The int64-plane screen (forced) and the 32-bit-plane screen give the same result."""
    import workloads as WL
    from paper_1707_05647_b200 import screen
    from paper_1707_05647_b200.screening import get_engine

    wl = WL.CONFIGS[0]
    c = WL.make_cases(wl)[0]
    kw = {"alpha": 0.6, "beta": 1.6, "ladder_ratio": 1.2, "quantizer": (6.0, 5.0, 7.0)}
    a = screen(c.image, c.template, pcfg(kw))
    eng = get_engine(c.image.shape[1], c.image.shape[0])
    eng.force_int64 = True
    try:
        b = screen(c.image, c.template, pcfg(kw))
    finally:
        eng.force_int64 = False
    assert a.candidates == b.candidates
    for m in a.ladder:
        assert np.array_equal(a.size_masks.packed(m), b.size_masks.packed(m)), m
    assert np.array_equal(a.region_packed(), b.region_packed())


@pytest.mark.parametrize("side", [256, 258])
def test_32bit_boundary_sizes(cuda, side):
    """m = 256 (ring-0 n = 128: 32-bit planes) and m = 258 (n = 129: int64 planes) vs the oracle."""
    from paper_1707_05647_b200 import _native
    import workloads as WL

    n0 = side // 2
    plan = O.ring_plan(side, 3)
    rn = np.array([p[0] for p in plan], np.int32)
    rd = np.array([p[1] for p in plan], np.int32)
    assert bool(_native.lib().ss_screen_fits32(len(plan), rn.ctypes.data, rd.ctypes.data)) == (n0 <= 128)
    img = WL.make_image(640, 560, seed=41, sigma=4.0, noise=3.0)
    case = WL.make_template(img, 43, side, (1.0, 1.0), std_threshold=10.0)
    compare_with_oracle(img, case.template, {"alpha": 1.0, "beta": 1.0, "quantizer": (4.0, 4.0, 4.0)})


@pytest.mark.parametrize("mode", ["0", "1"])
def test_list_modes_vs_oracle(cuda, monkeypatch, mode):
    """Both candidate-list modes of K3 (one (x, y) list; partitioned sub-lists
    carrying the ring-0 sums) on the same inputs, 32-bit and int64 planes."""
    import workloads as WL
    from paper_1707_05647_b200.screening import get_engine

    monkeypatch.setenv("SS_LIST_MODE", mode)
    img = WL.make_image(700, 380, seed=61, sigma=2.5, noise=2.0)
    case = WL.make_template(img, 62, 40, (0.8, 1.3), std_threshold=10.0)
    kw = {"alpha": 0.5, "beta": 1.8, "ladder_ratio": 1.25, "quantizer": (6.0, 6.0, 6.0)}
    compare_with_oracle(img, case.template, kw)
    eng = get_engine(img.shape[1], img.shape[0])
    eng.force_int64 = True
    try:
        compare_with_oracle(img, case.template, kw)
    finally:
        eng.force_int64 = False


@pytest.mark.parametrize("session", ["1", "0"])
def test_screen_batch_matches_screen(cuda, monkeypatch, session):
    """screen_batch (native sessions on host threads, or the engine pool's
    overlapped streams; engine reuse) == screen() per image."""
    import workloads as WL
    from paper_1707_05647_b200 import screen, screen_batch

    monkeypatch.setenv("SS_SESSION", session)

    imgs, tpls = [], []
    for i in range(7):
        img = WL.make_image(400, 300, seed=300 + i, sigma=2.5, noise=1.0)
        case = WL.make_template(img, 400 + i, 32, (0.8, 1.2), std_threshold=10.0)
        imgs.append(img)
        tpls.append(case.template)
    cfg = pcfg({"alpha": 0.7, "beta": 1.4, "quantizer": (6.0, 6.0, 6.0)})
    batch = screen_batch(imgs, tpls, cfg, engines=3)
    assert len(batch) == len(imgs)
    for img, tpl, b in zip(imgs, tpls, batch):
        a = screen(img, tpl, cfg)
        assert a.candidates == b.candidates
        assert a.stats.patches_tested == b.stats.patches_tested
        assert a.stats.region_pixels_kept == b.stats.region_pixels_kept
        for m in a.ladder:
            assert np.array_equal(a.size_masks.packed(m), b.size_masks.packed(m)), m
    with pytest.raises(ValueError):
        screen_batch(imgs[:2], tpls[:1], cfg)


@pytest.mark.parametrize("world", [2, 3])
def test_row_bands_on_device_assemble_to_full_screen(cuda, world):
    """The multi-GPU data path (sharding.py) run band by band on one GPU: band
    tables + screens (halo'd bands, border status in global rows), the mask
    halo rows the neighbour exchange would deliver, K5 over band + halo
    (ss_region_ladder_rows) and the device assembly of the padded survivor
    rows equal the single-image screen's masks, region and candidates."""
    import torch

    import workloads as WL
    from paper_1707_05647_b200 import screen
    from paper_1707_05647_b200.engine import prepare_template
    from paper_1707_05647_b200.screening import unpack_bits
    from paper_1707_05647_b200.sharding import (assemble_rows, band_engine, halo_counts, plan_bands,
                                                region_rows_device)

    img = WL.make_image(500, 431, seed=71, sigma=2.5, noise=2.0)
    case = WL.make_template(img, 72, 40, (0.8, 1.3), std_threshold=10.0)
    cfg = pcfg({"alpha": 0.5, "beta": 1.8, "ladder_ratio": 1.25, "quantizer": (6.0, 6.0, 6.0)})
    full = screen(img, case.template, cfg)
    H, W = img.shape
    tp = prepare_template(case.template, cfg, cuda)
    L = len(tp.sizes)
    bands = plan_bands(H, world, tp.ladder)
    masks, counts, rows = [], [], []
    for b in bands:
        eng = band_engine(W, H, b, cuda)
        sub = torch.from_numpy(np.ascontiguousarray(img[b.y_origin:b.y_origin + b.rows])).to(cuda)
        eng.run(sub, tp, region=False, capacity=1 << 16)
        masks.append(eng.masks[:L].clone())
        counts.append(eng.size_counts[:L].clone())
        rows.append(eng.xy[: 1 << 16].clone())
    for r, b in enumerate(bands):
        assert np.array_equal(masks[r].cpu().numpy().view(np.uint32),
                              full.size_masks.packed_all()[:, b.y_begin:b.y_end])
        top, bot = halo_counts(bands, r, H, tp.ladder)
        parts = ([masks[r - 1][:, masks[r - 1].shape[1] - top:]] if top else []) + [masks[r]] + \
                ([masks[r + 1][:, :bot]] if bot else [])
        stack = torch.cat(parts, 1)
        reg = region_rows_device(stack, W, b.y_begin - top, H, tp.ladder, cfg.stride)
        got = unpack_bits(reg[top: top + b.y_end - b.y_begin].cpu().numpy().view(np.uint32), W)
        assert np.array_equal(got, full.region_mask[b.y_begin:b.y_end]), r
    out = assemble_rows(torch.stack(rows), torch.stack(counts))
    n = full.stats.patches_kept
    assert int(torch.stack(counts).sum()) == n
    assert np.array_equal(out[:n].cpu().numpy(), full.candidates.array())


def _boundary_image(seed):
    """Flat blocks at mean-cell boundaries (v = 8k + 4), exact ramps,
    checkerboards and stripes: many centres whose mean / std / gradient sit
    exactly on or within rounding of a quantizer boundary."""
    rng = np.random.default_rng(seed)
    H, W = 300, 360
    img = np.zeros((H, W), np.uint8)
    for by in range(0, H, 60):
        for bx in range(0, W, 60):
            img[by:by + 60, bx:bx + 60] = 8 * int(rng.integers(0, 32)) + 4
    yy, xx = np.mgrid[0:60, 0:60]
    img[0:60, 0:60] = (xx * 4) % 256
    img[60:120, 120:180] = (yy * 2 + xx * 2) % 256
    img[120:180, 240:300] = ((xx + yy) % 2) * 255
    img[180:240, 0:60] = 4 + 8 * ((xx // 8) % 2)
    img[240:300, 300:360] = 12 + 16 * ((yy // 4) % 2)
    return img


@pytest.mark.parametrize("q", [(8.0, 8.0, 8.0), (2.0, 0.5, 0.25), (3.0, 1e-3, 0.7), (16.0, 4.0, 1e-3)])
def test_boundary_heavy_image_vs_oracle(cuda, q):
    """The fused rings decide cells from fp32 estimates and defer to the fp64
    sequence only near a boundary: on an image built to put features on
    boundaries the masks must still equal the oracle's bit for bit."""
    img = _boundary_image(5)
    tpl = np.ascontiguousarray(img[30:70, 30:70])
    compare_with_oracle(img, tpl, {"alpha": 0.6, "beta": 1.6, "ladder_ratio": 1.2, "quantizer": q})


@pytest.mark.parametrize("q", [(8.0, 8.0, 8.0), (5.0, 3.0, 2.5)])
def test_fused_ladder_equals_per_size_path(cuda, monkeypatch, q):
    """The fused ladder (lock-step sizes, fp32-estimated cells) and the
    per-size kernels (fp64 sequence everywhere) on the same inputs."""
    import workloads as WL
    from paper_1707_05647_b200 import screen

    img = WL.make_image(900, 700, seed=81, sigma=3.0, noise=2.0)
    case = WL.make_template(img, 82, 48, (0.7, 1.4), std_threshold=10.0)
    cfg = pcfg({"alpha": 0.5, "beta": 2.0, "ladder_ratio": 1.15, "quantizer": q})
    monkeypatch.setenv("SS_FUSED", "1")
    a = screen(img, case.template, cfg)
    monkeypatch.setenv("SS_FUSED", "0")
    b = screen(img, case.template, cfg)
    assert a.candidates == b.candidates
    assert (a.stats.patches_tested, a.stats.patches_kept, a.stats.region_pixels_kept) == (
        b.stats.patches_tested, b.stats.patches_kept, b.stats.region_pixels_kept)
    for m in a.ladder:
        assert np.array_equal(a.size_masks.packed(m), b.size_masks.packed(m)), m


def test_fused_ladder_declines_to_per_size_path(cuda):
    """A ladder whose rings exceed the fused parameter block (37 sizes, 111
    rings > 104) is screened size by size on the same stream: still equal to
    the oracle."""
    import workloads as WL

    img = WL.make_image(320, 280, seed=91, sigma=2.5, noise=2.0)
    case = WL.make_template(img, 92, 48, (0.8, 1.3), std_threshold=10.0)
    compare_with_oracle(img, case.template, {"alpha": 0.5, "beta": 2.0, "ladder_ratio": 1.04,
                                             "quantizer": (8.0, 8.0, 8.0)})


@pytest.mark.parametrize("cap_mb", [20, 40])
def test_fused_ladder_row_bands_vs_oracle(cuda, monkeypatch, cap_mb):
    """A workspace too small for the whole candidate list makes the fused
    ladder screen the image in several row bands (tables, masks and counts
    shared, lists per band): still equal to the oracle."""
    import workloads as WL
    from paper_1707_05647_b200.screening import _engine_cache

    monkeypatch.setenv("SS_LADDER_WS_BYTES", str(cap_mb << 20))
    _engine_cache.clear()
    try:
        img = WL.make_image(900, 640, seed=101, sigma=2.5, noise=2.0)
        case = WL.make_template(img, 102, 48, (0.8, 1.3), std_threshold=10.0)
        compare_with_oracle(img, case.template, {"alpha": 0.5, "beta": 2.0, "ladder_ratio": 1.2,
                                                 "quantizer": (8.0, 8.0, 8.0)})
    finally:
        _engine_cache.clear()


def test_streamed_mask_readback_in_chunks(cuda, monkeypatch):
    """screen() streams each finished row chunk of every size mask to pinned
    host memory while later chunks are screened (Engine.run(host_masks=...)):
    force several chunks (one ss_screen_ladder call each, mask rows starting at
    the chunk's first row) and compare the whole result with the oracle."""
    import workloads as WL
    from paper_1707_05647_b200.engine import Engine

    monkeypatch.setattr(Engine, "READBACK_CHUNK_BYTES", 1 << 14)
    monkeypatch.setenv("SS_SESSION", "0")  # the Python engine's streamed readback
    img = WL.make_image(700, 1100, seed=41, sigma=2.5, noise=3.0)
    case = WL.make_template(img, 42, 40, (0.8, 1.3), std_threshold=10.0)
    res = compare_with_oracle(img, case.template, {"alpha": 0.5, "beta": 1.8, "ladder_ratio": 1.2})
    from paper_1707_05647_b200.screening import get_engine

    eng = get_engine(700, 1100, cuda)
    assert len(eng.readback_chunks(len(res.ladder))) >= 4


def _stage_counts(img, tpl, cfg, cuda):
    """(interior centres evaluated, ring-0 mean passers, ring-0 passers,
    survivors) of one fused screen, from the kernels' stage counters."""
    import torch

    from paper_1707_05647_b200.engine import Engine, fill_keysets, plan_ladder

    h, w = img.shape
    eng = Engine(w, h, cuda)
    eng.stage_counts = torch.zeros(32, dtype=torch.int64, device=cuda)
    tp = plan_ladder(tpl.shape[1], cfg)
    fill_keysets(tp, tpl, cuda)
    eng.run(torch.from_numpy(np.ascontiguousarray(img)).to(cuda), tp)
    torch.cuda.synchronize()
    return eng.stage_counts[:4].tolist(), eng.masks[: len(tp.sizes)].cpu().numpy(), eng.coarse_shifts


@pytest.mark.parametrize("q", [(8.0, 8.0, 8.0), (2.0, 0.5, 0.25), (16.0, 4.0, 1e-3), (0.6, 8.0, 8.0)])
@pytest.mark.parametrize("which", ["boundary", "smooth"])
def test_coarse_stage1_equals_exact_stage1(cuda, monkeypatch, q, which):
    """Stage 1 from the u16 bit-slice planes (coarse estimate; centres within
    its error bound of a membership boundary go on to the rings kernel, whose
    level 0 tests ring 0's exact mean cell) gives exactly the 32-bit stage 1's
    results: same evaluated centres, ring-0 passers, survivors and masks; its
    candidate list is a superset."""
    import workloads as WL

    if which == "boundary":
        img = _boundary_image(9)
        tpl = np.ascontiguousarray(img[100:140, 40:80])
    else:
        img = WL.make_image(640, 480, seed=91, sigma=3.0, noise=1.0)
        tpl = WL.make_template(img, 92, 40, (0.7, 1.4), std_threshold=10.0).template
    cfg = pcfg({"alpha": 0.5, "beta": 2.0, "ladder_ratio": 1.2, "quantizer": q})
    monkeypatch.setenv("SS_COARSE", "1")
    ca, ma, shifts = _stage_counts(img, tpl, cfg, cuda)
    monkeypatch.setenv("SS_COARSE", "0")
    cb, mb, none = _stage_counts(img, tpl, cfg, cuda)
    assert shifts and not none
    assert (ca[0], ca[2], ca[3]) == (cb[0], cb[2], cb[3])
    assert ca[1] >= cb[1]
    assert np.array_equal(ma, mb)


def _step_image(which, seed=3):
    """Images whose ring-0 mean moves as fast as it can from one centre row to
    the next (the row-step bound of stage 1 is the worst case over images)."""
    import workloads as WL

    rng = np.random.default_rng(seed)
    h, w = 520, 640
    if which == "stripes":  # full-contrast horizontal stripes of many periods + a little noise
        img = np.zeros((h, w), np.int32)
        y = 0
        while y < h:
            t = int(rng.integers(3, 90))
            img[y:y + t] = int(rng.integers(0, 2)) * 255
            y += t
        img[:, w // 2:] = 255 - img[:, w // 2:]
        img = np.clip(img + rng.integers(-6, 7, size=img.shape), 0, 255).astype(np.uint8)
    elif which == "blocks":
        img = np.kron(rng.integers(0, 2, size=(h // 20, w // 20)) * 255, np.ones((20, 20))).astype(np.uint8)
        img = np.clip(img.astype(np.int32) + rng.integers(-20, 21, size=img.shape), 0, 255).astype(np.uint8)
    else:
        img = WL.make_image(w, h, seed=seed, sigma=3.0, noise=1.0)
    return np.ascontiguousarray(img)


@pytest.mark.parametrize("slack", ["0.4", "1.5", "12.0"])
@pytest.mark.parametrize("which", ["stripes", "blocks", "smooth"])
def test_stage1_row_steps_keep_every_ring0_passer(cuda, monkeypatch, which, slack):
    """Coarse stage 1 may test one centre row per group of 2 or 4 rows for
    sizes whose ring-0 mean cannot move by more than SS_S1_SLACK cells inside
    a group (window widened by the worst-case bound), sending the whole
    group's columns on as candidates.  With std / gradient steps so large that
    membership is the mean test alone, the ring-0 passer count would drop if
    any true passer were skipped: counts and masks must equal those of the
    every-row stage 1 (slack 0), on images built for the bound's worst case."""
    img = _step_image(which)
    tpl = np.ascontiguousarray(img[200:264, 300:364])
    for q in ((8.0, 1e6, 1e6), (16.0, 8.0, 1e6)):
        cfg = pcfg({"alpha": 0.5, "beta": 2.0, "ladder_ratio": 1.25, "quantizer": q})
        monkeypatch.setenv("SS_S1_SLACK", "0")
        monkeypatch.delenv("SS_S1_FORCE", raising=False)
        cb, mb, _ = _stage_counts(img, tpl, cfg, cuda)
        # forced: the largest row step the slack allows for each size;
        # planned: the step ladder_plan_kernel picks from its image sample
        for force in ("1", "0"):
            monkeypatch.setenv("SS_S1_SLACK", slack)
            monkeypatch.setenv("SS_S1_FORCE", force)
            monkeypatch.setenv("SS_S1_MIN_WORK", "0")  # plan even this small image
            ca, ma, shifts = _stage_counts(img, tpl, cfg, cuda)
            assert shifts
            assert (ca[0], ca[2], ca[3]) == (cb[0], cb[2], cb[3]), (q, force, ca, cb)
            assert ca[1] >= cb[1]
            if force == "1" and float(slack) > 1.0:
                assert ca[1] > cb[1]  # groups were formed (more candidates than the every-row test)
            assert np.array_equal(ma, mb)
        if q[1] > 1e5:
            assert cb[2] > 0  # the comparison is not vacuous


def test_dense_candidates_with_partitioned_lists(cuda):
    """A periodic texture screened with one of its periods: ring 0's mean is
    the same almost everywhere, so nearly every centre of every size passes
    stage 1 -- the candidate lists (8 partitions from 32768 tiles) fill close
    to their capacity and the row-step plan picks its largest steps.  Masks,
    candidates and region must still equal the oracle's."""
    import workloads as WL

    rng = np.random.default_rng(77)
    period = WL.make_image(64, 64, seed=78, sigma=2.0, noise=0.0)
    img = np.tile(period, (64, 64))  # 4096 x 4096
    img = np.clip(img.astype(np.int32) + rng.integers(-2, 3, size=img.shape), 0, 255).astype(np.uint8)
    tpl = np.ascontiguousarray(img[1024:1088, 2048:2112])
    res = compare_with_oracle(img, tpl, {"alpha": 0.7, "beta": 1.5, "ladder_ratio": 1.15,
                                         "quantizer": (8.0, 8.0, 8.0)})
    assert len(res.ladder) >= 5


def test_coarse_planes_are_bit_slices(cuda):
    """ss_build_tables3's u16 planes are (cell >> shift) & 0xffff of the
    SAT / E / O PLAIN cells for every shift."""
    import torch

    from paper_1707_05647_b200 import _native

    L = _native.lib()
    img = np.random.default_rng(3).integers(0, 256, (777, 1234), dtype=np.uint8)
    H, W = img.shape
    pitch = int(L.ss_plane_pitch(W))
    shifts = np.array([1, 4, 7, 10, 13], np.int32)
    p32 = torch.empty(int(L.ss_tables32_bytes(W, H)) // 4, dtype=torch.int32, device=cuda)
    co = torch.empty(int(L.ss_coarse_bytes(W, H, 5)) // 2, dtype=torch.int16, device=cuda)
    ws = torch.empty(int(L.ss_build_workspace_bytes(W, H)), dtype=torch.uint8, device=cuda)
    d_img = torch.from_numpy(img).to(cuda)
    _native.check(L.ss_build_tables3(d_img.data_ptr(), W, H, W, None, p32.data_ptr(), None, pitch, co.data_ptr(), 5,
                                     shifts.ctypes.data, ws.data_ptr(), ws.numel(),
                                     torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    planes = p32.view(12, H + 1, pitch).cpu().numpy().view(np.uint32)
    coarse = co[: 5 * 3 * (H + 1) * pitch].view(5, 3, H + 1, pitch).cpu().numpy().view(np.uint16)  # (+ 4 rows of padding)
    for c, k in enumerate(shifts):
        for t, p in enumerate((0, 4, 8)):  # PLAIN SAT, E, O
            want = ((planes[p] >> np.uint32(k)) & np.uint32(0xFFFF)).astype(np.uint16)
            assert np.array_equal(coarse[c, t, :, : W + 1], want[:, : W + 1]), (k, t)


def test_wide48_rings_equal_int64_planes(cuda, monkeypatch):
    """Sizes whose ring sums exceed 32 bits: the fused rings read 32-bit +
    hi16 cells (mod 2^48) by default (native session and Python engine) and
    the int64 planes when forced; all must give the oracle's result."""
    import workloads as WL
    from paper_1707_05647_b200 import screen
    from paper_1707_05647_b200.screening import get_engine

    img = WL.make_image(900, 720, seed=71, sigma=4.0, noise=2.0)
    case = WL.make_template(img, 72, 160, (0.9, 1.1), std_threshold=10.0)
    kw = {"alpha": 1.0, "beta": 2.0, "ladder_ratio": 1.3, "quantizer": (6.0, 5.0, 7.0)}
    a = compare_with_oracle(img, case.template, kw)  # the session
    monkeypatch.setenv("SS_SESSION", "0")
    c = screen(img, case.template, pcfg(kw))
    eng = get_engine(900, 720)
    assert eng.built_hi16 and not eng.built_int64
    assert a.candidates == c.candidates
    eng.force_int64 = True
    try:
        b = screen(img, case.template, pcfg(kw))
        assert eng.built_int64 and not eng.built_hi16
    finally:
        eng.force_int64 = False
    assert a.candidates == b.candidates
    for m in a.ladder:
        assert np.array_equal(a.size_masks.packed(m), b.size_masks.packed(m)), m


def test_pipelined_upload_build_screen(cuda, monkeypatch):
    """screen() on a large image uploads it, builds its tables and screens it
    row chunk by row chunk (Engine.run_pipelined, ss_build_tables_rows): force
    that path on a mid-size image (several build chunks, a ladder with a
    large lower margin) and compare with the oracle."""
    import workloads as WL
    from paper_1707_05647_b200.engine import Engine

    monkeypatch.setattr(Engine, "PIPELINE_MIN_BYTES", 1 << 10)
    monkeypatch.setattr(Engine, "PIPELINE_CHUNKS", 6)
    img = WL.make_image(600, 1500, seed=51, sigma=3.0, noise=2.0)
    case = WL.make_template(img, 52, 64, (0.8, 1.3), std_threshold=10.0)
    compare_with_oracle(img, case.template, {"alpha": 0.5, "beta": 2.0, "ladder_ratio": 1.25})
    # the same with a wide (hi16) size in the ladder
    case = WL.make_template(img, 53, 150, (0.9, 1.1), std_threshold=10.0)
    compare_with_oracle(img, case.template, {"alpha": 1.0, "beta": 1.8, "ladder_ratio": 1.3})


def test_build_tables_rows_equals_whole_build(cuda):
    """ss_build_tables_rows over consecutive band runs == one ss_build_tables3."""
    import torch

    from paper_1707_05647_b200 import _native

    L = _native.lib()
    rng = np.random.default_rng(12)
    for (H, W, exact) in ((1000, 777, 0), (2100, 513, 1)):
        img = rng.integers(0, 256, (H, W), dtype=np.uint8)
        pitch = int(L.ss_plane_pitch(W))
        ws = torch.empty(int(L.ss_build_workspace_bytes(W, H)), dtype=torch.uint8, device=cuda)
        d_img = torch.from_numpy(img).to(cuda)
        sh = np.array([1, 4, 7], np.int32)
        outs = []
        for chunked in (False, True):
            p32 = torch.zeros(int(L.ss_tables32_bytes(W, H)) // 4, dtype=torch.int32, device=cuda)
            h16 = torch.zeros(int(L.ss_tables_hi16_bytes(W, H)) // 2, dtype=torch.int16, device=cuda) if exact else None
            co = torch.zeros(int(L.ss_coarse_bytes(W, H, 3)) // 2, dtype=torch.int16, device=cuda)
            s = torch.cuda.current_stream().cuda_stream
            if not chunked:
                _native.check(L.ss_build_tables3(d_img.data_ptr(), W, H, W, None, p32.data_ptr(),
                                                 None if h16 is None else h16.data_ptr(), pitch, co.data_ptr(), 3,
                                                 sh.ctypes.data, ws.data_ptr(), ws.numel(), s))
            else:
                rb = int(L.ss_build_band_rows(W, H, exact))
                edges = sorted({0, H, *range(3 * rb, H, 5 * rb), *range(7 * rb, H, 7 * rb)})
                for y0, y1 in zip(edges[:-1], edges[1:]):
                    _native.check(L.ss_build_tables_rows(d_img.data_ptr(), W, H, W, None, p32.data_ptr(),
                                                         None if h16 is None else h16.data_ptr(), pitch,
                                                         co.data_ptr(), 3, sh.ctypes.data, y0, y1, ws.data_ptr(),
                                                         ws.numel(), s))
            torch.cuda.synchronize()
            outs.append([t.cpu().numpy() for t in (p32, h16, co) if t is not None])
        for a, b in zip(*outs):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("chain", ["1", "0"])
def test_region_chain_equals_union_of_footprints(cuda, monkeypatch, chain):
    """K5: the chained dilation (descending sizes, telescoping footprints,
    steps cut to <= 31 each way) and the per-size row / column passes both
    give the union of every evaluated survivor's m x m footprint, over
    ladders with large gaps, a single size, and odd / even sizes."""
    import workloads as WL

    monkeypatch.setenv("SS_REGION_CHAIN", chain)
    img = WL.make_image(500, 420, seed=31, sigma=2.5, noise=3.0)
    for seed, side, kw in ((32, 24, {"alpha": 0.4, "beta": 3.0, "ladder_ratio": 1.7}),
                           (33, 47, {"alpha": 1.0, "beta": 1.0}),
                           (34, 64, {"alpha": 0.5, "beta": 2.0, "ladder_ratio": 1.1, "stride": 2}),
                           (35, 100, {"alpha": 0.5, "beta": 2.0, "ladder_ratio": 2.0})):  # gaps > 31
        case = WL.make_template(img, seed, side, (0.9, 1.1), std_threshold=10.0)
        compare_with_oracle(img, case.template, kw)


def test_region_with_and_without_row_counts(cuda):
    """K5 skips rows whose K3 survivor count is zero without reading them
    (ss_region_ladder2); without the counts (ss_region_ladder: it finds the
    empty rows itself) the region must be the same, on a sparse result (most
    rows empty) and a dense one."""
    import torch
    import workloads as WL
    from paper_1707_05647_b200 import _native
    from paper_1707_05647_b200.engine import Engine, fill_keysets, plan_ladder

    L = _native.lib()
    img = WL.make_image(900, 700, seed=41, sigma=3.0, noise=1.0)
    for seed, q in ((42, (8.0, 8.0, 8.0)), (43, (64.0, 64.0, 64.0))):
        tpl = WL.make_template(img, seed, 48, (0.8, 1.3), std_threshold=10.0).template
        cfg = pcfg({"alpha": 0.5, "beta": 2.0, "ladder_ratio": 1.2, "quantizer": q})
        h, w = img.shape
        eng = Engine(w, h, cuda)
        tp = plan_ladder(tpl.shape[1], cfg)
        fill_keysets(tp, tpl, cuda)
        eng.run(torch.from_numpy(np.ascontiguousarray(img)).to(cuda), tp)
        torch.cuda.synchronize()
        with_counts = eng.region.clone()
        ms = np.array([sp.m for sp in tp.sizes], np.int32)
        other = torch.full_like(eng.region, -1)
        _native.check(L.ss_region_ladder(eng.masks.data_ptr(), eng.words, eng.mrows * eng.words, w, h, len(ms),
                                         ms.ctypes.data, cfg.stride, other.data_ptr(), eng.region_ws.data_ptr(),
                                         eng.region_ws.numel(), torch.cuda.current_stream().cuda_stream), "region")
        torch.cuda.synchronize()
        assert torch.equal(with_counts, other)
        empty = int((eng.row_counts[: len(ms)] == 0).sum())
        assert 0 < empty < eng.row_counts[: len(ms)].numel()  # both kinds of rows occur


def _same_result(a, b):
    assert tuple(a.ladder) == tuple(b.ladder)
    assert np.array_equal(a.candidates.array(), b.candidates.array())
    for m in a.ladder:
        assert np.array_equal(a.size_masks.packed(m), b.size_masks.packed(m)), m
    assert np.array_equal(a.region_packed(), b.region_packed())
    assert (a.stats.patches_tested, a.stats.patches_kept, a.stats.region_pixels_kept, a.stats.total_pixels) == (
        b.stats.patches_tested, b.stats.patches_kept, b.stats.region_pixels_kept, b.stats.total_pixels)
    assert a.candidates_per_size() == b.candidates_per_size()


@pytest.mark.parametrize("case", ["config0", "stride", "tiny", "wide", "everything", "no_coarse"])
def test_session_equals_engine_path(cuda, monkeypatch, case):
    """screen() through the native session (ss_session_screen: one C call) and
    through the Python engine (stream-level entry points) on the same inputs:
    identical results, including a ladder of sizes beyond 32 bits (hi16
    planes), tiny sizes (whole-grid keeps), stride 3, no coarse stage 1, and a
    screen keeping almost every centre (the survivor buffer and the output
    rows both overflow on the first call: K4 redone, rows fetched after)."""
    import workloads as WL
    from paper_1707_05647_b200 import screen
    from paper_1707_05647_b200.screening import _session_cache

    if case == "config0":
        wl = WL.CONFIGS[0]
        c = WL.make_cases(wl)[0]
        img, tpl = c.image, c.template
        kw = {"alpha": wl.alpha, "beta": wl.beta, "ladder_ratio": wl.ladder_ratio, "quantizer": wl.q}
    else:
        img = WL.make_image(640, 400, seed=501, sigma=3.0, noise=2.0)
        side = {"wide": 160, "tiny": 12}.get(case, 40)
        tpl = WL.make_template(img, 502, side, (0.9, 1.1), std_threshold=8.0).template
        kw = {"alpha": 0.5, "beta": 2.0, "ladder_ratio": 1.3}
        if case == "stride":
            kw["stride"] = 3
        if case == "tiny":
            kw.update(alpha=0.3, beta=1.0)
        if case == "wide":
            kw.update(alpha=1.0, beta=2.0, quantizer=(6.0, 5.0, 7.0))
        if case == "everything":
            kw.update(quantizer=(400.0, 400.0, 400.0))
        if case == "no_coarse":
            monkeypatch.setenv("SS_COARSE", "0")
    _session_cache.clear()  # a fresh session: first-call capacities
    a = screen(img, tpl, pcfg(kw))
    a2 = screen(img, tpl, pcfg(kw))  # the same session again (buffers reused)
    monkeypatch.setenv("SS_SESSION", "0")
    b = screen(img, tpl, pcfg(kw))
    _same_result(a, b)
    _same_result(a2, b)
    if case == "everything":
        assert a.stats.patches_kept > max(1 << 16, a.stats.patches_tested // 50)
    if case == "config0":
        compare_with_oracle(img, tpl, kw)


def test_session_threads_equal_serial(cuda):
    """Several native sessions driven from host threads at once (the GIL is
    released inside ss_session_screen) give the serial results."""
    import concurrent.futures

    import workloads as WL
    from paper_1707_05647_b200.session import Session

    cfg = pcfg({"alpha": 0.6, "beta": 1.5, "quantizer": (6.0, 6.0, 6.0)})
    cases = []
    for i in range(6):
        img = WL.make_image(480, 360, seed=600 + i, sigma=2.5, noise=1.0)
        cases.append((img, WL.make_template(img, 700 + i, 32, (0.8, 1.2), std_threshold=10.0).template))
    sessions = [Session(480, 360, cuda) for _ in range(3)]

    def run(i):
        _, r = sessions[i % 3].run(*cases[i], cfg)
        return r.rows[: r.kept].numpy().copy(), r.masks.numpy().copy(), r.region_pixels

    serial = [run(i) for i in range(len(cases))]
    with concurrent.futures.ThreadPoolExecutor(3) as ex:
        par = list(ex.map(run, range(len(cases))))
    for (ra, ma, pa), (rb, mb, pb) in zip(serial, par):
        assert np.array_equal(ra, rb) and np.array_equal(ma, mb) and pa == pb
