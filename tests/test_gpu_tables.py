"""K1/K2 parity: the 12 device planes vs the oracle's reference-layout tables.

SAT planes must equal Sat.cells exactly; E / O planes must equal the
reference Rsat H(u, v) at the mapped indices (include/starscreen_b200.h).
Cells outside the reference table's (u, v) domain are checked against the
brute-force quadrant-prefix definition instead.
"""

import numpy as np
import pytest

import oracle as O
from conftest import golden

pytestmark = pytest.mark.gpu


def device_planes(img, cuda):
    import torch

    from paper_1707_05647_b200.engine import Engine

    h, w = img.shape
    eng = Engine(w, h, cuda)
    eng.build_tables(torch.from_numpy(np.ascontiguousarray(img)).to(cuda), int64=True)
    torch.cuda.synchronize()
    p = eng.planes.view(12, h + 1, eng.pitch).cpu().numpy()
    # the 32-bit planes written by the same pass are the cells mod 2^32
    p32 = eng.planes32.view(12, h + 1, eng.pitch).cpu().numpy().view(np.uint32)
    assert np.array_equal(p32[:, :, : w + 1], p[:, :, : w + 1].astype(np.uint32)), "32-bit planes != int64 mod 2^32"
    return p[:, :, : w + 1]


def check_planes(img, planes, brute_extra=False):
    h, w = img.shape
    for k in range(4):
        assert np.array_equal(planes[k], O.build_sat(img, k)), f"SAT kind {k}"
        rs = O.build_rsat(img, k)

        def H(u, v):
            return rs[u + 1, v + h - 1]

        E = planes[4 + k]
        Op = planes[8 + k]
        ys, xs = np.mgrid[-1:h, 0:w]
        assert np.array_equal(E[ys + 1, xs + 1], H(xs + ys, xs - ys)), f"E kind {k}"
        ys, xs = np.mgrid[-1 : h - 1, -1:w]
        assert np.array_equal(Op[ys + 1, xs + 1], H(xs + ys + 1, xs - ys)), f"O kind {k}"
        if brute_extra:
            # every cell, including E col x=-1 and O row y=H-1, from the definition
            wm = img.astype(np.int64)
            jj, ii = np.mgrid[0:h, 0:w]
            if k == 1:
                wm = wm * (ii + 1)
            elif k == 2:
                wm = wm * (jj + 1)
            elif k == 3:
                wm = wm * wm
            s = ii + jj
            d = ii - jj
            for y in range(-1, h):
                for x in range(-1, w):
                    e = wm[(s <= x + y) & (d >= x - y)].sum()
                    o = wm[(s <= x + y + 1) & (d >= x - y)].sum()
                    assert E[y + 1, x + 1] == e and Op[y + 1, x + 1] == o, (k, x, y)


def test_golden_images(cuda):
    z = golden("tables.npz")
    for i in range(int(z["n"])):
        img = z[f"img{i}"]
        planes = device_planes(img, cuda)
        for k in range(4):
            assert np.array_equal(planes[k], z[f"sat{i}_{k}"]), (i, k)
        check_planes(img, planes, brute_extra=img.size <= 400)


@pytest.mark.parametrize("band_rows", [15, 31, 63])
@pytest.mark.parametrize("shape", [(15, 479), (16, 480), (31, 447), (63, 383), (64, 384), (126, 385), (127, 767),
                                   (200, 1000), (517, 130), (1, 2000), (1300, 3), (190, 961)])
def test_band_and_chunk_boundaries(cuda, shape, band_rows, monkeypatch):
    """Shapes straddling the band (15/31/63 rows) and chunk (480/448/384 columns) seams."""
    monkeypatch.setenv("SS_BAND_ROWS", str(band_rows))
    rng = np.random.default_rng(sum(shape) + band_rows)
    img = rng.integers(0, 256, shape, dtype=np.uint8)
    check_planes(img, device_planes(img, cuda))


def test_saturated_image(cuda):
    img = np.full((300, 900), 255, np.uint8)
    check_planes(img, device_planes(img, cuda))


def test_overflow_guard_rejected(cuda):
    import torch

    from paper_1707_05647_b200 import _native

    L = _native.lib()
    with pytest.raises(ValueError, match="too large"):
        _native.check(L.ss_build_tables(1, 300000, 300000, 300000, 16, L.ss_plane_pitch(300000), 0, 0, None))


def test_division_routine_matches_ieee(cuda):
    """The screen divides by per-size constants with a reciprocal and two FMA
    corrections; it must equal IEEE division for every operand family the
    features produce (integer sums, half-integer gradient numerators, wide doubles)."""
    import torch

    from paper_1707_05647_b200 import _native

    L = _native.lib()
    bad = torch.zeros(1, dtype=torch.int64, device=cuda)
    s = torch.cuda.current_stream().cuda_stream
    divisors = [4.0 * n * n for n in (4, 5, 11, 16, 64, 181, 256)]
    divisors += [2.0 * d * d + 2 * d + 1 for d in (3, 6, 15, 23, 181, 255)]
    divisors += [2.0 * n ** 3 for n in (4, 11, 64, 256)]
    divisors += [2.0 * d * d + d * (d - 1) * (2 * d - 1) // 3 for d in (3, 15, 255)]
    divisors += [8.0, 3.0, 0.75, 1e-3, 1e6, 6.25, 7.123456789]
    for i, b in enumerate(divisors):
        for mode in range(4):
            _native.check(L.ss_selftest_div(1 << 22, 1000 * i + mode, b, mode, bad.data_ptr(), s))
    torch.cuda.synchronize()
    assert int(bad.item()) == 0


@pytest.mark.parametrize("q", [(8.0, 8.0, 8.0), (6.0, 6.0, 6.0), (3.0, 0.7, 2.5), (8.0, 1e-3, 1e-3), (2.0, 0.25, 1e6)])
def test_fp32_estimated_cells_match_fp64(cuda, q):
    """The fused rings decide std / gradient cells from fp32 estimates and fall
    back to the fp64 sequence near a boundary: on 2^22 random region sums
    per ring (3 in 4 aimed within ~1e-6 of a boundary) the cells must equal
    the fp64 reference sequence's, for small to int64-sized rings."""
    import torch

    from paper_1707_05647_b200 import _native

    L = _native.lib()
    counts = torch.zeros(2, dtype=torch.int64, device=cuda)
    s = torch.cuda.current_stream().cuda_stream
    rings = [(4, 5), (8, 11), (11, 15), (16, 15), (32, 45), (45, 63), (64, 63), (91, 128), (128, 181), (181, 255),
             (256, 255)]
    for i, (n, d) in enumerate(rings):
        _native.check(L.ss_selftest_cells(1 << 22, 7919 * i + 1, n, d, q[0], q[1], q[2], counts.data_ptr(), s))
    torch.cuda.synchronize()
    assert counts.tolist() == [0, 0]


def test_template_features_device_bitwise(cuda):
    """f2: GPU rescale features == host C++ (== reference, test_native_lib) bit for bit."""
    import torch

    from paper_1707_05647_b200 import Quantizer, ScreeningConfig, build_feature_set, ring_plan
    from paper_1707_05647_b200.featureset import build_feature_sets_device, template_ring_features

    rng = np.random.default_rng(11)
    for trial in range(12):
        n = int(rng.integers(8, 96))
        tpl = rng.integers(0, 256, (n, n), dtype=np.uint8)
        ratio = float(rng.uniform(1.05, 1.5))
        cfg = ScreeningConfig(ladder_ratio=ratio, ring_count=int(rng.integers(1, 6)),
                              quantizer=Quantizer(*rng.uniform(0.5, 10, 3)))
        ms = sorted({int(rng.integers(8, 3 * n)) for _ in range(3)})
        dev = build_feature_sets_device(tpl, ms, cfg, cuda)
        for m in ms:
            host = build_feature_set(tpl, m, cfg)
            for a, b in zip(dev[m].ring_keys(), host.ring_keys()):
                assert np.array_equal(a, b), (trial, m)
    # raw features, every rescale of a 512 patch (config 4's largest size)
    n = 128
    tpl = rng.integers(0, 256, (n, n), dtype=np.uint8)
    from paper_1707_05647_b200 import _native

    plan = ring_plan(512, 3)
    rows = []
    for k in (512, 530, 560):
        d = np.zeros(36, np.int32)
        d[0], d[1], d[2] = 512, k, len(plan)
        for r, (nr, dr) in enumerate(plan):
            d[4 + 2 * r], d[5 + 2 * r] = nr, dr
        rows.append(d)
    out = torch.empty((3, 16, 3), dtype=torch.float64, device=cuda)
    # keep the device copies referenced until the kernel has run (a temporary's
    # memory goes back to the caching allocator as soon as data_ptr() returns)
    d_tpl = torch.from_numpy(tpl).to(cuda)
    d_desc = torch.from_numpy(np.stack(rows)).to(cuda)
    _native.check(_native.lib().ss_template_features_device(
        d_tpl.data_ptr(), n, 3, d_desc.data_ptr(), 36, out.data_ptr(), torch.cuda.current_stream().cuda_stream))
    got = out.cpu().numpy()
    for i, k in enumerate((512, 530, 560)):
        want = template_ring_features(tpl, k, 512, plan)
        assert np.array_equal(got[i, :3].view(np.int64), want.view(np.int64))


def _check_sat_rsat_fast(img, planes):
    """check_planes without the brute-force pass, one kind at a time (the
    reference-layout Rsat of a 4096^2 image is 0.5 GB per kind)."""
    h, w = img.shape
    for k in range(4):
        assert np.array_equal(planes[k], O.build_sat(img, k)), f"SAT kind {k}"
        rs = O.build_rsat(img, k)
        ys, xs = np.mgrid[-1:h, 0:w]
        assert np.array_equal(planes[4 + k][ys + 1, xs + 1], rs[xs + ys + 1, xs - ys + h - 1]), f"E kind {k}"
        ys, xs = np.mgrid[-1:h - 1, -1:w]
        assert np.array_equal(planes[8 + k][ys + 1, xs + 1], rs[xs + ys + 2, xs - ys + h - 1]), f"O kind {k}"
        del rs


@pytest.mark.parametrize("case", ["config1_2048sq", "random_4096x640", "bright_4096sq"])
def test_config_scale_tables(cuda, case):
    """K1/K2 at BASELINE scale, where the many-band carries and the u32
    wraparound actually occur (at 4096^2 the SQUARED SAT reaches ~1.1e12 >
    2^32): int64 planes == the oracle's Sat.cells / Rsat._h, and the 32-bit
    planes == int64 mod 2^32 (device_planes)."""
    if case == "config1_2048sq":
        import workloads as WL

        img = WL.make_cases(WL.CONFIGS[1])[0].image
    elif case == "random_4096x640":
        img = np.random.default_rng(4096).integers(0, 256, (640, 4096), dtype=np.uint8)
    else:
        img = np.random.default_rng(4097).integers(200, 256, (4096, 4096), dtype=np.uint8)
    planes = device_planes(img, cuda)
    if case == "bright_4096sq":
        assert planes[3, -1, img.shape[1]] > 2 ** 32  # the SQUARED plane wraps mod 2^32
    _check_sat_rsat_fast(img, planes)


def test_hi16_planes_are_bits_32_to_47(cuda):
    """ss_build_tables3's hi16 planes = bits 32..47 of the exact int64 cells
    (kinds X, Y, SQUARED; the PLAIN kind needs none)."""
    import torch

    from paper_1707_05647_b200 import _native

    L = _native.lib()
    img = np.random.default_rng(8).integers(150, 256, (1500, 1900), dtype=np.uint8)
    H, W = img.shape
    pitch = int(L.ss_plane_pitch(W))
    p64 = torch.empty(int(L.ss_tables_bytes(W, H)) // 8, dtype=torch.int64, device=cuda)
    p32 = torch.empty(int(L.ss_tables32_bytes(W, H)) // 4, dtype=torch.int32, device=cuda)
    h16 = torch.empty(int(L.ss_tables_hi16_bytes(W, H)) // 2, dtype=torch.int16, device=cuda)
    ws = torch.empty(int(L.ss_build_workspace_bytes(W, H)), dtype=torch.uint8, device=cuda)
    d_img = torch.from_numpy(img).to(cuda)
    sh = np.zeros(1, np.int32)
    _native.check(L.ss_build_tables3(d_img.data_ptr(), W, H, W, p64.data_ptr(), p32.data_ptr(), h16.data_ptr(),
                                     pitch, None, 0, sh.ctypes.data, ws.data_ptr(), ws.numel(),
                                     torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    full = p64.view(12, H + 1, pitch).cpu().numpy()[:, :, : W + 1]
    hi = h16.view(12, H + 1, pitch).cpu().numpy().view(np.uint16)[:, :, : W + 1]
    lo = p32.view(12, H + 1, pitch).cpu().numpy().view(np.uint32)[:, :, : W + 1]
    assert full.max() >= 1 << 32  # the SQUARED / weighted cells do reach past 32 bits here
    kinds = [p for p in range(12) if p % 4 != 0]  # PLAIN ring sums stay below 2^32: no hi16 for kind 0
    assert np.array_equal(hi[kinds], ((full[kinds] >> 32) & 0xFFFF).astype(np.uint16))
    assert np.array_equal(lo, (full & 0xFFFFFFFF).astype(np.uint32))
