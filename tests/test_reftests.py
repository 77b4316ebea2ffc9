"""The reference's own hot-path screen tests, replayed through this repo.

Source tests (the reference's assertions, restated here over fixtures the
reference generated -- tests/golden/reftests.npz, make_golden.py
`reftests_fixture`):
  * pkg/tests/test_screening.py:265-397 (TestScreen): result structure,
    never-miss exact crops, pasted templates at the borders, candidate
    ordering, masks / region consistency, border keeps, tiny-ladder keeps,
    the tested-count formula, scan == exhaustive scalar membership, stride
    subset, determinism;
  * pkg/tests/test_acceptance.py:205-234 (criterion 4: the exact-crop centre
    survives in 100/100 screens) and :270-282 (criterion 6: median screen time
    on a 640x480 scene <= 1 s).

Each case runs twice: through the CPU oracle (no GPU; pins the checker) and,
under ``-m gpu``, through the drop-in ``paper_1707_05647_b200.screen`` (the
CUDA path over the C ABI).  Besides the reference's own assertions, every
result must equal the reference's stored result bit for bit (candidates,
every size mask, region, stats); the 100 criterion-4 screens are compared by
sha256 digest of the same fields.
"""

import hashlib
import json
import time

import numpy as np
import pytest

import oracle as O
from conftest import golden, packbits

IMPLS = ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)]
MIN_PATCH_SIDE = 8


class R:
    """One screen result in plain arrays (oracle or GPU)."""

    def __init__(self, ladder, cands, masks, region, stats):
        self.ladder = tuple(int(m) for m in ladder)
        self.cands = np.asarray(cands, np.int32).reshape(-1, 3)
        self.masks = masks
        self.region = region
        self.tested, self.kept, self.region_px, self.total = (int(v) for v in stats)

    def cand_set(self):
        return {tuple(int(v) for v in c) for c in self.cands}

    def digest(self):
        h = hashlib.sha256()
        h.update(self.cands.tobytes())
        for m in self.ladder:
            h.update(packbits(self.masks[m]).tobytes())
        h.update(packbits(self.region).tobytes())
        return h.hexdigest()


def _run(impl, image, template, kw, cuda=None):
    kw = dict(kw)
    if impl == "oracle":
        if "quantizer" in kw:
            kw["quantizer"] = O.Quantizer(*kw["quantizer"])
        r = O.screen(image, template, O.ScreeningConfig(**kw), nthreads=4)
        return R(r.ladder, np.array(r.candidates, np.int32), r.size_masks, r.region_mask,
                 (r.patches_tested, r.patches_kept, r.region_pixels_kept, r.total_pixels))
    from paper_1707_05647_b200 import Quantizer, ScreeningConfig, screen

    if "quantizer" in kw:
        kw["quantizer"] = Quantizer(*kw["quantizer"])
    r = screen(image, template, ScreeningConfig(**kw), device=cuda)
    st = r.stats
    assert st.patches_kept == len(r.candidates)
    return R(r.ladder, r.candidates.array(), {m: r.size_masks[m] for m in r.ladder}, r.region_mask,
             (st.patches_tested, st.patches_kept, st.region_pixels_kept, st.total_pixels))


@pytest.fixture(scope="module")
def z():
    return golden("reftests.npz")


def _case(z, key):
    return z[f"{key}/image"], z[f"{key}/template"], json.loads(str(z[f"{key}/cfg"]))


def _golden_eq(z, key, r):
    assert r.ladder == tuple(int(m) for m in z[f"{key}/ladder"])
    assert np.array_equal(r.cands, z[f"{key}/candidates"])
    for m in r.ladder:
        assert np.array_equal(packbits(r.masks[m]), z[f"{key}/mask_{m}"]), f"{key}: mask m={m}"
    assert np.array_equal(packbits(r.region), z[f"{key}/region"]), f"{key}: region"
    assert (r.tested, r.kept, r.region_px, r.total) == tuple(int(v) for v in z[f"{key}/stats"])


def run(impl, z, key, request):
    cuda = request.getfixturevalue("cuda") if impl == "gpu" else None
    img, tpl, kw = _case(z, key)
    r = _run(impl, img, tpl, kw, cuda)
    _golden_eq(z, key, r)
    return r


def margins(m):
    return (m - 1) // 2, m // 2


@pytest.mark.parametrize("impl", IMPLS)
def test_result_structure(impl, z, request):  # test_screening.py:265-276
    r = run(impl, z, "structure", request)
    assert r.ladder == (64, 45, 32, 23, 16)
    assert set(r.masks) == set(r.ladder)
    assert r.region.shape == (72, 96)
    assert r.kept == len(r.cands)
    assert r.total == 96 * 72


@pytest.mark.parametrize("impl", IMPLS)
def test_never_misses_exact_crop(impl, z, request):  # test_screening.py:278-289
    for i, (cx, cy) in enumerate(z["crop_xy"]):
        r = run(impl, z, f"crop{i}", request)
        assert (cx, cy, 32) in r.cand_set()
        assert r.masks[32][cy, cx]
        assert r.region[cy, cx]


@pytest.mark.parametrize("impl", IMPLS)
def test_pasted_template_found_at_borders(impl, z, request):  # test_screening.py:291-297
    for i, (cx, cy) in enumerate(z["paste_xy"]):
        r = run(impl, z, f"paste{i}", request)
        assert (cx, cy, 32) in r.cand_set()


@pytest.mark.parametrize("impl", IMPLS)
def test_candidate_ordering(impl, z, request):  # test_screening.py:299-308
    r = run(impl, z, "ordering", request)
    order = {m: i for i, m in enumerate(r.ladder)}
    sizes = [int(m) for m in r.cands[:, 2]]
    assert sizes == sorted(sizes, key=lambda m: order[m])
    for m in r.ladder:
        pts = [(int(cy), int(cx)) for cx, cy, mm in r.cands if mm == m]
        assert pts == sorted(pts)


@pytest.mark.parametrize("impl", IMPLS)
def test_masks_and_region_consistent(impl, z, request):  # test_screening.py:310-323
    r = run(impl, z, "region", request)
    want = np.zeros_like(r.region)
    for cx, cy, m in r.cands:
        assert r.masks[int(m)][cy, cx]
        lo, hi = margins(int(m))
        want[cy - lo:cy + hi + 1, cx - lo:cx + hi + 1] = True
    assert np.array_equal(r.region, want)
    assert r.region_px == int(want.sum())


@pytest.mark.parametrize("impl", IMPLS)
def test_border_centers_kept_in_size_masks_only(impl, z, request):  # test_screening.py:325-334
    r = run(impl, z, "border", request)
    for m in r.ladder:
        if m < MIN_PATCH_SIDE:
            continue
        assert r.masks[m][0, :].all() and r.masks[m][:, 0].all()
    assert all(cx > 0 and cy > 0 for cx, cy, _ in r.cands)


@pytest.mark.parametrize("impl", IMPLS)
def test_tiny_ladder_sizes_keep_everything(impl, z, request):  # test_screening.py:336-345
    r = run(impl, z, "tiny", request)
    assert r.ladder == (16, 11, 8, 6, 4)
    for m in (6, 4):
        assert r.masks[m].all()
        assert not (r.cands[:, 2] == m).any()


@pytest.mark.parametrize("impl", IMPLS)
def test_tested_count_matches_grid(impl, z, request):  # test_screening.py:347-358
    r = run(impl, z, "tested", request)
    want = 0
    for m in r.ladder:
        if m < MIN_PATCH_SIDE:
            continue
        lo, hi = margins(m)
        want += max(0, 96 - hi - lo) * max(0, 80 - hi - lo)
    assert r.tested == want


@pytest.mark.parametrize("impl", IMPLS)
def test_scan_equals_exhaustive_membership(impl, z, request):  # test_screening.py:360-377
    """The reference's scalar path (ring_features + FeatureSet.contains at
    every interior centre, stored by the generator) decides the same set."""
    r = run(impl, z, "exhaustive", request)
    assert r.ladder == (32,)
    got = {(int(cx), int(cy)) for cx, cy, _ in r.cands}
    want = {(int(cx), int(cy)) for cx, cy in z["exhaustive_want"]}
    assert got == want


@pytest.mark.parametrize("impl", IMPLS)
def test_stride(impl, z, request):  # test_screening.py:379-387
    r1 = run(impl, z, "stride1", request)
    r3 = run(impl, z, "stride3", request)
    assert all(cx % 3 == 0 and cy % 3 == 0 for cx, cy, _ in r3.cands)
    assert r3.tested < r1.tested
    sub = {c for c in r1.cand_set() if c[0] % 3 == 0 and c[1] % 3 == 0}
    assert r3.cand_set() == sub


@pytest.mark.parametrize("impl", IMPLS)
def test_determinism(impl, z, request):  # test_screening.py:389-397
    a = run(impl, z, "determinism", request)
    b = run(impl, z, "determinism", request)
    assert np.array_equal(a.cands, b.cands)
    assert np.array_equal(a.region, b.region)
    for m in a.ladder:
        assert np.array_equal(a.masks[m], b.masks[m])


@pytest.mark.parametrize("impl", IMPLS)
def test_criterion_4_never_miss(impl, z, request):  # test_acceptance.py:205-234
    """100 exact-crop screens (10 scenes x 10 crops): the crop centre is kept
    in every one, and each full result equals the reference's (digest)."""
    cuda = request.getfixturevalue("cuda") if impl == "gpu" else None
    kept = 0
    for i, (si, cx, cy, ref_kept, n_cand, tested, region_px) in enumerate(z["c4_cases"]):
        scene = z[f"c4_scene{si}"]
        r = _run(impl, scene, scene[cy - 15:cy + 17, cx - 15:cx + 17], {}, cuda)
        kept += int((int(cx), int(cy), 32) in r.cand_set())
        assert (len(r.cands), r.tested, r.region_px) == (n_cand, tested, region_px)
        assert r.digest() == str(z[f"c4_digest{i}"]), f"case {i}"
    assert kept == len(z["c4_cases"]) == int(z["c4_cases"][:, 3].sum()) == 100


@pytest.mark.gpu
def test_criterion_6_screen_speed(z, cuda):  # test_acceptance.py:270-282
    from paper_1707_05647_b200 import screen

    img, tpl, kw = _case(z, "speed640")
    r = _run("gpu", img, tpl, kw, cuda)
    _golden_eq(z, "speed640", r)
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        screen(img, tpl)
        times.append(time.perf_counter() - t0)
    assert sorted(times)[1] <= 1.0
