"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Every array written here comes from the reference's own code
(/root/reference/pkg/src/starscreen): integral tables, ring features,
feature-set keys, complete screen() results, and the survivor counts of
pkg/demos/out/report.json (re-derived through run_benchmark's own case
generator).  The config-0 case uses this repo's workloads.py generator for
the input image, screened by the reference.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from starscreen import integral as I  # noqa: E402
from starscreen import features as F  # noqa: E402
from starscreen import screening as S  # noqa: E402
from starscreen.synth_bench import _case_seed, make_case, make_textured_scene  # noqa: E402

KINDS = list(I.WeightKind)


def packbits(mask: np.ndarray) -> np.ndarray:
    return np.packbits(mask.astype(np.uint8), axis=-1, bitorder="little")


def tables_fixture():
    rng = np.random.default_rng(20261019)
    imgs = [np.array([[1, 2], [3, 4]], np.uint8), np.full((1, 1), 255, np.uint8),
            rng.integers(0, 256, (1, 9), dtype=np.uint8), rng.integers(0, 256, (9, 1), dtype=np.uint8),
            rng.integers(0, 256, (5, 7), dtype=np.uint8), rng.integers(0, 256, (17, 13), dtype=np.uint8),
            rng.integers(0, 256, (20, 33), dtype=np.uint8), np.full((11, 6), 255, np.uint8),
            make_textured_scene(70, 45, seed=3)]
    out = {}
    for i, img in enumerate(imgs):
        t = I.build_tables(img)
        out[f"img{i}"] = img
        for k, kind in enumerate(KINDS):
            out[f"sat{i}_{k}"] = t.sats[kind].cells
            out[f"rsat{i}_{k}"] = t.rsats[kind].table
    out["n"] = np.array(len(imgs))
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **out)


def features_fixture():
    scene = make_textured_scene(64, 48, seed=1)
    t = I.build_tables(scene)
    out = {"scene": scene}
    for m in (32, 17, 8):
        plan = F.ring_plan(m, 3)
        lo, hi = F.patch_center_margins(m)
        cys, cxs = np.mgrid[lo:48 - hi, lo:64 - hi]
        maps = F.ring_feature_maps(t, cxs.ravel(), cys.ravel(), plan)
        out[f"plan_{m}"] = np.array(plan, np.int32)
        out[f"centers_{m}"] = np.stack([cxs.ravel(), cys.ravel()], 1).astype(np.int32)
        out[f"feat_{m}"] = np.stack([np.stack(mp, 1) for mp in maps], 1)  # (N, rings, 3)
    np.savez_compressed(os.path.join(HERE, "features.npz"), **out)


FS_CASES = [
    # (template seed, side, m, ladder_ratio, quantizer)
    (3, 32, 32, math.sqrt(2.0), (8.0, 8.0, 8.0)),
    (3, 32, 45, math.sqrt(2.0), (8.0, 8.0, 8.0)),
    (4, 20, 8, math.sqrt(2.0), (8.0, 8.0, 8.0)),
    (5, 64, 128, 4.0 ** (1 / 7), (8.0, 8.0, 8.0)),
    (6, 48, 33, (8 / 3) ** (1 / 7), (8.0, 8.0, 8.0)),
    (7, 32, 32, math.sqrt(2.0), (8.0, 8.0, 1e6)),
    (8, 24, 24, 1.05, (2.5, 0.75, 0.001)),
]


def featuresets_fixture():
    out = {}
    for i, (seed, side, m, ratio, q) in enumerate(FS_CASES):
        tpl = make_textured_scene(side, side, seed=seed)
        cfg = S.ScreeningConfig(ladder_ratio=ratio, quantizer=S.Quantizer(*q))
        fs = S.build_feature_set(tpl, m, cfg)
        out[f"tpl{i}"] = tpl
        out[f"meta{i}"] = np.array([m, ratio, *q], np.float64)
        for r, keys in enumerate(fs.ring_keys()):
            out[f"keys{i}_{r}"] = keys
        out[f"nrings{i}"] = np.array(len(fs.plan))
    out["n"] = np.array(len(FS_CASES))
    np.savez_compressed(os.path.join(HERE, "featuresets.npz"), **out)


def screen_cases():
    """(name, image, template, cfg kwargs) -- the reference tests' scenes plus extras."""
    cases = []
    s = make_textured_scene(96, 72, seed=4)
    cases.append(("t4_default", s, s[20:52, 30:62].copy(), {}))
    s = make_textured_scene(72, 56, seed=13)
    cases.append(("t13_single", s, s[12:44, 20:52].copy(), {"alpha": 1.0, "beta": 1.0}))
    s = make_textured_scene(96, 80, seed=14)
    cases.append(("t14_stride3", s, s[24:56, 24:56].copy(), {"stride": 3}))
    s = make_textured_scene(64, 64, seed=11)
    cases.append(("t11_tiny", s, s[28:36, 28:36].copy(), {}))
    s = make_textured_scene(160, 120, seed=5)
    cases.append(("t5_q", s, s[40:72, 50:82].copy(), {"quantizer": (6.0, 4.0, 3.0), "ladder_ratio": 1.25}))
    s = make_textured_scene(131, 97, seed=21)
    cases.append(("t21_odd", s, s[30:57, 40:67].copy(), {"alpha": 0.6, "beta": 1.7, "ring_count": 4}))
    s = make_textured_scene(40, 200, seed=22)
    cases.append(("t22_tall", s, s[100:116, 10:26].copy(), {"stride": 2}))
    s = make_textured_scene(100, 100, seed=6)
    cases.append(("t6_big_m", s, make_textured_scene(32, 32, seed=7), {"beta": 3.5, "alpha": 0.3}))
    # config-0-like input from this repo's generator (BASELINE config 0)
    import workloads as WL

    c0 = WL.make_cases(WL.CONFIGS[0])[0]
    cases.append(("config0", c0.image, c0.template,
                   {"alpha": 1.0, "beta": 1.0, "quantizer": (8.0, 8.0, 1e6)}))
    return cases


def _cfg(kw):
    kw = dict(kw)
    if "quantizer" in kw:
        kw["quantizer"] = S.Quantizer(*kw["quantizer"])
    return S.ScreeningConfig(**kw)


def screens_fixture():
    out = {}
    names = []
    for name, img, tpl, kw in screen_cases():
        res = S.screen(img, tpl, _cfg(kw))
        names.append(name)
        out[f"{name}/image"] = img
        out[f"{name}/template"] = tpl
        out[f"{name}/cfg"] = np.array(json.dumps(kw))
        out[f"{name}/ladder"] = np.array(res.ladder, np.int32)
        out[f"{name}/candidates"] = np.array(res.candidates, np.int32).reshape(-1, 3)
        for m in res.ladder:
            out[f"{name}/mask_{m}"] = packbits(res.size_masks[m])
        out[f"{name}/region"] = packbits(res.region_mask)
        st = res.stats
        out[f"{name}/stats"] = np.array([st.patches_tested, st.patches_kept, st.region_pixels_kept, st.total_pixels],
                                        np.int64)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "screens.npz"), **out)


def report_fixture():
    """pkg/demos/out/report.json cases: 6 scenes x 2 cases, run_benchmark(seed=1)."""
    with open("/root/reference/pkg/demos/out/report.json") as fh:
        report = json.load(fh)
    out = {}
    idx = 0
    for img_idx in range(6):
        scene = make_textured_scene(320, 240, seed=600 + img_idx)
        out[f"scene{img_idx}"] = scene
        for case_idx in range(2):
            tpl, truth = make_case(scene, _case_seed(1, img_idx, case_idx))
            rec = report["cases"][idx]
            assert rec["image"] == f"scene{img_idx}.pgm" and rec["case"] == case_idx
            res = S.screen(scene, tpl)
            assert len(res.candidates) == rec["candidates"], (idx, len(res.candidates), rec["candidates"])
            assert res.stats.patch_pruning == rec["patch_pruning"]
            assert res.stats.region_pruning == rec["region_pruning"]
            out[f"tpl{idx}"] = tpl
            out[f"expect{idx}"] = np.array([img_idx, rec["candidates"], res.stats.patches_tested,
                                            res.stats.region_pixels_kept], np.int64)
            out[f"pruning{idx}"] = np.array([rec["patch_pruning"], rec["region_pruning"]], np.float64)
            idx += 1
    out["n"] = np.array(idx)
    np.savez_compressed(os.path.join(HERE, "report_cases.npz"), **out)


def frozen_fixture():
    """Small frozen values the reference tests pin (ladders, plans, radii, quantize)."""
    cfg = S.ScreeningConfig()
    out = {
        "ladders": {str(n): list(S.ladder_sizes(n, cfg)) for n in (8, 20, 32, 48, 64, 96, 128)},
        "ladders_cfg": {
            "a1b1": list(S.ladder_sizes(32, S.ScreeningConfig(alpha=1.0, beta=1.0))),
            "a09b11": list(S.ladder_sizes(32, S.ScreeningConfig(alpha=0.9, beta=1.1))),
            "a2b2": list(S.ladder_sizes(32, S.ScreeningConfig(alpha=2.0, beta=2.0))),
        },
        "plans": {str(m): [list(p) for p in F.ring_plan(m, 3)] for m in (8, 11, 16, 17, 32, 45, 64, 128, 512)},
        "plans5": {str(m): [list(p) for p in F.ring_plan(m, 5)] for m in (32, 77, 512)},
        "radius": {str(n): F.default_star_radius(n) for n in (4, 8, 11, 16, 64, 181)},
        "quantize": [[v, q, S.quantize(v, q)] for v, q in ((12.0, 8.0), (11.999, 8.0), (4.0, 8.0), (3.999, 8.0),
                                                         (0.0, 8.0), (-3.0, 8.0), (7.5, 5.0), (1e6 - 1, 1e6))],
    }
    import workloads as WL

    out["config_ladders"] = {}
    for i, wl in WL.CONFIGS.items():
        c = S.ScreeningConfig(alpha=wl.alpha, beta=wl.beta, ladder_ratio=wl.ladder_ratio,
                              quantizer=S.Quantizer(*wl.q))
        out["config_ladders"][str(i)] = list(S.ladder_sizes(wl.template_side, c))
    with open(os.path.join(HERE, "frozen.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def io_fixture():
    """f4 wire formats, written by the reference's own functions: the stats
    JSON of `starscreen screen` (cli.py:101-134, write_json_atomic
    synth_bench.py:314-326; screen_time zeroed -- the only run-dependent
    field), the region / size-mask PGM files (cli.py:97-98, save_pgm
    image_io.py:108-128), and load_pgm on the header variants the reference
    tests parse (pkg/tests/test_image_io.py:61-109)."""
    import dataclasses
    import tempfile

    from starscreen import cli as C
    from starscreen import image_io as IO
    from starscreen.synth_bench import write_json_atomic

    out = {}
    cases = {name: (img, tpl, kw) for name, img, tpl, kw in screen_cases()}
    names = ["t4_default", "t21_odd", "t22_tall"]
    with tempfile.TemporaryDirectory() as d:
        for name in names:
            img, tpl, kw = cases[name]
            res = S.screen(img, tpl, _cfg(kw))
            res = dataclasses.replace(res, stats=dataclasses.replace(res.stats, wall_time_s=0.0))
            payload = C._screen_stats_payload("scene.pgm", "template.pgm", res)
            write_json_atomic(os.path.join(d, "stats.json"), payload)
            out[f"{name}/stats_json"] = np.frombuffer(open(os.path.join(d, "stats.json"), "rb").read(), np.uint8)
            IO.save_pgm(os.path.join(d, "region.pgm"), C._mask_to_pgm(res.region_mask))
            out[f"{name}/region_pgm"] = np.frombuffer(open(os.path.join(d, "region.pgm"), "rb").read(), np.uint8)
            for m in (res.ladder[0], res.ladder[-1]):
                IO.save_pgm(os.path.join(d, "m.pgm"), C._mask_to_pgm(res.size_masks[m]))
                out[f"{name}/mask_pgm_{m}"] = np.frombuffer(open(os.path.join(d, "m.pgm"), "rb").read(), np.uint8)
        blobs = [b"P5 # magic\n# a comment line\n  3\t2 # dims\n255\n" + bytes(range(6)),
                 b"P5\n2 1\n15\n" + bytes([3, 15]),
                 b"P5\n7 3\n255\n" + bytes(range(21)),
                 b"P2\n2 2\n255\n" + b"\x00" * 4, b"P5\n2 2\n300\n" + b"\x00" * 4, b"P5\n2 2\n0\n" + b"\x00" * 4,
                 b"P5\n0 2\n255\n", b"P5\n2 2\n255\n\x00\x00", b"P5\n2\n", b"P5\nab 2\n255\n" + b"\x00" * 4,
                 b"P6 junk"]
        for i, blob in enumerate(blobs):
            path = os.path.join(d, "in.pgm")
            open(path, "wb").write(blob)
            out[f"pgm_in{i}"] = np.frombuffer(blob, np.uint8)
            try:
                out[f"pgm_out{i}"] = IO.load_pgm(path)
            except IO.PgmError as e:
                out[f"pgm_err{i}"] = np.array(str(e))
        out["pgm_n"] = np.array(len(blobs))
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "io.npz"), **out)


def match_fixture():
    """f3: the reference's match_candidates (second_stage.py:168-204) on the
    reference's own screens -- golden screen cases and report.json scenes."""
    from starscreen import second_stage as M

    out = {}
    names = []
    cases = {name: (img, tpl, kw) for name, img, tpl, kw in screen_cases()}
    jobs = [("t4_default", 10.0), ("t5_q", 10.0), ("t21_odd", 30.0), ("t14_stride3", 45.0), ("t13_single", 10.0),
            ("t6_big_m", 10.0), ("t22_tall", 20.0), ("t6_big_m", 5.0), ("t21_odd", 4.0)]
    for name, step in jobs:
        img, tpl, kw = cases[name]
        res = S.screen(img, tpl, _cfg(kw))
        r = M.match_candidates(img, tpl, res, angle_step=step)
        key = f"{name}@{step:g}"
        names.append(key)
        out[f"{key}/step"] = np.array(step)
        out[f"{key}/result"] = np.array([r.cx, r.cy, r.scale, r.angle, r.score], np.float64)
    for img_idx, case_idx in ((0, 0), (3, 1), (5, 0), (2, 1)):
        scene = make_textured_scene(320, 240, seed=600 + img_idx)
        tpl, _ = make_case(scene, _case_seed(1, img_idx, case_idx))
        res = S.screen(scene, tpl)
        r = M.match_candidates(scene, tpl, res)
        key = f"scene{img_idx}_case{case_idx}"
        names.append(key)
        out[f"{key}/image"] = scene
        out[f"{key}/template"] = tpl
        out[f"{key}/step"] = np.array(10.0)
        out[f"{key}/result"] = np.array([r.cx, r.cy, r.scale, r.angle, r.score], np.float64)
    # ladder sizes whose I x P dot products pass 2^31 (m >= 182): the GPU
    # kernel drains that accumulator into int64 every few window rows
    flush = {"flush192": (300, 260, 777, 80, 100, 96, 30.0), "flush264": (380, 330, 778, 100, 120, 132, 45.0)}
    for key, (w, h, seed, y0, x0, side, step) in flush.items():
        scene = make_textured_scene(w, h, seed=seed)
        tpl = np.ascontiguousarray(scene[y0:y0 + side, x0:x0 + side])
        kw = {"alpha": 1.9, "beta": 2.0, "quantizer": (16.0, 16.0, 16.0)}
        res = S.screen(scene, tpl, _cfg(kw))
        r = M.match_candidates(scene, tpl, res, angle_step=step)
        names.append(key)
        out[f"{key}/image"] = scene
        out[f"{key}/template"] = tpl
        out[f"{key}/cfg"] = np.array(json.dumps(kw))
        out[f"{key}/step"] = np.array(step)
        out[f"{key}/result"] = np.array([r.cx, r.cy, r.scale, r.angle, r.score], np.float64)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "match.npz"), **out)


def _digest(res):
    """sha256 over the reference result's candidates, packed size masks (ladder
    order) and packed region -- compact pin for the 100 criterion-4 screens."""
    import hashlib

    h = hashlib.sha256()
    h.update(np.array(res.candidates, np.int32).reshape(-1, 3).tobytes())
    for m in res.ladder:
        h.update(packbits(res.size_masks[m]).tobytes())
    h.update(packbits(res.region_mask).tobytes())
    return h.hexdigest()


def _paste(scene, tpl, cx, cy):
    """pkg/tests/test_screening.py:_paste -- tpl's window centre lands on (cx, cy)."""
    out = scene.copy()
    m = tpl.shape[0]
    lo, _ = F.patch_center_margins(m)
    out[cy - lo:cy - lo + m, cx - lo:cx - lo + m] = tpl
    return out


def reftests_fixture():
    """The reference's own hot-path screen tests, as input/output fixtures:
    pkg/tests/test_screening.py:265-397 (TestScreen: structure, never-miss
    exact crops, pasted templates at the borders, ordering, masks/region
    consistency, border keeps, tiny ladder, tested-count formula, scan ==
    exhaustive scalar membership, stride subset, determinism) and
    pkg/tests/test_acceptance.py:205-234 (criterion 4: 100 exact-crop screens,
    10 scenes x 10 crops) and :270-282 (criterion 6 scene).  Every screen is
    run through the REFERENCE; its full result (or, for the 100 criterion-4
    screens, a sha256 digest of it) is stored with the inputs."""
    out = {}
    full = []  # (key, image, template, cfg kwargs): full results stored

    def add(key, img, tpl, kw=None):
        kw = kw or {}
        res = S.screen(img, tpl, _cfg(kw))
        full.append(key)
        out[f"{key}/image"] = img
        out[f"{key}/template"] = tpl
        out[f"{key}/cfg"] = np.array(json.dumps(kw))
        out[f"{key}/ladder"] = np.array(res.ladder, np.int32)
        out[f"{key}/candidates"] = np.array(res.candidates, np.int32).reshape(-1, 3)
        for m in res.ladder:
            out[f"{key}/mask_{m}"] = packbits(res.size_masks[m])
        out[f"{key}/region"] = packbits(res.region_mask)
        st = res.stats
        out[f"{key}/stats"] = np.array([st.patches_tested, st.patches_kept, st.region_pixels_kept, st.total_pixels],
                                       np.int64)
        return res

    s = make_textured_scene(96, 72, seed=4)  # test_result_structure
    add("structure", s, s[20:52, 30:62].copy())
    # test_never_misses_exact_crop: 10 crops, rng 34
    s = make_textured_scene(160, 120, seed=5)
    rng = np.random.default_rng(34)
    lo, hi = F.patch_center_margins(32)
    crops = []
    for i in range(10):
        cx = int(rng.integers(lo, 160 - hi))
        cy = int(rng.integers(lo, 120 - hi))
        add(f"crop{i}", s, s[cy - lo:cy - lo + 32, cx - lo:cx - lo + 32].copy())
        crops.append((cx, cy))
    out["crop_xy"] = np.array(crops, np.int32)
    # test_pasted_template_found_at_borders
    s = make_textured_scene(100, 100, seed=6)
    tpl = make_textured_scene(32, 32, seed=7)
    pasted = [(lo, lo), (99 - hi, lo), (lo, 99 - hi), (99 - hi, 99 - hi)]
    for i, (cx, cy) in enumerate(pasted):
        add(f"paste{i}", _paste(s, tpl, cx, cy), tpl)
    out["paste_xy"] = np.array(pasted, np.int32)
    s = make_textured_scene(128, 96, seed=8)  # test_candidate_ordering
    add("ordering", s, s[30:62, 40:72].copy())
    s = make_textured_scene(96, 80, seed=9)  # test_masks_and_region_consistent
    add("region", s, s[24:56, 24:56].copy())
    s = make_textured_scene(90, 70, seed=10)  # test_border_centers_kept_in_size_masks_only
    add("border", s, s[20:52, 20:52].copy())
    s = make_textured_scene(64, 64, seed=11)  # test_tiny_ladder_sizes_keep_everything
    add("tiny", s, s[28:36, 28:36].copy())
    s = make_textured_scene(96, 80, seed=12)  # test_tested_count_matches_grid
    add("tested", s, s[24:56, 24:56].copy())
    # test_scan_equals_exhaustive_membership: the scalar path's survivor set
    s = make_textured_scene(72, 56, seed=13)
    tpl = s[12:44, 20:52].copy()
    kw = {"alpha": 1.0, "beta": 1.0}
    add("exhaustive", s, tpl, kw)
    fs = S.build_feature_set(tpl, 32, _cfg(kw))
    t = I.build_tables(s)
    want = [(cx, cy) for cy in range(lo, 56 - hi) for cx in range(lo, 72 - hi)
            if fs.contains(F.ring_features(t, cx, cy, 32))]
    out["exhaustive_want"] = np.array(want, np.int32).reshape(-1, 2)
    s = make_textured_scene(96, 80, seed=14)  # test_stride
    add("stride1", s, s[24:56, 24:56].copy(), {"stride": 1})
    add("stride3", s, s[24:56, 24:56].copy(), {"stride": 3})
    s = make_textured_scene(100, 90, seed=15)  # test_determinism
    add("determinism", s, s[30:62, 30:62].copy())
    s = make_textured_scene(640, 480, seed=99)  # test_criterion_6_screen_speed
    tpl, _ = make_case(s, seed=1, scale_range=(1.0, 1.0))
    add("speed640", s, tpl)
    # criterion 4 (test_acceptance.py:205-234): 100 screens, digests only
    c4 = []
    for si in range(10):
        scene = make_textured_scene(160, 120, seed=7000 + si)
        out[f"c4_scene{si}"] = scene
        rng = np.random.default_rng(np.random.SeedSequence([7100, si]))
        for c in range(10):
            cx = int(rng.integers(15, 144))
            cy = int(rng.integers(15, 104))
            res = S.screen(scene, scene[cy - 15:cy + 17, cx - 15:cx + 17])
            kept = (cx, cy, 32) in set(res.candidates)
            c4.append((si, cx, cy, int(kept), len(res.candidates), res.stats.patches_tested,
                       res.stats.region_pixels_kept))
            out[f"c4_digest{len(c4) - 1}"] = np.array(_digest(res))
    out["c4_cases"] = np.array(c4, np.int64)
    out["full"] = np.array(full)
    np.savez_compressed(os.path.join(HERE, "reftests.npz"), **out)


FIXTURES = {"tables": tables_fixture, "features": features_fixture, "featuresets": featuresets_fixture,
            "screens": screens_fixture, "report": report_fixture, "frozen": frozen_fixture, "io": io_fixture,
            "match": match_fixture, "reftests": reftests_fixture}

if __name__ == "__main__":
    for name in (sys.argv[1:] or list(FIXTURES)):
        FIXTURES[name]()
    print("golden fixtures written to", HERE)
