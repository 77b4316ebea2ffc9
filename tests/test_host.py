"""Host logic of the drop-in: config, ladder, ring plans, quantize,
FeatureSet semantics and validation -- the reference tests' frozen values
(pkg/tests/test_screening.py, test_features.py) on this package."""

import numpy as np
import pytest

from conftest import frozen

import paper_1707_05647_b200 as P


def test_frozen_ladders_plans_radii_quantize():
    f = frozen()
    cfg = P.ScreeningConfig()
    for n, lad in f["ladders"].items():
        assert list(P.ladder_sizes(int(n), cfg)) == lad
    assert list(P.ladder_sizes(32, P.ScreeningConfig(alpha=1.0, beta=1.0))) == f["ladders_cfg"]["a1b1"] == [32]
    assert list(P.ladder_sizes(32, P.ScreeningConfig(alpha=0.9, beta=1.1))) == f["ladders_cfg"]["a09b11"] == [35, 32]
    assert list(P.ladder_sizes(32, P.ScreeningConfig(alpha=2.0, beta=2.0))) == f["ladders_cfg"]["a2b2"] == [64]
    for m, plan in f["plans"].items():
        assert [list(p) for p in P.ring_plan(int(m), 3)] == plan
    assert P.ring_plan(32, 3) == ((16, 15), (11, 15), (8, 11))
    for m, plan in f["plans5"].items():
        assert [list(p) for p in P.ring_plan(int(m), 5)] == plan
    for n, r in f["radius"].items():
        assert P.default_star_radius(int(n)) == r
    for v, q, c in f["quantize"]:
        assert P.quantize(v, q) == c


def test_config_ladders_of_the_five_workloads():
    import workloads as WL

    f = frozen()
    for i, wl in WL.CONFIGS.items():
        assert list(P.ladder_sizes(wl.template_side, WL.screening_config(wl))) == f["config_ladders"][str(i)]
    assert len(f["config_ladders"]["4"]) == 33 and len(f["config_ladders"]["2"]) == 17


def test_config_validation():
    with pytest.raises(ValueError):
        P.ScreeningConfig(alpha=2.0, beta=1.0)
    with pytest.raises(ValueError):
        P.ScreeningConfig(alpha=0.0)
    with pytest.raises(ValueError):
        P.ScreeningConfig(ladder_ratio=1.0)
    with pytest.raises(ValueError):
        P.ScreeningConfig(ring_count=0)
    with pytest.raises(ValueError):
        P.ScreeningConfig(stride=0)
    with pytest.raises(ValueError):
        P.ladder_sizes(0, P.ScreeningConfig())
    with pytest.raises(ValueError):
        P.Quantizer(q_mean=0.0)
    assert P.Quantizer().factors() == (8.0, 8.0, 8.0)


def test_feature_set_guard_band_and_contains():
    plan = P.ring_plan(32, 3)
    fs = P.FeatureSet(plan, P.Quantizer())
    fv = P.RingFeatureVector(tuple(P.RingBand(n, d, 100.0 + n, 20.0, 5.0) for n, d in plan))
    assert not fs.contains(fv)
    fs.insert(fv)
    assert fs.contains(fv)
    assert all(1 <= s <= 27 for s in fs.ring_sizes())
    rng = np.random.default_rng(30)
    for _ in range(500):
        d = rng.uniform(-4.0, 4.0, 3)
        near = P.RingFeatureVector(tuple(P.RingBand(n, r, 100.0 + n + d[0], 20.0 + d[1], 5.0 + d[2]) for n, r in plan))
        assert fs.contains(near)
    far = P.RingFeatureVector(tuple(P.RingBand(n, r, 100.0 + n + 16.0, 20.0, 5.0) for n, r in plan))
    assert not fs.contains(far)
    with pytest.raises(ValueError):
        P.FeatureSet([], P.Quantizer())
    big = P.FeatureSet([(8, 11)], P.Quantizer(q_mean=0.001))
    with pytest.raises(ValueError, match="capacity"):
        big.insert(P.RingFeatureVector((P.RingBand(8, 11, 0.001 * (P.config.KEY_BASE + 10), 1.0, 1.0),)))


def test_validation_errors_before_any_device_work():
    scene = np.random.default_rng(1).integers(0, 256, (64, 64), dtype=np.uint8)
    with pytest.raises(P.FlatTemplateError, match="too flat"):
        P.screen(scene, np.full((32, 32), 128, np.uint8))
    assert issubclass(P.FlatTemplateError, ValueError)
    with pytest.raises(ValueError, match="square"):
        P.screen(scene, scene[:16, :20])
    with pytest.raises(ValueError, match="below minimum"):
        P.screen(scene, scene[:4, :4])
    with pytest.raises(ValueError, match="2-D"):
        P.screen(scene[None], scene[:16, :16])
    with pytest.raises(ValueError, match="outside"):
        P.screen(scene.astype(np.int32) + 300, scene[:16, :16])
    assert P.std_dev(np.full((4, 4), 7, np.uint8)) == 0.0


def test_prune_stats_ratios():
    s = P.PruneStats(1000, 50, 1024, 307200, 0.1)
    assert s.patch_pruning == 1.0 - 50 / 1000
    assert s.region_pruning == 1.0 - 1024 / 307200
    e = P.PruneStats(0, 0, 0, 0, 0.0)
    assert e.patch_pruning == 1.0 and e.region_pruning == 1.0


def test_candidate_list_semantics():
    from paper_1707_05647_b200.screening import CandidateList

    xy = np.array([[5, 1], [7, 1], [3, 2], [9, 9]], np.int32)
    cl = CandidateList.build(xy, (64, 32), [3, 1])
    assert len(cl) == 4
    assert list(cl) == [(5, 1, 64), (7, 1, 64), (3, 2, 64), (9, 9, 32)]
    assert (3, 2, 64) in cl and (3, 2, 32) not in cl
    assert cl == [(5, 1, 64), (7, 1, 64), (3, 2, 64), (9, 9, 32)]
    assert cl[1] == (7, 1, 64) and cl[-1] == (9, 9, 32)
