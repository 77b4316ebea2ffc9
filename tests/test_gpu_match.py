"""f3: match_candidates (second_stage.py:168-204) on the GPU vs the
reference's own results on the same screens (tests/golden/match.npz):
winner position, scale, angle and the float64 score, bit for bit."""

import json

import numpy as np
import pytest

from conftest import golden, load_screen_case

pytestmark = pytest.mark.gpu


def _cfg(kw):
    from paper_1707_05647_b200 import Quantizer, ScreeningConfig

    kw = dict(kw)
    if "quantizer" in kw:
        kw["quantizer"] = Quantizer(*kw["quantizer"])
    return ScreeningConfig(**kw)


def _names():
    return [str(n) for n in golden("match.npz")["names"]]


@pytest.mark.parametrize("key", _names())
def test_match_candidates_matches_reference(cuda, key):
    from paper_1707_05647_b200 import ScreeningConfig, match_candidates, screen

    z = golden("match.npz")
    step = float(z[f"{key}/step"])
    if f"{key}/image" in z.files:
        img, tpl = z[f"{key}/image"], z[f"{key}/template"]
        cfg = _cfg(json.loads(str(z[f"{key}/cfg"]))) if f"{key}/cfg" in z.files else ScreeningConfig()
    else:
        c = load_screen_case(key.split("@")[0])
        img, tpl, cfg = c["image"], c["template"], _cfg(c["cfg"])
    res = screen(img, tpl, cfg)
    r = match_candidates(img, tpl, res, angle_step=step)
    exp = z[f"{key}/result"]
    assert (r.cx, r.cy) == (int(exp[0]), int(exp[1]))
    assert r.scale == exp[2] and r.angle == exp[3]
    assert r.score == exp[4], (r.score, exp[4])  # bit-exact float64


def test_match_edge_cases(cuda):
    from paper_1707_05647_b200 import match_candidates, screen
    from paper_1707_05647_b200.second_stage import _angle_grid

    c = load_screen_case("t4_default")
    res = screen(c["image"], c["template"], _cfg(c["cfg"]))
    with pytest.raises(ValueError):
        _angle_grid(7.0)
    with pytest.raises(ValueError):
        _angle_grid(0.0)
    assert _angle_grid(90.0) == [0.0, 90.0, 180.0, 270.0]
    # no candidates -> None
    small = c["image"][:10, :14].copy()
    empty = screen(small, c["template"])
    assert len(empty.candidates) == 0
    assert match_candidates(small, c["template"], empty) is None
    # more than one angle group (40 per launch) gives the same winner as the golden
    r = match_candidates(c["image"], c["template"], res, angle_step=2.0)
    assert r is not None and r.angle % 2.0 == 0.0
