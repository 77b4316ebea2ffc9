"""f4: PGM masks and the stats JSON of `starscreen screen` (cli.py:97-166,
image_io.py:43-128, synth_bench.py:314-326), byte for byte against files the
reference wrote (tests/golden/io.npz, tests/golden/make_golden.py io)."""

import dataclasses
import json

import numpy as np
import pytest

from conftest import golden, load_screen_case, packbits


def _cfg(kw):
    from paper_1707_05647_b200 import Quantizer, ScreeningConfig

    kw = dict(kw)
    if "quantizer" in kw:
        kw["quantizer"] = Quantizer(*kw["quantizer"])
    return ScreeningConfig(**kw)


def _host_result(name):
    """A ScreeningResult assembled on the host from the reference's golden screen."""
    from paper_1707_05647_b200.screening import CandidateList, PruneStats, ScreeningResult, SizeMasks

    c = load_screen_case(name)
    W = c["image"].shape[1]
    H = c["image"].shape[0]
    words = (W + 31) // 32

    def words_of(packed_bytes):
        b = np.zeros((packed_bytes.shape[0], words * 4), np.uint8)
        b[:, : packed_bytes.shape[1]] = packed_bytes
        return b.view(np.uint32)

    masks = np.stack([words_of(c["masks"][m]) for m in c["ladder"]])
    cand = np.asarray(c["candidates"], np.int32).reshape(-1, 3)
    st = c["stats"]
    stats = PruneStats(int(st[0]), int(st[1]), int(st[2]), int(st[3]), 0.0)
    return ScreeningResult(W, H, c["template"].shape[0], _cfg(c["cfg"]), c["ladder"],
                           CandidateList(cand, cand.shape[0]), SizeMasks(c["ladder"], masks, W),
                           words_of(c["region"]), stats)


def test_load_pgm_matches_reference(tmp_path):
    from paper_1707_05647_b200.pgm import PgmError, load_pgm

    z = golden("io.npz")
    for i in range(int(z["pgm_n"])):
        p = tmp_path / f"in{i}.pgm"
        p.write_bytes(bytes(z[f"pgm_in{i}"]))
        if f"pgm_out{i}" in z.files:
            assert np.array_equal(load_pgm(p), z[f"pgm_out{i}"]), i
        else:
            with pytest.raises(PgmError) as e:
                load_pgm(p)
            assert str(e.value) == str(z[f"pgm_err{i}"]), i
            assert isinstance(e.value, ValueError)
    with pytest.raises(FileNotFoundError):
        load_pgm(tmp_path / "nope.pgm")


def test_save_pgm_roundtrip_and_header(tmp_path):
    from paper_1707_05647_b200.pgm import load_pgm, save_pgm

    rng = np.random.default_rng(11)
    for w, h in [(1, 1), (7, 3), (2, 9), (64, 64), (33, 17)]:
        img = rng.integers(0, 256, size=(h, w), dtype=np.uint8)
        p = tmp_path / f"rt_{w}x{h}.pgm"
        save_pgm(p, img)
        assert p.read_bytes() == f"P5\n{w} {h}\n255\n".encode() + img.tobytes()
        assert np.array_equal(load_pgm(p), img)
    save_pgm(tmp_path / "x.pgm", np.full((2, 2), 9, np.uint8))
    assert not [q for q in tmp_path.iterdir() if q.suffix == ".tmp"]


@pytest.mark.parametrize("name", ["t4_default", "t21_odd", "t22_tall"])
def test_stats_json_matches_reference(tmp_path, name):
    from paper_1707_05647_b200.pgm import screen_stats_payload, write_json_atomic

    res = _host_result(name)
    write_json_atomic(tmp_path / "s.json", screen_stats_payload("scene.pgm", "template.pgm", res))
    assert (tmp_path / "s.json").read_bytes() == bytes(golden("io.npz")[f"{name}/stats_json"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["t4_default", "t21_odd", "t22_tall"])
def test_screen_outputs_match_reference(cuda, tmp_path, name):
    """screen() on the GPU, masks expanded on the device: every file
    `starscreen screen --out-mask --out-size-masks --out-stats` writes."""
    from paper_1707_05647_b200 import screen
    from paper_1707_05647_b200.pgm import save_screen_outputs

    z = golden("io.npz")
    c = load_screen_case(name)
    res = screen(c["image"], c["template"], _cfg(c["cfg"]))
    res.stats = dataclasses.replace(res.stats, wall_time_s=0.0)
    payload = save_screen_outputs(res, "scene.pgm", "template.pgm", out_mask=tmp_path / "region.pgm",
                                  out_stats=tmp_path / "stats.json", out_size_masks=str(tmp_path / "mask"))
    assert (tmp_path / "stats.json").read_bytes() == bytes(z[f"{name}/stats_json"])
    assert payload == json.loads(bytes(z[f"{name}/stats_json"]).decode())
    assert (tmp_path / "region.pgm").read_bytes() == bytes(z[f"{name}/region_pgm"])
    for key in z.files:
        if key.startswith(f"{name}/mask_pgm_"):
            m = int(key.rsplit("_", 1)[1])
            assert (tmp_path / f"mask_m{m:03d}.pgm").read_bytes() == bytes(z[key]), m
    # the device raster equals the unpacked mask
    assert np.array_equal(res.region_pgm() == 255, res.region_mask)
    m = res.ladder[len(res.ladder) // 2]
    assert np.array_equal(res.size_mask_pgm(m) == 255, res.size_masks[m])
    assert np.array_equal(packbits(res.size_mask_pgm(m) == 255), c["masks"][m])
