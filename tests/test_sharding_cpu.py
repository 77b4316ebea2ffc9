"""Multi-process (gloo, world_size 2) test of the row-band sharding host logic.

The per-band screen is a CPU stand-in built from the pinned oracle (test
infrastructure; the product's band screen is the GPU kernel, covered by the
GPU tests): it sees only its halo'd band's tables, in the band's local frame,
and decides border status in global coordinates -- the same contract
ss_screen_size implements.  The gathered, assembled result must equal the
oracle's single-image screen: candidates (order included), every size mask,
patches_tested, the kept region.
"""

import os
import socket

import numpy as np
import torch
import pytest
import torch.multiprocessing as mp

import oracle as O
from conftest import packbits


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _member(keys, key):
    i = np.searchsorted(keys, key)
    return i < len(keys) and keys[i] == key


def oracle_band(img, tp, band, dev):
    from paper_1707_05647_b200.config import KEY_BASE, patch_center_margins, quantize
    from paper_1707_05647_b200.sharding import BandResult

    H, W = img.shape
    stride = tp.config.stride
    qm, qs, qg = tp.config.quantizer.factors()
    sub = img[band.y_origin:band.y_origin + band.rows]
    t = O.build_tables(sub)
    rows = band.y_end - band.y_begin
    L = len(tp.sizes)
    masks = np.zeros((L, rows, W), bool)
    xy, counts, tested = [], [], 0
    for k, sp in enumerate(tp.sizes):
        m = sp.m
        if m < 8:
            for y in range(band.y_begin, band.y_end):
                if y % stride == 0:
                    masks[k, y - band.y_begin, ::stride] = True
            counts.append(0)
            continue
        lo, hi = patch_center_margins(m)
        keys = sp.feature_set.ring_keys()
        c = 0
        for y in range(band.y_begin, band.y_end):
            if y % stride:
                continue
            for x in range(0, W, stride):
                if not (lo <= x <= W - 1 - hi and lo <= y <= H - 1 - hi):
                    masks[k, y - band.y_begin, x] = True
                    continue
                tested += 1
                f = O.ring_features_at(t, x, y - band.y_origin, sp.plan)
                ok = True
                for r in range(len(sp.plan)):
                    key = (quantize(f[r, 0], qm) * KEY_BASE + quantize(f[r, 1], qs)) * KEY_BASE + quantize(f[r, 2], qg)
                    if not _member(keys[r], key):
                        ok = False
                        break
                if ok:
                    masks[k, y - band.y_begin, x] = True
                    xy.append((x, y, m))
                    c += 1
        counts.append(c)
    words = (W + 31) // 32
    packed = np.zeros((L, rows, words * 4), np.uint8)
    if rows:
        b = np.packbits(masks.astype(np.uint8), axis=2, bitorder="little")
        packed[:, :, : b.shape[2]] = b
    return BandResult(band, torch.tensor(counts, dtype=torch.int64),
                      torch.from_numpy(np.array(xy, np.int32).reshape(-1, 3)),
                      torch.from_numpy(packed.view(np.int32).copy()), tested)


def oracle_region(masks, W, H, ladder, stride, dev):
    from paper_1707_05647_b200.screening import unpack_bits

    region = np.zeros((H, W), bool)
    for k, m in enumerate(ladder):
        if m < 8:
            continue
        lo, hi = (m - 1) // 2, m // 2
        full = unpack_bits(masks[k], W)
        surv = np.zeros_like(full)
        surv[lo:H - hi, lo:W - hi] = full[lo:H - hi, lo:W - hi]
        O.footprint_union(surv, m, region)
    words = (W + 31) // 32
    b = np.packbits(region.astype(np.uint8), axis=1, bitorder="little")
    packed = np.zeros((H, words * 4), np.uint8)
    packed[:, : b.shape[1]] = b
    return packed.view(np.uint32), int(region.sum())


def _worker(rank, world, port, img, tpl, cfg_kw, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1707_05647_b200 import Quantizer, ScreeningConfig
    from paper_1707_05647_b200.sharding import screen_sharded

    dist.init_process_group("gloo", rank=rank, world_size=world)
    kw = dict(cfg_kw)
    if "quantizer" in kw:
        kw["quantizer"] = Quantizer(*kw["quantizer"])
    res = screen_sharded(img, tpl, ScreeningConfig(**kw), band_fn=oracle_band, region_fn=oracle_region)
    if rank == 0:
        out_q.put((res.candidates.array(), {m: packbits(res.size_masks[m]) for m in res.ladder},
                   packbits(res.region_mask), res.stats.patches_tested, res.stats.region_pixels_kept))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg_kw", [(2, {}), (3, {"stride": 2, "alpha": 0.7, "beta": 1.5})])
def test_row_band_sharding_matches_single_image(world, cfg_kw):
    import workloads as WL

    img = WL.make_image(150, 117, seed=3)
    case = WL.make_template(img, 4, 24, (0.9, 1.2), std_threshold=10.0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, img, case.template, cfg_kw, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    cands, masks, region, tested, region_px = got
    kw = dict(cfg_kw)
    ref = O.screen(img, case.template, O.ScreeningConfig(**kw), nthreads=2)
    assert np.array_equal(cands, np.array(ref.candidates, np.int32).reshape(-1, 3))
    for m in ref.ladder:
        assert np.array_equal(masks[m], packbits(ref.size_masks[m])), m
    assert np.array_equal(region, packbits(ref.region_mask))
    assert tested == ref.patches_tested and region_px == ref.region_pixels_kept


def test_plan_bands_cover_rows_with_halo():
    from paper_1707_05647_b200.sharding import ladder_margins, plan_bands

    ladder = (512, 300, 128, 33, 7)
    lo, hi = ladder_margins(ladder)
    assert (lo, hi) == (255, 256)
    for H, world in [(16384, 8), (1000, 3), (10, 4), (1080, 7)]:
        bands = plan_bands(H, world, ladder)
        assert bands[0].y_begin == 0 and bands[-1].y_end == H
        for a, b in zip(bands, bands[1:]):
            assert a.y_end == b.y_begin
        for b in bands:
            assert b.y_origin == max(0, b.y_begin - lo)
            assert b.y_origin + b.rows == min(H, b.y_end + hi) or b.rows == 1
