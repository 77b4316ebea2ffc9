"""Multi-process (gloo, world_size 2 and 3) test of the row-band sharding logic.

The per-band screen and the band's region pass are CPU stand-ins built from
the pinned oracle (test infrastructure; the product's are the GPU kernels,
covered by the GPU tests): the band screen sees only its halo'd band's
tables, in the band's local frame, and decides border status in global
coordinates -- the contract ss_screen_ladder implements; the region pass
sees only the band's mask rows plus the halo rows the neighbour exchange
delivered -- the contract of ss_region_ladder_rows.  Everything between them
is the product's code: band planning, the halo exchange (send / recv), the
all-gather of counts and padded survivor rows, the device-style assembly of
the candidate order.  The result must equal the oracle's single-image
screen: candidates (order included), every band's size masks and region
rows, patches_tested, patches_kept, region_pixels_kept.
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
    xy, counts = [], []
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
                      torch.from_numpy(packed.view(np.int32).copy()))


def oracle_region(stack, W, y0, H, ladder, stride):
    """Region rows of a window of mask rows (global row y0 first): footprints
    of the interior (evaluated) survivors in the window, clipped to it."""
    from paper_1707_05647_b200.screening import unpack_bits

    rows = stack.shape[1]
    region = np.zeros((rows, W), bool)
    for k, m in enumerate(ladder):
        if m < 8:
            continue
        lo, hi = (m - 1) // 2, m // 2
        full = unpack_bits(stack[k].numpy().view(np.uint32), W)
        surv = np.zeros_like(full)
        ys = np.arange(rows) + y0
        live = (ys >= lo) & (ys <= H - 1 - hi)
        surv[live, lo:W - hi] = full[live, lo:W - hi]
        O.footprint_union(surv, m, region)
    words = (W + 31) // 32
    b = np.packbits(region.astype(np.uint8), axis=1, bitorder="little")
    packed = np.zeros((rows, words * 4), np.uint8)
    packed[:, : b.shape[1]] = b
    return packed.view(np.int32)


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
    out_q.put((rank, res.size_masks.rows, res.candidates.array(), {m: packbits(res.size_masks[m]) for m in res.ladder},
               packbits(res.region_mask), res.stats.patches_tested, res.stats.patches_kept,
               res.stats.region_pixels_kept))
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
    got = []
    while len(got) < world:  # fail fast if a worker dies instead of waiting out the queue timeout
        try:
            got.append(q.get(timeout=2))
        except Exception:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            assert not dead, f"worker exit codes {dead}"
    got.sort(key=lambda g: g[0])
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    kw = dict(cfg_kw)
    ref = O.screen(img, case.template, O.ScreeningConfig(**kw), nthreads=2)
    want_c = np.array(ref.candidates, np.int32).reshape(-1, 3)
    covered = 0
    for rank, (y0, y1), cands, masks, region, tested, kept, region_px in got:
        assert covered == y0
        covered = y1
        assert np.array_equal(cands, want_c), rank  # every rank holds the whole list
        for m in ref.ladder:
            assert np.array_equal(masks[m], packbits(ref.size_masks[m][y0:y1])), (rank, m)
        assert np.array_equal(region, packbits(ref.region_mask[y0:y1])), rank
        assert (tested, kept, region_px) == (ref.patches_tested, len(ref.candidates), ref.region_pixels_kept)
    assert covered == img.shape[0]


def test_plan_bands_cover_rows_with_halo():
    from paper_1707_05647_b200.sharding import ladder_margins, plan_bands

    ladder = (512, 300, 128, 33, 7)
    lo, hi = ladder_margins(ladder)
    assert (lo, hi) == (255, 256)
    with pytest.raises(ValueError):
        plan_bands(1000, 8, ladder)  # bands thinner than the halo
    for H, world in [(16384, 8), (1000, 3), (10, 1), (1080, 4)]:
        bands = plan_bands(H, world, ladder)
        assert bands[0].y_begin == 0 and bands[-1].y_end == H
        for a, b in zip(bands, bands[1:]):
            assert a.y_end == b.y_begin
        for b in bands:
            assert b.y_origin == max(0, b.y_begin - lo)
            assert b.y_origin + b.rows == min(H, b.y_end + hi) or b.rows == 1


def test_assemble_rows_orders_by_size_then_rank():
    from paper_1707_05647_b200.sharding import assemble_rows

    rng = np.random.default_rng(0)
    world, L, cap = 3, 4, 9
    counts = rng.integers(0, 3, size=(world, L))
    rows = np.full((world, cap, 3), -7, np.int32)
    want = []
    for k in range(L):
        for r in range(world):
            for j in range(counts[r, k]):
                want.append((r * 100 + j, k, r))
    for r in range(world):
        i = 0
        for k in range(L):
            for j in range(counts[r, k]):
                rows[r, i] = (r * 100 + j, k, r)
                i += 1
    out = assemble_rows(torch.from_numpy(rows), torch.from_numpy(counts))
    assert np.array_equal(out[: len(want)].numpy(), np.array(want, np.int32).reshape(-1, 3))
