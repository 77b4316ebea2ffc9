"""Multi-GPU screening: row bands of one image, or images of a batch.

SURVEY.md 8(e): the work shards with no exchange before the final gather.

* Row bands (configs 2 and 4): rank r decides rows [y_begin, y_end) and
  builds its tables over the halo'd band [y_begin - lo_max, y_end + hi_max)
  (lo_max / hi_max = the largest ladder size's centre margins,
  features.py:214-217).  Tables are local to the band -- no prefix carry
  crosses GPUs, because only region differences are used and the weighted
  numerators are frame-invariant -- and border status
  is decided in global coordinates (ss_screen_size's y_origin / y_begin /
  y_end).  Duplicated work is only the halo part of the table build.
* Images of a batch (config 3): image i goes to rank i % world.

The only collective is the final gather: an all-gather of per-size survivor
counts, then of the compacted (cx, cy) lists and packed mask rows, padded to
the largest rank (NCCL has no gather primitive).  Concatenating bands in rank
order keeps global row-major order, so the gathered candidate list equals the
single-GPU one.  The kept region is computed after the gather from the full
survivor masks (it needs neighbour bands' survivors within the margins).

Host-side planning and assembly are plain functions so they can be tested
with the gloo backend on CPU (tests/test_sharding_cpu.py).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

from .config import MIN_PATCH_SIDE, patch_center_margins


@dataclass(frozen=True)
class Band:
    rank: int
    y_begin: int  # first decided row (global)
    y_end: int  # one past the last decided row
    y_origin: int  # first table row (global)
    rows: int  # table rows


def ladder_margins(ladder: Sequence[int]) -> Tuple[int, int]:
    """(lo_max, hi_max) over the evaluated sizes (features.py:214-217)."""
    ev = [m for m in ladder if m >= MIN_PATCH_SIDE]
    if not ev:
        return 0, 0
    return max(patch_center_margins(m)[0] for m in ev), max(patch_center_margins(m)[1] for m in ev)


def plan_bands(height: int, world: int, ladder: Sequence[int]) -> List[Band]:
    """Balanced row bands with the halo the largest ladder size needs."""
    lo, hi = ladder_margins(ladder)
    out = []
    for r in range(world):
        yb = r * height // world
        ye = (r + 1) * height // world
        y0 = max(0, yb - lo)
        y1 = min(height, ye + hi)
        out.append(Band(r, yb, ye, y0, max(y1 - y0, 1)))
    return out


@dataclass
class BandResult:
    """One rank's share: survivors in global coordinates, packed mask rows."""

    band: Band
    counts: "torch.Tensor"  # (L,) int64 survivors per ladder size
    rows: "torch.Tensor"  # (k, 3) int32 (cx, cy, m), ladder order then row-major
    masks: "torch.Tensor"  # (L, y_end - y_begin, words) int32 (bit-packed rows)
    tested: int


def _coll_device(group=None) -> torch.device:
    backend = dist.get_backend(group)
    return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")


def _all_gather_padded(t: torch.Tensor, group=None) -> List[torch.Tensor]:
    """All-gather tensors whose first dimension differs per rank."""
    dev = _coll_device(group)
    world = dist.get_world_size(group)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=dev)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(v.item()) for v in ns]
    mx = max(ns) if ns else 0
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
    pad[: t.shape[0]] = t.to(dev)
    outs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return [o[:k] for o, k in zip(outs, ns)]


def gather_band_results(local: BandResult, group=None) -> List[BandResult]:
    """All ranks' BandResults, in rank order (every rank receives all); the
    tensors stay on the collective's device (NCCL: the GPU)."""
    world = dist.get_world_size(group)
    dev = _coll_device(group)
    counts = torch.as_tensor(local.counts, dtype=torch.int64).to(dev)
    allc = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(allc, counts, group=group)
    rows = _all_gather_padded(torch.as_tensor(local.rows, dtype=torch.int32).reshape(-1, 3), group)
    m = torch.as_tensor(local.masks).view(torch.int32)
    ms = _all_gather_padded(m.permute(1, 0, 2).contiguous(), group)  # rows first
    tested = torch.tensor([local.tested], dtype=torch.int64, device=dev)
    allt = [torch.zeros_like(tested) for _ in range(world)]
    dist.all_gather(allt, tested, group=group)
    bands = plan_bands_from(local.band, world, group)
    return [BandResult(bands[r], allc[r], rows[r], ms[r].permute(1, 0, 2), int(allt[r].item())) for r in range(world)]


def plan_bands_from(band: Band, world: int, group=None) -> List[Band]:
    dev = _coll_device(group)
    t = torch.tensor([band.rank, band.y_begin, band.y_end, band.y_origin, band.rows], dtype=torch.int64, device=dev)
    allb = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(allb, t, group=group)
    return [Band(*[int(v) for v in b.cpu().tolist()]) for b in allb]


def assemble(parts: List[BandResult], width: int, height: int, ladder: Sequence[int]):
    """Concatenate band results into full-image tensors on the parts' device
    (ladder order, then row-major): masks (L, H, words) int32, rows (K, 3)
    int32, counts (L,) int64 (host), tested."""
    L = len(ladder)
    words = (width + 31) // 32
    dev = parts[0].rows.device if parts else torch.device("cpu")
    masks = torch.zeros((L, height, words), dtype=torch.int32, device=dev)
    per_size = [[] for _ in range(L)]
    for p in sorted(parts, key=lambda p: p.band.y_begin):
        masks[:, p.band.y_begin:p.band.y_end] = p.masks
        cnts = [int(c) for c in p.counts.tolist()]
        for k, chunk in enumerate(torch.split(p.rows, cnts)):
            per_size[k].append(chunk)
    counts = np.array([sum(int(c.shape[0]) for c in per_size[k]) for k in range(L)], np.int64)
    empty = torch.zeros((0, 3), dtype=torch.int32, device=dev)
    rows = torch.cat([torch.cat(per_size[k]) if per_size[k] else empty for k in range(L)]) if L else empty
    tested = sum(p.tested for p in parts)
    return masks, rows, counts, tested


_band_engines: dict = {}


def band_engine(W: int, H: int, band: Band, device):
    """One cached engine per (shape, band, device) -- the most recent only:
    an engine's tables and workspaces are allocated once, not per call."""
    from .engine import Engine

    key = (W, H, band.y_origin, band.rows, band.y_begin, band.y_end, str(torch.device(device)))
    eng = _band_engines.get(key)
    if eng is None:
        _band_engines.clear()
        eng = Engine(W, H, device, band=(band.y_origin, band.rows, band.y_begin, band.y_end))
        _band_engines[key] = eng
    return eng


def screen_band_device(image: np.ndarray, tp, band: Band, device) -> BandResult:
    """This rank's band on its GPU (libstarscreen through engine.Engine)."""
    H, W = image.shape
    eng = band_engine(W, H, band, device)
    sub = torch.from_numpy(np.ascontiguousarray(image[band.y_origin:band.y_origin + band.rows])).to(eng.device)
    eng.run(sub, tp, region=False)
    totals = eng.totals.cpu()
    kept = int(totals[0])
    if kept > eng.capacity:
        eng.recompact(tp, kept)
    counts = eng.size_counts[: len(tp.sizes)].clone()
    rows = eng.xy[:kept].clone()  # (cx, cy, m) on the device
    masks = eng.masks[: len(tp.sizes)].clone()
    return BandResult(band, counts, rows, masks, eng.tested(tp))


def region_from_masks(masks, width: int, height: int, ladder: Sequence[int], stride: int, device):
    """Kept region (K5, ladder form) on the device from the gathered full
    survivor masks ((L, H, words) int32 tensor); returns (packed region
    tensor on the device, kept pixels)."""
    from . import _native

    L = _native.lib()
    dev = torch.device(device)
    words = (width + 31) // 32
    mk = torch.as_tensor(masks).to(dev).view(torch.int32).contiguous()
    ms = np.asarray(ladder, np.int32)
    region = torch.empty((height, words), dtype=torch.int32, device=dev)
    ws = torch.empty(int(L.ss_region_ladder_workspace_bytes(width, height, len(ms))), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream(dev).cuda_stream
    _native.check(L.ss_region_ladder(mk.data_ptr(), words, height * words, width, height, len(ms), ms.ctypes.data,
                                     stride, region.data_ptr(), ws.data_ptr(), ws.numel(), s), "region")
    _native.check(L.ss_popcount(region.data_ptr(), words, width, height, cnt.data_ptr(), s), "popcount")
    return region, int(cnt.item())


def screen_sharded(image: np.ndarray, template: np.ndarray, cfg=None, group=None, device=None,
                   band_fn: Optional[Callable] = None, region_fn: Optional[Callable] = None):
    """Row-band sharded screen() over the ranks of `group`; every rank gets the result.

    band_fn / region_fn default to the GPU implementations (tests substitute a
    CPU stand-in to exercise the planning, gather and assembly logic on gloo).
    """
    import time

    from .config import ScreeningConfig
    from .engine import prepare_template
    from .screening import CandidateList, PruneStats, ScreeningResult, SizeMasks, validate

    cfg = cfg or ScreeningConfig()
    img, tpl = validate(image, template, cfg)
    H, W = img.shape
    start = time.perf_counter()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if torch.cuda.is_available() else None)
    tp = prepare_template(tpl, cfg, dev if band_fn is None else torch.device("cpu"))
    band = plan_bands(H, world, tp.ladder)[rank]
    local = (band_fn or screen_band_device)(img, tp, band, dev)
    parts = gather_band_results(local, group)
    masks, rows, counts, tested = assemble(parts, W, H, tp.ladder)
    if region_fn is None:
        region, kept_px = region_from_masks(masks, W, H, tp.ladder, cfg.stride, dev)
    else:  # host stand-in (tests)
        region, kept_px = region_fn(masks.cpu().numpy().view(np.uint32), W, H, tp.ladder, cfg.stride, dev)
    stats = PruneStats(tested, int(counts.sum()), kept_px, W * H, time.perf_counter() - start)
    return ScreeningResult(W, H, tp.template_side, cfg, tp.ladder, CandidateList(rows, int(rows.shape[0])),
                           SizeMasks(tp.ladder, masks, W), region, stats, counts.tolist())
