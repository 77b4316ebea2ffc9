"""Multi-GPU screening: row bands of one image (configs 2 and 4).

SURVEY.md 8(e): the work shards with no exchange inside the hot path.

* Rank r decides rows [y_begin, y_end) and builds its tables over the halo'd
  band [y_begin - lo_max, y_end + hi_max) (lo_max / hi_max = the largest
  ladder size's centre margins, features.py:214-217).  Tables are local to
  the band -- no prefix carry crosses GPUs, because only region differences
  are used and the weighted numerators are frame-invariant (SURVEY.md
  App. B.1) -- and border status is decided in global coordinates
  (y_origin / y_begin / y_end of ss_screen_ladder).  Duplicated work is the
  halo part of the table build only.
* Kept region (screening.py:316-330): a region row p is covered by survivors
  in rows [p - hi_max, p + lo_max], so a band's region rows need hi_max mask
  rows of the band above and lo_max of the band below.  They come from a
  neighbour halo exchange (NCCL send / recv, every size's rows, ~17 MB per
  neighbour at config 4), and K5 runs over the band plus halo in global
  coordinates (ss_region_ladder_rows).  The full masks are never gathered.
* The only other collective is the final gather: an all-gather of per-size
  survivor counts (+ the band's kept-region pixels) and of the compacted
  (cx, cy, m) survivor rows, padded to a fixed row capacity, so the step has
  no host synchronisation (NCCL has no gather primitive).  The rows are then
  placed in ladder order, rank order within a size (= global row-major
  order) on the device (``assemble_rows``): the gathered list equals the
  single-GPU one.

Bytes over NVLink at config 4, N = 8 (measured survivor count 22.45 M):
counts 8 x 34 x 8 B; rows 8 x ~2.8 M x 12 B ~ 270 MB received per rank with
the capacity at the largest band's count + 25%; halo 2 x 33 x 256 x 512 x 4 B
~ 34 MB per rank.

The collective and host logic is plain torch, so the gloo tests on CPU
exercise it with oracle stand-ins for the band screen and the region
(tests/test_sharding_cpu.py).
"""

from __future__ import annotations

import time
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
    """Balanced row bands with the halo the largest ladder size needs.
    Raises ValueError when a band would be thinner than the halo (its
    neighbours' region rows would need rows of bands further away)."""
    lo, hi = ladder_margins(ladder)
    out = []
    for r in range(world):
        yb = r * height // world
        ye = (r + 1) * height // world
        if world > 1 and ye - yb < max(lo, hi):
            raise ValueError(f"{world} row bands of a {height}-row image are thinner than the halo ({max(lo, hi)})")
        y0 = max(0, yb - lo)
        y1 = min(height, ye + hi)
        out.append(Band(r, yb, ye, y0, max(y1 - y0, 1)))
    return out


def halo_counts(bands: Sequence[Band], r: int, height: int, ladder: Sequence[int]) -> Tuple[int, int]:
    """(rows above, rows below) of mask halo band r needs for its region rows."""
    lo, hi = ladder_margins(ladder)
    b = bands[r]
    top = b.y_begin - max(0, b.y_begin - hi) if r > 0 else 0
    bot = min(height, b.y_end + lo) - b.y_end if r + 1 < len(bands) else 0
    return top, bot


def _coll_device(group=None) -> torch.device:
    backend = dist.get_backend(group)
    return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")


def _peer(group, r: int) -> int:
    return r if group is None else dist.get_global_rank(group, r)


def exchange_halo(masks: torch.Tensor, bands: Sequence[Band], height: int, ladder: Sequence[int],
                  group=None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Neighbour exchange of packed mask rows (every size): returns (rows from
    the band above, rows from the band below), each (L, k, words)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    L, _, words = masks.shape
    top_n, bot_n = halo_counts(bands, rank, height, ladder)
    top = torch.empty((L, top_n, words), dtype=masks.dtype, device=masks.device)
    bot = torch.empty((L, bot_n, words), dtype=masks.dtype, device=masks.device)
    ops = []
    if rank > 0:
        send_n = halo_counts(bands, rank - 1, height, ladder)[1]  # the band above needs my first rows
        ops.append(dist.P2POp(dist.isend, masks[:, :send_n].contiguous(), _peer(group, rank - 1), group))
        ops.append(dist.P2POp(dist.irecv, top, _peer(group, rank - 1), group))
    if rank + 1 < world:
        send_n = halo_counts(bands, rank + 1, height, ladder)[0]  # the band below needs my last rows
        ops.append(dist.P2POp(dist.isend, masks[:, masks.shape[1] - send_n:].contiguous(), _peer(group, rank + 1),
                              group))
        ops.append(dist.P2POp(dist.irecv, bot, _peer(group, rank + 1), group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return top, bot


def all_gather_stacked(t: torch.Tensor, group=None) -> torch.Tensor:
    """(world, *t.shape): every rank's equally shaped tensor, rank order."""
    world = dist.get_world_size(group)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t.contiguous(), group=group)
    return torch.stack(outs)


def assemble_rows(rows_g: torch.Tensor, counts_g: torch.Tensor) -> torch.Tensor:
    """Gathered survivor rows -> the single-GPU candidate order, on the device
    without a host sync.  rows_g: (world, cap, 3) int32, each rank's rows in
    ladder order then row-major (its first sum(counts_g[r]) rows valid);
    counts_g: (world, L) int64.  Returns (world * cap, 3): ladder order, rank
    order within a size (bands are row-ordered), the total = counts_g.sum()
    rows first."""
    world, cap, _ = rows_g.shape
    dev = rows_g.device
    cum = counts_g.cumsum(1)  # (world, L) end of size k in rank r's rows
    start = cum - counts_g
    tot_k = counts_g.sum(0)
    base_k = tot_k.cumsum(0) - tot_k  # start of size k in the output
    rank_off = counts_g.cumsum(0) - counts_g  # rank r's offset inside size k
    i = torch.arange(cap, device=dev, dtype=torch.int64).expand(world, cap).contiguous()
    k = torch.searchsorted(cum, i, right=True)  # size of row i of rank r (L: past the valid rows)
    L = counts_g.shape[1]
    valid = k < L
    kk = k.clamp(max=max(L - 1, 0))
    dest = (base_k[kk] + rank_off.gather(1, kk) + i - start.gather(1, kk))
    dest = torch.where(valid, dest, torch.full_like(dest, world * cap))  # invalid rows -> a spare slot
    out = torch.zeros((world * cap + 1, 3), dtype=rows_g.dtype, device=dev)
    out.index_copy_(0, dest.reshape(-1), rows_g.reshape(-1, 3))
    return out[: world * cap]


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


def region_rows_device(stack: torch.Tensor, W: int, y0: int, H: int, ladder: Sequence[int], stride: int,
                       ws: Optional[torch.Tensor] = None) -> torch.Tensor:
    """K5 over a window of mask rows (global row y0 first) on the device:
    packed region rows (rows, words) int32 (ss_region_ladder_rows)."""
    from . import _native

    L = _native.lib()
    Ls, rows, words = stack.shape
    ms = np.asarray(ladder, np.int32)
    need = int(L.ss_region_ladder_workspace_bytes(W, rows, Ls))
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=stack.device)
    region = torch.empty((rows, words), dtype=torch.int32, device=stack.device)
    s = torch.cuda.current_stream(stack.device).cuda_stream
    _native.check(L.ss_region_ladder_rows(stack.data_ptr(), words, rows * words, W, rows, y0, H, Ls, ms.ctypes.data,
                                          stride, region.data_ptr(), ws.data_ptr(), ws.numel(), s), "region")
    return region


def popcount_device(region: torch.Tensor, W: int, out: torch.Tensor) -> None:
    """out[0] = set bits of the packed (rows, words) region (ss_popcount)."""
    from . import _native

    rows, words = region.shape
    s = torch.cuda.current_stream(region.device).cuda_stream
    _native.check(_native.lib().ss_popcount(region.data_ptr(), words, W, rows, out.data_ptr(), s), "popcount")


class ShardedScreener:
    """One rank's share of a row-band sharded screen, enqueued without host
    synchronisation: band tables + K3 + K4 (engine.Engine with a band frame),
    the halo exchange, the band's region rows (K5) and popcount, the
    all-gather of counts and of the survivor rows padded to ``gather_rows``,
    and the device-side assembly of the gathered rows.  ``result()`` syncs
    once and builds the ScreeningResult."""

    def __init__(self, width: int, height: int, tp, device=None, group=None):
        self.W, self.H = int(width), int(height)
        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.ladder = tuple(tp.ladder)
        self.bands = plan_bands(self.H, self.world, self.ladder)
        self.band = self.bands[self.rank]
        self.top, self.bot = halo_counts(self.bands, self.rank, self.H, self.ladder)
        self.engine = band_engine(self.W, self.H, self.band, self.device)
        self.gather_rows = 1 << 16
        self.region_ws = None
        self.px = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.counts_g = self.rows_g = self.rows_out = self.region = None

    def upload_band(self, image: np.ndarray) -> torch.Tensor:
        b = self.band
        return torch.from_numpy(np.ascontiguousarray(image[b.y_origin:b.y_origin + b.rows])).to(self.device)

    def set_capacity(self, rows: int) -> None:
        """Survivor rows per rank: the engine's compaction capacity and the
        padded row count of the all-gather."""
        self.gather_rows = max(int(rows), 1)

    def step(self, img: torch.Tensor, tp, capacity: Optional[int] = None) -> None:
        eng = self.engine
        L = len(tp.sizes)
        with torch.cuda.device(self.device):
            eng.run(img, tp, region=False, capacity=max(capacity or 0, self.gather_rows))
            masks = eng.masks[:L]
            top, bot = exchange_halo(masks, self.bands, self.H, self.ladder, self.group)
            stack = torch.cat([top, masks, bot], 1) if (self.top or self.bot) else masks
            if self.region_ws is None:
                rws = int(eng.L.ss_region_ladder_workspace_bytes(self.W, stack.shape[1], L))
                self.region_ws = torch.empty(rws, dtype=torch.uint8, device=self.device)
            reg = region_rows_device(stack, self.W, self.band.y_begin - self.top, self.H, self.ladder,
                                     tp.config.stride, self.region_ws)
            self.region = reg[self.top: self.top + (self.band.y_end - self.band.y_begin)]
            popcount_device(self.region, self.W, self.px)
            local = torch.cat([eng.size_counts[:L], self.px])
            self.counts_g = all_gather_stacked(local, self.group)  # (world, L + 1)
            self.rows_g = all_gather_stacked(eng.xy[: self.gather_rows], self.group)
            self.rows_out = assemble_rows(self.rows_g, self.counts_g[:, :L])
            self.masks = masks

    def result(self, tp, start: float):
        """Host sync, overflow handling (every rank sees the same gathered
        counts, so all re-gather together), ScreeningResult."""
        from .screening import BandSizeMasks, CandidateList, PruneStats, ScreeningResult

        L = len(tp.sizes)
        cg = self.counts_g.cpu()
        per_rank = cg[:, :L].sum(1)
        need = int(per_rank.max()) if self.world else 0
        if need > self.gather_rows:  # a rank kept more rows than the gather carried: redo K4 + the row gather
            eng = self.engine
            if need > eng.capacity:
                eng.recompact(tp, need)
            self.gather_rows = need
            with torch.cuda.device(self.device):
                self.rows_g = all_gather_stacked(eng.xy[:need], self.group)
                self.rows_out = assemble_rows(self.rows_g, self.counts_g[:, :L].to(self.rows_g.device))
        counts = cg[:, :L].sum(0).numpy().astype(np.int64)
        total = int(counts.sum())
        tested = sum(band_tested(self.W, self.H, b, tp) for b in self.bands)
        stats = PruneStats(tested, total, int(cg[:, L].sum()), self.W * self.H, time.perf_counter() - start)
        rows = self.rows_out[:total].clone()
        masks = BandSizeMasks(tp.ladder, self.masks.clone(), self.W, (self.band.y_begin, self.band.y_end))
        return ScreeningResult(self.W, self.H, tp.template_side, tp.config, tp.ladder, CandidateList(rows, total),
                               masks, self.region.clone(), stats, counts.tolist(),
                               region_rows=(self.band.y_begin, self.band.y_end))


def band_tested(W: int, H: int, band: Band, tp) -> int:
    """patches_tested of a band's decided rows (screening.py:446, 513)."""
    from .config import grid_count

    s = tp.config.stride
    out = 0
    for m in tp.ladder:
        if m < MIN_PATCH_SIDE:
            continue
        lo, hi = patch_center_margins(m)
        nx = grid_count(W, lo, hi, s)
        ylo, yhi = max(band.y_begin, lo), min(band.y_end - 1, H - 1 - hi)
        if yhi >= ylo:
            first = ((ylo + s - 1) // s) * s
            out += nx * (0 if first > yhi else (yhi - first) // s + 1)
    return out


@dataclass
class BandResult:
    """A band screen's output (the stand-in interface of the CPU tests):
    per-size counts (L,) int64, survivor rows (k, 3) int32 in global
    coordinates (ladder order, row-major), packed mask rows (L, rows, words)."""

    band: Band
    counts: torch.Tensor
    rows: torch.Tensor
    masks: torch.Tensor


def screen_sharded(image: np.ndarray, template: np.ndarray, cfg=None, group=None, device=None,
                   band_fn: Optional[Callable] = None, region_fn: Optional[Callable] = None):
    """Row-band sharded screen() over the ranks of `group`.

    Every rank receives the whole candidate list and the whole PruneStats;
    ``size_masks`` and the region hold the rank's own band rows
    (``result.region_rows``) -- the masks are not gathered.

    band_fn(image, tp, band, device) -> BandResult and region_fn(stack, W, y0,
    H, ladder, stride) -> packed region rows replace the GPU band screen and
    K5 (tests run the collective logic on gloo with CPU stand-ins).
    """
    from .config import ScreeningConfig
    from .engine import prepare_template
    from .screening import BandSizeMasks, CandidateList, PruneStats, ScreeningResult, validate

    cfg = cfg or ScreeningConfig()
    img, tpl = validate(image, template, cfg)
    H, W = img.shape
    start = time.perf_counter()
    if band_fn is None:
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.device(dev):
            tp = prepare_template(tpl, cfg, dev)
            sh = ShardedScreener(W, H, tp, dev, group)
            eng = sh.engine
            sh.set_capacity(max(eng.last_kept or 0, 1 << 16))
            sh.step(sh.upload_band(img), tp)
            return sh.result(tp, start)
    # CPU stand-ins (tests): the same halo / gather / assembly logic
    tp = prepare_template(tpl, cfg, torch.device("cpu"))
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    bands = plan_bands(H, world, tp.ladder)
    band = bands[rank]
    local = band_fn(img, tp, band, device)
    masks = torch.as_tensor(local.masks).view(torch.int32)
    top, bot = exchange_halo(masks, bands, H, tp.ladder, group)
    t_n = top.shape[1]
    stack = torch.cat([top, masks, bot], 1)
    reg = torch.as_tensor(region_fn(stack, W, band.y_begin - t_n, H, tp.ladder, cfg.stride)).view(torch.int32)
    region = reg[t_n: t_n + band.y_end - band.y_begin]
    px = int(np.unpackbits(region.numpy().view(np.uint8), bitorder="little").sum())
    L = len(tp.sizes)
    local_c = torch.cat([torch.as_tensor(local.counts, dtype=torch.int64), torch.tensor([px], dtype=torch.int64)])
    counts_g = all_gather_stacked(local_c, group)
    cap = int(all_gather_stacked(torch.tensor([local.rows.shape[0]], dtype=torch.int64), group).max())
    padded = torch.zeros((max(cap, 1), 3), dtype=torch.int32)
    padded[: local.rows.shape[0]] = torch.as_tensor(local.rows, dtype=torch.int32).reshape(-1, 3)
    rows = assemble_rows(all_gather_stacked(padded, group), counts_g[:, :L])
    counts = counts_g[:, :L].sum(0).numpy().astype(np.int64)
    total = int(counts.sum())
    tested = sum(band_tested(W, H, b, tp) for b in bands)
    stats = PruneStats(tested, total, int(counts_g[:, L].sum()), W * H, time.perf_counter() - start)
    return ScreeningResult(W, H, tp.template_side, cfg, tp.ladder, CandidateList(rows[:total], total),
                           BandSizeMasks(tp.ladder, masks, W, (band.y_begin, band.y_end)), region, stats,
                           counts.tolist(), region_rows=(band.y_begin, band.y_end))
