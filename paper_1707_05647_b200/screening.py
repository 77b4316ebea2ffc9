"""The drop-in screening entry point: ``screen(image, template, cfg) -> ScreeningResult``.

Mirrors screening.py:474-539 (same signature, validation order, error
classes and messages, result fields) with the per-pixel work on the GPU:
tables (K1/K2), ring features + membership + mask (K3), survivor list (K4)
and the kept region (K5), all through libstarscreen_b200 (engine.py).  The
template side computes every rescale's ring features in one GPU launch (f2)
and builds the guard-banded key sets on the host (featureset.py).

Results stay on the device, bit-packed, until a caller looks: the counts
(PruneStats) are read back by screen(); ``candidates`` copies the compacted
int32 survivor list on first use; ``size_masks[m]`` / ``region_mask`` copy
and unpack one mask on first access -- a 16384^2 x 33-size screen never
materialises 8.8 GB of bools or 10^7 Python tuples it is not asked for.
"""

from __future__ import annotations

import os
import threading
import time
from collections.abc import Mapping, Sequence
from dataclasses import dataclass
from typing import Dict, Iterator, List, Optional, Tuple

import numpy as np
import torch

from .config import MIN_PATCH_SIDE, ScreeningConfig
from .engine import (Engine, EnginePool, TemplatePlan, fill_keysets, launch_features, plan_ladder, prepare_template,
                     upload_keysets)
from .image import as_gray, std_dev
from .session import Session


class FlatTemplateError(ValueError):
    """Template has too little variance to be screened (screening.py:60-61)."""


@dataclass(frozen=True)
class PruneStats:
    """screening.py:253-273."""

    patches_tested: int
    patches_kept: int
    region_pixels_kept: int
    total_pixels: int
    wall_time_s: float

    @property
    def patch_pruning(self) -> float:
        if self.patches_tested == 0:
            return 1.0
        return 1.0 - self.patches_kept / self.patches_tested

    @property
    def region_pruning(self) -> float:
        if self.total_pixels == 0:
            return 1.0
        return 1.0 - self.region_pixels_kept / self.total_pixels


def unpack_bits(words: np.ndarray, width: int) -> np.ndarray:
    """(rows, ceil(W/32)) little-endian bit words -> (rows, W) bool."""
    w = np.ascontiguousarray(words).view(np.uint8)
    bits = np.unpackbits(w.reshape(words.shape[0], -1), axis=1, bitorder="little")
    return bits[:, :width].astype(bool)


def _to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> numpy through a pinned staging buffer (torch's caching
    host allocator): the D2H runs at full PCIe/C2C rate instead of the
    pageable path's bounce copies."""
    if not t.is_cuda:
        return t.numpy()
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return out.numpy()


_UPLOAD_CHUNK = 16 << 20


def upload_image(img: np.ndarray, device) -> torch.Tensor:
    """Host uint8 image -> device, through pinned staging chunks: a
    multi-threaded host copy into one chunk overlaps the DMA of the previous
    one (the pageable path moves ~11 GB/s)."""
    dev = torch.device(device)
    src = torch.from_numpy(np.ascontiguousarray(img))
    if src.numel() < 2 * _UPLOAD_CHUNK:
        return src.pin_memory().to(dev, non_blocking=True)
    out = torch.empty(src.shape, dtype=torch.uint8, device=dev)
    flat_src, flat_dst = src.view(-1), out.view(-1)
    stream = torch.cuda.current_stream(dev)
    bufs = [torch.empty(_UPLOAD_CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    done = [None, None]
    for i, off in enumerate(range(0, src.numel(), _UPLOAD_CHUNK)):
        b = i & 1
        if done[b] is not None:
            done[b].synchronize()  # the DMA that last read this buffer has finished
        n = min(_UPLOAD_CHUNK, src.numel() - off)
        bufs[b][:n].copy_(flat_src[off:off + n])
        flat_dst[off:off + n].copy_(bufs[b][:n], non_blocking=True)
        done[b] = torch.cuda.Event()
        done[b].record(stream)
    return out


def _host_words(t) -> np.ndarray:
    """Bit-packed words as uint32 numpy (from a torch tensor or an array)."""
    if isinstance(t, torch.Tensor):
        return _to_host(t).view(np.uint32)
    return np.asarray(t).view(np.uint32)


class SizeMasks(Mapping):
    """Dict[m, bool (H, W)] view over bit-packed per-size keep masks.

    The packed masks may stay on the device; a size is copied to the host on
    first access to .packed(m) and unpacked on first access to [m].
    """

    def __init__(self, ladder: Tuple[int, ...], packed, width: int, pending=None):
        self._ladder = tuple(ladder)
        # (L, H, words) uint32 array, int32 CUDA tensor, or a pinned int32 CPU
        # tensor that a stream copy is still filling (screen() streams each
        # finished row chunk to the host while later chunks are screened);
        # `pending` is that copy's completion event
        self._packed = packed
        self._pending = pending
        self._width = width
        self._host: Dict[int, np.ndarray] = {}
        self._cache: Dict[int, np.ndarray] = {}

    def _ready(self) -> None:
        if self._pending is not None:
            self._pending.synchronize()
            self._pending = None

    def packed_all(self) -> np.ndarray:
        """(L, H, ceil(W/32)) uint32: every size's bit-packed rows in ladder
        order, copied to the host in one transfer."""
        if len(self._host) < len(self._ladder):
            self._ready()
            allw = _host_words(self._packed)
            for k, m in enumerate(self._ladder):
                self._host[m] = allw[k]
            return allw
        return np.stack([self._host[m] for m in self._ladder])

    def packed(self, m: int) -> np.ndarray:
        if m not in self._host:
            self._ready()
            k = self._ladder.index(m)
            self._host[m] = _host_words(self._packed[k])
        return self._host[m]

    def source(self, m: int):
        """Size m's packed rows where they live: a CUDA tensor, or host words."""
        self._ready()
        k = self._ladder.index(m)
        p = self._packed
        if isinstance(p, torch.Tensor):
            return p[k] if p.is_cuda else p[k].numpy().view(np.uint32)
        return np.asarray(p)[k]

    def __getitem__(self, m: int) -> np.ndarray:
        if m not in self._ladder:
            raise KeyError(m)
        if m not in self._cache:
            self._cache[m] = unpack_bits(self.packed(m), self._width)
        return self._cache[m]

    def __contains__(self, m) -> bool:
        return m in self._ladder

    def __iter__(self) -> Iterator[int]:
        return iter(self._ladder)

    def __len__(self) -> int:
        return len(self._ladder)


class BandSizeMasks(SizeMasks):
    """SizeMasks of a row-band sharded screen (sharding.py): each rank holds
    the rows [y_begin, y_end) it decided; .packed(m) / [m] are those rows."""

    def __init__(self, ladder: Tuple[int, ...], packed, width: int, rows: Tuple[int, int]):
        super().__init__(ladder, packed, width)
        self.rows = (int(rows[0]), int(rows[1]))


class CandidateList(Sequence):
    """List[(cx, cy, m)] view: ladder order, then row-major (screening.py:280-283).

    Backed by the compacted int32 (cx, cy, m) rows -- on the device until
    first use, then copied once -- and the per-size counts.
    """

    def __init__(self, rows, n: int, host=None):
        self._rows = rows  # (k, 3) int32 array or CUDA tensor
        self._n = int(n)
        # optional (pinned (cap, 3) tensor, event): the rows already on their
        # way to the host (Engine.start_readback), used when they cover n
        self._host = host if host is not None and host[0].shape[0] >= self._n else None

    @staticmethod
    def build(xy, ladder: Tuple[int, ...], counts: List[int]) -> "CandidateList":
        """From host (k, 2) (cx, cy) pairs and per-size counts."""
        xy = np.asarray(xy, np.int32).reshape(-1, 2)
        rows = np.empty((xy.shape[0], 3), np.int32)
        rows[:, :2] = xy
        rows[:, 2] = np.repeat(np.asarray(ladder, np.int32), counts)
        return CandidateList(rows, rows.shape[0])

    def array(self) -> np.ndarray:
        """(k, 3) int32 [cx, cy, m]."""
        if isinstance(self._rows, torch.Tensor):
            if self._host is not None:
                buf, done = self._host
                done.synchronize()
                self._rows = buf[: self._n].numpy()  # a view: buf stays referenced by the array base
            else:
                self._rows = _to_host(self._rows).reshape(-1, 3)
        return self._rows

    @property
    def xy(self) -> np.ndarray:
        return self.array()[:, :2]

    @property
    def m(self) -> np.ndarray:
        return self.array()[:, 2]

    def __len__(self) -> int:
        return self._n

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        r = self.array()[i]
        return (int(r[0]), int(r[1]), int(r[2]))

    def __iter__(self):
        return iter(map(tuple, self.array().tolist()))

    def __contains__(self, item) -> bool:
        try:
            cx, cy, m = item
        except (TypeError, ValueError):
            return False
        a = self.array()
        return bool(np.any((a[:, 0] == cx) & (a[:, 1] == cy) & (a[:, 2] == m)))

    def __eq__(self, other) -> bool:
        if isinstance(other, CandidateList):
            return np.array_equal(self.array(), other.array())
        if isinstance(other, (list, tuple)):
            return list(self) == [tuple(t) for t in other]
        return NotImplemented

    def __repr__(self) -> str:
        return f"CandidateList(len={len(self)})"


class ScreeningResult:
    """screening.py:276-298: everything the second stage needs from the screen."""

    def __init__(self, width, height, template_side, config, ladder, candidates, size_masks, region_packed, stats,
                 size_counts=None, region_rows=None):
        self._size_counts = None if size_counts is None else [int(c) for c in size_counts]
        # row-band sharded results hold the region rows [y0, y1) of their band only
        self.region_rows = (0, height) if region_rows is None else (int(region_rows[0]), int(region_rows[1]))
        self.width = width
        self.height = height
        self.template_side = template_side
        self.config = config
        self.ladder = ladder
        self.candidates = candidates
        self.size_masks = size_masks
        self._region_packed = region_packed
        self._region_event = None  # pending copy into a host _region_packed (fetch_result(to_host=True))
        self._region = None
        self.stats = stats

    def region_packed(self) -> np.ndarray:
        """Bit-packed region rows (H, ceil(W/32)) uint32."""
        if self._region_packed is None:
            return np.zeros((self.region_rows[1] - self.region_rows[0], (self.width + 31) // 32), np.uint32)
        if isinstance(self._region_packed, torch.Tensor):
            if self._region_event is not None:
                self._region_event.synchronize()
                self._region_event = None
            self._region_packed = _host_words(self._region_packed)
        return self._region_packed

    @property
    def region_mask(self) -> np.ndarray:
        if self._region is None:
            self._region = unpack_bits(self.region_packed(), self.width)
        return self._region

    def candidates_per_size(self) -> List[int]:
        """Survivors per ladder size, in ladder order (cli.py:104-106)."""
        if self._size_counts is None:
            ms = self.candidates.m if len(self.candidates) else np.zeros(0, np.int32)
            self._size_counts = [int(np.count_nonzero(ms == m)) for m in self.ladder]
        return list(self._size_counts)

    def region_pgm(self) -> np.ndarray:
        """The kept region as a 0/255 uint8 raster (cli.py:97-98, 159-160), built on the device."""
        from .pgm import packed_to_pgm

        src = self._region_packed
        if isinstance(src, torch.Tensor) and not src.is_cuda:
            src = self.region_packed()  # a host copy (waits for it)
        if src is None:
            return np.zeros((self.region_rows[1] - self.region_rows[0], self.width), np.uint8)
        return packed_to_pgm(src, self.width)

    def size_mask_pgm(self, m: int) -> np.ndarray:
        """One size's centre mask as a 0/255 uint8 raster (cli.py:161-163), built on the device."""
        from .pgm import packed_to_pgm

        if m not in self.ladder:
            raise KeyError(m)
        return packed_to_pgm(self.size_masks.source(m), self.width)

    def __repr__(self) -> str:
        return (f"ScreeningResult({self.width}x{self.height}, n={self.template_side}, ladder={self.ladder}, "
                f"candidates={len(self.candidates)}, stats={self.stats})")


def prune_stats(result: ScreeningResult) -> PruneStats:
    """screening.py:301-309."""
    return PruneStats(
        patches_tested=result.stats.patches_tested,
        patches_kept=len(result.candidates),
        region_pixels_kept=int(result.region_mask.sum()),
        total_pixels=result.width * result.height,
        wall_time_s=result.stats.wall_time_s,
    )


_engine_lock = threading.Lock()
_engine_cache: Dict[Tuple[int, int, str], Engine] = {}


def get_engine(width: int, height: int, device=None) -> Engine:
    """One cached engine per (W, H, device); the most recent shape only."""
    dev = torch.device(device if device is not None else "cuda")
    if dev.type == "cuda" and dev.index is None:  # "cuda" and "cuda:<current>" are one engine
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (width, height, str(dev))
    with _engine_lock:
        eng = _engine_cache.get(key)
        if eng is None:
            _engine_cache.clear()
            eng = Engine(width, height, dev)
            _engine_cache[key] = eng
        return eng


def validate(image, template, cfg: ScreeningConfig):
    """Validation prologue of screen() (screening.py:481-494)."""
    img = as_gray(image)
    tpl = as_gray(template)
    th, tw = tpl.shape
    if th != tw:
        raise ValueError(f"template must be square, got {tw}x{th}")
    n = tw
    if n < MIN_PATCH_SIDE:
        raise ValueError(f"template side {n} below minimum {MIN_PATCH_SIDE}")
    if std_dev(tpl) < cfg.min_template_std:
        raise FlatTemplateError(f"template too flat: std {std_dev(tpl):.3f} below {cfg.min_template_std}")
    return img, tpl


def fetch_result(eng: Engine, tp: TemplatePlan, start: float, readback=None, masks=None,
                 to_host: bool = False, region_host=None) -> ScreeningResult:
    """Counts to the host; survivor list, masks and region stay on the device
    (private copies, the engine's buffers are reused) until first accessed;
    `readback` (Engine.start_readback) carries the survivor rows' host copy
    that started right after compaction; `masks` = (pinned host tensor,
    event) of the size masks streamed to the host during the screen
    (Engine.run(host_masks=...)), used instead of a device copy.  to_host:
    every array goes straight to pinned host memory (asynchronous on the
    current stream, one event) instead of a device copy -- no device
    allocation per result (screen_batch)."""
    cur = torch.cuda.current_stream(eng.device)
    totals = eng.totals.cpu()  # synchronises the stream
    kept = int(totals[0])
    if kept > eng.capacity:
        eng.recompact(tp, kept)
        totals = eng.totals.cpu()
    size_counts = eng.size_counts[: len(tp.sizes)].cpu().tolist()
    eng.last_kept = kept
    region_event = None
    if to_host:
        rows = torch.empty((kept, 3), dtype=torch.int32, pin_memory=True)
        rows.copy_(eng.xy[:kept], non_blocking=True)
        packed = None
        if masks is None:
            packed = torch.empty(eng.masks[: len(tp.sizes)].shape, dtype=torch.int32, pin_memory=True)
            packed.copy_(eng.masks[: len(tp.sizes)], non_blocking=True)
        region = None
        if eng.region is not None:
            region = torch.empty(eng.region.shape, dtype=torch.int32, pin_memory=True)
            region.copy_(eng.region, non_blocking=True)
        done = torch.cuda.Event()
        done.record(cur)
        readback = (rows, done)
        if masks is None:
            masks = (packed, done)
        region_event = done
    else:
        rows = eng.xy[:kept].clone()
        packed = eng.masks[: len(tp.sizes)].clone() if masks is None else None
        if region_host is not None:  # already on its way to pinned host memory (start_region_readback)
            region, region_event = region_host
        else:
            region = eng.region.clone() if eng.region is not None else None
        # the copies are ordered on this stream; a caller reading them on another
        # stream must wait for it (screen_batch), and their memory must not be
        # reused before those streams are done with it
        for t in (rows, packed, region):
            if t is not None and t.is_cuda:
                t.record_stream(cur)
    elapsed = time.perf_counter() - start
    W, H = eng.W, eng.H
    stats = PruneStats(
        patches_tested=eng.tested(tp),
        patches_kept=kept,
        region_pixels_kept=int(totals[1]),
        total_pixels=W * H,
        wall_time_s=elapsed,
    )
    cands = CandidateList(rows, kept, readback)
    sm = SizeMasks(tp.ladder, packed, W) if masks is None else SizeMasks(tp.ladder, masks[0], W, pending=masks[1])
    out = ScreeningResult(W, H, tp.template_side, tp.config, tp.ladder, cands, sm, region, stats, size_counts)
    out._region_event = region_event
    return out


def screen(image: np.ndarray, template: np.ndarray, cfg: Optional[ScreeningConfig] = None,
           device=None) -> ScreeningResult:
    """Run the full first stage: ladder, feature sets, and the scan (screening.py:474-539).

    Raises FlatTemplateError when the template's standard deviation is
    below cfg.min_template_std, and ValueError for non-square or too-small
    templates.
    """
    cfg = cfg or ScreeningConfig()
    img, tpl = validate(image, template, cfg)
    h, w = img.shape
    start = time.perf_counter()
    if img.nbytes < Engine.PIPELINE_MIN_BYTES and _session_path(w, h, device):
        return _screen_session(img, tpl, cfg, device, start)
    eng = get_engine(w, h, device)
    # The template's f2 features start first (engine's template stream), the
    # image side (upload + K1/K2 on the current stream) overlaps them, then
    # the host builds the key sets.  The engine is held for the whole call
    # (concurrent screen() calls of one shape take turns).
    with eng.lock, torch.cuda.device(eng.device):
        tp = plan_ladder(tpl.shape[1], cfg)
        pending = launch_features(tp, tpl, eng.device, eng.template_stream)
        # the size masks go to pinned host memory chunk by chunk while the
        # later row chunks are still being screened (the reference returns
        # host masks; at 16384^2 x 33 sizes that is 1.1 GB of D2H)
        host_masks = eng.host_mask_buffer(len(tp.sizes))
        if img.nbytes >= eng.PIPELINE_MIN_BYTES:
            # large image: upload, table build and screen overlap by row chunk
            eng.run_pipelined(img, tp, host_masks,
                              lambda: fill_keysets(tp, tpl, eng.device, eng.template_stream, pending))
        else:
            img_dev = upload_image(img, eng.device)
            eng.build_tables(img_dev, int64=eng.needs_int64(tp), tp=tp)
            fill_keysets(tp, tpl, eng.device, eng.template_stream, pending)
            eng.run(img_dev, tp, build=False, host_masks=host_masks)
        readback = eng.start_readback()  # the survivor rows' D2H overlaps K5 and the result bookkeeping
        region = eng.start_region_readback()  # and the region's right after K5
        return fetch_result(eng, tp, start, readback, masks=(host_masks, eng.masks_done), region_host=region)


def _device_key(device) -> torch.device:
    dev = torch.device(device if device is not None else "cuda")
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


_session_cache: Dict[Tuple[int, int, str], Session] = {}


def get_session(width: int, height: int, device=None) -> Session:
    """One cached native session per (W, H, device); the most recent shape only."""
    dev = _device_key(device)
    key = (width, height, str(dev))
    with _engine_lock:
        ses = _session_cache.get(key)
        if ses is None:
            _session_cache.clear()
            ses = Session(width, height, dev)
            _session_cache[key] = ses
        return ses


def _session_path(width: int, height: int, device) -> bool:
    """screen() runs through the native session unless an experiment / test
    hook asks for the Python engine: SS_SESSION=0, SS_FUSED=0,
    SS_LADDER_WS_BYTES, or the cached engine of this shape carrying
    force_int64 / stage_counts / hooks."""
    env = os.environ
    if env.get("SS_SESSION", "1") == "0" or env.get("SS_FUSED", "1") == "0" or env.get("SS_LADDER_WS_BYTES"):
        return False
    eng = _engine_cache.get((width, height, str(_device_key(device))))
    return eng is None or not (eng.force_int64 or eng.stage_counts is not None or eng.hooks is not None)


def _screen_session(img: np.ndarray, tpl: np.ndarray, cfg: ScreeningConfig, device, start: float,
                    session: Optional[Session] = None) -> ScreeningResult:
    """screen() through one ss_session_screen call; every result lands in
    pinned host memory before it returns."""
    h, w = img.shape
    geo, r = (session or get_session(w, h, device)).run(img, tpl, cfg)
    stats = PruneStats(patches_tested=r.tested, patches_kept=r.kept, region_pixels_kept=r.region_pixels,
                       total_pixels=w * h, wall_time_s=time.perf_counter() - start)
    cands = CandidateList(r.rows[: r.kept].numpy(), r.kept)
    masks = SizeMasks(geo.ladder, r.masks.numpy().view(np.uint32), w)
    return ScreeningResult(w, h, tpl.shape[1], cfg, geo.ladder, cands, masks, r.region.numpy().view(np.uint32),
                           stats, r.size_counts.tolist())


_pool_cache: Dict[Tuple[int, int, str, int], EnginePool] = {}


def get_pool(width: int, height: int, device=None, n: int = 4) -> EnginePool:
    """One cached engine pool per (W, H, device, n); the most recent shape only."""
    dev = torch.device(device if device is not None else "cuda")
    key = (width, height, str(dev), n)
    with _engine_lock:
        pool = _pool_cache.get(key)
        if pool is None:
            _pool_cache.clear()
            pool = EnginePool(width, height, dev, n)
            _pool_cache[key] = pool
        return pool


def screen_batch(images: Sequence[np.ndarray], templates: Sequence[np.ndarray],
                 cfg: Optional[ScreeningConfig] = None, device=None, engines: int = 4) -> List[ScreeningResult]:
    """screen(images[i], templates[i], cfg) for a batch of same-shape images
    (the benchmark loop of synth_bench.py:400-410 over independent cases).

    Image i runs on engine i % engines of a pool, each engine on its own
    stream: while the GPU screens image i, the host prepares image i + 1's
    template side and image i - engines' results are read back.  Results are
    identical to calling screen() per image; wall_time_s of each result is
    measured from the start of its own preparation to its read-back.
    """
    cfg = cfg or ScreeningConfig()
    if len(images) != len(templates):
        raise ValueError(f"{len(images)} images but {len(templates)} templates")
    if not len(images):
        return []
    checked = [validate(img, tpl, cfg) for img, tpl in zip(images, templates)]
    h, w = checked[0][0].shape
    if any(img.shape != (h, w) for img, _ in checked):
        raise ValueError("screen_batch needs images of one shape")
    n = max(1, min(engines, len(images)))
    if img_bytes(checked) < Engine.PIPELINE_MIN_BYTES and _session_path(w, h, device):
        return _screen_batch_sessions(get_session_pool(w, h, device, n), checked, cfg)
    pool = get_pool(w, h, device, n)
    with pool.lock, torch.cuda.device(pool.device):
        return _screen_batch(pool, checked, cfg)


def img_bytes(checked) -> int:
    return checked[0][0].nbytes


_session_pool_cache: Dict[Tuple[int, int, str, int], List[Session]] = {}
_session_pool_lock = threading.Lock()


def get_session_pool(width: int, height: int, device=None, n: int = 4) -> List[Session]:
    """n native sessions of one shape (screen_batch), cached; the most recent (shape, n) only."""
    dev = _device_key(device)
    key = (width, height, str(dev), n)
    with _engine_lock:
        pool = _session_pool_cache.get(key)
        if pool is None:
            _session_pool_cache.clear()
            pool = [Session(width, height, dev) for _ in range(n)]
            _session_pool_cache[key] = pool
        return pool


def _screen_batch_sessions(sessions: List[Session], checked, cfg: ScreeningConfig) -> List[ScreeningResult]:
    """screen_batch over native sessions: host thread j screens images j, j +
    n, ... through session j (ss_session_screen releases the GIL), so n
    screens overlap on the GPU -- each on its session's streams -- while the
    other threads copy their inputs and results."""
    n = len(sessions)
    results: List[Optional[ScreeningResult]] = [None] * len(checked)

    def work(j: int) -> None:
        for i in range(j, len(checked), n):
            img, tpl = checked[i]
            results[i] = _screen_session(img, tpl, cfg, None, time.perf_counter(), sessions[j])

    with _session_pool_lock:  # one batch at a time over these sessions
        futs = [_batch_workers(n).submit(work, j) for j in range(n)]
        for f in futs:
            f.result()
    return results  # type: ignore[return-value]


_batch_pool = None


def _batch_workers(n: int):
    global _batch_pool
    if _batch_pool is None or _batch_pool._max_workers < n:
        import concurrent.futures

        _batch_pool = concurrent.futures.ThreadPoolExecutor(max_workers=max(n, 4))
    return _batch_pool


def _screen_batch(pool: EnginePool, checked, cfg: ScreeningConfig) -> List[ScreeningResult]:
    n = len(pool)
    results: List[Optional[ScreeningResult]] = [None] * len(checked)
    pending: List[Optional[Tuple[int, TemplatePlan, float]]] = [None] * n

    caller = torch.cuda.current_stream(pool.device)

    def collect(j: int) -> None:
        if pending[j] is None:
            return
        i, tp, start = pending[j]
        with torch.cuda.stream(pool.streams[j]):
            results[i] = fetch_result(pool.engines[j], tp, start, to_host=True)
        caller.wait_stream(pool.streams[j])
        pending[j] = None

    # Template side first, for the whole batch: every template's f2 features
    # (own buffers, one stream), then the host key sets on a thread pool (the
    # native call releases the GIL) while the loop below screens.
    starts = [time.perf_counter()] * len(checked)
    tps = [plan_ladder(tpl.shape[1], cfg) for _, tpl in checked]
    tstream = pool.engines[0].template_stream
    feats = [launch_features(tp, tpl, pool.device, tstream, owned=True) for tp, (_, tpl) in zip(tps, checked)]
    workers = _keyset_workers()
    futs = [workers.submit(fill_keysets, tp, tpl, pool.device, None, f, False)
            for tp, (_, tpl), f in zip(tps, checked, feats)]
    for i, (img, tpl) in enumerate(checked):
        j = i % n
        collect(j)  # the engine's previous image leaves before its buffers are reused
        eng = pool.engines[j]
        tp = tps[i]
        with torch.cuda.stream(pool.streams[j]):
            img_dev = upload_image(img, eng.device)
            eng.build_tables(img_dev, int64=eng.needs_int64(tp), tp=tp)
            futs[i].result()  # this template's key sets (host)
            upload_keysets(tp, eng.device)
            eng.run(img_dev, tp, build=False)
        pending[j] = (i, tp, starts[i])
    for j in range(n):
        collect(j)
    return results  # type: ignore[return-value]


_keyset_pool = None


def _keyset_workers():
    """Host threads for screen_batch's key sets (ss_ladder_keysets releases the GIL)."""
    global _keyset_pool
    if _keyset_pool is None:
        import concurrent.futures
        import os

        _keyset_pool = concurrent.futures.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1))
    return _keyset_pool
