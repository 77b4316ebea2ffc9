"""The drop-in screening entry point: ``screen(image, template, cfg) -> ScreeningResult``.

Mirrors screening.py:474-539 (same signature, validation order, error
classes and messages, result fields) with the per-pixel work on the GPU:
tables (K1/K2), ring features + membership + mask (K3), survivor list (K4)
and the kept region (K5), all through libstarscreen_b200 (engine.py).  The
template side (ladder, ring plans, guard-banded key sets) runs on the host
(featureset.py, native C++).

Results stay bit-packed until a caller looks: ``size_masks[m]`` and
``region_mask`` unpack on first access and ``candidates`` is a sequence
view over the compacted int32 survivor list, so a 16384^2 x 33-size screen
does not materialise 8.8 GB of bools or 10^7 Python tuples.
"""

from __future__ import annotations

import threading
import time
from collections.abc import Mapping, Sequence
from dataclasses import dataclass
from typing import Dict, Iterator, List, Optional, Tuple

import numpy as np
import torch

from .config import MIN_PATCH_SIDE, ScreeningConfig
from .engine import Engine, TemplatePlan, prepare_template
from .image import as_gray, std_dev


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


class SizeMasks(Mapping):
    """Dict[m, bool (H, W)] view over bit-packed per-size keep masks."""

    def __init__(self, ladder: Tuple[int, ...], packed: np.ndarray, width: int):
        self._ladder = tuple(ladder)
        self._packed = packed  # (L, H, words) uint32
        self._width = width
        self._cache: Dict[int, np.ndarray] = {}

    def __getitem__(self, m: int) -> np.ndarray:
        if m not in self._cache:
            k = self._ladder.index(m)  # ValueError -> KeyError below
            self._cache[m] = unpack_bits(self._packed[k], self._width)
        return self._cache[m]

    def packed(self, m: int) -> np.ndarray:
        return self._packed[self._ladder.index(m)]

    def __contains__(self, m) -> bool:
        return m in self._ladder

    def __iter__(self) -> Iterator[int]:
        return iter(self._ladder)

    def __len__(self) -> int:
        return len(self._ladder)

    def __missing__(self, m):  # pragma: no cover - Mapping protocol
        raise KeyError(m)


class CandidateList(Sequence):
    """List[(cx, cy, m)] view: ladder order, then row-major (screening.py:280-283)."""

    def __init__(self, xy: np.ndarray, sizes: np.ndarray):
        self.xy = xy  # (k, 2) int32
        self.m = sizes  # (k,) int32

    @staticmethod
    def build(xy: np.ndarray, ladder: Tuple[int, ...], counts: List[int]) -> "CandidateList":
        return CandidateList(xy, np.repeat(np.asarray(ladder, np.int32), counts))

    def __len__(self) -> int:
        return int(self.xy.shape[0])

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        return (int(self.xy[i, 0]), int(self.xy[i, 1]), int(self.m[i]))

    def __iter__(self):
        return iter(zip(self.xy[:, 0].tolist(), self.xy[:, 1].tolist(), self.m.tolist()))

    def __contains__(self, item) -> bool:
        try:
            cx, cy, m = item
        except (TypeError, ValueError):
            return False
        return bool(np.any((self.xy[:, 0] == cx) & (self.xy[:, 1] == cy) & (self.m == m)))

    def __eq__(self, other) -> bool:
        if isinstance(other, CandidateList):
            return np.array_equal(self.xy, other.xy) and np.array_equal(self.m, other.m)
        if isinstance(other, (list, tuple)):
            return list(self) == list(other)
        return NotImplemented

    def array(self) -> np.ndarray:
        """(k, 3) int32 [cx, cy, m]."""
        return np.concatenate([self.xy, self.m[:, None]], axis=1)

    def __repr__(self) -> str:
        return f"CandidateList(len={len(self)})"


class ScreeningResult:
    """screening.py:276-298: everything the second stage needs from the screen."""

    def __init__(self, width, height, template_side, config, ladder, candidates, size_masks, region_packed, stats):
        self.width = width
        self.height = height
        self.template_side = template_side
        self.config = config
        self.ladder = ladder
        self.candidates = candidates
        self.size_masks = size_masks
        self._region_packed = region_packed
        self._region = None
        self.stats = stats

    @property
    def region_mask(self) -> np.ndarray:
        if self._region is None:
            if self._region_packed is None:
                self._region = np.zeros((self.height, self.width), dtype=bool)
            else:
                self._region = unpack_bits(self._region_packed, self.width)
        return self._region

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


def fetch_result(eng: Engine, tp: TemplatePlan, start: float) -> ScreeningResult:
    """Device -> host: per-size counts, survivor list, packed masks, region."""
    totals = eng.totals.cpu()  # synchronises the stream
    kept = int(totals[0])
    if kept > eng.capacity:
        eng.recompact(tp, kept)
        totals = eng.totals.cpu()
    counts = eng.size_counts[: len(tp.sizes)].cpu().numpy().astype(np.int64)
    xy = eng.xy[:kept].cpu().numpy()
    packed = eng.masks[: len(tp.sizes)].cpu().numpy().view(np.uint32)
    region = eng.region.cpu().numpy().view(np.uint32) if eng.region is not None else None
    elapsed = time.perf_counter() - start
    W, H = eng.W, eng.H
    stats = PruneStats(
        patches_tested=eng.tested(tp),
        patches_kept=kept,
        region_pixels_kept=int(totals[1]),
        total_pixels=W * H,
        wall_time_s=elapsed,
    )
    cands = CandidateList.build(xy, tp.ladder, counts.tolist())
    return ScreeningResult(W, H, tp.template_side, tp.config, tp.ladder, cands, SizeMasks(tp.ladder, packed, W),
                           region, stats)


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
    eng = get_engine(w, h, device)
    tp = prepare_template(tpl, cfg, eng.device)
    img_dev = torch.from_numpy(img).to(eng.device)
    eng.run(img_dev, tp)
    return fetch_result(eng, tp, start)
