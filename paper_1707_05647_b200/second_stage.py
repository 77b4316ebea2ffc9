"""f3: the second stage -- masked zero-mean NCC over the screened candidates.

Mirrors ``starscreen.second_stage.match_candidates`` (second_stage.py:168-204)
and ``MatchResult`` (:29-37) on the GPU: same hypothesis grid (every screened
(cx, cy, m) x the angle grid {0, step, ..., 360 - step}), same scores, same
winner and tie-break (highest score; exact ties to the smallest (scale,
angle, cy, cx) order the reference's loops produce).

Per ladder size (ascending, as the reference iterates ``sorted(by_size)``):

* ``ss_match_probes`` resamples the template to m x m and rotates it for
  every angle with its support mask (image_io.py:164-203), on the device;
  the rotation's cos / sin come from NumPy, as in the reference, so the
  probes are bit-identical;
* ``ss_match_fused`` gathers the candidates' windows straight from the
  image into shared memory (the UMMA canonical layout) and computes
  ``W @ [P | M]`` and ``(W * W) @ M`` (second_stage.py:136-150; W^2 as its
  high and low bytes) with tcgen05.mma kind::i8 (u8 x u8 -> s32, TMEM
  accumulators) -- exact integers, like the reference's float64 products of
  integer data -- then replays the reference's float64 score sequence op for
  op and reduces to the best candidate per angle.

There is no CPU fallback.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _native
from .image import as_gray

_GROUP = 40  # angles per fused launch (csrc/ss_match.cu MAX_GROUP_ANGLES)


@dataclass(frozen=True)
class MatchResult:
    """Best hypothesis found; ties broken by (scale, angle, cy, cx) ascending (second_stage.py:29-37)."""

    cx: int
    cy: int
    scale: float
    angle: float
    score: float


def _angle_grid(angle_step: float) -> List[float]:
    """second_stage.py:40-46."""
    if angle_step <= 0:
        raise ValueError("angle_step must be positive")
    steps = 360.0 / angle_step
    if abs(steps - round(steps)) > 1e-9:
        raise ValueError(f"angle_step must divide 360, got {angle_step}")
    return [i * angle_step for i in range(int(round(steps)))]


def _round_up(v: int, a: int) -> int:
    return (v + a - 1) // a * a


def _rotation_cos_sin(angles: Sequence[float]) -> Tuple[np.ndarray, np.ndarray]:
    """cos / sin of each angle exactly as image_io.py:190-191 computes them."""
    c = np.empty(len(angles), np.float64)
    s = np.empty(len(angles), np.float64)
    for i, angle in enumerate(angles):
        theta = np.deg2rad(angle)
        c[i], s[i] = np.cos(theta), np.sin(theta)
    return c, s


def _best_per_angle(planes: torch.Tensor, W: int, H: int, pitch: int, tpl_dev: torch.Tensor, n: int,
                    rows: torch.Tensor, first: int, count: int, m: int, cs_dev: torch.Tensor, sn_dev: torch.Tensor,
                    na: int, stream) -> Tuple[np.ndarray, np.ndarray]:
    """Per angle, the best (score, candidate index within the size) over the
    size's `count` candidates starting at row `first` of `rows`
    (second_stage.py:106-165)."""
    L = _native.lib()
    dev = planes.device
    bfrag = torch.empty(int(L.ss_match_probe_bytes(m, na)), dtype=torch.uint8, device=dev)
    stats = torch.empty((na, 3), dtype=torch.int64, device=dev)
    base = torch.empty(m * m, dtype=torch.uint8, device=dev)
    _native.check(L.ss_match_probes(tpl_dev.data_ptr(), n, m, na, cs_dev.data_ptr(), sn_dev.data_ptr(),
                                    bfrag.data_ptr(), stats.data_ptr(), base.data_ptr(), stream), "match probes")
    parts = int(L.ss_match_parts(count))
    part_s = torch.empty((parts, _GROUP), dtype=torch.float64, device=dev)
    part_i = torch.empty((parts, _GROUP), dtype=torch.int64, device=dev)
    best_s = torch.empty(na, dtype=torch.float64, device=dev)
    best_i = torch.empty(na, dtype=torch.int64, device=dev)
    for g in range((na + _GROUP - 1) // _GROUP):
        _native.check(L.ss_match_fused(planes.data_ptr(), W, H, pitch, rows.data_ptr(), rows.shape[1], first, count,
                                       m, bfrag.data_ptr(), na, g, stats.data_ptr(), part_s.data_ptr(),
                                       part_i.data_ptr(), best_s.data_ptr(), best_i.data_ptr(), stream), "match")
    return best_s.cpu().numpy(), best_i.cpu().numpy()


def match_candidates(image: np.ndarray, template: np.ndarray, screened, angle_step: float = 10.0,
                     device=None) -> Optional[MatchResult]:
    """Evaluate every screened candidate over the angle grid and return the
    best hypothesis (second_stage.py:168-204); None for an empty candidate set."""
    img = as_gray(image)
    tpl = as_gray(template)
    angles = _angle_grid(angle_step)
    if not len(screened.candidates):
        return None
    if not torch.cuda.is_available():
        raise RuntimeError("match_candidates needs a CUDA device (no CPU fallback)")
    dev = torch.device(device if device is not None else "cuda")
    with torch.cuda.device(dev):  # launches go to `dev`'s streams whatever device is current
        return _match(img, tpl, screened, angles, dev)


def _match(img, tpl, screened, angles, dev) -> MatchResult:
    n = tpl.shape[0]
    na = len(angles)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    # candidate rows (cx, cy, m), ladder order then row-major; per-size blocks
    cand = screened.candidates
    rows = cand._rows if isinstance(cand._rows, torch.Tensor) else torch.from_numpy(cand.array())
    rows = rows.to(dev).contiguous()
    counts = screened.candidates_per_size()
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
    cs, sn = _rotation_cos_sin(angles)
    cs_dev = torch.from_numpy(cs).to(dev)
    sn_dev = torch.from_numpy(sn).to(dev)
    H, W = img.shape
    img_dev = torch.from_numpy(img).to(dev)
    tpl_dev = torch.from_numpy(tpl).to(dev)
    pitch = int(_native.lib().ss_match_plane_pitch(W))
    planes = torch.empty(3 * H * pitch, dtype=torch.uint8, device=dev)
    _native.check(_native.lib().ss_match_planes(img_dev.data_ptr(), W, H, planes.data_ptr(), pitch, sh), "match planes")
    best: Optional[MatchResult] = None
    for k in sorted(range(len(screened.ladder)), key=lambda k: screened.ladder[k]):
        m, count, first = screened.ladder[k], int(counts[k]), int(starts[k])
        if count == 0:
            continue
        top, idx = _best_per_angle(planes, W, H, pitch, tpl_dev, n, rows, first, count, m, cs_dev, sn_dev, na, sh)
        # second_stage.py:153-162: angles in order, exact ties to the smallest (angle, candidate)
        best_score, best_angle, best_cand = -math.inf, 0, 0
        for a in range(na):
            sc = float(top[a])
            c = int(idx[a])
            if sc > best_score or (sc == best_score and (a, c) < (best_angle, best_cand)):
                best_score, best_angle, best_cand = sc, a, c
        if best is None or best_score > best.score:
            cx, cy, _ = (int(v) for v in rows[first + best_cand].cpu().tolist())
            best = MatchResult(cx=cx, cy=cy, scale=m / n, angle=angles[best_angle], score=best_score)
    return best
