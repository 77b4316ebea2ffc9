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
* ``ss_match_gather`` lays the candidates' windows out as int8 GEMM operands;
* the dot products ``W @ [P | M]`` and ``(W * W) @ M`` (second_stage.py:
  136-150) run as int8 tensor-core GEMMs (``torch._int_mm``, cuBLASLt) on
  value-128 offset operands -- exact integers, like the reference's float64
  products of integer data;
* ``ss_match_scores`` undoes the offsets and replays the reference's float64
  score sequence op for op, reducing to the best candidate per angle.

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

_CHUNK_BYTES = 768 << 20  # A-operand bytes per chunk of candidates (3 int8 matrices)


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


class _SizeProbes:
    """Probe operands of one ladder size (second_stage.py:124-135)."""

    def __init__(self, tpl_dev: torch.Tensor, n: int, m: int, cs_dev, sn_dev, na: int, stream):
        self.m = m
        self.k_pad = _round_up(m * m, 16)
        self.n1 = _round_up(2 * na, 8)
        self.n2 = _round_up(na, 8)
        dev = tpl_dev.device
        self.b1 = torch.empty((self.k_pad, self.n1), dtype=torch.int8, device=dev)
        self.b2 = torch.empty((self.k_pad, self.n2), dtype=torch.int8, device=dev)
        self.stats = torch.empty((na, 3), dtype=torch.int64, device=dev)
        base = torch.empty(m * m, dtype=torch.uint8, device=dev)
        _native.check(_native.lib().ss_match_probes(
            tpl_dev.data_ptr(), n, m, na, cs_dev.data_ptr(), sn_dev.data_ptr(), self.b1.data_ptr(), self.n1,
            self.b2.data_ptr(), self.n2, self.k_pad, self.stats.data_ptr(), base.data_ptr(), stream), "match probes")


def _best_of_size(img_dev: torch.Tensor, rows: torch.Tensor, first: int, count: int, probes: _SizeProbes, na: int,
                  stream) -> Tuple[np.ndarray, np.ndarray]:
    """Per angle, the best (score, candidate index within the size) over the
    size's `count` candidates starting at row `first` of `rows`."""
    H, W = img_dev.shape
    dev = img_dev.device
    L = _native.lib()
    per_cand = 3 * probes.k_pad
    chunk = max(32, min(_round_up(count, 32), (_CHUNK_BYTES // per_cand) // 32 * 32))
    scores, idxs = [], []
    a1 = torch.empty((chunk, probes.k_pad), dtype=torch.int8, device=dev)
    a2 = torch.empty_like(a1)
    a3 = torch.empty_like(a1)
    rsum = torch.empty((chunk, 3), dtype=torch.int64, device=dev)
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        n_pad = max(32, _round_up(e - s, 32))
        _native.check(L.ss_match_gather(img_dev.data_ptr(), W, H, rows.data_ptr(), rows.shape[1], first + s, e - s,
                                        n_pad, probes.m, probes.k_pad, a1.data_ptr(), a2.data_ptr(), a3.data_ptr(),
                                        rsum.data_ptr(), stream), "match gather")
        c1 = torch._int_mm(a1[:n_pad], probes.b1)
        c2 = torch._int_mm(a2[:n_pad], probes.b2)
        c3 = torch._int_mm(a3[:n_pad], probes.b2)
        bs = torch.empty(na, dtype=torch.float64, device=dev)
        bi = torch.empty(na, dtype=torch.int64, device=dev)
        _native.check(L.ss_match_scores(c1.data_ptr(), probes.n1, c2.data_ptr(), c3.data_ptr(), probes.n2,
                                        rsum.data_ptr(), probes.stats.data_ptr(), e - s, na, probes.k_pad, s,
                                        bs.data_ptr(), bi.data_ptr(), stream), "match scores")
        scores.append(bs)
        idxs.append(bi)
    sc = torch.stack(scores).cpu().numpy()
    ix = torch.stack(idxs).cpu().numpy()
    # chunks in candidate order: per angle the highest score, first candidate on ties
    best_s = sc[0].copy()
    best_i = ix[0].copy()
    for k in range(1, sc.shape[0]):
        upd = sc[k] > best_s
        best_s[upd] = sc[k][upd]
        best_i[upd] = ix[k][upd]
    return best_s, best_i


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
    img_dev = torch.from_numpy(img).to(dev)
    tpl_dev = torch.from_numpy(tpl).to(dev)
    best: Optional[MatchResult] = None
    for k in sorted(range(len(screened.ladder)), key=lambda k: screened.ladder[k]):
        m, count, first = screened.ladder[k], int(counts[k]), int(starts[k])
        if count == 0:
            continue
        probes = _SizeProbes(tpl_dev, n, m, cs_dev, sn_dev, na, sh)
        top, idx = _best_of_size(img_dev, rows, first, count, probes, na, sh)
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
