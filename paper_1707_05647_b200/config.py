"""Screening configuration and host-side integer geometry.

Mirrors the reference's config surface so callers switch by changing the
import: Quantizer (screening.py:64-78), ScreeningConfig (:181-199),
ladder_sizes (:202-219), quantize (:81-83), ring_plan / default_star_radius /
round_half_up / patch_center_margins (features.py:44-47, 145-148, 190-217).
Same names, argument meaning, defaults, error classes and messages.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Tuple

MIN_RING_HALF_SIZE = 4  # features.py:40
MIN_PATCH_SIDE = 2 * MIN_RING_HALF_SIZE  # screening.py:55
SQRT2 = math.sqrt(2.0)  # features.py:41
KEY_BASE = 1 << 21  # screening.py:57 _KEY_BASE


def round_half_up(x: float) -> int:
    """features.py:44-47: always round .5 upward."""
    return int(math.floor(x + 0.5))


def default_star_radius(n: int) -> int:
    """features.py:145-148: same-area diamond radius round(sqrt2 * n)."""
    return round_half_up(SQRT2 * n)


def ring_plan(m: int, ring_count: int) -> Tuple[Tuple[int, int], ...]:
    """features.py:190-211: (half_size, diamond_radius) per ring of an m x m patch."""
    if m < 2 * MIN_RING_HALF_SIZE:
        raise ValueError(f"patch side {m} too small for any ring")
    if ring_count < 1:
        raise ValueError("ring_count must be >= 1")
    cap = (m - 1) // 2
    plan: List[Tuple[int, int]] = []
    for r in range(ring_count):
        n = int(math.floor(m / (2.0 * 2.0 ** (r / 2.0))))
        if n < MIN_RING_HALF_SIZE:
            break
        plan.append((n, min(default_star_radius(n), cap)))
    return tuple(plan)


def patch_center_margins(m: int) -> Tuple[int, int]:
    """features.py:214-217: (left/top, right/bottom) centre margins."""
    return (m - 1) // 2, m // 2


@dataclass(frozen=True)
class Quantizer:
    """screening.py:64-78: per-channel quantization factors."""

    q_mean: float = 8.0
    q_std: float = 8.0
    q_grad: float = 8.0

    def __post_init__(self) -> None:
        for name, q in (("q_mean", self.q_mean), ("q_std", self.q_std), ("q_grad", self.q_grad)):
            if not (q >= 1e-3):
                raise ValueError(f"{name} must be >= 0.001, got {q}")

    def factors(self) -> Tuple[float, float, float]:
        return (self.q_mean, self.q_std, self.q_grad)


def quantize(value: float, q: float) -> int:
    """screening.py:81-83: floor(value / q + 1/2)."""
    return int(math.floor(value / q + 0.5))


@dataclass(frozen=True)
class ScreeningConfig:
    """screening.py:181-199."""

    alpha: float = 0.5
    beta: float = 2.0
    ladder_ratio: float = SQRT2
    ring_count: int = 3
    quantizer: Quantizer = Quantizer()
    stride: int = 1
    min_template_std: float = 5.0

    def __post_init__(self) -> None:
        if not (0.0 < self.alpha <= self.beta):
            raise ValueError(f"need 0 < alpha <= beta, got {self.alpha}, {self.beta}")
        if self.ladder_ratio <= 1.0:
            raise ValueError("ladder_ratio must exceed 1")
        if self.ring_count < 1:
            raise ValueError("ring_count must be >= 1")
        if self.stride < 1:
            raise ValueError("stride must be >= 1")


def ladder_sizes(n: int, cfg: ScreeningConfig) -> Tuple[int, ...]:
    """screening.py:202-219: descending patch sizes for an n x n template."""
    if n < 1:
        raise ValueError("template side must be >= 1")
    sizes: List[int] = []
    floor_raw = cfg.alpha * n * (1.0 - 1e-12)
    t = 0
    while True:
        raw = cfg.beta * n * cfg.ladder_ratio ** (-t)
        if raw < floor_raw:
            break
        m = round_half_up(raw)
        if m >= 1 and m not in sizes:
            sizes.append(m)
        t += 1
    if cfg.alpha <= 1.0 <= cfg.beta and n not in sizes:
        sizes.append(n)
    return tuple(sorted(sizes, reverse=True))


def grid_count(limit: int, lo: int, hi: int, stride: int) -> int:
    """Number of stride-grid coordinates in [lo, limit-1-hi] (screening.py:433-437)."""
    top = limit - 1 - hi
    if top < lo:
        return 0
    first = ((lo + stride - 1) // stride) * stride
    if first > top:
        return 0
    return (top - first) // stride + 1
