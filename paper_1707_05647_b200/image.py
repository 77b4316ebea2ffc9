"""Image validation (image_io.py:25-40 as_gray, :231-242 std_dev)."""

from __future__ import annotations

import numpy as np

MAX_LEVEL = 255


def as_gray(img) -> np.ndarray:
    """Validate a 2-D grayscale array and return it as C-contiguous uint8."""
    arr = np.asarray(img)
    if arr.ndim != 2:
        raise ValueError(f"expected a 2-D grayscale array, got shape {arr.shape}")
    if arr.size == 0:
        raise ValueError("empty image")
    if arr.dtype != np.uint8:
        if arr.min() < 0 or arr.max() > MAX_LEVEL:
            raise ValueError("pixel values outside [0, 255]")
        arr = arr.astype(np.uint8)
    return np.ascontiguousarray(arr)


def std_dev(img) -> float:
    """Population standard deviation from exact integer sums (bit-identical)."""
    arr = as_gray(img)
    n = arr.size
    s1 = int(arr.sum(dtype=np.int64))
    s2 = int((arr.astype(np.int64) ** 2).sum(dtype=np.int64))
    var = s2 / n - (s1 / n) ** 2
    return float(np.sqrt(max(var, 0.0)))
