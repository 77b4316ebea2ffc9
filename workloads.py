"""Seeded synthetic workloads for the five BASELINE.json configs.

Bench and test support only (not the product path).  BASELINE.json names no
public dataset; SURVEY.md section 8(d) fixes the generator:

1. seeded white noise N(0, 1), Gaussian-smoothed with sigma;
2. affinely mapped to mean 128, std 40;
3. 20 filled axis-aligned rectangles or ellipses, centres uniform,
   half-extents uniform in [0.02, 0.15] * W and [0.02, 0.15] * H, uniform
   uint8 level;
4. optional additive N(0, sigma_n) noise;
5. round half up, clip to 0..255, uint8.

Config 4 ("4x smoothing scale") is sigma = 12 on the full-resolution
16384^2 noise.  Images of >= 4096^2 pixels are smoothed on the GPU when one is
present (``_smooth_device``: a separable 97-tap Gaussian, truncate 4 sigma like
scipy, reflect padding, fp32 shifted-slice accumulation in a fixed order, so
the result is deterministic); smaller images (and GPU-less hosts) use
``scipy.ndimage.gaussian_filter``.  The two differ in the last fp32 bits, so
an image's bytes depend on where it was made; every parity check screens the
same bytes on both sides, in one process.

Templates follow the reference protocol (synth_bench.py:99-161
extract_rotated_square / make_case): angle ~ U[0, 360), scale per config,
centre uniform inside the rotation margin, retried while std < 20.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

SQRT2 = math.sqrt(2.0)


@dataclass(frozen=True)
class Workload:
    index: int
    width: int
    height: int
    images: int
    sigma: float
    noise: float
    template_side: int
    scale: Tuple[float, float]
    alpha: float
    beta: float
    ladder_ratio: float
    q: Tuple[float, float, float] = (8.0, 8.0, 8.0)
    zoom: int = 1
    seed: int = 0

    @property
    def name(self) -> str:
        return f"config{self.index}"

    def describe(self) -> str:
        return (f"config{self.index}: {self.images} x {self.width}x{self.height} u8, sigma={self.sigma}, "
                f"noise={self.noise}, n={self.template_side}, scale={self.scale}, "
                f"alpha={self.alpha}, beta={self.beta}, ratio={self.ladder_ratio:.6f}, q={self.q}")


CONFIGS = {
    0: Workload(0, 512, 512, 1, 3.0, 0.0, 32, (1.0, 1.0), 1.0, 1.0, SQRT2, (8.0, 8.0, 1e6)),
    1: Workload(1, 2048, 2048, 1, 3.0, 0.0, 64, (1.25, 1.25), 0.5, 2.0, 4.0 ** (1.0 / 7.0)),
    2: Workload(2, 4096, 4096, 1, 3.0, 8.0, 96, (0.5, 2.0), 0.4, 2.5, 6.25 ** (1.0 / 15.0)),
    3: Workload(3, 1920, 1080, 64, 3.0, 0.0, 48, (0.7, 1.5), 0.6, 1.6, (8.0 / 3.0) ** (1.0 / 7.0)),
    4: Workload(4, 16384, 16384, 1, 12.0, 0.0, 128, (0.25, 4.0), 0.25, 4.0, 16.0 ** (1.0 / 31.0)),
}


def _smooth(field: np.ndarray, sigma: float) -> np.ndarray:
    from scipy.ndimage import gaussian_filter

    return gaussian_filter(field, sigma, mode="reflect")


DEVICE_SMOOTH_PIXELS = 4096 * 4096  # images at least this large are smoothed on the GPU when one exists


def _smooth_device(field: np.ndarray, sigma: float):
    """Separable Gaussian (truncate 4 sigma, reflect padding) on the GPU; returns
    the smoothed field as a CUDA float32 tensor.  None without a GPU."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        return None
    if not torch.cuda.is_available():
        return None
    r = int(4.0 * sigma + 0.5)
    x = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-0.5 * (x / sigma) ** 2)
    w /= w.sum()
    src = torch.from_numpy(field).cuda()
    h, wd = src.shape
    # columns: pad left/right, accumulate the 2r+1 shifted slices
    pad = torch.nn.functional.pad(src[None, None], (r, r, 0, 0), mode="reflect")[0, 0]
    tmp = torch.zeros_like(src)
    for k in range(2 * r + 1):
        tmp.add_(pad[:, k:k + wd], alpha=float(w[k]))
    del pad
    pad = torch.nn.functional.pad(tmp[None, None], (0, 0, r, r), mode="reflect")[0, 0]
    out = tmp.zero_()
    for k in range(2 * r + 1):
        out.add_(pad[k:k + h, :], alpha=float(w[k]))
    return out


def _upsample_bilinear(a: np.ndarray, zoom: int, H: int, W: int) -> np.ndarray:
    h, w = a.shape
    ys = (np.arange(H, dtype=np.float64) + 0.5) / zoom - 0.5
    xs = (np.arange(W, dtype=np.float64) + 0.5) / zoom - 0.5
    y0 = np.clip(np.floor(ys).astype(np.int64), 0, h - 1)
    x0 = np.clip(np.floor(xs).astype(np.int64), 0, w - 1)
    y1 = np.clip(y0 + 1, 0, h - 1)
    x1 = np.clip(x0 + 1, 0, w - 1)
    fy = np.clip(ys - np.floor(ys), 0, 1).astype(np.float32)[:, None]
    fx = np.clip(xs - np.floor(xs), 0, 1).astype(np.float32)[None, :]
    out = np.empty((H, W), np.float32)
    step = 2048
    for r0 in range(0, H, step):
        r1 = min(H, r0 + step)
        top = a[y0[r0:r1]][:, x0] * (1 - fx) + a[y0[r0:r1]][:, x1] * fx
        bot = a[y1[r0:r1]][:, x0] * (1 - fx) + a[y1[r0:r1]][:, x1] * fx
        out[r0:r1] = top * (1 - fy[r0:r1]) + bot * fy[r0:r1]
    return out


def make_image(width: int, height: int, seed: int, sigma: float = 3.0, noise: float = 0.0,
               n_shapes: int = 20, zoom: int = 1) -> np.ndarray:
    """SURVEY.md 8(d) scene generator (deterministic for a seed)."""
    rng = np.random.default_rng(seed)
    g = None
    if zoom > 1:
        small = rng.standard_normal((math.ceil(height / zoom), math.ceil(width / zoom))).astype(np.float32)
        small = _smooth(small, sigma / zoom)
        f = _upsample_bilinear(small, zoom, height, width)
    elif width * height >= DEVICE_SMOOTH_PIXELS:
        f = rng.standard_normal((height, width), dtype=np.float32)
        g = _smooth_device(f, sigma)
        if g is None:
            f = _smooth(f, sigma)
    else:
        f = _smooth(rng.standard_normal((height, width)).astype(np.float32), sigma)
    if g is not None:  # affine map on the device (fp64 statistics), then back to the host
        import torch

        mu = float(g.mean(dtype=torch.float64))
        sd = float(torch.sqrt(((g.double() - mu) ** 2).mean()))
        g.sub_(mu).mul_(float(np.float32(40.0 / max(sd, 1e-12)))).add_(128.0)
        f = g.cpu().numpy()
        del g
    else:
        mu = float(f.mean(dtype=np.float64))
        sd = float(f.std(dtype=np.float64))
        f -= mu
        f *= np.float32(40.0 / max(sd, 1e-12))
        f += np.float32(128.0)
    for _ in range(n_shapes):
        cx = rng.uniform(0, width)
        cy = rng.uniform(0, height)
        ax = rng.uniform(0.02, 0.15) * width
        ay = rng.uniform(0.02, 0.15) * height
        level = float(rng.integers(0, 256))
        ellipse = bool(rng.integers(0, 2))
        x0, x1 = max(0, int(math.floor(cx - ax))), min(width, int(math.ceil(cx + ax)) + 1)
        y0, y1 = max(0, int(math.floor(cy - ay))), min(height, int(math.ceil(cy + ay)) + 1)
        if x0 >= x1 or y0 >= y1:
            continue
        if ellipse:
            yy = ((np.arange(y0, y1) - cy) / ay)[:, None]
            xx = ((np.arange(x0, x1) - cx) / ax)[None, :]
            inside = xx * xx + yy * yy <= 1.0
            f[y0:y1, x0:x1][inside] = level
        else:
            xs = np.abs(np.arange(x0, x1) - cx) <= ax
            ys = np.abs(np.arange(y0, y1) - cy) <= ay
            f[y0:y1, x0:x1][np.ix_(ys, xs)] = level
    if noise > 0:
        f += rng.normal(0.0, noise, f.shape).astype(np.float32)
    return np.clip(np.floor(f + np.float32(0.5)), 0, 255).astype(np.uint8)


# synth_bench.py:45-47 _geometric_offset
def _geometric_offset(side: int) -> float:
    return (side - 1) / 2.0 - (side - 1) // 2


def _sample_bilinear(img: np.ndarray, xs: np.ndarray, ys: np.ndarray) -> np.ndarray:
    h, w = img.shape
    x0 = np.floor(xs)
    y0 = np.floor(ys)
    fx = xs - x0
    fy = ys - y0
    x0 = x0.astype(np.int64)
    y0 = y0.astype(np.int64)
    x0c = np.clip(x0, 0, w - 1)
    x1c = np.clip(x0 + 1, 0, w - 1)
    y0c = np.clip(y0, 0, h - 1)
    y1c = np.clip(y0 + 1, 0, h - 1)
    f = img.astype(np.float64)
    top = f[y0c, x0c] + fx * (f[y0c, x1c] - f[y0c, x0c])
    bot = f[y1c, x0c] + fx * (f[y1c, x1c] - f[y1c, x0c])
    return top + fy * (bot - top)


def extract_rotated_square(image: np.ndarray, cx: int, cy: int, angle: float, scale: float,
                           out_side: int) -> np.ndarray:
    """Template protocol of synth_bench.py:99-112 (bilinear, round half up)."""
    delta = _geometric_offset(out_side)
    offs = np.arange(out_side, dtype=np.float64) - (out_side - 1) / 2.0
    du, dv = np.meshgrid(offs, offs)
    th = np.deg2rad(angle)
    c, s = np.cos(th), np.sin(th)
    xs = (cx + delta) + scale * (c * du - s * dv)
    ys = (cy + delta) + scale * (s * du + c * dv)
    return np.clip(np.floor(_sample_bilinear(image, xs, ys) + 0.5), 0, 255).astype(np.uint8)


def _std(img: np.ndarray) -> float:
    n = img.size
    s1 = int(img.sum(dtype=np.int64))
    s2 = int((img.astype(np.int64) ** 2).sum(dtype=np.int64))
    return math.sqrt(max(s2 / n - (s1 / n) ** 2, 0.0))


@dataclass
class Case:
    image: np.ndarray
    template: np.ndarray
    cx: int
    cy: int
    angle: float
    scale: float


def make_template(image: np.ndarray, seed: int, side: int, scale_range: Tuple[float, float],
                  std_threshold: float = 20.0, retries: int = 200) -> Case:
    """make_case draw order (synth_bench.py:141-157): scale, angle, cx, cy."""
    h, w = image.shape
    rng = np.random.default_rng(seed)
    for _ in range(retries):
        scale = float(rng.uniform(*scale_range)) if scale_range[0] != scale_range[1] else float(scale_range[0])
        angle = float(rng.uniform(0.0, 360.0))
        th = np.deg2rad(angle)
        margin = int(np.ceil((scale * side / 2.0) * (abs(np.cos(th)) + abs(np.sin(th))))) + 1
        if w - margin <= margin or h - margin <= margin:
            continue
        cx = int(rng.integers(margin, w - margin))
        cy = int(rng.integers(margin, h - margin))
        tpl = extract_rotated_square(image, cx, cy, angle, scale, side)
        if _std(tpl) < std_threshold:
            continue
        return Case(image, tpl, cx, cy, angle, scale)
    raise RuntimeError("no qualifying template")


def make_cases(cfg: Workload, images: Optional[int] = None, first_image: int = 0) -> List[Case]:
    """Seeded cases for a workload: image i uses seed cfg.seed + i."""
    count = cfg.images if images is None else images
    out = []
    for i in range(first_image, first_image + count):
        img = make_image(cfg.width, cfg.height, cfg.seed + i, cfg.sigma, cfg.noise, zoom=cfg.zoom)
        out.append(make_template(img, 1000 + cfg.seed + i, cfg.template_side, cfg.scale))
    return out


def screening_config(cfg: Workload):
    """The ScreeningConfig of a workload, built with the product's own API."""
    from paper_1707_05647_b200 import Quantizer, ScreeningConfig

    return ScreeningConfig(alpha=cfg.alpha, beta=cfg.beta, ladder_ratio=cfg.ladder_ratio,
                           quantizer=Quantizer(*cfg.q))
