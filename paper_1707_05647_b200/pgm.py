"""f4: the result wire formats of the screen -- PGM masks and the stats JSON.

Mirrors the reference's file surface for this path:
``load_pgm`` / ``save_pgm`` / ``PgmError`` (image_io.py:21-22, 43-128: binary
P5 only, atomic replace), ``write_json_atomic`` (synth_bench.py:314-326) and
what ``starscreen screen --out-mask / --out-size-masks / --out-stats`` writes
(cli.py:97-166): 0/255 PGM masks and the stats payload.

The masks are produced on the device from the bit-packed results
(ss_bits_to_bytes): a size mask or the region never goes through a NumPy
bool array on the way to its PGM raster.
"""

from __future__ import annotations

import json
import os
import re
import tempfile
from pathlib import Path
from typing import Dict, Optional, Tuple, Union

import numpy as np
import torch

from . import _native
from .image import as_gray

MAX_LEVEL = 255
PathLike = Union[str, Path]


class PgmError(ValueError):
    """Raised for malformed or unsupported PGM input (image_io.py:21-22)."""


# One header field: any run of whitespace and '#' comments (to end of line),
# then the field itself (a maximal run of non-whitespace bytes).
_FIELD = re.compile(rb"(?:[ \t\n\r\v\f]|#[^\n\r]*)*([^ \t\n\r\v\f]*)")


def load_pgm(path: PathLike) -> np.ndarray:
    """Binary P5 PGM -> (height, width) uint8 array; same acceptance rules and
    PgmError cases as image_io.py:63-105 (header fields separated by
    whitespace / comments, maxval 1..255, one whitespace byte before the
    raster, trailing bytes ignored)."""
    data = Path(path).read_bytes()
    if not data.startswith(b"P5"):
        raise PgmError(f"unsupported PNM magic {data[:2]!r}, only binary P5 is handled")
    fields, pos = [], 2
    while len(fields) < 3:
        m = _FIELD.match(data, pos)
        tok, pos = m.group(1), m.end()
        if not tok:
            raise PgmError("truncated PGM header")
        if not tok.isdigit():
            raise PgmError(f"malformed PGM header field {tok!r}")
        fields.append(int(tok))
    width, height, maxval = fields
    if min(width, height) <= 0:
        raise PgmError(f"bad PGM dimensions {width}x{height}")
    if maxval > MAX_LEVEL:
        raise PgmError(f"maxval {maxval} above 255 is not supported")
    if maxval <= 0:
        raise PgmError(f"bad PGM maxval {maxval}")
    body = memoryview(data)[pos + 1:]
    need = width * height
    if len(body) < need:
        raise PgmError("truncated PGM raster")
    return np.array(body[:need], dtype=np.uint8).reshape(height, width)


def _write_atomic(path: PathLike, parts, mode: str = "wb", suffix: str = ".tmp") -> None:
    path = Path(path)
    fd, tmp = tempfile.mkstemp(dir=str(path.parent) or ".", suffix=suffix)
    try:
        with os.fdopen(fd, mode) as fh:
            for p in parts:
                fh.write(p)
        os.replace(tmp, str(path))
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def save_pgm(path: PathLike, img: np.ndarray) -> None:
    """Write a binary (P5) PGM with maxval 255, atomically (image_io.py:108-128)."""
    arr = as_gray(img)
    h, w = arr.shape
    header = f"P5\n{w} {h}\n{MAX_LEVEL}\n".encode("ascii")
    _write_atomic(path, (header, arr.tobytes()), suffix=".pgm.tmp")


def write_json_atomic(path: PathLike, payload: Dict[str, object]) -> None:
    """synth_bench.py:314-326: sorted, indented JSON, replaced in one step."""
    text = json.dumps(payload, sort_keys=True, indent=2) + "\n"
    _write_atomic(path, (text,), mode="w")


def packed_to_pgm(packed, width: int) -> np.ndarray:
    """Bit-packed mask rows (H, ceil(W/32)) -> (H, W) uint8 0/255 raster,
    expanded on the device (ss_bits_to_bytes; cli.py:97-98 _mask_to_pgm)."""
    if isinstance(packed, np.ndarray):
        if not torch.cuda.is_available():
            raise RuntimeError("PGM rasters are expanded on the GPU (no CPU fallback)")
        packed = torch.from_numpy(np.ascontiguousarray(packed).view(np.int32)).cuda()
    packed = packed.contiguous()
    H, words = packed.shape
    out = torch.empty((H, width), dtype=torch.uint8, device=packed.device)
    _native.check(_native.lib().ss_bits_to_bytes(packed.data_ptr(), words, width, H, out.data_ptr(),
                                                  torch.cuda.current_stream(packed.device).cuda_stream),
                  "bits_to_bytes")
    host = torch.empty(out.shape, dtype=torch.uint8, pin_memory=True)
    host.copy_(out, non_blocking=True)
    torch.cuda.current_stream(packed.device).synchronize()
    return host.numpy()


def screen_stats_payload(image: str, template: str, result) -> dict:
    """cli.py:101-134 _screen_stats_payload, from the result's per-size counts
    (no candidate tuples are materialised)."""
    per_size = {str(m): int(c) for m, c in zip(result.ladder, result.candidates_per_size())}
    s = result.stats
    cfg = result.config
    return {
        "image": image,
        "template": template,
        "template_side": result.template_side,
        "image_size": [result.width, result.height],
        "ladder": list(result.ladder),
        "config": {
            "alpha": cfg.alpha,
            "beta": cfg.beta,
            "ladder_ratio": cfg.ladder_ratio,
            "ring_count": cfg.ring_count,
            "q_mean": cfg.quantizer.q_mean,
            "q_std": cfg.quantizer.q_std,
            "q_grad": cfg.quantizer.q_grad,
            "stride": cfg.stride,
        },
        "stats": {
            "patches_tested": s.patches_tested,
            "patches_kept": s.patches_kept,
            "patch_pruning": s.patch_pruning,
            "region_pixels_kept": s.region_pixels_kept,
            "total_pixels": s.total_pixels,
            "region_pruning": s.region_pruning,
            "screen_time": s.wall_time_s,
        },
        "candidates_per_size": per_size,
    }


def save_screen_outputs(result, image: str = "", template: str = "", out_mask: Optional[PathLike] = None,
                        out_stats: Optional[PathLike] = None, out_size_masks: Optional[str] = None) -> dict:
    """The files `starscreen screen` writes (cli.py:142-166): the merged
    kept-region mask, per-size centre masks PREFIX_mNNN.pgm, the stats JSON.
    Returns the stats payload."""
    payload = screen_stats_payload(image, template, result)
    if out_mask:
        save_pgm(out_mask, result.region_pgm())
    if out_size_masks:
        for m in result.ladder:
            save_pgm(f"{out_size_masks}_m{m:03d}.pgm", result.size_mask_pgm(m))
    if out_stats:
        write_json_atomic(out_stats, payload)
    return payload
