"""Template-side feature sets (host).

FeatureSet mirrors screening.py:100-170 (per-ring guard-banded key sets,
ring_keys(), contains()); build_feature_set mirrors screening.py:222-250 and
runs its per-rescale work (resize, crop, patch tables, ring features, guard
cells) in native C++ (csrc/ss_template.cpp) over the host's threads.
keyset_blob packs one size's keys for the device screen.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native
from .config import KEY_BASE, MIN_PATCH_SIDE, Quantizer, ScreeningConfig, quantize, ring_plan
from .image import as_gray


@dataclass(frozen=True)
class RingBand:
    """features.py:70-76."""

    half_size: int
    radius: int
    mean: float
    std: float
    grad_mag: float


@dataclass(frozen=True)
class RingFeatureVector:
    """features.py:79-91: per-ring triples, outermost ring first."""

    rings: Tuple[RingBand, ...]

    def __post_init__(self) -> None:
        sizes = [b.half_size for b in self.rings]
        if any(inner >= outer for outer, inner in zip(sizes, sizes[1:])):
            raise ValueError(f"ring half-sizes must strictly decrease, got {sizes}")

    def __len__(self) -> int:
        return len(self.rings)


class FeatureSet:
    """screening.py:100-170: per-ring sets of packed quantized feature keys."""

    def __init__(self, plan: Sequence[Tuple[int, int]], quantizer: Quantizer):
        if not plan:
            raise ValueError("empty ring plan")
        self.plan = tuple(plan)
        self.quantizer = quantizer
        self._rings: List[set] = [set() for _ in plan]
        self._sorted: Optional[List[np.ndarray]] = None

    def __len__(self) -> int:
        return sum(len(s) for s in self._rings)

    def ring_sizes(self) -> Tuple[int, ...]:
        return tuple(len(s) for s in self._rings)

    def _guard_cells(self, value: float, q: float) -> List[int]:
        half = q / 2.0
        return sorted({quantize(value - half, q), quantize(value, q), quantize(value + half, q)})

    def insert(self, fv: RingFeatureVector) -> None:
        """Insert one template instance with the guard band (screening.py:127-145)."""
        if len(fv) != len(self.plan):
            raise ValueError(f"expected {len(self.plan)} rings, got {len(fv)}")
        qm, qs, qg = self.quantizer.factors()
        for ring, band in zip(self._rings, fv.rings):
            for cm in self._guard_cells(band.mean, qm):
                for cs in self._guard_cells(band.std, qs):
                    for cg in self._guard_cells(band.grad_mag, qg):
                        if cm >= KEY_BASE or cs >= KEY_BASE or cg >= KEY_BASE:
                            raise ValueError("quantized cell exceeds key capacity, quantizer too fine")
                        if cm < 0 or cs < 0 or cg < 0:
                            raise ValueError("negative quantized cell; features must be non-negative")
                        ring.add((cm * KEY_BASE + cs) * KEY_BASE + cg)
        self._sorted = None

    def _set_sorted(self, arrays: List[np.ndarray]) -> None:
        self._rings = [set(a.tolist()) for a in arrays]
        self._sorted = [np.ascontiguousarray(a, dtype=np.int64) for a in arrays]

    def ring_keys(self) -> List[np.ndarray]:
        """Sorted key arrays, one per ring (screening.py:147-155)."""
        if self._sorted is None:
            self._sorted = [np.fromiter(s, dtype=np.int64, count=len(s)) for s in self._rings]
            for a in self._sorted:
                a.sort()
        return self._sorted

    def contains(self, fv: RingFeatureVector) -> bool:
        """True when every ring's quantized key is marked (screening.py:157-170)."""
        if len(fv) != len(self.plan):
            raise ValueError(f"expected {len(self.plan)} rings, got {len(fv)}")
        qm, qs, qg = self.quantizer.factors()
        for ring, band in zip(self._rings, fv.rings):
            cm, cs, cg = quantize(band.mean, qm), quantize(band.std, qs), quantize(band.grad_mag, qg)
            if cm < 0 or cs < 0 or cg < 0:
                return False
            if (cm * KEY_BASE + cs) * KEY_BASE + cg not in ring:
                return False
        return True


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def template_ring_features(template: np.ndarray, k: int, m: int, plan) -> np.ndarray:
    """Ring features (n_rings, 3) of rescale k of the template (screening.py:238-248 body)."""
    tpl = as_gray(template)
    rn = np.array([p[0] for p in plan], np.int32)
    rd = np.array([p[1] for p in plan], np.int32)
    out = np.empty((len(plan), 3), np.float64)
    _native.check(_native.lib().ss_template_ring_features(_ptr(tpl), tpl.shape[0], k, m, len(plan), _ptr(rn),
                                                          _ptr(rd), _ptr(out)), "template features")
    return out


def build_feature_set(template: np.ndarray, m: int, cfg: ScreeningConfig) -> FeatureSet:
    """screening.py:222-250: feature set of every template rescale k = m .. ceil(m * ratio)."""
    tpl = as_gray(template)
    if m < MIN_PATCH_SIDE:
        raise ValueError(f"patch side {m} below minimum {MIN_PATCH_SIDE}")
    plan = ring_plan(m, cfg.ring_count)
    fs = FeatureSet(plan, cfg.quantizer)
    k_hi = math.ceil(m * cfg.ladder_ratio)
    n = tpl.shape[0]
    if tpl.shape[0] != tpl.shape[1]:
        raise ValueError(f"template must be square, got {tpl.shape[1]}x{tpl.shape[0]}")
    rn = np.array([p[0] for p in plan], np.int32)
    rd = np.array([p[1] for p in plan], np.int32)
    cap = len(plan) * 27 * (k_hi - m + 1)
    keys = np.empty(cap, np.int64)
    off = np.empty(len(plan) + 1, np.int64)
    qm, qs, qg = cfg.quantizer.factors()
    _native.check(_native.lib().ss_feature_set_keys(_ptr(tpl), n, m, k_hi, len(plan), _ptr(rn), _ptr(rd), qm, qs, qg,
                                                    _ptr(keys), _ptr(off)), "feature set")
    fs._set_sorted([keys[off[r]:off[r + 1]].copy() for r in range(len(plan))])
    return fs


SS_MAX_RINGS = 16
DESC_STRIDE = 4 + 2 * SS_MAX_RINGS


def instance_descriptors(ms, ring_count: int, ladder_ratio: float):
    """Rescale instances (m, k = m .. ceil(m * ratio), screening.py:236-238) of
    every size in `ms` as the f2 kernel's descriptor rows
    [m, k, n_rings, 0, n_0, d_0, ...]; returns (desc (n_inst, DESC_STRIDE)
    int32, nk (len(ms),) int32 instances per size)."""
    rows, nk = [], []
    for m in ms:
        if m < MIN_PATCH_SIDE:
            raise ValueError(f"patch side {m} below minimum {MIN_PATCH_SIDE}")
        plan = ring_plan(m, ring_count)
        k_hi = math.ceil(m * ladder_ratio)
        d = np.zeros((k_hi - m + 1, DESC_STRIDE), np.int32)
        d[:, 0] = m
        d[:, 1] = np.arange(m, k_hi + 1)
        d[:, 2] = len(plan)
        for r, (nr, dr) in enumerate(plan):
            d[:, 4 + 2 * r], d[:, 5 + 2 * r] = nr, dr
        rows.append(d)
        nk.append(k_hi - m + 1)
    desc = np.concatenate(rows) if rows else np.zeros((0, DESC_STRIDE), np.int32)
    return np.ascontiguousarray(desc), np.array(nk, np.int32)


_desc_cache: dict = {}


def _device_desc(desc: np.ndarray, dev):
    """Device copy of a (read-only, geometry-cached) descriptor array, kept
    per (array, device): the descriptors of a ladder geometry never change."""
    key = (id(desc), str(dev))
    hit = _desc_cache.get(key)
    if hit is not None and hit[0] is desc:
        return hit[1]
    if len(_desc_cache) > 64:
        _desc_cache.clear()
    import torch

    t = torch.from_numpy(np.ascontiguousarray(desc)).to(dev)  # synchronous: complete before any stream uses it
    _desc_cache[key] = (desc, t)
    return t


def launch_template_features(template: np.ndarray, desc: np.ndarray, device, stream=None, owned: bool = False):
    """Enqueue the ring features of the rescale instances `desc`
    (instance_descriptors) of the template: one GPU launch (f2,
    csrc/ss_featureset.cu) on `stream` (default: the current stream) and the
    copy of the result into pinned host memory.  Returns a handle for
    wait_template_features.  owned=True: the round trip gets its own buffers
    (several may be in flight on one stream: screen_batch), else the
    stream's cached staging buffers."""
    import torch

    tpl = as_gray(template)
    n = tpl.shape[0]
    if tpl.shape[0] != tpl.shape[1]:
        raise ValueError(f"template must be square, got {tpl.shape[1]}x{tpl.shape[0]}")
    if desc.shape[0] == 0:
        return None
    dev = torch.device(device)
    stream = stream or torch.cuda.current_stream(dev)
    d_desc = _device_desc(desc, dev)
    st = _staging(dev, stream, n * n, desc.shape[0]) if not owned else _owned_staging(dev, n * n, desc.shape[0])
    _native.check(_native.lib().ss_template_features_async(
        tpl.ctypes.data, n, desc.shape[0], d_desc.data_ptr(), DESC_STRIDE, st["tpl"].data_ptr(), st["out"].data_ptr(),
        st["host"].data_ptr(), stream.cuda_stream, st["event"].cuda_event), "template features")
    return st["host"][: desc.shape[0]], st["event"]


_staging_cache: dict = {}


def _owned_staging(dev, tpl_bytes: int, n_inst: int) -> dict:
    """Fresh f2 round-trip buffers (the caller's handle keeps them alive)."""
    import torch

    event = torch.cuda.Event()
    return {"tpl": torch.empty(max(tpl_bytes, 1), dtype=torch.uint8, device=dev),
            "out": torch.empty((n_inst, SS_MAX_RINGS, 3), dtype=torch.float64, device=dev),
            "host": torch.empty((n_inst, SS_MAX_RINGS, 3), dtype=torch.float64, pin_memory=True),
            "event": event}


def _staging(dev, stream, tpl_bytes: int, n_inst: int) -> dict:
    """Per-stream buffers of the f2 round trip (device template and features,
    pinned host features, an event), grown on demand.  A stream's previous
    round trip has been consumed (wait_template_features) before the next
    one is enqueued on it (engine order)."""
    import torch

    key = (str(dev), stream.cuda_stream)
    st = _staging_cache.get(key)
    if st is None or st["tpl"].numel() < tpl_bytes or st["out"].shape[0] < n_inst:
        tb = max(tpl_bytes, 128 * 128, st["tpl"].numel() if st else 0)
        ni = max(n_inst, 64, st["out"].shape[0] if st else 0)
        event = torch.cuda.Event()
        event.record(stream)  # creates the handle
        st = {"tpl": torch.empty(tb, dtype=torch.uint8, device=dev),
              "out": torch.empty((ni, SS_MAX_RINGS, 3), dtype=torch.float64, device=dev),
              "host": torch.empty((ni, SS_MAX_RINGS, 3), dtype=torch.float64, pin_memory=True),
              "event": event}
        if len(_staging_cache) > 32:
            _staging_cache.clear()
        _staging_cache[key] = st
    return st


def wait_template_features(handle) -> np.ndarray:
    """(n_inst, SS_MAX_RINGS, 3) float64 host features of a launch_template_features handle."""
    if handle is None:
        return np.zeros((0, SS_MAX_RINGS, 3))
    host, done = handle
    done.synchronize()
    return host.numpy()


def template_features_device(template: np.ndarray, desc: np.ndarray, device, stream=None) -> np.ndarray:
    """Ring features of the rescale instances `desc` (instance_descriptors) of
    the template from one GPU launch (f2); (n_inst, SS_MAX_RINGS, 3) float64."""
    return wait_template_features(launch_template_features(template, desc, device, stream))


def build_feature_sets_device(template: np.ndarray, ms, cfg: ScreeningConfig, device) -> dict:
    """build_feature_set for every size in `ms` with the rescale features on the GPU (f2).

    The guard-banded key sets are built on the host from the returned
    features, in k order, exactly as build_feature_set (screening.py:222-250)
    does.
    """
    desc, nks = instance_descriptors(ms, cfg.ring_count, cfg.ladder_ratio)
    feats_all = template_features_device(template, desc, device)
    out = {}
    qm, qs, qg = cfg.quantizer.factors()
    first = 0
    for m, nk in zip(ms, nks):
        nk = int(nk)
        plan = ring_plan(m, cfg.ring_count)
        feats = np.ascontiguousarray(feats_all[first:first + nk, :len(plan), :])
        first += nk
        keys = np.empty(len(plan) * 27 * nk, np.int64)
        off = np.empty(len(plan) + 1, np.int64)
        _native.check(_native.lib().ss_keys_from_features(_ptr(feats), nk, len(plan), qm, qs, qg, _ptr(keys),
                                                          _ptr(off)), "feature set")
        fs = FeatureSet(plan, cfg.quantizer)
        fs._set_sorted([keys[off[r]:off[r + 1]].copy() for r in range(len(plan))])
        out[m] = fs
    return out


def keyset_blob(fs: FeatureSet) -> np.ndarray:
    """Device-ready membership blob of one size (keys + mean / (mean,std) projections)."""
    arrays = fs.ring_keys()
    keys = np.ascontiguousarray(np.concatenate(arrays) if arrays else np.zeros(0, np.int64), dtype=np.int64)
    off = np.zeros(len(arrays) + 1, np.int64)
    off[1:] = np.cumsum([len(a) for a in arrays])
    size = ctypes.c_size_t(0)
    L = _native.lib()
    _native.check(L.ss_keyset_blob(_ptr(keys), _ptr(off), len(arrays), None, ctypes.byref(size)), "keyset")
    blob = np.empty(size.value // 8, np.int64)
    _native.check(L.ss_keyset_blob(_ptr(keys), _ptr(off), len(arrays), _ptr(blob), ctypes.byref(size)), "keyset")
    return blob
