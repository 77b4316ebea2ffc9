"""Device-resident screening engine (torch owns the memory, libstarscreen does the work).

One Engine holds the 12 integral planes, workspaces and result buffers for
images of one (W, H) on one device.  ``run`` enqueues the whole hot path on
the current CUDA stream -- table build (K1/K2), then per ladder size the
screen (K3), survivor compaction (K4) and footprint union (K5), then the
region popcount -- with no host synchronisation, so a run can be captured in
a CUDA graph.  Row-band shards use the same engine with a band frame
(y_origin, y_begin, y_end); see sharding.py.
"""

from __future__ import annotations

import ctypes
import functools
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _native
from ._native import SS_BLOB_MAX_BITMAP_WORDS, SS_MAX_RINGS
from .config import MIN_PATCH_SIDE, ScreeningConfig, grid_count, ladder_sizes, patch_center_margins, ring_plan
from .featureset import (FeatureSet, build_feature_set, instance_descriptors, keyset_blob, launch_template_features,
                         wait_template_features)


import os

# Ladder sizes run on up to N_STREAMS side streams (fork/join around K3):
# for images whose 32-bit tables fit in a few GB, three sizes in flight fill
# the launch tails and overlap one size's compute-bound stage 1 with
# another's memory-bound rings (measured: config 1 -19%, config 2 -12%);
# for larger images two sizes' working sets thrash L2 (config 4 +27%), so
# they run one at a time.  SS_STREAMS overrides (experiments).
N_STREAMS = 3
STREAMS_MAX_TABLE_BYTES = 4 << 30


# Fused ladder (ss_ladder_screen.cu): every size sharing a plane width is
# screened in lock-step, two launches per row band, so each plane row is read
# from HBM about once per band instead of once per size.  SS_FUSED=0 selects
# the per-size kernels on side streams (experiments, tests).
def fused_enabled() -> bool:
    return os.environ.get("SS_FUSED", "1") != "0"


def streams_for(table_bytes: int) -> int:
    env = os.environ.get("SS_STREAMS")
    if env:
        return max(1, int(env))
    return N_STREAMS if table_bytes <= STREAMS_MAX_TABLE_BYTES else 1


def _p(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream_handle(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


@dataclass
class SizePlan:
    m: int
    plan: Tuple[Tuple[int, int], ...] = ()
    keys: Optional[List[np.ndarray]] = None  # per-ring sorted keys (FeatureSet.ring_keys())
    blob: Optional[np.ndarray] = None  # host key blob (kernel parameters are read from it)
    ring_n: Optional[np.ndarray] = None
    ring_d: Optional[np.ndarray] = None
    fits32: bool = True  # ring sums recoverable from the 32-bit planes (ss_screen_fits32)
    quantizer: Optional[object] = None
    _fs: Optional[FeatureSet] = None

    @property
    def feature_set(self) -> Optional[FeatureSet]:
        """The reference's FeatureSet for this size (built on first access)."""
        if self._fs is None and self.keys is not None:
            fs = FeatureSet(self.plan, self.quantizer)
            fs._set_sorted(self.keys)
            self._fs = fs
        return self._fs


@dataclass
class TemplatePlan:
    """Everything the device needs about one template and config: per size the
    ring plan and key blob, and the whole ladder as flat arrays for
    ss_screen_ladder (one call per screen)."""

    template_side: int
    config: ScreeningConfig
    ladder: Tuple[int, ...]
    sizes: List[SizePlan] = field(default_factory=list)
    m_arr: Optional[np.ndarray] = None  # (L,) int32
    n_rings: Optional[np.ndarray] = None  # (L,) int32, 0 for m < MIN_PATCH_SIDE
    ring_n: Optional[np.ndarray] = None  # (L, SS_MAX_RINGS) int32
    ring_d: Optional[np.ndarray] = None
    blobs: Optional[np.ndarray] = None  # all sizes' key blobs, int64
    blob_off: Optional[np.ndarray] = None  # (L + 1,) int64 slot offsets
    blobs_dev: Optional[torch.Tensor] = None
    geometry: Optional["LadderGeometry"] = None

    @property
    def max_m(self) -> int:
        return max(self.ladder) if self.ladder else 1


@dataclass(frozen=True)
class LadderGeometry:
    """Config-derived constants of one (template side, config): ladder, ring
    plans, the flat per-size arrays ss_screen_ladder reads and the f2
    instance descriptors.  Pure functions of (n, alpha, beta, ladder_ratio,
    ring_count), computed once and shared (read-only) by every TemplatePlan."""

    ladder: Tuple[int, ...]
    plans: Tuple[Tuple[Tuple[int, int], ...], ...]
    m_arr: np.ndarray
    n_rings: np.ndarray
    ring_n: np.ndarray
    ring_d: np.ndarray
    fits32: Tuple[bool, ...]
    evaluated: Tuple[int, ...]
    desc: np.ndarray  # (n_inst, DESC_STRIDE) int32 rescale instances of the evaluated sizes
    nk: np.ndarray  # (len(evaluated),) int32 instances per evaluated size


@functools.lru_cache(maxsize=64)
def ladder_geometry(n: int, alpha: float, beta: float, ladder_ratio: float, ring_count: int) -> LadderGeometry:
    cfg = ScreeningConfig(alpha=alpha, beta=beta, ladder_ratio=ladder_ratio, ring_count=ring_count)
    ladder = ladder_sizes(n, cfg)
    L = len(ladder)
    plans = tuple(ring_plan(m, ring_count) if m >= MIN_PATCH_SIDE else () for m in ladder)
    m_arr = np.array(ladder, np.int32)
    n_rings = np.array([len(p) for p in plans], np.int32)
    ring_n = np.zeros((max(L, 1), SS_MAX_RINGS), np.int32)
    ring_d = np.zeros((max(L, 1), SS_MAX_RINGS), np.int32)
    fits = []
    lib = _native.lib()
    for k, plan in enumerate(plans):
        for r, (nr, dr) in enumerate(plan):
            ring_n[k, r], ring_d[k, r] = nr, dr
        fits.append(bool(plan) and bool(lib.ss_screen_fits32(len(plan), ring_n[k].ctypes.data, ring_d[k].ctypes.data)))
    evaluated = tuple(m for m in ladder if m >= MIN_PATCH_SIDE)
    desc, nk = instance_descriptors(evaluated, ring_count, ladder_ratio)
    for a in (m_arr, n_rings, ring_n, ring_d, nk):
        a.setflags(write=False)
    return LadderGeometry(ladder, plans, m_arr, n_rings, ring_n, ring_d, tuple(fits), evaluated, desc, nk)


def plan_ladder(n: int, cfg: ScreeningConfig) -> TemplatePlan:
    """The template-independent part of prepare_template: ladder, ring plans,
    flat arrays (ladder_sizes screening.py:202-219, ring_plan
    features.py:190-211)."""
    geo = ladder_geometry(n, cfg.alpha, cfg.beta, cfg.ladder_ratio, cfg.ring_count)
    tp = TemplatePlan(n, cfg, geo.ladder)
    tp.geometry = geo
    tp.m_arr, tp.n_rings, tp.ring_n, tp.ring_d = geo.m_arr, geo.n_rings, geo.ring_n, geo.ring_d
    for k, m in enumerate(geo.ladder):
        plan = geo.plans[k]
        sp = SizePlan(m, plan, quantizer=cfg.quantizer, fits32=geo.fits32[k] if plan else True)
        if plan:
            sp.ring_n = geo.ring_n[k, : len(plan)]
            sp.ring_d = geo.ring_d[k, : len(plan)]
        tp.sizes.append(sp)
    return tp


def launch_features(tp: TemplatePlan, template: np.ndarray, device, stream: Optional[torch.cuda.Stream] = None,
                    owned: bool = False):
    """Start fill_keysets' GPU part early (f2 rescale features, async on
    `stream`; owned: with its own buffers, see launch_template_features);
    pass the handle to fill_keysets.  None off the GPU path."""
    dev = torch.device(device) if device is not None else torch.device("cpu")
    geo = getattr(tp, "geometry", None)
    if dev.type != "cuda" or geo is None or not geo.evaluated:
        return None
    return launch_template_features(template, geo.desc, dev, stream, owned=owned)


def upload_keysets(tp: TemplatePlan, device) -> None:
    """The key blobs to the device on the current stream (a few KB-MB: a
    pageable copy costs less host time than pinning a fresh buffer)."""
    tp.blobs_dev = torch.from_numpy(tp.blobs).to(torch.device(device), non_blocking=True)


def fill_keysets(tp: TemplatePlan, template: np.ndarray, device, stream: Optional[torch.cuda.Stream] = None,
                 pending=None, upload: bool = True) -> None:
    """The template-dependent part of prepare_template (build_feature_set,
    screening.py:222-250, for every size).

    On a CUDA device: the rescale features of every size from one GPU launch
    on `stream` (f2; only that stream is synchronised), the key sets and
    device blobs of every size from one host call (ss_ladder_keysets), and
    one upload of the blobs on the current stream.  Otherwise each size goes
    through the host C++ build_feature_set.
    """
    cfg = tp.config
    dev = torch.device(device) if device is not None else torch.device("cpu")
    L = len(tp.sizes)
    geo = getattr(tp, "geometry", None)
    if dev.type == "cuda" and geo is not None and geo.evaluated:
        if pending is None:
            pending = launch_template_features(template, geo.desc, dev, stream)
        feats = wait_template_features(pending)
        nk = geo.nk
        n_r = tp.n_rings[tp.n_rings > 0]
        keys_cap = int(27 * (nk.astype(np.int64) * n_r).sum())
        blobs_cap = int(sum(1 + 16 * int(r) + int(r) * (81 * int(k) + SS_BLOB_MAX_BITMAP_WORDS // 2 + 2)
                            for k, r in zip(nk, n_r)))
        keys = np.empty(max(keys_cap, 1), np.int64)
        key_off = np.empty(int(n_r.sum()) + len(n_r), np.int64)
        blobs = np.empty(max(blobs_cap, 1), np.int64)
        boff = np.empty(len(n_r) + 1, np.int64)
        q = cfg.quantizer.factors()
        _native.check(_native.lib().ss_ladder_keysets(
            feats.ctypes.data, SS_MAX_RINGS, len(n_r), nk.ctypes.data, n_r.ctypes.data, q[0], q[1], q[2],
            keys.ctypes.data, keys.size, key_off.ctypes.data, blobs.ctypes.data, blobs.size, boff.ctypes.data),
            "feature sets")
        tp.blobs = blobs[: int(boff[-1])]
        tp.blob_off = np.zeros(L + 1, np.int64)
        i = ko = kp = 0
        for k, sp in enumerate(tp.sizes):
            if sp.plan:
                r = len(sp.plan)
                off = key_off[ko: ko + r + 1]
                sp.keys = [keys[kp + off[j]: kp + off[j + 1]] for j in range(r)]
                kp += int(off[r])
                ko += r + 1
                sp.blob = tp.blobs[int(boff[i]): int(boff[i + 1])]
                i += 1
            tp.blob_off[k + 1] = boff[i]
    else:
        parts = []
        tp.blob_off = np.zeros(L + 1, np.int64)
        for k, sp in enumerate(tp.sizes):
            if sp.plan:
                fs = build_feature_set(template, sp.m, cfg)
                sp._fs = fs
                sp.keys = fs.ring_keys()
                sp.blob = keyset_blob(fs)
                parts.append(sp.blob)
            tp.blob_off[k + 1] = tp.blob_off[k] + (len(sp.blob) if sp.plan else 0)
        tp.blobs = np.concatenate(parts) if parts else np.zeros(0, np.int64)
    if not tp.blobs.size:
        tp.blobs = np.zeros(1, np.int64)
    if dev.type == "cuda" and upload:
        upload_keysets(tp, dev)


def prepare_template(template: np.ndarray, cfg: ScreeningConfig, device,
                     stream: Optional[torch.cuda.Stream] = None) -> TemplatePlan:
    """Template side of screen() (screening.py:497, 511): ladder + per-size key sets."""
    tp = plan_ladder(template.shape[1], cfg)
    fill_keysets(tp, template, device, stream)
    return tp


class Engine:
    def __init__(self, width: int, height: int, device=None, band: Optional[Tuple[int, int, int, int]] = None):
        """band = (y_origin, rows, y_begin, y_end): the tables cover global rows
        [y_origin, y_origin + rows) and rows [y_begin, y_end) are decided.
        Default: the full image."""
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1707_05647_b200 needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device if device is not None else "cuda")
        self.L = _native.lib()
        self.W, self.H = int(width), int(height)
        if band is None:
            band = (0, self.H, 0, self.H)
        self.y_origin, self.rows, self.y_begin, self.y_end = (int(v) for v in band)
        self.pitch = int(self.L.ss_plane_pitch(self.W))
        # 32-bit planes (cells mod 2^32) serve every size whose ring sums fit
        # (ss_screen_fits32); the int64 planes are allocated and built only
        # for templates with a larger size (see run())
        tb32 = int(self.L.ss_tables32_bytes(self.W, self.rows))
        self.planes32 = torch.empty(tb32 // 4, dtype=torch.int32, device=self.device)
        self.planes = None
        self.build_ws = torch.empty(max(1, int(self.L.ss_build_workspace_bytes(self.W, self.rows))), dtype=torch.uint8,
                                    device=self.device)
        self.words = (self.W + 31) // 32
        self.mrows = self.y_end - self.y_begin
        self.compact_ws = None
        # ladder sizes are independent: they run on N_STREAMS side streams
        # (fork/join around the K3 region), each with its own screen workspace
        self.n_streams = streams_for(tb32)
        self.streams = [torch.cuda.Stream(self.device) for _ in range(self.n_streams)]
        self.template_stream = torch.cuda.Stream(self.device)  # f2 features, overlapping the table build
        self.screen_ws = None  # per-size workspaces, one per side stream (allocated when the per-size path runs)
        self.ladder_ws = None  # fused ladder workspace (allocated for the first ladder that needs it)
        self.region_stream = None  # K5 beside K4
        self.copy_stream = None  # survivor-row readback (start_readback)
        self.compact_event = None  # recorded after K4 of the last run
        self.readback_done = None  # the last readback's completion (K4 of the next run waits on it)
        self.last_kept = None  # survivors of the last fetched screen (sizes the next readback)
        self.totals = torch.zeros(2, dtype=torch.int64, device=self.device)  # [0] survivors, [1] region pixels
        self.n_sizes = 0
        self.masks = None
        self.row_counts = None
        self.size_counts = None
        self.region = None
        self.region_ws = None
        self._region_m = 0
        self.capacity = 0
        self.xy = None
        self.hi16 = None  # bits 32..47 of the cells (the fused rings' wide path, instead of the int64 planes)
        self.built_int64 = False  # what the last build wrote beyond the 32-bit planes
        self.built_hi16 = False
        self.coarse = None  # stage 1's coarse planes (u16 bit slices, ss_build_tables3)
        self.coarse_shifts: List[int] = []  # the shifts the last build wrote
        self.masks_done = None  # completion of the last run's streamed mask copy (run(host_masks=...))
        self.region_event = None  # K5 of the last run done (start_region_readback)
        self._host_masks_inflight = None  # (pinned buffer, event) of that copy, kept alive until it has landed
        self.stage_counts = None  # set to a (4,) int64 device tensor to instrument the cascade
        self.force_int64 = False  # test hook: screen every size from the int64 planes
        self.hooks = None  # optional (before, after) callables(main_stream) around the K3 region
        # one screen at a time per engine: its tables, masks and result buffers are shared state
        self.lock = threading.RLock()

    # ── buffers ────────────────────────────────────────────────────────────
    def _ensure(self, n_sizes: int, max_m: int, capacity: int, region: bool) -> None:
        if self.masks is None or self.n_sizes != n_sizes:
            self.n_sizes = n_sizes
            self.masks = torch.empty((n_sizes, self.mrows, self.words), dtype=torch.int32, device=self.device)
            self.row_counts = torch.empty((n_sizes, max(self.mrows, 1)), dtype=torch.int32, device=self.device)
            self.size_counts = torch.zeros(n_sizes, dtype=torch.int64, device=self.device)
            self.compact_ws = torch.empty(int(self.L.ss_compact_ladder_workspace_bytes(max(self.mrows, 1), n_sizes)),
                                          dtype=torch.uint8, device=self.device)
            self.region_ws = None
        if region and (self.region is None or self.region_ws is None):
            self.region = torch.empty((self.H, self.words), dtype=torch.int32, device=self.device)
            self.region_ws = torch.empty(int(self.L.ss_region_ladder_workspace_bytes(self.W, self.H, n_sizes)),
                                         dtype=torch.uint8, device=self.device)
        if self.xy is None or self.capacity < capacity:
            self.capacity = max(capacity, 1)
            self.xy = torch.empty((self.capacity, 3), dtype=torch.int32, device=self.device)

    def default_capacity(self, tp: TemplatePlan) -> int:
        # Start at 2% of the decided positions (measured survivor rates are
        # 0.1-17%); fetch() grows the buffer and re-compacts on overflow.
        tested = self.tested(tp)
        return max(1 << 16, tested // 50)

    def tested(self, tp: TemplatePlan) -> int:
        """patches_tested of the decided rows (screening.py:446, 513)."""
        return sum(self.tested_per_size(tp))

    def tested_per_size(self, tp: TemplatePlan) -> List[int]:
        out = []
        for sp in tp.sizes:
            if sp.m < MIN_PATCH_SIDE:
                out.append(0)
                continue
            lo, hi = patch_center_margins(sp.m)
            nx = grid_count(self.W, lo, hi, tp.config.stride)
            ylo, yhi = max(self.y_begin, lo), min(self.y_end - 1, self.H - 1 - hi)
            ny = 0
            if yhi >= ylo:
                s = tp.config.stride
                first = ((ylo + s - 1) // s) * s
                ny = 0 if first > yhi else (yhi - first) // s + 1
            out.append(nx * ny)
        return out

    # ── the hot path ───────────────────────────────────────────────────────
    def needs_int64(self, tp: TemplatePlan) -> bool:
        """True when some size's ring sums exceed the 32-bit planes."""
        if self.force_int64:
            return True
        for sp in tp.sizes:
            if sp.plan and not sp.fits32:
                return True
        return False

    def coarse_shifts_for(self, tp: Optional[TemplatePlan]) -> List[int]:
        """The coarse-plane shifts stage 1 needs for this ladder: ss_coarse_shift
        of every evaluated size's ring-0 square (4 n^2) and diamond
        (2 d^2 + 2 d + 1) pixel counts ([] when a count has none, more than
        SS_MAX_COARSE are needed, or SS_COARSE=0)."""
        if tp is None or os.environ.get("SS_COARSE", "1") == "0":
            return []
        need = set()
        for sp in tp.sizes:
            if not sp.plan:
                continue
            n, d = sp.plan[0]
            for count in (4 * n * n, 2 * d * d + 2 * d + 1):
                k = int(self.L.ss_coarse_shift(count))
                if k < 0:
                    return []
                need.add(k)
        return sorted(need) if len(need) <= _native.SS_MAX_COARSE else []

    def wide_as_hi16(self, tp: Optional[TemplatePlan]) -> bool:
        """Sizes beyond 32 bits read 32-bit + hi16 cells (mod 2^48) in the
        fused rings when the fused ladder takes their group (ss_ladder_screen.cu:
        <= 64 sizes, <= 104 rings, <= 8 rings per size, H < 2^24), every ring
        sum stays below 2^48 and ring 0's PLAIN sums below 2^32; otherwise
        (and under SS_FUSED=0 / force_int64) the int64 planes are built."""
        if tp is None or self.force_int64 or not fused_enabled() or self.H >= (1 << 24) or self.W > (1 << 30):
            return False
        wide = [sp for sp in tp.sizes if sp.plan and not sp.fits32]
        if not wide or len(wide) > 64 or sum(len(sp.plan) for sp in wide) > 104:
            return False
        span = max(self.W, self.H) + 1
        for sp in wide:
            if len(sp.plan) > 8:
                return False
            for r, (n, d) in enumerate(sp.plan):
                cq, cd = 4 * n * n, 2 * d * d + 2 * d + 1
                if 255 * max(cq, cd) * span >= 1 << 48:
                    return False
                if r == 0 and 255 * max(cq, cd) >= 1 << 32:
                    return False
        return True

    def build_tables(self, img: torch.Tensor, int64: bool = False, tp: Optional[TemplatePlan] = None) -> None:
        """K1/K2 on the current stream.  img: (rows, W) uint8 on the device.
        Writes the 32-bit planes, the int64 planes too when `int64`, and --
        given the template plan -- the coarse planes its stage 1 reads."""
        with torch.cuda.device(self.device):
            self._build_tables(img, int64, tp)

    def _build_tables(self, img: torch.Tensor, int64: bool, tp: Optional[TemplatePlan] = None) -> None:
        assert img.dtype == torch.uint8 and img.is_cuda and img.shape == (self.rows, self.W)
        img = img.contiguous()
        hi16 = int64 and self.wide_as_hi16(tp)
        int64 = int64 and not hi16
        if int64 and self.planes is None:
            tb = int(self.L.ss_tables_bytes(self.W, self.rows))
            self.planes = torch.empty(tb // 8, dtype=torch.int64, device=self.device)
        if hi16 and self.hi16 is None:
            self.hi16 = torch.empty(int(self.L.ss_tables_hi16_bytes(self.W, self.rows)) // 2, dtype=torch.int16,
                                    device=self.device)
        shifts = self.coarse_shifts_for(tp)
        if shifts:
            nb = int(self.L.ss_coarse_bytes(self.W, self.rows, len(shifts)))
            if self.coarse is None or self.coarse.numel() < nb:
                self.coarse = None
                self.coarse = torch.empty(nb, dtype=torch.uint8, device=self.device)
        sh = np.array(shifts or [0], np.int32)
        _native.check(self.L.ss_build_tables3(img.data_ptr(), self.W, self.rows, self.W,
                                              _p(self.planes) if int64 else None, self.planes32.data_ptr(),
                                              _p(self.hi16) if hi16 else None,
                                              self.pitch, _p(self.coarse) if shifts else None, len(shifts),
                                              sh.ctypes.data, self.build_ws.data_ptr(), self.build_ws.numel(),
                                              _stream_handle(self.device)), "build_tables")
        self.coarse_shifts = list(shifts)
        self.built_int64, self.built_hi16 = int64, hi16

    def screen_ladder(self, tp: TemplatePlan, main: Optional[torch.cuda.Stream] = None,
                      rows: Optional[Tuple[int, int]] = None) -> None:
        """K3 for every ladder size in one ss_screen_ladder call (sizes spread
        over the side streams, event fork/join around them); `rows` = the
        global rows [y0, y1) to decide (default: all of this engine's)."""
        main = main or torch.cuda.current_stream(self.device)
        y0, y1 = rows if rows is not None else (self.y_begin, self.y_end)
        cfg = tp.config
        q = cfg.quantizer.factors()
        L = len(tp.sizes)
        flags = 1 if self.force_int64 else 0
        if fused_enabled():
            need = int(self.L.ss_ladder_workspace_bytes(self.W, max(self.mrows, 1), max(L, 1)))
            cap = os.environ.get("SS_LADDER_WS_BYTES")  # test hook: a smaller workspace forces row bands
            if cap:
                need = int(cap)
            if self.ladder_ws is None or self.ladder_ws.numel() < need:
                self.ladder_ws = None
                self.ladder_ws = torch.empty(need, dtype=torch.uint8, device=self.device)
            flags |= 2
            handles = (ctypes.c_void_p * 1)(main.cuda_stream)
            wss = (ctypes.c_void_p * 1)(self.ladder_ws.data_ptr())
            n_streams, ws_bytes = 1, self.ladder_ws.numel()
        else:
            if self.screen_ws is None:
                ws = int(self.L.ss_screen_workspace_bytes(self.W, max(self.mrows, 1)))
                self.screen_ws = [torch.empty(ws, dtype=torch.uint8, device=self.device)
                                  for _ in range(self.n_streams)]
            handles = (ctypes.c_void_p * (1 + self.n_streams))(main.cuda_stream,
                                                                *[st.cuda_stream for st in self.streams])
            wss = (ctypes.c_void_p * (1 + self.n_streams))(self.screen_ws[0].data_ptr(),
                                                            *[w.data_ptr() for w in self.screen_ws])
            n_streams, ws_bytes = 1 + self.n_streams, self.screen_ws[0].numel()
        shifts = np.array(self.coarse_shifts or [0], np.int32)
        _native.check(self.L.ss_screen_ladder2(
            _p(self.planes) if self.built_int64 else None, None if self.force_int64 else self.planes32.data_ptr(),
            self.W, self.rows, self.pitch,
            self.W, self.H, self.y_origin, y0, y1, cfg.stride, L, tp.m_arr.ctypes.data,
            tp.n_rings.ctypes.data, tp.ring_n.ctypes.data, tp.ring_d.ctypes.data, tp.blobs_dev.data_ptr(),
            tp.blobs.ctypes.data, tp.blob_off.ctypes.data, q[0], q[1], q[2],
            # the ABI's mask / row-count row 0 is global row y0
            self.masks.data_ptr() + (y0 - self.y_begin) * self.words * 4, self.words, self.mrows * self.words,
            self.row_counts.data_ptr() + (y0 - self.y_begin) * 4, self.row_counts.shape[1], _p(self.stage_counts),
            flags, n_streams, handles, wss, ws_bytes,
            _p(self.coarse) if self.coarse_shifts else None, len(self.coarse_shifts), shifts.ctypes.data,
            _p(self.hi16) if self.built_hi16 else None),
            "screen")

    def _ladder_array(self, tp: TemplatePlan) -> np.ndarray:
        return np.array([sp.m for sp in tp.sizes], np.int32)

    def compact_all(self, tp: TemplatePlan) -> None:
        """K4 for every size in one pass (ladder order, then row-major)."""
        ms = tp.m_arr if tp.m_arr is not None else self._ladder_array(tp)
        _native.check(self.L.ss_compact_ladder(
            self.masks.data_ptr(), self.words, self.mrows * self.words, self.W, self.H, self.y_begin, self.y_end,
            len(ms), ms.ctypes.data, tp.config.stride, self.row_counts.data_ptr(), self.xy.data_ptr(), 3, self.capacity,
            self.totals.data_ptr(), self.size_counts.data_ptr(), self.compact_ws.data_ptr(), self.compact_ws.numel(),
            _stream_handle(self.device)), "compact")

    def region_all(self, tp: TemplatePlan) -> None:
        """K5 for every size in one pass, then the region popcount."""
        ms = tp.m_arr if tp.m_arr is not None else self._ladder_array(tp)
        _native.check(self.L.ss_region_ladder2(
            self.masks.data_ptr(), self.words, self.mrows * self.words, self.W, self.H, len(ms), ms.ctypes.data,
            tp.config.stride, self.row_counts.data_ptr(), self.row_counts.shape[1], self.region.data_ptr(),
            self.region_ws.data_ptr(), self.region_ws.numel(), _stream_handle(self.device)), "region")
        _native.check(self.L.ss_popcount(self.region.data_ptr(), self.words, self.W, self.H,
                                         self.totals[1:].data_ptr(), _stream_handle(self.device)), "popcount")

    # Streamed mask readback (run(host_masks=...)): row chunks of about this
    # many mask bytes (all sizes) each, so a chunk's D2H overlaps the next
    # chunks' screening; smaller results go in one piece after the ladder.
    READBACK_CHUNK_BYTES = 128 << 20

    def host_mask_buffer(self, n_sizes: int) -> torch.Tensor:
        """A pinned (n_sizes, rows, words) int32 host buffer for
        run(host_masks=...).  The buffer of the previous streamed copy is
        released only once that copy has landed."""
        if self._host_masks_inflight is not None:
            buf, ev = self._host_masks_inflight
            if not ev.query():
                ev.synchronize()
            self._host_masks_inflight = None
        return torch.empty((n_sizes, self.mrows, self.words), dtype=torch.int32, pin_memory=True)

    def readback_chunks(self, n_sizes: int) -> List[Tuple[int, int]]:
        """Global row ranges [a, b) screened one ss_screen_ladder call each
        when the masks are streamed to the host (multiples of 16 rows)."""
        total = n_sizes * self.mrows * self.words * 4
        n = max(1, min(16, total // self.READBACK_CHUNK_BYTES))
        per = -(-self.mrows // n)  # ceil
        step = max(256, -(-per // 16) * 16)
        return [(a, min(self.y_end, a + step)) for a in range(self.y_begin, self.y_end, step)]

    def run(self, img: torch.Tensor, tp: TemplatePlan, *, build: bool = True, region: bool = True,
            capacity: Optional[int] = None, host_masks: Optional[torch.Tensor] = None) -> None:
        """Enqueue the whole screen of one image (no host sync) on this
        engine's device (its current stream).  host_masks (a pinned
        host_mask_buffer): every size's packed mask rows are copied there on
        the engine's copy stream, row chunk by row chunk as each chunk's
        screen finishes; `masks_done` records the last copy."""
        with torch.cuda.device(self.device):
            self._run(img, tp, build=build, region=region, capacity=capacity, host_masks=host_masks)

    def _screen_streamed(self, tp: TemplatePlan, main: torch.cuda.Stream, host: torch.Tensor,
                         chunks: Optional[List[Tuple[int, int]]] = None, before=None) -> None:
        """K3 row chunk by row chunk, each chunk's mask rows (every size) copied
        to the pinned `host` on the copy stream as soon as it is screened.
        before(k): called before chunk k is enqueued (the pipelined path
        enqueues the table build it needs there)."""
        L = len(tp.sizes)
        assert host.shape == (L, self.mrows, self.words) and host.dtype == torch.int32 and host.is_pinned()
        if self.copy_stream is None:
            self.copy_stream = torch.cuda.Stream(self.device)
        cs = self.copy_stream
        pitch = self.mrows * self.words * 4
        for k, (a, b) in enumerate(chunks if chunks is not None else self.readback_chunks(L)):
            if before is not None:
                before(k)
            if b <= a:
                continue
            self.screen_ladder(tp, main, (a, b))
            ev = torch.cuda.Event()
            ev.record(main)
            cs.wait_event(ev)
            off = (a - self.y_begin) * self.words * 4
            _native.check(self.L.ss_copy_rows_async(host.data_ptr() + off, pitch, self.masks.data_ptr() + off, pitch,
                                                    (b - a) * self.words * 4, L, cs.cuda_stream), "mask readback")
        done = torch.cuda.Event()
        done.record(cs)
        self.masks_done = done
        self._host_masks_inflight = (host, done)

    # ── upload, build and screen overlapped (large images, screen()) ─────
    PIPELINE_MIN_BYTES = 32 << 20  # images from this size take run_pipelined
    PIPELINE_CHUNKS = 10  # measured at config 4 (e2e ms): 4: 27.6, 5: 26.7, 8: 26.4, 10: 26.2, 12+: 31 (two pieces per chunk)

    def run_pipelined(self, img: np.ndarray, tp: TemplatePlan, host_masks: torch.Tensor, keysets) -> None:
        """screen() for a large host image: the image goes up in row chunks
        (pinned staging, its own stream), each chunk's tables are built as it
        lands (ss_build_tables_rows: the recurrences only look up), and the
        rows whose tables are complete (those more than the largest size's
        lower margin above the built edge) are screened right after, their
        masks streamed back -- upload, K1/K2, K3 and the mask D2H overlap.
        keysets(): builds the template's key sets on the host (called once
        the first chunk is enqueued, while the GPU works on it).  Whole-image
        engines only; then K5 / K4 as run()."""
        with torch.cuda.device(self.device):
            self._run_pipelined(img, tp, host_masks, keysets)

    def _run_pipelined(self, img: np.ndarray, tp: TemplatePlan, host_masks: torch.Tensor, keysets) -> None:
        assert (self.y_begin, self.y_end, self.y_origin, self.rows) == (0, self.H, 0, self.H)
        assert img.shape == (self.H, self.W) and img.dtype == np.uint8
        H, W = self.H, self.W
        self._ensure(len(tp.sizes), tp.max_m, self.default_capacity(tp), True)
        main = torch.cuda.current_stream(self.device)
        for ev in (self.readback_done, self.masks_done):
            if ev is not None:
                main.wait_event(ev)
        self.readback_done = self.masks_done = None
        # table planes for this template (as _build_tables)
        wide = self.needs_int64(tp)
        hi16 = wide and self.wide_as_hi16(tp)
        int64 = wide and not hi16
        if int64 and self.planes is None:
            self.planes = torch.empty(int(self.L.ss_tables_bytes(W, H)) // 8, dtype=torch.int64, device=self.device)
        if hi16 and self.hi16 is None:
            self.hi16 = torch.empty(int(self.L.ss_tables_hi16_bytes(W, H)) // 2, dtype=torch.int16,
                                    device=self.device)
        shifts = self.coarse_shifts_for(tp)
        if shifts:
            nb = int(self.L.ss_coarse_bytes(W, H, len(shifts)))
            if self.coarse is None or self.coarse.numel() < nb:
                self.coarse = None
                self.coarse = torch.empty(nb, dtype=torch.uint8, device=self.device)
        sh = np.array(shifts or [0], np.int32)
        self.coarse_shifts = list(shifts)
        self.built_int64, self.built_hi16 = int64, hi16
        # image buffers: device image and pinned staging, kept by the engine
        if getattr(self, "_img_dev", None) is None:
            self._img_dev = torch.empty((H, W), dtype=torch.uint8, device=self.device)
            self._img_stage = torch.empty((H, W), dtype=torch.uint8, pin_memory=True)
            self.upload_stream = torch.cuda.Stream(self.device)
        img_dev, stage, us = self._img_dev, self._img_stage, self.upload_stream
        us.wait_stream(main)  # the previous screen is done reading the device image
        # build chunks: whole bands; screen chunks: rows whose tables are final
        rb = int(self.L.ss_build_band_rows(W, H, 1 if (int64 or hi16) else 0))
        n_chunks = int(os.environ.get("SS_PIPE_CHUNKS", self.PIPELINE_CHUNKS))  # experiment hooks
        last_parts = int(os.environ.get("SS_PIPE_LAST_PARTS", 2))
        mid_parts = int(os.environ.get("SS_PIPE_MID_PARTS", 1))
        per = -(-H // n_chunks)  # ceil
        step = max(rb, -(-per // rb) * rb)
        ends = list(range(step, H, step)) + [H]
        hi_max = max(((sp.m // 2) for sp in tp.sizes if sp.plan), default=0)
        # screen chunk k = the rows build chunk k completes; the last chunk
        # in two pieces so that the copy left after the last piece is short
        # (every piece costs launches and pipeline ramps: more pieces measured
        # slower)
        dec, owner, prev = [], [], 0
        for k, e in enumerate(ends):
            # cuts on multiples of 16 rows: stage 1 decides groups of up to 16
            # rows from one tested row, and a group cut by a piece's end falls
            # back to "every column is a candidate"
            d = H if e == H else max(prev, (e - hi_max - 1) // 16 * 16)
            parts = last_parts if e == H else mid_parts
            cuts = [prev] + [max(prev, (prev + (d - prev) * i // parts) // 16 * 16) for i in range(1, parts)] + [d]
            for a, b in zip(cuts[:-1], cuts[1:]):
                if b > a:
                    dec.append((a, b))
                    owner.append(k)
            prev = d
        src = torch.from_numpy(img)
        pinned_src = src.is_pinned()

        built = []

        def build(i: int) -> None:
            # screen piece i needs the build chunks up to owner[i] (chunks go up in order)
            for k in range(len(built), owner[i] + 1):
                build_chunk(k)

        def build_chunk(k: int) -> None:
            built.append(k)
            r0, r1 = (0 if k == 0 else ends[k - 1]), ends[k]
            if pinned_src:  # the caller's buffer is pinned: DMA straight from it
                part = src[r0:r1]
            else:
                stage[r0:r1].copy_(src[r0:r1])  # host copy into pinned staging (torch: multi-threaded)
                part = stage[r0:r1]
            with torch.cuda.stream(us):
                img_dev[r0:r1].copy_(part, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(us)
            main.wait_event(ev)
            _native.check(self.L.ss_build_tables_rows(
                img_dev.data_ptr(), W, H, W, _p(self.planes) if int64 else None, self.planes32.data_ptr(),
                _p(self.hi16) if hi16 else None, self.pitch, _p(self.coarse) if shifts else None, len(shifts),
                sh.ctypes.data, r0, r1, self.build_ws.data_ptr(), self.build_ws.numel(), main.cuda_stream),
                "build_tables")
            if k == 0:
                keysets()  # host work while the GPU builds the first chunk

        self._screen_streamed(tp, main, host_masks, dec, before=build)
        rs = self.region_stream = self.region_stream or torch.cuda.Stream(self.device)
        rs.wait_stream(main)
        with torch.cuda.stream(rs):
            self.region_all(tp)
            self.region_event = torch.cuda.Event()
            self.region_event.record(rs)
        self.compact_all(tp)
        if self.compact_event is None:
            self.compact_event = torch.cuda.Event()
        self.compact_event.record(main)
        main.wait_stream(rs)

    def _run(self, img: torch.Tensor, tp: TemplatePlan, *, build: bool, region: bool,
             capacity: Optional[int], host_masks: Optional[torch.Tensor] = None) -> None:
        full = (self.y_begin, self.y_end, self.y_origin, self.rows) == (0, self.H, 0, self.H)
        region = region and full
        self._ensure(len(tp.sizes), tp.max_m, capacity or self.default_capacity(tp), region)
        if build:
            self._build_tables(img, self.needs_int64(tp), tp)
        main = torch.cuda.current_stream(self.device)
        if self.readback_done is not None:  # the previous run's rows must have left before K4 rewrites them
            main.wait_event(self.readback_done)
            self.readback_done = None
        if self.masks_done is not None:  # likewise its streamed masks before K3 rewrites them
            main.wait_event(self.masks_done)
            self.masks_done = None
        if self.hooks is not None:
            self.hooks[0](main)
        if host_masks is None:
            self.screen_ladder(tp, main)
        else:
            self._screen_streamed(tp, main, host_masks)
        if self.hooks is not None:
            self.hooks[1](main)
        if region:
            # K5 reads only the masks: it runs beside K4 on a side stream
            # (both are small latency-bound passes), joined back before return
            if self.region_stream is None:
                self.region_stream = torch.cuda.Stream(self.device)
            rs = self.region_stream
            rs.wait_stream(main)
            with torch.cuda.stream(rs):
                self.region_all(tp)
                self.region_event = torch.cuda.Event()
                self.region_event.record(rs)
        self.compact_all(tp)
        if self.compact_event is None:
            self.compact_event = torch.cuda.Event()
        self.compact_event.record(main)
        if region:
            main.wait_stream(rs)

    def start_readback(self):
        """Start copying the survivor rows (int32 (cx, cy, m); as many as the
        last screen kept plus a margin) into a fresh pinned buffer on a copy
        stream, right after the last run's K4 -- overlapping K5 and the host's
        result bookkeeping.  Returns (buffer, event) for CandidateList (which
        falls back to its own copy when the survivors outnumber the buffer)."""
        if self.compact_event is None or self.last_kept is None:
            return None  # no estimate of the survivor count yet
        rows = min(self.capacity, int(self.last_kept * 1.25) + 4096)  # last screen's count + margin
        if self.copy_stream is None:
            self.copy_stream = torch.cuda.Stream(self.device)
        cs = self.copy_stream
        host = torch.empty((rows, 3), dtype=torch.int32, pin_memory=True)
        cs.wait_event(self.compact_event)
        with torch.cuda.stream(cs):
            host.copy_(self.xy[:rows], non_blocking=True)
            done = torch.cuda.Event()
            done.record(cs)
        self.readback_done = done
        return host, done

    def start_region_readback(self):
        """Start copying the kept region (bit-packed rows) into a fresh pinned
        buffer on the copy stream right after K5 (beside K4 and the rows'
        copy).  Returns (buffer, event), or None without a region."""
        ev = getattr(self, "region_event", None)
        if ev is None or self.region is None:
            return None
        if self.copy_stream is None:
            self.copy_stream = torch.cuda.Stream(self.device)
        cs = self.copy_stream
        host = torch.empty(self.region.shape, dtype=torch.int32, pin_memory=True)
        cs.wait_event(ev)
        with torch.cuda.stream(cs):
            host.copy_(self.region, non_blocking=True)
            done = torch.cuda.Event()
            done.record(cs)
        self.readback_done = done  # (the copy stream is in order: this also covers the rows' copy)
        self.region_event = None
        return host, done

    def recompact(self, tp: TemplatePlan, capacity: int) -> None:
        """Grow the survivor buffer and redo K4 only (after an overflow)."""
        with torch.cuda.device(self.device):
            self.capacity = capacity
            self.xy = torch.empty((capacity, 3), dtype=torch.int32, device=self.device)
            self.compact_all(tp)


class EnginePool:
    """Several engines of one image shape, each on its own stream, for
    batches of independent images (config 3: 64 x 1920x1080).  Image i goes
    to engine i % n; the engines' work overlaps on the GPU, filling the SMs
    that one small image's ladder leaves idle.  ``run`` forks from and joins
    back to the current stream (CUDA-graph capturable); an engine reused for
    a later image overwrites its buffers, so callers that need every image's
    results fetch them between uses (screening.screen_batch)."""

    def __init__(self, width: int, height: int, device=None, n: int = 4):
        if n < 1:
            raise ValueError("an engine pool needs at least one engine")
        self.engines = [Engine(width, height, device) for _ in range(n)]
        self.device = self.engines[0].device
        self.lock = threading.RLock()  # one batch at a time per pool
        self.streams = [torch.cuda.Stream(self.device) for _ in range(n)]

    def __len__(self) -> int:
        return len(self.engines)

    def run(self, imgs: Sequence[torch.Tensor], tps: Sequence[TemplatePlan], **kw) -> None:
        with torch.cuda.device(self.device):
            self._run(imgs, tps, **kw)

    def _run(self, imgs: Sequence[torch.Tensor], tps: Sequence[TemplatePlan], **kw) -> None:
        main = torch.cuda.current_stream(self.device)
        fork = torch.cuda.Event()
        fork.record(main)
        used = min(len(self.engines), len(imgs))
        for j in range(used):
            self.streams[j].wait_event(fork)
        for i, (img, tp) in enumerate(zip(imgs, tps)):
            j = i % len(self.engines)
            with torch.cuda.stream(self.streams[j]):
                self.engines[j].run(img, tp, **kw)
        for j in range(used):
            main.wait_stream(self.streams[j])
