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
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _native
from .config import MIN_PATCH_SIDE, ScreeningConfig, grid_count, ladder_sizes, patch_center_margins, ring_plan
from .featureset import FeatureSet, build_feature_set, build_feature_sets_device, keyset_blob


import os

# Ladder sizes run on up to N_STREAMS side streams (fork/join around K3):
# for images whose 32-bit tables fit in a few GB, three sizes in flight fill
# the launch tails and overlap one size's compute-bound stage 1 with
# another's memory-bound rings (measured: config 1 -19%, config 2 -12%);
# for larger images two sizes' working sets thrash L2 (config 4 +27%), so
# they run one at a time.  SS_STREAMS overrides (experiments).
N_STREAMS = 3
STREAMS_MAX_TABLE_BYTES = 4 << 30


def streams_for(table_bytes: int) -> int:
    env = os.environ.get("SS_STREAMS")
    if env:
        return max(1, int(env))
    return N_STREAMS if table_bytes <= STREAMS_MAX_TABLE_BYTES else 1


def _p(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


@dataclass
class SizePlan:
    m: int
    plan: Tuple[Tuple[int, int], ...] = ()
    feature_set: Optional[FeatureSet] = None
    blob: Optional[np.ndarray] = None  # host copy (kernel parameters are read from it)
    blob_dev: Optional[torch.Tensor] = None
    ring_n: Optional[np.ndarray] = None
    ring_d: Optional[np.ndarray] = None
    fits32: bool = True  # ring sums recoverable from the 32-bit planes (ss_screen_fits32)


@dataclass
class TemplatePlan:
    """Everything the device needs about one template and config."""

    template_side: int
    config: ScreeningConfig
    ladder: Tuple[int, ...]
    sizes: List[SizePlan] = field(default_factory=list)

    @property
    def max_m(self) -> int:
        return max(self.ladder) if self.ladder else 1


def prepare_template(template: np.ndarray, cfg: ScreeningConfig, device) -> TemplatePlan:
    """Template side of screen() (screening.py:497, 511): ladder + per-size key sets.

    On a CUDA device the rescale features of every size come from one GPU
    launch (f2, build_feature_sets_device); otherwise from the host C++ path.
    """
    n = template.shape[1]
    ladder = ladder_sizes(n, cfg)
    tp = TemplatePlan(n, cfg, ladder)
    dev = torch.device(device) if device is not None else torch.device("cpu")
    evaluated = [m for m in ladder if m >= MIN_PATCH_SIDE]
    fsets = build_feature_sets_device(template, evaluated, cfg, dev) if dev.type == "cuda" else {}
    for m in ladder:
        sp = SizePlan(m)
        if m >= MIN_PATCH_SIDE:
            fs = fsets[m] if m in fsets else build_feature_set(template, m, cfg)
            sp.plan = fs.plan
            sp.feature_set = fs
            sp.blob = keyset_blob(fs)
            sp.blob_dev = torch.from_numpy(sp.blob).to(device)
            sp.ring_n = np.array([p[0] for p in fs.plan], np.int32)
            sp.ring_d = np.array([p[1] for p in fs.plan], np.int32)
            sp.fits32 = bool(_native.lib().ss_screen_fits32(len(fs.plan), sp.ring_n.ctypes.data,
                                                            sp.ring_d.ctypes.data))
        tp.sizes.append(sp)
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
        ws = int(self.L.ss_screen_workspace_bytes(self.W, max(self.mrows, 1)))
        self.screen_ws = [torch.empty(ws, dtype=torch.uint8, device=self.device) for _ in range(self.n_streams)]
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
        self.stage_counts = None  # set to a (4,) int64 device tensor to instrument the cascade
        self.force_int64 = False  # test hook: screen every size from the int64 planes
        self.hooks = None  # optional (before, after) callables(main_stream) around the K3 region

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

    def build_tables(self, img: torch.Tensor, int64: bool = False) -> None:
        """K1/K2 on the current stream.  img: (rows, W) uint8 on the device.
        Writes the 32-bit planes, and the int64 planes too when `int64`."""
        assert img.dtype == torch.uint8 and img.is_cuda and img.shape == (self.rows, self.W)
        img = img.contiguous()
        if int64 and self.planes is None:
            tb = int(self.L.ss_tables_bytes(self.W, self.rows))
            self.planes = torch.empty(tb // 8, dtype=torch.int64, device=self.device)
        _native.check(self.L.ss_build_tables2(img.data_ptr(), self.W, self.rows, self.W,
                                              _p(self.planes) if int64 else None, self.planes32.data_ptr(),
                                              self.pitch, self.build_ws.data_ptr(), self.build_ws.numel(),
                                              _stream_handle()), "build_tables")

    def screen_size(self, k: int, tp: TemplatePlan, ws: Optional[torch.Tensor] = None) -> None:
        ws = self.screen_ws[0] if ws is None else ws
        sp = tp.sizes[k]
        cfg = tp.config
        mask = self.masks[k]
        rc = self.row_counts[k]
        s = _stream_handle()
        if sp.m < MIN_PATCH_SIDE:
            _native.check(self.L.ss_fill_grid(self.W, self.y_begin, self.y_end, cfg.stride, mask.data_ptr(),
                                              self.words, rc.data_ptr(), s), "fill_grid")
            return
        q = cfg.quantizer.factors()
        _native.check(self.L.ss_screen_size(
            _p(self.planes) if (self.force_int64 or not sp.fits32) else None,
            None if self.force_int64 else self.planes32.data_ptr(), self.W, self.rows, self.pitch, self.W, self.H, self.y_origin, self.y_begin,
            self.y_end, sp.m, cfg.stride, len(sp.plan), sp.ring_n.ctypes.data, sp.ring_d.ctypes.data,
            sp.blob_dev.data_ptr(), sp.blob.ctypes.data, q[0], q[1], q[2], mask.data_ptr(), self.words, rc.data_ptr(),
            _p(self.stage_counts), ws.data_ptr(), ws.numel(), s), "screen_size")

    def _ladder_array(self, tp: TemplatePlan) -> np.ndarray:
        return np.array([sp.m for sp in tp.sizes], np.int32)

    def compact_all(self, tp: TemplatePlan) -> None:
        """K4 for every size in one pass (ladder order, then row-major)."""
        ms = self._ladder_array(tp)
        _native.check(self.L.ss_compact_ladder(
            self.masks.data_ptr(), self.words, self.mrows * self.words, self.W, self.H, self.y_begin, self.y_end,
            len(ms), ms.ctypes.data, tp.config.stride, self.row_counts.data_ptr(), self.xy.data_ptr(), 3, self.capacity,
            self.totals.data_ptr(), self.size_counts.data_ptr(), self.compact_ws.data_ptr(), self.compact_ws.numel(),
            _stream_handle()), "compact")

    def region_all(self, tp: TemplatePlan) -> None:
        """K5 for every size in one pass, then the region popcount."""
        ms = self._ladder_array(tp)
        _native.check(self.L.ss_region_ladder(
            self.masks.data_ptr(), self.words, self.mrows * self.words, self.W, self.H, len(ms), ms.ctypes.data,
            tp.config.stride, self.region.data_ptr(), self.region_ws.data_ptr(), self.region_ws.numel(),
            _stream_handle()), "region")
        _native.check(self.L.ss_popcount(self.region.data_ptr(), self.words, self.W, self.H,
                                         self.totals[1:].data_ptr(), _stream_handle()), "popcount")

    def run(self, img: torch.Tensor, tp: TemplatePlan, *, build: bool = True, region: bool = True,
            capacity: Optional[int] = None) -> None:
        """Enqueue the whole screen of one image (no host sync)."""
        full = (self.y_begin, self.y_end, self.y_origin, self.rows) == (0, self.H, 0, self.H)
        region = region and full
        self._ensure(len(tp.sizes), tp.max_m, capacity or self.default_capacity(tp), region)
        if build:
            self.build_tables(img, int64=self.needs_int64(tp))
        if region:
            self.region.zero_()
            self.totals[1:].zero_()
        main = torch.cuda.current_stream(self.device)
        if self.hooks is not None:
            self.hooks[0](main)
        fork = torch.cuda.Event()
        fork.record(main)
        used = set()
        for k in range(len(tp.sizes)):
            j = k % self.n_streams
            st = self.streams[j]
            if j not in used:
                st.wait_event(fork)
                used.add(j)
            with torch.cuda.stream(st):
                self.screen_size(k, tp, self.screen_ws[j])
        for j in used:
            main.wait_stream(self.streams[j])
        if self.hooks is not None:
            self.hooks[1](main)
        self.compact_all(tp)
        if region:
            self.region_all(tp)

    def recompact(self, tp: TemplatePlan, capacity: int) -> None:
        """Grow the survivor buffer and redo K4 only (after an overflow)."""
        self.capacity = capacity
        self.xy = torch.empty((capacity, 3), dtype=torch.int32, device=self.device)
        self.compact_all(tp)
