"""Native screening sessions: one screen() in one C call (csrc/ss_session.cpp).

A Session owns, for one (W, H) on one device, the device tables, workspaces,
result buffers, pinned staging and streams of the whole screen; ``run`` hands
it the host image and template plus the ladder plan and gets every result
back in pinned host memory -- the template features (f2), upload, K1/K2, key
sets, K3, K4 beside K5 and the D2H all happen inside ss_session_screen with
one host synchronisation, instead of a few hundred Python-level CUDA calls.
The Python Engine (engine.py) stays the stream-level API (CUDA graphs, row
bands, engine pools, the pipelined path for very large images).
"""

from __future__ import annotations

import ctypes
import functools
import threading
from typing import Tuple

import numpy as np
import torch

from . import _native
from ._native import SS_ECAPACITY, SS_ECUDA, LadderPlan, ScreenOut
from .config import ScreeningConfig
from .engine import LadderGeometry, ladder_geometry
from .featureset import DESC_STRIDE


@functools.lru_cache(maxsize=64)
def _plan(n: int, alpha: float, beta: float, ratio: float, ring_count: int, q: Tuple[float, float, float],
          stride: int) -> Tuple[LadderGeometry, LadderPlan]:
    geo = ladder_geometry(n, alpha, beta, ratio, ring_count)  # read-only arrays, kept alive by the cache
    p = LadderPlan(len(geo.ladder), geo.m_arr.ctypes.data, geo.n_rings.ctypes.data, geo.ring_n.ctypes.data,
                   geo.ring_d.ctypes.data, geo.desc.shape[0], geo.desc.ctypes.data if geo.desc.size else None,
                   DESC_STRIDE, geo.nk.ctypes.data if geo.nk.size else None, q[0], q[1], q[2], stride)
    return geo, p


def ladder_plan(n: int, cfg: ScreeningConfig) -> Tuple[LadderGeometry, LadderPlan]:
    """(geometry, ss_ladder_plan) of a template side and config (cached)."""
    return _plan(n, cfg.alpha, cfg.beta, cfg.ladder_ratio, cfg.ring_count, tuple(cfg.quantizer.factors()),
                 cfg.stride)


class SessionResult:
    __slots__ = ("masks", "region", "rows", "kept", "region_pixels", "tested", "size_counts")


class Session:
    def __init__(self, width: int, height: int, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1707_05647_b200 needs a CUDA device (no CPU fallback)")
        dev = torch.device(device if device is not None else "cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.W, self.H = int(width), int(height)
        self.words = (self.W + 31) // 32
        self.L = _native.lib()
        self._ptr = ctypes.c_void_p()
        self.last_kept = 0
        self.lock = threading.Lock()
        _native.check(self.L.ss_session_create(dev.index, self.W, self.H, ctypes.byref(self._ptr)), "session")

    def __del__(self):
        ptr = getattr(self, "_ptr", None)
        if ptr is not None and ptr.value:
            self.L.ss_session_destroy(ptr)
            self._ptr = None

    def run(self, img: np.ndarray, tpl: np.ndarray, cfg: ScreeningConfig) -> Tuple[LadderGeometry, SessionResult]:
        """Screen one C-contiguous u8 (H, W) image with one u8 (n, n) template."""
        assert img.shape == (self.H, self.W) and img.dtype == np.uint8 and img.flags.c_contiguous
        n = tpl.shape[0]
        geo, plan = ladder_plan(n, cfg)
        L = len(geo.ladder)
        r = SessionResult()
        with self.lock:
            r.masks = torch.empty((L, self.H, self.words), dtype=torch.int32, pin_memory=True)
            r.region = torch.empty((self.H, self.words), dtype=torch.int32, pin_memory=True)
            cap = self.last_kept + self.last_kept // 4 + 4096
            r.rows = torch.empty((cap, 3), dtype=torch.int32, pin_memory=True)
            r.size_counts = np.zeros(L, np.int64)
            out = ScreenOut(r.masks.data_ptr(), r.region.data_ptr(), r.rows.data_ptr(), cap,
                            r.size_counts.ctypes.data, 0, 0, 0)
            st = self._screen(img, tpl, n, plan, out)
            if st == SS_ECAPACITY and out.kept > cap:
                r.rows = torch.empty((out.kept, 3), dtype=torch.int32, pin_memory=True)
                _native.check(self.L.ss_session_rows(self._ptr, r.rows.data_ptr(), 0, out.kept), "survivor rows")
            else:
                _native.check(st, "screen")
            self.last_kept = int(out.kept)
        r.kept, r.region_pixels, r.tested = int(out.kept), int(out.region_pixels), int(out.tested)
        return geo, r

    def _screen(self, img, tpl, n, plan, out) -> int:
        st = self.L.ss_session_screen(self._ptr, img.ctypes.data, tpl.ctypes.data, n, ctypes.byref(plan),
                                      ctypes.byref(out))
        if st == SS_ECUDA and b"out of device memory" in self.L.ss_last_error():
            torch.cuda.empty_cache()  # memory cached by torch's allocator, then once more
            st = self.L.ss_session_screen(self._ptr, img.ctypes.data, tpl.ctypes.data, n, ctypes.byref(plan),
                                          ctypes.byref(out))
        return st
