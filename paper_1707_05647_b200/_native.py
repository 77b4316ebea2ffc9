"""ctypes binding of libstarscreen_b200.so (the C ABI in include/starscreen_b200.h).

This is the binding a maintainer of the reference would add:
every call returns an SS_* status that is mapped to the reference's error
classes -- ValueError for bad arguments / capacity, RuntimeError for CUDA
failures.  There is no fallback: if the library is missing or fails to load,
importing the GPU path raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SS_LIB_PATH: experiment hook (an alternative build of the same library)
LIB_PATH = os.environ.get("SS_LIB_PATH") or os.path.join(_HERE, "libstarscreen_b200.so")

SS_OK, SS_EINVAL, SS_ECAPACITY, SS_ECUDA = 0, 1, 2, 3
SS_MAX_RINGS = 16
SS_BLOB_MAX_BITMAP_WORDS = 8192
SS_MAX_COARSE = 5
KEY_BASE = 1 << 21

_lib = None

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_p = ctypes.c_void_p
c_sz = ctypes.c_size_t
c_d = ctypes.c_double

_SIGS = {
    "ss_last_error": (ctypes.c_char_p, []),
    "ss_version": (ctypes.c_int, []),
    "ss_launch_count": (ctypes.c_uint64, []),
    "ss_plane_pitch": (c_i64, [c_i64]),
    "ss_tables_bytes": (c_sz, [c_i64, c_i64]),
    "ss_build_workspace_bytes": (c_sz, [c_i64, c_i64]),
    "ss_build_tables": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_p, c_i64, c_p, c_sz, c_p]),
    "ss_tables32_bytes": (c_sz, [c_i64, c_i64]),
    "ss_build_tables2": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_p, c_p, c_i64, c_p, c_sz, c_p]),
    "ss_screen_fits32": (ctypes.c_int, [c_i32, c_p, c_p]),
    "ss_coarse_shift": (c_i32, [c_i64]),
    "ss_coarse_bytes": (c_sz, [c_i64, c_i64, c_i32]),
    "ss_tables_hi16_bytes": (c_sz, [c_i64, c_i64]),
    "ss_build_band_rows": (c_i32, [c_i64, c_i64, c_i32]),
    "ss_build_tables_rows": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_p, c_p, c_p, c_i64, c_p, c_i32, c_p, c_i64,
                                            c_i64, c_p, c_sz, c_p]),
    "ss_build_tables3": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_p, c_p, c_p, c_i64, c_p, c_i32, c_p, c_p, c_sz,
                                        c_p]),
    "ss_keyset_blob": (ctypes.c_int, [c_p, c_p, c_i32, c_p, ctypes.POINTER(c_sz)]),
    "ss_screen_size": (ctypes.c_int, [c_p, c_p, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i32, c_i32,
                                      c_i32, c_p, c_p, c_p, c_p, c_d, c_d, c_d, c_p, c_i64, c_p, c_p, c_p, c_sz, c_p]),
    "ss_screen_workspace_bytes": (c_sz, [c_i64, c_i64]),
    "ss_ladder_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32]),
    "ss_selftest_div": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, c_d, c_i32, c_p, c_p]),
    "ss_selftest_cells": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, c_i32, c_i32, c_d, c_d, c_d, c_p, c_p]),
    "ss_fill_grid": (ctypes.c_int, [c_i64, c_i64, c_i64, c_i32, c_p, c_i64, c_p, c_p]),
    "ss_screen_ladder": (ctypes.c_int, [c_p, c_p, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i32, c_i32,
                                        c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_d, c_d, c_d, c_p, c_i64, c_i64, c_p, c_i64,
                                        c_p, c_i32, c_i32, c_p, c_p, c_sz]),
    "ss_screen_ladder2": (ctypes.c_int, [c_p, c_p, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i32,
                                         c_i32, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_d, c_d, c_d, c_p, c_i64, c_i64,
                                         c_p, c_i64, c_p, c_i32, c_i32, c_p, c_p, c_sz, c_p, c_i32, c_p, c_p]),
    "ss_ladder_keysets": (ctypes.c_int, [c_p, c_i32, c_i32, c_p, c_p, c_d, c_d, c_d, c_p, c_i64, c_p, c_p, c_i64,
                                         c_p]),
    "ss_compact_workspace_bytes": (c_sz, [c_i64]),
    "ss_compact": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_i64, c_i64, c_i32, c_i32, c_p, c_p, c_i64, c_p, c_p,
                                  c_p, c_sz, c_p]),
    "ss_compact_ladder_workspace_bytes": (c_sz, [c_i64, c_i32]),
    "ss_compact_ladder": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i32, c_p, c_i32, c_p, c_p,
                                         c_i32, c_i64, c_p, c_p, c_p, c_sz, c_p]),
    "ss_region_ladder_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32]),
    "ss_region_ladder": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_i64, c_i32, c_p, c_i32, c_p, c_p, c_sz, c_p]),
    "ss_region_ladder2": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_i64, c_i32, c_p, c_i32, c_p, c_i64, c_p, c_p, c_sz,
                                         c_p]),
    "ss_region_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32]),
    "ss_region_accumulate": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_i32, c_i32, c_p, c_p, c_sz, c_p]),
    "ss_region_ladder_rows": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i32, c_p, c_i32, c_p,
                                             c_p, c_sz, c_p]),
    "ss_popcount": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_p, c_p]),
    "ss_bits_to_bytes": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_p, c_p]),
    "ss_copy_rows_async": (ctypes.c_int, [c_p, c_i64, c_p, c_i64, c_i64, c_i64, c_p]),
    "ss_match_plane_pitch": (c_i64, [c_i64]),
    "ss_match_planes": (ctypes.c_int, [c_p, c_i64, c_i64, c_p, c_i64, c_p]),
    "ss_match_probe_bytes": (c_sz, [c_i32, c_i32]),
    "ss_match_probes": (ctypes.c_int, [c_p, c_i32, c_i32, c_i32, c_p, c_p, c_p, c_p, c_p, c_p]),
    "ss_match_parts": (c_i64, [c_i64]),
    "ss_match_fused": (ctypes.c_int, [c_p, c_i64, c_i64, c_i64, c_p, c_i32, c_i64, c_i64, c_i32, c_p, c_i32, c_i32,
                                      c_p, c_p, c_p, c_p, c_p, c_p]),
    "ss_feature_set_keys": (ctypes.c_int, [c_p, c_i32, c_i32, c_i32, c_i32, c_p, c_p, c_d, c_d, c_d, c_p, c_p]),
    "ss_keys_from_features": (ctypes.c_int, [c_p, c_i32, c_i32, c_d, c_d, c_d, c_p, c_p]),
    "ss_template_features_device": (ctypes.c_int, [c_p, c_i32, c_i32, c_p, c_i32, c_p, c_p]),
    "ss_template_features_async": (ctypes.c_int, [c_p, c_i32, c_i32, c_p, c_i32, c_p, c_p, c_p, c_p, c_p]),
    "ss_template_ring_features": (ctypes.c_int, [c_p, c_i32, c_i32, c_i32, c_i32, c_p, c_p, c_p]),
    "ss_session_create": (ctypes.c_int, [c_i32, c_i64, c_i64, c_p]),
    "ss_session_destroy": (None, [c_p]),
    "ss_session_screen": (ctypes.c_int, [c_p, c_p, c_p, c_i32, c_p, c_p]),
    "ss_session_rows": (ctypes.c_int, [c_p, c_p, c_i64, c_i64]),
}


class LadderPlan(ctypes.Structure):
    """struct ss_ladder_plan (include/starscreen_b200.h)."""

    _fields_ = [("n_sizes", c_i32), ("m", c_p), ("n_rings", c_p), ("ring_n", c_p), ("ring_d", c_p),
                ("n_inst", c_i32), ("desc", c_p), ("desc_stride", c_i32), ("nk", c_p),
                ("q_mean", c_d), ("q_std", c_d), ("q_grad", c_d), ("stride", c_i32)]


class ScreenOut(ctypes.Structure):
    """struct ss_screen_out (include/starscreen_b200.h)."""

    _fields_ = [("masks", c_p), ("region", c_p), ("rows", c_p), ("rows_cap", c_i64), ("size_counts", c_p),
                ("kept", c_i64), ("region_pixels", c_i64), ("tested", c_i64)]


def lib() -> ctypes.CDLL:
    """Load the native library (raises if it is missing: no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(status: int, what: str = "") -> None:
    """Map an SS_* status to the reference's exception classes."""
    if status == SS_OK:
        return
    msg = lib().ss_last_error().decode(errors="replace")
    if status in (SS_EINVAL, SS_ECAPACITY):
        raise ValueError(msg or what)
    raise RuntimeError(f"{what}: {msg}" if what else msg)


def launch_count() -> int:
    return int(lib().ss_launch_count())
