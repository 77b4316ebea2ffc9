"""The C-ABI library: loads on a GPU-less host, exports every symbol the
header declares, and its host-only entry points behave (no GPU compute)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

HEADER = os.path.join(ROOT, "include", "starscreen_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1707_05647_b200 import _native

    lib = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.exported_symbols())


def test_layout_queries():
    from paper_1707_05647_b200 import _native

    L = _native.lib()
    for W in (1, 31, 32, 2047, 16384):
        p = L.ss_plane_pitch(W)
        assert p >= W + 1 and p % 32 == 0
        assert L.ss_tables_bytes(W, 10) == 12 * 11 * p * 8
    assert L.ss_build_workspace_bytes(2048, 2048) > 0
    assert L.ss_version() == 1


def test_ladder_workspace_query():
    """The fused ladder's workspace: at least the per-size screen's (the
    fallback shares it), grows with the sizes screened in lock-step, and is
    capped (taller images run in row bands)."""
    from paper_1707_05647_b200 import _native

    L = _native.lib()
    for W, H in ((512, 512), (2048, 2048), (1920, 1080)):
        one = L.ss_ladder_workspace_bytes(W, H, 1)
        assert one >= L.ss_screen_workspace_bytes(W, H)
        assert L.ss_ladder_workspace_bytes(W, H, 9) > one
    big = L.ss_ladder_workspace_bytes(16384, 16384, 33)  # config 4: 16 GiB cap, row bands of 2048 rows
    assert big <= max(17 << 30, L.ss_screen_workspace_bytes(16384, 16384))
    assert big < 33 * 16384 * 16384 * 8  # less than one entry per centre of the whole image


def test_argument_errors_map_to_value_error():
    from paper_1707_05647_b200 import _native

    L = _native.lib()
    with pytest.raises(ValueError, match="empty image"):
        _native.check(L.ss_build_tables(None, 0, 5, 0, None, 32, None, 0, None))
    with pytest.raises(ValueError, match="too large"):
        _native.check(L.ss_build_tables(1, 300000, 300000, 300000, 16, L.ss_plane_pitch(300000), None, 0, None))
    with pytest.raises(ValueError, match="pitch"):
        _native.check(L.ss_build_tables(1, 100, 100, 100, 16, 7, None, 0, None))


def test_keyset_blob_layout():
    from paper_1707_05647_b200 import _native

    KB = _native.KEY_BASE
    HDR = 16
    keys = [np.array([(1 * KB + 2) * KB + 3, (1 * KB + 2) * KB + 4, (5 * KB + 0) * KB + 0], np.int64),
            np.array([], np.int64)]
    allk = np.concatenate(keys)
    off = np.array([0, 3, 3], np.int64)
    size = ctypes.c_size_t(0)
    L = _native.lib()
    _native.check(L.ss_keyset_blob(allk.ctypes.data, off.ctypes.data, 2, None, ctypes.byref(size)))
    blob = np.empty(size.value // 8, np.int64)
    _native.check(L.ss_keyset_blob(allk.ctypes.data, off.ctypes.data, 2, blob.ctypes.data, ctypes.byref(size)))
    assert blob[0] == 2
    h = blob[1:1 + HDR]
    om, nm, oms, nms, ok, nk = h[:6]
    assert list(blob[om:om + nm]) == [1, 5]
    assert list(blob[oms:oms + nms]) == [1 * KB + 2, 5 * KB]
    assert list(blob[ok:ok + nk]) == list(keys[0])
    # bounding box cm in [1,5], cs in [0,2], cg in [0,4]
    assert list(h[6:12]) == [1, 5, 0, 3, 0, 5]
    ob, wm, wms, wfull = h[12:16]
    assert ob > 0 and (wm, wms, wfull) == (1, 1, 3)
    words = blob[ob:].view(np.uint32)
    bits = lambda base, i: (int(words[base + i // 32]) >> (i % 32)) & 1
    assert [bits(0, i) for i in range(5)] == [1, 0, 0, 0, 1]
    assert bits(wm, 0 * 3 + 2) and bits(wm, 4 * 3 + 0) and not bits(wm, 0 * 3 + 0)
    assert bits(wm + wms, (0 * 3 + 2) * 5 + 3) and bits(wm + wms, (0 * 3 + 2) * 5 + 4)
    assert bits(wm + wms, (4 * 3 + 0) * 5 + 0) and not bits(wm + wms, (0 * 3 + 2) * 5 + 2)
    h2 = blob[1 + HDR:1 + 2 * HDR]
    assert h2[1] == h2[3] == h2[5] == 0 and h2[12] == -1
    bad = np.array([5, 3], np.int64)
    with pytest.raises(ValueError, match="sorted"):
        _native.check(L.ss_keyset_blob(bad.ctypes.data, np.array([0, 2], np.int64).ctypes.data, 1, None,
                                       ctypes.byref(size)))


def test_host_feature_sets_match_reference_golden():
    """Template side (native C++ host code) vs the reference's ring_keys()."""
    from paper_1707_05647_b200 import Quantizer, ScreeningConfig, build_feature_set

    z = golden("featuresets.npz")
    for i in range(int(z["n"])):
        meta = z[f"meta{i}"]
        m, ratio, q = int(meta[0]), float(meta[1]), tuple(float(v) for v in meta[2:])
        fs = build_feature_set(z[f"tpl{i}"], m, ScreeningConfig(ladder_ratio=ratio, quantizer=Quantizer(*q)))
        keys = fs.ring_keys()
        assert len(keys) == int(z[f"nrings{i}"])
        for r, k in enumerate(keys):
            assert np.array_equal(k, z[f"keys{i}_{r}"]), (i, r)


def test_template_ring_features_bitwise_vs_oracle():
    import oracle as O
    from paper_1707_05647_b200 import ring_plan
    from paper_1707_05647_b200.featureset import template_ring_features

    rng = np.random.default_rng(5)
    for _ in range(20):
        n = int(rng.integers(8, 70))
        tpl = rng.integers(0, 256, (n, n), dtype=np.uint8)
        m = int(rng.integers(8, 2 * n))
        k = m + int(rng.integers(0, 10))
        plan = ring_plan(m, 3)
        a = template_ring_features(tpl, k, m, plan)
        b = O.template_ring_features(tpl, k, m, plan)
        assert np.array_equal(a.view(np.int64), b.view(np.int64))
