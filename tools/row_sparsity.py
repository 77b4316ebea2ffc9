"""Fraction of (size, row) pairs whose interior survivor bits are all zero
(how much of K5's row pass is skippable).  usage: python tools/row_sparsity.py [CONFIG]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as WL  # noqa: E402
from paper_1707_05647_b200 import screen  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
wl = WL.CONFIGS[idx]
case = WL.make_cases(wl, images=1)[0]
res = screen(case.image, case.template, WL.screening_config(wl))
H, W = case.image.shape
tot = empty = 0
for m in res.ladder:
    lo, hi = (m - 1) // 2, m // 2
    p = res.size_masks.packed(m)  # (H, words) uint32
    bits = np.unpackbits(p.view(np.uint8), axis=1, bitorder="little")[:, :W]
    inner = bits[lo:H - hi, lo:W - hi]
    live = inner.any(axis=1)
    tot += H
    empty += H - int(live.sum())
    # 32-row blocks without any survivor
print(f"config {idx}: {empty}/{tot} (size, row) pairs empty = {empty / tot:.3f}; survivors {len(res.candidates)}")
