"""One-off evidence: a BASELINE config's WHOLE image on the GPU against the
tiled oracle (row bands screened with their halo decide
every centre exactly as the full image does) -- every size mask, the
candidate list, the tested count and the kept region; SURVEY.md 8(d)'s
threshold-band positions counted from the oracle's fp64 features.  The same
check as tests/test_gpu_configs.py::test_config2_full_image_vs_tiled_oracle,
at a size the test suite cannot afford (config 4: 8.7e9 positions x scales,
~15 min of 16 host threads).

usage: python tools/full_parity.py [CONFIG] [BANDS] > summary.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import workloads as WL  # noqa: E402
from paper_1707_05647_b200 import screen  # noqa: E402
from paper_1707_05647_b200.screening import unpack_bits  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
bands = int(sys.argv[2]) if len(sys.argv) > 2 else 32
wl = WL.CONFIGS[idx]
case = WL.make_cases(wl, images=1)[0]
cfg = WL.screening_config(wl)
ocfg = O.ScreeningConfig(alpha=wl.alpha, beta=wl.beta, ladder_ratio=wl.ladder_ratio, quantizer=O.Quantizer(*wl.q))
t0 = time.time()
res = screen(case.image, case.template, cfg)
H, W = case.image.shape
nthreads = os.cpu_count() or 1
cand = res.candidates.array()
region = res.region_packed()
out = {"config": wl.name, "image": f"{W}x{H}", "ladder": list(res.ladder), "row_bands": bands, "host_threads": nthreads,
       "mask_bit_disagreements": 0, "disagreements_outside_band": 0, "band_positions": 0, "positions": 0,
       "region_rows_differing": 0}
cands = []
for i in range(bands):
    y0, y1 = i * H // bands, (i + 1) * H // bands
    t = O.screen_tile(case.image, case.template, ocfg, y0, y1, 0, W, nthreads=nthreads, band=True)
    assert tuple(t.ladder) == tuple(res.ladder)
    for m in res.ladder:
        got = unpack_bits(res.size_masks.packed(m)[y0:y1], W)
        d = got != t.size_masks[m]
        out["mask_bit_disagreements"] += int(d.sum())
        out["disagreements_outside_band"] += int((d & ~t.band_masks[m]).sum())
        out["band_positions"] += int(t.band_masks[m].sum())
    ry0, ry1, rx0, rx1 = t.region_window
    same = np.array_equal(unpack_bits(region[ry0:ry1], W)[:, rx0:rx1], t.region)
    out["region_rows_differing"] += 0 if same else (ry1 - ry0)
    out["positions"] += int(t.patches_tested)
    cands.append(np.asarray(t.candidates, np.int32).reshape(-1, 3))
    print(f"band {i + 1}/{bands} rows [{y0},{y1}): {out['mask_bit_disagreements']} disagreements so far, "
          f"{time.time() - t0:.0f} s", file=sys.stderr, flush=True)
want = np.concatenate(cands)
order = {m: k for k, m in enumerate(res.ladder)}
want = want[np.argsort([order[int(m)] for m in want[:, 2]], kind="stable")]
out["candidates"] = int(len(cand))
out["candidates_identical"] = bool(np.array_equal(cand, want))
out["tested_identical"] = bool(res.stats.patches_tested == out["positions"])
out["seconds"] = round(time.time() - t0, 1)
print(json.dumps(out))
