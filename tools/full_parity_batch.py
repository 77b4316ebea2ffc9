"""One-off evidence: every image of BASELINE config 3 (64 x 1920x1080, one
template each) through screen_batch on the GPU against the untiled oracle --
every size mask, the candidate list, the tested count and the kept region
(the test suite compares images 0 and 63).

usage: python tools/full_parity_batch.py > summary.json
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
from paper_1707_05647_b200 import screen_batch  # noqa: E402

wl = WL.CONFIGS[3]
cfg = WL.screening_config(wl)
ocfg = O.ScreeningConfig(alpha=wl.alpha, beta=wl.beta, ladder_ratio=wl.ladder_ratio, quantizer=O.Quantizer(*wl.q))
cases = [WL.make_cases(wl, images=1, first_image=i)[0] for i in range(wl.images)]
t0 = time.time()
results = screen_batch([c.image for c in cases], [c.template for c in cases], cfg)
out = {"config": wl.name, "images": wl.images, "host_threads": os.cpu_count(), "mask_bit_disagreements": 0,
       "disagreements_outside_band": 0, "band_positions": 0, "positions": 0, "candidates": 0,
       "images_with_identical_candidates": 0, "images_with_identical_region": 0, "images_with_identical_tested": 0}
for i, (c, res) in enumerate(zip(cases, results)):
    ref = O.screen(c.image, c.template, ocfg, nthreads=os.cpu_count() or 1, band=True)
    assert tuple(res.ladder) == tuple(ref.ladder)
    for m in res.ladder:
        d = res.size_masks[m] != ref.size_masks[m]
        b = ref.band_masks.get(m)
        out["mask_bit_disagreements"] += int(d.sum())
        if b is not None:
            out["band_positions"] += int(b.sum())
            out["disagreements_outside_band"] += int((d & ~b).sum())
        else:
            out["disagreements_outside_band"] += int(d.sum())
    out["positions"] += int(ref.patches_tested)
    out["candidates"] += len(res.candidates)
    out["images_with_identical_candidates"] += int(np.array_equal(res.candidates.array(),
                                                                  np.array(ref.candidates, np.int32).reshape(-1, 3)))
    out["images_with_identical_region"] += int(np.array_equal(res.region_mask, ref.region_mask))
    out["images_with_identical_tested"] += int(res.stats.patches_tested == ref.patches_tested)
    print(f"image {i + 1}/{wl.images}: {out['mask_bit_disagreements']} disagreements so far, {time.time() - t0:.0f} s",
          file=sys.stderr, flush=True)
out["seconds"] = round(time.time() - t0, 1)
print(json.dumps(out))
