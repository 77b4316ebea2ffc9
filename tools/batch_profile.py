"""cProfile of screen_batch on config 3 (64 x 1920x1080): where the host time goes."""
import cProfile
import os
import pstats
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as WL  # noqa: E402
from paper_1707_05647_b200 import screen_batch  # noqa: E402

wl = WL.CONFIGS[3]
cases = WL.make_cases(wl)
cfg = WL.screening_config(wl)
imgs = [c.image for c in cases]
tpls = [c.template for c in cases]


def call():
    res = screen_batch(imgs, tpls, cfg)
    for r in res:
        r.candidates.array(), r.size_masks.packed_all(), r.region_packed()
    return res


for _ in range(2):
    call()
torch.cuda.synchronize()
t0 = time.perf_counter()
res = call()
print("screen_batch + readback", 1e3 * (time.perf_counter() - t0), "ms")
t0 = time.perf_counter()
res = screen_batch(imgs, tpls, cfg)
torch.cuda.synchronize()
print("screen_batch only", 1e3 * (time.perf_counter() - t0), "ms")
pr = cProfile.Profile()
pr.enable()
call()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
