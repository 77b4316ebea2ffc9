"""cProfile of repeated screen() calls (host overhead of the public API).

usage: python tools/screen_profile.py [CONFIG] [CALLS] [pinned]
(pinned: the inputs in pinned host memory, as bench.py's e2e)
"""
import cProfile
import os
import pstats
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as WL  # noqa: E402
from paper_1707_05647_b200 import screen  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 50
wl = WL.CONFIGS[idx]
case = WL.make_cases(wl, images=1)[0]
cfg = WL.screening_config(wl)
if len(sys.argv) > 3 and sys.argv[3] == "pinned":
    for name in ("image", "template"):
        a = getattr(case, name)
        t = torch.empty(a.shape, dtype=torch.uint8, pin_memory=True)
        t.numpy()[...] = a
        setattr(case, name, t.numpy())


def call():
    r = screen(case.image, case.template, cfg)
    r.candidates.array(), r.size_masks.packed_all(), r.region_packed()


for _ in range(5):
    call()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(calls):
    call()
print(f"{1e3 * (time.perf_counter() - t0) / calls:.3f} ms per call")
pr = cProfile.Profile()
pr.enable()
for _ in range(calls):
    call()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
