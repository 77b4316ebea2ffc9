"""GPU timeline of the pipelined screen() of a large image (config 4): the
completion time of every table-build chunk, screen piece and mask copy,
relative to the call's start, from CUDA events recorded behind each.

usage: python tools/pipe_trace.py [CONFIG]
"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as WL  # noqa: E402
from paper_1707_05647_b200 import screen  # noqa: E402
from paper_1707_05647_b200.engine import Engine  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
wl = WL.CONFIGS[idx]
case = WL.make_cases(wl, images=1)[0]
cfg = WL.screening_config(wl)
for name in ("image", "template"):
    a = getattr(case, name)
    t = torch.empty(a.shape, dtype=torch.uint8, pin_memory=True)
    t.numpy()[...] = a
    setattr(case, name, t.numpy())


def call():
    r = screen(case.image, case.template, cfg)
    r.candidates.array(), r.size_masks.packed_all(), r.region_packed()
    return r


for _ in range(3):
    call()
torch.cuda.synchronize()
marks = []


def mark(label, stream=None):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream or torch.cuda.current_stream())
    marks.append((label, e, time.perf_counter()))


orig_ladder = Engine.screen_ladder
orig_region = Engine.region_all
orig_compact = Engine.compact_all


def ladder(self, tp, main, rows=None):
    r = orig_ladder(self, tp, main, rows)
    mark(f"screen {rows}", main)
    if self.copy_stream is not None and len(marks) > 2:
        pass
    return r


def region(self, tp):
    r = orig_region(self, tp)
    mark("region")
    return r


def compact(self, tp):
    r = orig_compact(self, tp)
    mark("compact")
    return r


Engine.screen_ladder, Engine.region_all, Engine.compact_all = ladder, region, compact
torch.cuda.synchronize()
t0 = time.perf_counter()
mark("start")
r = call()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"screen() + readback: {1e3 * (t1 - t0):.2f} ms")
for label, e, th in marks[1:]:
    print(f"{label:28s} gpu done {marks[0][1].elapsed_time(e):8.3f} ms   host enqueued {1e3 * (th - marks[0][2]):8.3f} ms")
