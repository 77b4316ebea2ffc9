"""Fine-grained host timeline of screen() for one config (no extra syncs)."""
import sys, time, functools
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as WL
import paper_1707_05647_b200.engine as E
import paper_1707_05647_b200.featureset as F
from paper_1707_05647_b200 import screen
from paper_1707_05647_b200.screening import get_engine, fetch_result, validate, upload_image

T = {}
def wrap(obj, name, label=None):
    f = getattr(obj, name)
    @functools.wraps(f)
    def g(*a, **k):
        t = time.perf_counter(); r = f(*a, **k); T[label or name] = T.get(label or name, 0) + time.perf_counter() - t; return r
    setattr(obj, name, g)
for n in ["screen_ladder", "compact_all", "region_all", "_ensure", "build_tables"]:
    wrap(E.Engine, n)
wrap(E, "launch_template_features"); wrap(E, "wait_template_features")
wrap(E.torch.Tensor, "pin_memory")
import paper_1707_05647_b200._native as N
lib = N.lib()
orig = lib.ss_ladder_keysets
wl = WL.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
case = WL.make_cases(wl, images=1)[0]
cfg = WL.screening_config(wl)
for _ in range(5):
    screen(case.image, case.template, cfg).candidates.array()
torch.cuda.synchronize()
for rep in range(4):
    T.clear()
    t0 = time.perf_counter()
    r = screen(case.image, case.template, cfg); a = r.candidates.array()
    tot = time.perf_counter() - t0
    print(f"total {1e3*tot:.3f} ms | " + " ".join(f"{k} {1e3*v:.3f}" for k, v in T.items()))
