import cProfile, pstats, sys, time, io
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as WL
from paper_1707_05647_b200 import screen
for cfg_i in [int(c) for c in sys.argv[1:]] or [1]:
    wl = WL.CONFIGS[cfg_i]
    case = WL.make_cases(wl, images=1)[0]
    cfg = WL.screening_config(wl)
    for _ in range(3):
        r = screen(case.image, case.template, cfg); r.candidates.array()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); r = screen(case.image, case.template, cfg); r.candidates.array(); ts.append(time.perf_counter() - t0)
    print(f"cfg{cfg_i} e2e ms: {[round(1e3*t, 2) for t in ts]}")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        r = screen(case.image, case.template, cfg); r.candidates.array()
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats('cumulative').print_stats(35)
    print(s.getvalue()[:6000])
