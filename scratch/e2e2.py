import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as WL
from paper_1707_05647_b200 import screen
wl = WL.CONFIGS[1]
case = WL.make_cases(wl, images=1)[0]
cfg = WL.screening_config(wl)
for rep in range(6):
    t0 = time.perf_counter()
    res = screen(case.image, case.template, cfg)
    t1 = time.perf_counter()
    a = res.candidates.array()
    t2 = time.perf_counter()
    print(f"screen {1e3*(t1-t0):.2f} ms  cand readback {1e3*(t2-t1):.2f} ms  n={len(a)}")
x = torch.empty((1139257, 2), dtype=torch.int32, device='cuda')
for pin in (False, True):
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        if pin:
            h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True); h.copy_(x); out = h.numpy()
        else:
            out = x.cpu().numpy()
        t1 = time.perf_counter()
        print('pin' if pin else 'pageable', f"{1e3*(t1-t0):.2f} ms")
