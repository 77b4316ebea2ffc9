"""Host time of the ladder C-ABI call (no syncs inside the loop)."""
import sys, time
sys.path.insert(0, '.')
import torch
import workloads as WL
from paper_1707_05647_b200.engine import prepare_template
from paper_1707_05647_b200.screening import get_engine, upload_image
wl = WL.CONFIGS[1]
case = WL.make_cases(wl, images=1)[0]
cfg = WL.screening_config(wl)
eng = get_engine(case.image.shape[1], case.image.shape[0])
tp = prepare_template(case.template, cfg, eng.device)
img = upload_image(case.image, eng.device)
eng.run(img, tp)
torch.cuda.synchronize()
for name, fn in [("screen_ladder", lambda: eng.screen_ladder(tp)), ("compact_all", lambda: eng.compact_all(tp)),
                 ("region_all", lambda: eng.region_all(tp)), ("build", lambda: eng.build_tables(img)),
                 ("run", lambda: eng.run(img, tp, build=False))]:
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(50):
            fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"{name:14s} host {1e6*(t1-t)/50:8.1f} us/call   (gpu+host {1e6*(time.perf_counter()-t)/50:8.1f})")
