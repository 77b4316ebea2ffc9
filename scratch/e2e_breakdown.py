import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as WL
from paper_1707_05647_b200 import screen
from paper_1707_05647_b200.engine import prepare_template
from paper_1707_05647_b200.screening import get_engine, fetch_result, validate
for cfg_i in (1, 4):
    wl = WL.CONFIGS[cfg_i]
    case = WL.make_cases(wl, images=1)[0]
    cfg = WL.screening_config(wl)
    for rep in range(3):
        t0 = time.perf_counter()
        img, tpl = validate(case.image, case.template, cfg)
        t1 = time.perf_counter()
        eng = get_engine(img.shape[1], img.shape[0], 'cuda')
        tp = prepare_template(tpl, cfg, eng.device)
        t2 = time.perf_counter()
        d = torch.from_numpy(img).to(eng.device)
        torch.cuda.synchronize(); t3 = time.perf_counter()
        eng.run(d, tp)
        torch.cuda.synchronize(); t4 = time.perf_counter()
        res = fetch_result(eng, tp, t0)
        t5 = time.perf_counter()
        _ = list(res.candidates)[:10]
        t6 = time.perf_counter()
        print(f"cfg{cfg_i} validate {1e3*(t1-t0):.2f} featuresets {1e3*(t2-t1):.2f} h2d {1e3*(t3-t2):.2f} gpu {1e3*(t4-t3):.2f} fetch {1e3*(t5-t4):.2f} total {1e3*(t5-t0):.2f} ms; cands={len(res.candidates)}")
