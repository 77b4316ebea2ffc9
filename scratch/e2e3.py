import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as WL
from paper_1707_05647_b200 import screen
from paper_1707_05647_b200.engine import prepare_template
from paper_1707_05647_b200.screening import get_engine, fetch_result, validate
for cfg_i in [int(a) for a in sys.argv[1:]] or (1, 4):
    wl = WL.CONFIGS[cfg_i]
    case = WL.make_cases(wl, images=1)[0]
    cfg = WL.screening_config(wl)
    for rep in range(4):
        t0 = time.perf_counter()
        img, tpl = validate(case.image, case.template, cfg)
        t1 = time.perf_counter()
        eng = get_engine(img.shape[1], img.shape[0], 'cuda')
        tp = prepare_template(tpl, cfg, eng.device)
        t2 = time.perf_counter()
        from paper_1707_05647_b200.screening import upload_image; d = upload_image(img, eng.device)
        torch.cuda.synchronize(); t3 = time.perf_counter()
        eng.run(d, tp)
        t3b = time.perf_counter()
        torch.cuda.synchronize(); t4 = time.perf_counter()
        res = fetch_result(eng, tp, t0)
        t5 = time.perf_counter()
        arr = res.candidates.array()
        t6 = time.perf_counter()
        print(f"cfg{cfg_i} validate {1e3*(t1-t0):.2f} prep {1e3*(t2-t1):.2f} h2d {1e3*(t3-t2):.2f} enqueue {1e3*(t3b-t3):.2f} gpu {1e3*(t4-t3):.2f} fetch {1e3*(t5-t4):.2f} array {1e3*(t6-t5):.2f} total {1e3*(t6-t0):.2f} ms; cands={len(arr)}")
    # prep breakdown
    import cProfile, pstats
    continue
    pr = cProfile.Profile(); pr.enable()
    for _ in range(3):
        tp = prepare_template(tpl, cfg, eng.device)
    pr.disable()
    pstats.Stats(pr).sort_stats('cumulative').print_stats(18)
