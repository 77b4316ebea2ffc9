import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as WL
from paper_1707_05647_b200 import screen
from paper_1707_05647_b200.screening import get_engine, fetch_result, validate, upload_image
from paper_1707_05647_b200.engine import plan_ladder, fill_keysets, launch_features
wl = WL.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
case = WL.make_cases(wl, images=1)[0]
cfg = WL.screening_config(wl)
for _ in range(5):
    screen(case.image, case.template, cfg).candidates.array()
torch.cuda.synchronize()
for rep in range(3):
    T = [time.perf_counter()]
    img, tpl = validate(case.image, case.template, cfg); T.append(time.perf_counter())
    eng = get_engine(img.shape[1], img.shape[0]); tp = plan_ladder(tpl.shape[1], cfg); feats = launch_features(tp, tpl, eng.device, eng.template_stream); T.append(time.perf_counter())
    img_dev = upload_image(img, eng.device); T.append(time.perf_counter())
    eng.build_tables(img_dev, int64=eng.needs_int64(tp)); T.append(time.perf_counter())
    fill_keysets(tp, tpl, eng.device, eng.template_stream, feats); T.append(time.perf_counter())
    eng.run(img_dev, tp, build=False); T.append(time.perf_counter())
    res = fetch_result(eng, tp, T[0]); T.append(time.perf_counter())
    a = res.candidates.array(); T.append(time.perf_counter())
    names = ["validate", "plan", "upload", "build_enq", "keysets", "run_enq", "fetch(sync)", "cand_d2h"]
    print(" ".join(f"{n} {1e3*(T[i+1]-T[i]):.3f}" for i, n in enumerate(names)), f"total {1e3*(T[-1]-T[0]):.3f} ms")
