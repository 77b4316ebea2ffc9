import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import torch
import workloads as WL
from paper_1707_05647_b200 import screen
from paper_1707_05647_b200.engine import plan_ladder, fill_keysets, launch_features
from paper_1707_05647_b200.screening import get_engine
wl = WL.CONFIGS[1]; case = WL.make_cases(wl, images=1)[0]; cfg = WL.screening_config(wl)
for _ in range(5):
    screen(case.image, case.template, cfg).candidates.array()
eng = get_engine(case.image.shape[1], case.image.shape[0])
torch.cuda.synchronize()
def once():
    tp = plan_ladder(case.template.shape[1], cfg)
    p = launch_features(tp, case.template, eng.device, eng.template_stream)
    torch.cuda.synchronize()
    t = time.perf_counter()
    fill_keysets(tp, case.template, eng.device, eng.template_stream, p)
    return time.perf_counter() - t
for _ in range(3): once()
print("fill_keysets alone (features ready):", [round(1e3 * once(), 3) for _ in range(5)], "ms")
pr = cProfile.Profile(); pr.enable()
for _ in range(50): screen(case.image, case.template, cfg).candidates.array()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
