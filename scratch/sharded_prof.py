import sys, time, cProfile, pstats, os
sys.path.insert(0, '.')
import torch, torch.distributed as dist
import workloads as WL
from paper_1707_05647_b200.sharding import screen_sharded
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29541", rank=0, world_size=1, device_id=torch.device("cuda", 0))
wl = WL.CONFIGS[2]; case = WL.make_cases(wl, images=1)[0]; cfg = WL.screening_config(wl)
for _ in range(2): screen_sharded(case.image, case.template, cfg, device="cuda:0")
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
t = time.perf_counter()
for _ in range(3): r = screen_sharded(case.image, case.template, cfg, device="cuda:0"); len(r.candidates)
print("per call ms", (time.perf_counter() - t) / 3 * 1e3)
pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(22)
