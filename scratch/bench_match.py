import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as WL
from paper_1707_05647_b200 import screen, match_candidates
for ci in [int(a) for a in sys.argv[1:]] or [1]:
    wl = WL.CONFIGS[ci]
    case = WL.make_cases(wl, images=1)[0]
    cfg = WL.screening_config(wl)
    res = screen(case.image, case.template, cfg)
    n_c = len(res.candidates)
    r = match_candidates(case.image, case.template, res)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); r = match_candidates(case.image, case.template, res); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    ms = min(ts) * 1e3
    # int8 GEMM ops: per size count x k_pad x (n1 + 2 n2) x 2
    ops = 0
    counts = res.candidates_per_size()
    for m, c in zip(res.ladder, counts):
        kp = (m * m + 15) // 16 * 16
        ops += c * kp * (72 + 2 * 40) * 2
    print(f"config {ci}: {n_c} candidates, match {ms:.2f} ms, {n_c * 36 / ms / 1e3:.2f} M hypotheses/s, int8 GEMM {ops / ms / 1e9:.1f} TOPS-equiv, result {r}")
