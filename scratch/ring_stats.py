import sys; sys.path.insert(0, '.')
import torch, numpy as np
import workloads as WL
from paper_1707_05647_b200.engine import prepare_template
from paper_1707_05647_b200.screening import get_engine, upload_image
for ci in (1, 2):
    wl = WL.CONFIGS[ci]; case = WL.make_cases(wl, images=1)[0]; cfg = WL.screening_config(wl)
    eng = get_engine(case.image.shape[1], case.image.shape[0]); tp = prepare_template(case.template, cfg, eng.device)
    img = upload_image(case.image, eng.device)
    eng.stage_counts = torch.zeros(24, dtype=torch.int64, device=eng.device)
    eng.run(img, tp); torch.cuda.synchronize()
    c = eng.stage_counts.cpu().numpy()
    print("config", ci, "stage1 evals", c[0], "mean pass", c[1], "ring0 pass", c[2], "surv", c[3])
    for l in range(3):
        print(f"  level {l}: evals {c[4+4*l]} mean-pass {c[5+4*l]} std-pass {c[6+4*l]} full-pass {c[7+4*l]}")
    print("  level0 entries whose deeper-ring means all pass:", c[20], " and ring0 passes too:", c[21])
    eng.stage_counts = None
