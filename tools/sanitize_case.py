"""One small screen per call, for compute-sanitizer (tools/sanitize.sh).

usage: python tools/sanitize_case.py CONFIG [SIDE]
Runs the drop-in screen() (every K1-K5 kernel, fused ladder) on BASELINE
config CONFIG's seeded input, cropped to SIDE x SIDE when given (config 1 at
full size takes minutes under racecheck), and checks the result against the
oracle so a sanitizer run that perturbs the kernels is also caught as a
parity failure.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402  (the checker)
import workloads as WL  # noqa: E402
from paper_1707_05647_b200 import screen  # noqa: E402


def main():
    idx = int(sys.argv[1])
    side = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    wl = WL.CONFIGS[idx]
    case = WL.make_cases(wl)[0]
    img = case.image if not side else np.ascontiguousarray(case.image[:side, :side])
    cfg = WL.screening_config(wl)
    res = screen(img, case.template, cfg)
    ref = O.screen(img, case.template, O.ScreeningConfig(alpha=wl.alpha, beta=wl.beta, ladder_ratio=wl.ladder_ratio,
                                                         quantizer=O.Quantizer(*wl.q)), nthreads=os.cpu_count() or 1)
    bad = sum(int((res.size_masks[m] != ref.size_masks[m]).sum()) for m in res.ladder)
    same = np.array_equal(res.candidates.array(), np.array(ref.candidates, np.int32).reshape(-1, 3))
    print(f"config {idx} {img.shape}: {len(res.ladder)} sizes, {len(res.candidates)} candidates, "
          f"mask disagreements {bad}, candidates identical {same}")
    sys.exit(0 if bad == 0 and same else 1)


if __name__ == "__main__":
    main()
