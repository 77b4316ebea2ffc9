"""Where the end-to-end screen() time goes (host view, synchronised phases).

usage: python tools/e2e_breakdown.py [CONFIG]
Replays screen()'s phases with a device synchronise after each (so phases do
not overlap the way they do inside screen()) and prints wall ms per phase,
then the real screen() + readback for comparison.
"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as WL  # noqa: E402
from paper_1707_05647_b200 import screen  # noqa: E402
from paper_1707_05647_b200.engine import fill_keysets, launch_features, plan_ladder  # noqa: E402
from paper_1707_05647_b200.screening import fetch_result, get_engine, upload_image  # noqa: E402


def main():
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    wl = WL.CONFIGS[idx]
    case = WL.make_cases(wl, images=1)[0]
    cfg = WL.screening_config(wl)
    img, tpl = case.image, case.template
    dev = torch.device("cuda:0")
    for it in range(3):
        t = {}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng = get_engine(img.shape[1], img.shape[0], dev)
        tp = plan_ladder(tpl.shape[1], cfg)
        t["plan"] = time.perf_counter()
        pending = launch_features(tp, tpl, dev, eng.template_stream)
        torch.cuda.synchronize()
        t["features(f2 gpu)"] = time.perf_counter()
        img_dev = upload_image(img, dev)
        torch.cuda.synchronize()
        t["upload"] = time.perf_counter()
        eng.build_tables(img_dev, int64=eng.needs_int64(tp), tp=tp)
        torch.cuda.synchronize()
        t["build K1/K2"] = time.perf_counter()
        fill_keysets(tp, tpl, dev, eng.template_stream, pending)
        torch.cuda.synchronize()
        t["keysets(host)"] = time.perf_counter()
        eng.run(img_dev, tp, build=False)
        torch.cuda.synchronize()
        t["run K3-K5"] = time.perf_counter()
        res = fetch_result(eng, tp, t0, None)
        t["fetch"] = time.perf_counter()
        a = res.candidates.array()
        t["rows d2h"] = time.perf_counter()
        p = res.size_masks.packed_all()
        t["masks d2h"] = time.perf_counter()
        r = res.region_packed()
        t["region d2h"] = time.perf_counter()
        prev = t0
        parts = []
        for k, v in t.items():
            parts.append(f"{k} {1e3 * (v - prev):.1f}")
            prev = v
        print(f"iter {it}: " + ", ".join(parts) + f" | total {1e3 * (prev - t0):.1f} ms "
              f"(masks {p.nbytes / 1e6:.0f} MB, rows {a.nbytes / 1e6:.1f} MB, region {r.nbytes / 1e6:.1f} MB)")
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = screen(img, tpl, cfg, device=dev)
        t1 = time.perf_counter()
        res.candidates.array()
        res.size_masks.packed_all()
        res.region_packed()
        t2 = time.perf_counter()
        print(f"screen() {1e3 * (t1 - t0):.1f} ms + readback {1e3 * (t2 - t1):.1f} ms = {1e3 * (t2 - t0):.1f} ms")


if __name__ == "__main__":
    main()
