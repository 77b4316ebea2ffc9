"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes) per kernel.

usage: python tools/launches.py launches.csv [runs] [--k3 CONFIG_NAME]
Times are converted to microseconds and bytes to GB regardless of the unit ncu
printed; `runs` divides the totals into per-run figures.  With --k3 the DRAM
bytes and warp instructions (smsp__inst_executed.sum) per run of the K3
kernels (border + stage 1 + rings) are recorded in
profiles/<round>/k3_traffic.json under CONFIG_NAME (bench.py's roofline
traffic / dram / issue entries).
"""
import json
import os
import csv
import re
import sys
from collections import defaultdict

SCALE_T = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
SCALE_B = {"byte": 1e-9, "KB": 1e-6, "MB": 1e-3, "GB": 1.0, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}


def main(path, runs=1):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    t = defaultdict(float)
    b = defaultdict(float)
    n = defaultdict(int)
    inst = defaultdict(float)
    l2 = defaultdict(float)
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        name = re.sub(r"\(.*", "", r[ix["Kernel Name"]]).replace("ss::(anonymous namespace)::", "")
        metric, unit, val = r[ix["Metric Name"]], r[ix["Metric Unit"]], float(r[ix["Metric Value"]].replace(",", ""))
        if metric == "gpu__time_duration.sum":
            t[name] += val * SCALE_T[unit]
            n[name] += 1
        elif metric.startswith("dram__bytes"):
            b[name] += val * SCALE_B[unit]
        elif metric == "smsp__inst_executed.sum":
            inst[name] += val
        elif metric == "lts__t_bytes.sum":
            l2[name] += val * SCALE_B[unit]
    tot = sum(t.values())
    print(f"{'kernel':40s} {'launch':>7s} {'ms/run':>9s} {'share':>6s} {'GB/run':>8s} {'GB/s':>7s}")
    for k in sorted(t, key=lambda k: -t[k]):
        ms = t[k] / 1e3 / runs
        gb = b[k] / runs
        print(f"{k[:40]:40s} {n[k] // runs:7d} {ms:9.3f} {t[k] / tot:6.1%} {gb:8.2f} {gb / (ms / 1e3) if ms else 0:7.0f}")
    print(f"total ms/run {tot / 1e3 / runs:.3f}")
    main.l2 = l2
    main.n = n
    return t, b, inst


def record_k3(path, runs, name, rnd="r2"):
    t, b, inst = main(path, runs)
    k3 = [k for k in t if "stage1" in k or "ring_kernel" in k or "rings_kernel" in k or "border_kernel" in k]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    rec = {"dram_bytes_per_step": sum(b[k] for k in k3) * 1e9 / runs,
           "k3_ms_per_step_under_ncu": sum(t[k] for k in k3) / 1e3 / runs,
           "source": os.path.relpath(os.path.abspath(path), root)}
    # images per step (config 3 screens 64): one rowpre launch per image build
    rec["images"] = max(1, sum(main.n[k] for k in main.n if "rowpre" in k) // runs)
    if inst:
        rec["inst_per_step"] = sum(inst[k] for k in k3) / runs
        rec["inst_stage1_per_step"] = sum(inst[k] for k in k3 if "stage1" in k) / runs
        rec["inst_rings_per_step"] = sum(inst[k] for k in k3 if "ring" in k) / runs
    # per-kernel-family times (ms per step under ncu) and stage 1's L2 bytes
    fam = {"stage1": "stage1", "rings": "ring", "border": "border_kernel", "build": "band_", "region": "region_",
           "rowpre": "rowpre", "compact": "_xy_", "plan": "plan_kernel"}
    rec["ms_per_step_under_ncu"] = {f: sum(t[k] for k in t if sub in k) / 1e3 / runs for f, sub in fam.items()}
    l2 = getattr(main, "l2", {})
    if l2:
        rec["l2_bytes_stage1_per_step"] = sum(l2[k] for k in l2 if "stage1" in k) * 1e9 / runs
        rec["l2_bytes_rings_per_step"] = sum(l2[k] for k in l2 if "ring" in k) * 1e9 / runs
    out = os.path.join(root, "profiles", rnd, "k3_traffic.json")
    data = json.load(open(out)) if os.path.exists(out) else {}
    data[name] = rec
    with open(out, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)
    print(name, rec)


if __name__ == "__main__":
    runs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    if "--k3" in sys.argv:
        record_k3(sys.argv[1], runs, sys.argv[sys.argv.index("--k3") + 1])
    else:
        main(sys.argv[1], runs)
