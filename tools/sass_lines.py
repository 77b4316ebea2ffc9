"""Join an ncu SASS source-page CSV (per-address instruction counts / stall
samples) with nvdisasm line info of the same kernel, and print the hottest
source lines.

usage: python tools/sass_lines.py NCU_SASS_CSV CUBIN FUNC_SUBSTRING [TOP]
(ncu -i rep --page source --csv --print-source sass -k regex:NAME > csv;
 cuobjdump -xelf all build/x.cu.o  ->  x.sm_100a.cubin)
"""
import csv
import re
import subprocess
import sys
from collections import defaultdict


def main():
    path, cubin, fsub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    h = rows[hi]
    ix = {k: i for i, k in enumerate(h)}
    data = [r for r in rows[hi + 1:] if r and r[0].startswith("0x")]
    base = int(data[0][0], 16)
    cnt = {int(r[0], 16) - base: (int(r[ix["Instructions Executed"]] or 0),
                                  int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)) for r in data}
    full = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
    # one section per function: ".text.<mangled>:"; pick the u32 (Ij) instance
    secs = re.split(r"\n\s*\.section\s+\.text\.", full)
    cands = [x for x in secs if x.split(",")[0].find(fsub) >= 0]
    pick = [x for x in cands if "Ij" in x.split(",")[0]] or cands
    fn = [pick[0].split(",")[0]]
    dis = pick[0]
    line = "?"
    agg = defaultdict(lambda: [0, 0])
    for l in dis.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            line = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m:
            a = int(m.group(1), 16)
            n, s = cnt.get(a, (0, 0))
            agg[line][0] += n
            agg[line][1] += s
    tot = sum(v[0] for v in agg.values()) or 1
    st = sum(v[1] for v in agg.values()) or 1
    print(f"function {fn[0][:80]}  instructions {tot}  samples {st}")
    for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * n / tot:5.1f}% inst {100 * s / st:5.1f}% stall  {k}")


if __name__ == "__main__":
    main()
