"""Summaries of ncu exports (run here, on the CPU box)."""
import collections
import csv
import re
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hi]
    ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r'\(.*', '', r[ki]).split('::')[-1][:40]
        v = float(r[vi].replace(',', ''))
        v *= {'nsecond': 1e-3, 'usecond': 1.0, 'msecond': 1e3, 'second': 1e6}.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:42s} n={n:4d} total={t:10.1f} us  mean={t/n:9.2f} us  share={t/tot*100:5.1f}%")
    return "\n".join(out)


def details(rep, kid=None):
    txt = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h = r[0]
    idx = {k: i for i, k in enumerate(h)}
    ids = sorted({row[idx['ID']] for row in r[1:]})
    kid = kid or ids[0]
    out = []
    for row in r[1:]:
        if row[idx['ID']] != kid or not row[idx['Metric Name']]:
            continue
        out.append(f"{row[idx['Section Name']][:28]:28s} {row[idx['Metric Name']][:48]:48s} {row[idx['Metric Value']]} {row[idx['Metric Unit']]}")
    return "\n".join(out)


def raw(rep, pattern):
    txt = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h, units = r[0], r[1]
    out = []
    for row in r[2:]:
        for i, k in enumerate(h):
            if re.search(pattern, k):
                out.append(f"{row[h.index('ID')]} {k} = {row[i]} {units[i]}")
    return "\n".join(out)


def sass_mix(rep):
    txt = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h = rows[1]
    d = [x for x in rows[2:] if len(x) == len(h)]
    i_src, i_s, i_ex = h.index('Source'), h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
    num = lambda x: int(x) if x.strip().isdigit() else 0
    tot_s = sum(num(x[i_s]) for x in d) or 1
    tot_ex = sum(num(x[i_ex]) for x in d) or 1
    ops, opsS = collections.Counter(), collections.Counter()
    for x in d:
        m = re.match(r'\s*(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)', x[i_src])
        if not m:
            continue
        op = m.group(1).split('.')[0]
        ops[op] += num(x[i_ex])
        opsS[op] += num(x[i_s])
    out = [f"total instr {tot_ex} samples {tot_s}"]
    for op, c in ops.most_common(25):
        out.append(f"{op:10s} exec={c:10d} ({c/tot_ex*100:5.1f}%) stall={opsS[op]/tot_s*100:5.1f}%")
    return "\n".join(out)


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "launches":
        print(launches(sys.argv[2]))
    elif cmd == "details":
        print(details(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None))
    elif cmd == "raw":
        print(raw(sys.argv[2], sys.argv[3]))
    elif cmd == "sass":
        print(sass_mix(sys.argv[2]))
