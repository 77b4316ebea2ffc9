"""One ncu report's details page as aligned text (what profiles/ keeps).

usage: python tools/ncu_summary.py REPORT.ncu-rep > summary.txt
"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
name = None
for r in rows[1:]:
    if name != r[ix["Kernel Name"]]:
        name = r[ix["Kernel Name"]]
        print(f"kernel: {name[:120]}")
    sec, met, unit, val = r[ix["Section Name"]], r[ix["Metric Name"]], r[ix["Metric Unit"]], r[ix["Metric Value"]]
    if met:
        print(f"{sec[:28]:28s} | {met[:45]:45s} | {val} {unit}")
