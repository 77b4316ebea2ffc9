"""Summarise an ncu source page (SASS): top instructions by stall samples, and stall reasons."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
S = ix["Warp Stall Sampling (All Samples)"]; E = ix["Instructions Executed"]; SRC = ix["Source"]
f = lambda v: float(v) if v not in ("", "-") else 0.0
ts = sum(f(r[S]) for r in data); te = sum(f(r[E]) for r in data)
print(f"instructions {len(data)}  samples {ts:.0f}  warp-inst executed {te:.0f}")
stall_cols = [h for h in hdr if h.startswith("stall_") or "Stall" in h and "Sampling" not in h]
order = sorted(range(len(data)), key=lambda i: -f(data[i][S]))
for i in order[:top]:
    r = data[i]
    print(f"{i:5d} {f(r[S])/ts*100:5.1f}% exec {f(r[E])/te*100:5.2f}%  {r[SRC][:90]}")
if "--dump" in sys.argv:
    for i, r in enumerate(data):
        print(f"{i:5d} {f(r[S])/ts*100:5.1f}% {f(r[E]):9.0f} {r[SRC][:100]}")
