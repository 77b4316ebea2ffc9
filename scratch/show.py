import json, sys
for c in sys.argv[1:]:
    d = json.loads(open(f"gpurun_out/bf_c{c}.json").read().strip().splitlines()[-1]); r = d["roofline"]
    print(c, round(d["value"] / 1e9, 2), "G/s", round(d["ms_per_step"], 3), "ms", "frac", round(r["frac"], 3), "k3ms",
          round(r.get("screen_ms_per_step", 0), 3), "e2e ms", round(d["e2e"]["ms_per_step"], 2), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
