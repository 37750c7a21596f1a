"""Summarise gpurun_out/<tag>_{new,old,new2}.json (+ _bench.json) A/B lines."""
import json, sys
tag = sys.argv[1]
for f in ("new", "old", "new2", "bench"):
    try:
        d = json.loads(open(f"gpurun_out/{tag}_{f}.json").read().strip().splitlines()[-1])
    except (OSError, IndexError, ValueError):
        continue
    c = d["config"]
    oc = {k: (round(v["ms_per_step"], 2), v["passes_per_step"]) for k, v in d.get("other_configs", {}).items()}
    print(f, round(d["value"], 2), round(d["ms_per_step"], 1), c["passes_per_step"], c.get("autotune_ms_per_step"),
          d["clocks"]["sm_mhz"], round(d["roofline"]["frac"], 3), d.get("parity", {}).get("max_abs_dpsi"), oc)
