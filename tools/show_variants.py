"""Summarise gpurun_out/<tag>_<name>.json bench lines of tools/gpu_variants.sh."""
import glob, json, sys
tag = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/{tag}_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except (OSError, IndexError, ValueError):
        print(f, "no line"); continue
    c = d["config"]
    print(f.split("/")[-1], round(d["value"], 2), round(d["ms_per_step"], 2), c["passes_per_step"],
          c.get("autotune_ms_per_step"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], round(d["roofline"]["frac"], 3),
          d.get("norm_error"))
