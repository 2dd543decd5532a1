"""Print a compact summary of a bench.py JSON line (developer tool)."""
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value", round(d["value"], 3), "e2e", round(d["e2e"]["value"], 3), "ms/step", d["ms_per_step"],
      "cycles/rhs", d.get("sequence", {}).get("mean_cycles_per_rhs"), "restarts", d.get("sequence", {}).get("restarts"),
      "launches", d.get("gpu_launches"), "clocks", d.get("clocks"))
tot = 0
for k, v in d.get("kernels", {}).items():
    tot += v["launches"] * v["avg_us"]
    print(f"  {k:17s} {v['launches']:6d} {v['avg_us']:9.2f} us {v['achieved_gbs']:8.1f} GB/s  frac {v['frac']:.3f}")
if d.get("steps"):
    print("  kernel ms/step", round(tot / 1e3 / d["steps"], 2))
if d.get("cpu_baseline"):
    print("  cpu", d["cpu_baseline"]["value"])
