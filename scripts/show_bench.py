"""Print the key fields of a bench.py JSON line (headline + secondaries)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])


def show(d, keys):
    for k in keys:
        if k in d:
            print(f"  {k}: {json.dumps(d.get(k))[:700]}")


print("HEADLINE", d.get("config", {}).get("workload"))
show(d, ["value", "ms_per_step", "e2e", "roofline", "host_roofline", "lane_busy_ms_per_step", "plan", "offload",
         "lanes_vs_sim", "calibration", "memory", "ps_gain", "grad", "clocks", "cpu_baseline"])
for k, v in d.get("secondary", {}).items():
    print("SECONDARY", k)
    show(v, ["value", "ms_per_step", "e2e", "roofline", "lane_busy_ms_per_step", "plan", "offload", "calibration",
             "memory", "ps_gain"])
