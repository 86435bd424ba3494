"""Print the key numbers of bench.py JSON lines read from stdin (one per line)."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    rf = d.get("roofline", {})
    print(d["config"].get("n"), d["config"].get("rule", ""), "%.3e" % d["value"],
          "ms/step %.4f" % d["ms_per_step"], "kernel %.4f" % rf.get("kernel_ms_per_generation", rf.get("kernel_ms_per_launch", 0)),
          "frac %.3f" % rf.get("frac", 0), "clk", (d.get("clocks") or {}).get("sm_mhz"),
          "W", (d.get("clocks") or {}).get("power_w"), (d.get("clocks") or {}).get("reasons"))
