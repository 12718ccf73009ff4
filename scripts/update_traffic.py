"""Rewrite profiles/traffic.json (the `roofline.traffic` of bench.py) from the
ncu launch lists of one profiles/<round> directory: per config, the DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum) of ONE bench step summed over
every kernel of the step -- the same scope as roofline.achieved (algorithmic
bytes of a step / the step's time) -- and the step's dominant kernel."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02"
out = {"_note": "DRAM bytes per bench step, summed over the step's kernels, from the ncu "
                f"launch lists in {d}/ncu_launches_<cfg>.csv (scripts/update_traffic.py)."}
for cfg in ("cfg4a", "cfg0", "cfg1", "cfg2", "cfg3", "cfg4b"):
    csv = os.path.join(ROOT, d, f"ncu_launches_{cfg}.csv")
    if not os.path.exists(csv):
        continue
    res = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "summarize_launches.py"),
                          csv], capture_output=True, text=True, check=True)
    rows = [json.loads(ln) for ln in res.stdout.splitlines() if ln.startswith("{")]
    steps = min(r["launches"] for r in rows)  # the rarest kernel runs once per step
    total = sum(r["launches"] * r["mean_dram_bytes"] for r in rows)
    out[cfg] = int(round(total / steps))
    out[cfg + "_kernel"] = rows[0]["kernel"]
    out[cfg + "_kernel_share"] = rows[0]["share"]
with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
